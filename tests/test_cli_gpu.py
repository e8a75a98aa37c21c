"""GPU: the harness end to end against the reference CLI's golden run
(tests/golden/make_golden_cli.py): same report schema and deterministic
fields, reconstructions and layer maps."""

import io
import json
import os

import numpy as np
import pytest

from paper_2205_11226_b200 import cli

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "aux", "cli")
RUNS = {
    "random": ["--pattern", "random", "--rate", "0.3", "--seed", "5", "--method", "skmmse,kmmse,brl,idl,hql",
               "--profile", "efficient", "--layer-map"],
    "dispersed_lost": ["--pattern", "dispersed", "--method", "skmmse", "--t-phi", "12", "--t-nu", "0.05",
                       "--psnr-lost-only"],
}


def _pgm(buf):
    from paper_2205_11226_b200.netpbm import read_pgm_bytes

    return read_pgm_bytes(bytes(buf))


@pytest.mark.parametrize("run", sorted(RUNS))
def test_cli_matches_reference_run(native, tmp_path, run):
    rc = cli.main(["--input", os.path.join(GOLD, "img_*.pgm"), "--out-dir", str(tmp_path), *RUNS[run]])
    assert rc == 0
    ours = json.load(open(tmp_path / "report.json"))
    ref = json.load(open(os.path.join(GOLD, f"{run}_report.json")))
    assert ours["schema_version"] == ref["schema_version"] == 1
    assert ours["config"] == ref["config"]
    assert len(ours["images"]) == len(ref["images"])
    for a, b in zip(ours["images"], ref["images"]):
        assert set(b) <= set(a)
        for k in ("image", "status", "method", "profile", "t_phi", "t_nu", "pattern", "rate", "seed", "psnr_scope",
                  "patches", "layer_counts", "deferred_fills"):
            assert a[k] == b[k], (k, a[k], b[k])
        assert abs(a["psnr_db"] - b["psnr_db"]) <= 0.05, (a["psnr_db"], b["psnr_db"])  # +-1 LSB on <=0.1% px
        assert abs(a["ssim"] - b["ssim"]) <= 1e-3
    files = np.load(os.path.join(GOLD, f"{run}_files.npz"))
    for name in files.files:
        got = np.fromfile(tmp_path / name, dtype=np.uint8)
        exp = files[name]
        assert got.shape == exp.shape, name
        if name.endswith(".recon.pgm"):
            # the +-1 LSB bar, except where a beta choice the reference itself made
            # at rounding level moved a few cells (decision-level parity, with the
            # tie rule, is tests/test_gpu.py's): those stay few and local
            g, e = _pgm(got).astype(int), _pgm(exp).astype(int)
            d = np.abs(g - e)
            big = d > 1
            cells = {(r // 16, c // 16) for r, c in zip(*np.nonzero(big))}
            assert (d > 0).mean() <= 0.01 and len(cells) <= 3, (name, int(d.max()), sorted(cells))
        else:
            assert np.array_equal(got, exp), name
    # CSV schema
    rc = cli.main(["--input", os.path.join(GOLD, "img_*.pgm"), "--out-dir", str(tmp_path / "csv"), "--report", "csv",
                   *RUNS[run]])
    assert rc == 0
    head = open(tmp_path / "csv" / "report.csv").readline().strip().split(",")
    assert head == cli.CSV_COLUMNS
