"""CPU: raster I/O (netpbm.py) and the harness's argument handling (cli.py)."""

import os

import numpy as np
import pytest

from paper_2205_11226_b200 import cli, netpbm
from paper_2205_11226_b200.errors import FormatError
from paper_2205_11226_b200.image import ImageBuffer, LossMask

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "aux", "cli")


def test_pgm_round_trip_and_quantize(tmp_path):
    a = (np.arange(48 * 64) * 7 % 256).astype(np.float64).reshape(48, 64)
    a[0, 0], a[0, 1], a[0, 2] = -3.2, 300.0, 127.5  # clamp + round half up
    netpbm.save_image(ImageBuffer(a), tmp_path / "x.pgm")
    b = netpbm.load_image(tmp_path / "x.pgm").pixels
    assert b[0, 0] == 0 and b[0, 1] == 255 and b[0, 2] == 128
    assert np.array_equal(b[1:], a[1:])


def test_pgm_header_comments_and_errors(tmp_path):
    p = tmp_path / "c.pgm"
    p.write_bytes(b"P5\n# comment\n3 2\n# more\n255\n" + bytes(range(6)))
    assert netpbm.load_image(p).pixels.tolist() == [[0, 1, 2], [3, 4, 5]]
    for body, msg in ((b"P2\n3 2\n255\n", "unsupported"), (b"P5\n3 2\n65535\n" + bytes(12), "bit depth"),
                      (b"P5\n3 2\n255\n" + bytes(3), "end of file"), (b"P5\n3 x\n255\n", "malformed"),
                      (b"P5\n0 2\n255\n", "positive")):
        p.write_bytes(body)
        with pytest.raises(FormatError, match=msg):
            netpbm.load_image(p)


def test_masks(tmp_path):
    st = np.zeros((40, 40), np.uint8)
    st[16:32, 16:32] = 1
    netpbm.save_mask(LossMask(st), tmp_path / "m.pgm")
    assert np.array_equal(netpbm.load_mask(tmp_path / "m.pgm").states, st)
    raw = np.full((40, 40), 255, np.uint8)
    raw[35, 5] = 0  # lost outside the full-block area
    (tmp_path / "bad.pgm").write_bytes(b"P5\n40 40\n255\n" + raw.tobytes())
    with pytest.raises(FormatError, match="outside"):
        netpbm.load_mask(tmp_path / "bad.pgm")
    raw[35, 5] = 7
    (tmp_path / "bad.pgm").write_bytes(b"P5\n40 40\n255\n" + raw.tobytes())
    with pytest.raises(FormatError, match="invalid mask sample"):
        netpbm.load_mask(tmp_path / "bad.pgm")
    with pytest.raises(ValueError):
        netpbm.save_mask(LossMask(np.full((16, 16), 2, np.uint8)), tmp_path / "r.pgm")


def test_ppm_and_png(tmp_path):
    rgb = np.zeros((4, 5, 3), np.uint8)
    rgb[..., 1] = 200
    netpbm.save_ppm(rgb, tmp_path / "x.ppm")
    assert (tmp_path / "x.ppm").read_bytes() == b"P6\n5 4\n255\n" + rgb.tobytes()
    with pytest.raises(ValueError):
        netpbm.save_ppm(rgb[..., :2], tmp_path / "y.ppm")
    from PIL import Image

    g = (np.arange(30 * 20) % 256).astype(np.uint8).reshape(30, 20)
    Image.fromarray(g, mode="L").save(tmp_path / "g.png")
    assert np.array_equal(netpbm.load_image(tmp_path / "g.png").pixels, g)
    Image.fromarray(rgb).save(tmp_path / "c.png")
    with pytest.raises(FormatError, match="mode"):
        netpbm.load_image(tmp_path / "c.png")


def test_golden_inputs_readable():
    for name in ("img_a", "img_b"):
        img = netpbm.load_image(os.path.join(GOLD, f"{name}.pgm"))
        assert img.pixels.dtype == np.float64 and img.pixels.ndim == 2


@pytest.mark.parametrize("args,msg", [
    (["--method", "foo"], "unknown method"),
    ([], "requires --profile"),
    (["--profile", "efficient", "--t-phi", "3"], "together"),
    (["--profile", "efficient", "--pattern", "zigzag"], "unknown pattern"),
])
def test_cli_validation(tmp_path, capsys, args, msg):
    rc = cli.main(["--input", str(tmp_path / "none.pgm"), "--out-dir", str(tmp_path / "o"), *args])
    assert rc == 2
    assert msg in capsys.readouterr().err


def test_cli_no_inputs(tmp_path, capsys):
    assert cli.main(["--input", str(tmp_path / "none*.pgm"), "--out-dir", str(tmp_path / "o"),
                     "--profile", "efficient"]) == 2
