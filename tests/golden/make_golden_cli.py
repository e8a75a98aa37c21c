"""Golden run of the REFERENCE CLI (blockmend/cli.py) for the harness tests:

    python tests/golden/make_golden_cli.py

Writes two seeded PGM inputs and the reference's report.json / reconstructions
(deterministic fields only are compared) under tests/golden/aux/cli/.
"""

from __future__ import annotations

import json
import os
import shutil
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

from blockmend import cli as rcli  # noqa: E402  (the reference)

from paper_2205_11226_b200.synth import synth_frame  # noqa: E402

OUT = os.path.join(HERE, "aux", "cli")
RUNS = {
    "random": ["--pattern", "random", "--rate", "0.3", "--seed", "5", "--method", "skmmse,kmmse,brl,idl,hql",
               "--profile", "efficient", "--layer-map"],
    "dispersed_lost": ["--pattern", "dispersed", "--method", "skmmse", "--t-phi", "12", "--t-nu", "0.05",
                       "--psnr-lost-only"],
}


def inputs(dirpath):
    paths = []
    for name, (h, w, seed, noise) in {"img_a": (64, 64, 11, 14.0), "img_b": (80, 96, 12, 20.0)}.items():
        px = synth_frame(h, w, seed, noise, 1.0)
        p = os.path.join(dirpath, f"{name}.pgm")
        with open(p, "wb") as fh:
            fh.write(f"P5\n{w} {h}\n255\n".encode())
            fh.write(px.tobytes())
        paths.append(p)
    return paths


def main():
    os.makedirs(OUT, exist_ok=True)
    inp = inputs(OUT)
    for run, args in RUNS.items():
        tmp = tempfile.mkdtemp()
        rc = rcli.main(["--input", os.path.join(OUT, "img_*.pgm"), "--out-dir", tmp, *args])
        assert rc == 0, rc
        rep = json.load(open(os.path.join(tmp, "report.json")))
        for r in rep["images"]:
            for k in ("mean_patch_ms", "total_s"):
                r.pop(k, None)
        for a in rep["aggregates"]:
            for k in ("mean_patch_ms", "time_vs_kmmse"):
                a.pop(k, None)
        rep.pop("timestamp")
        recons = {f: np.fromfile(os.path.join(tmp, f), dtype=np.uint8) for f in sorted(os.listdir(tmp))
                  if f.endswith(".recon.pgm") or f.endswith(".layers.ppm")}
        np.savez_compressed(os.path.join(OUT, f"{run}_files.npz"), **recons)
        with open(os.path.join(OUT, f"{run}_report.json"), "w") as fh:
            json.dump(rep, fh, indent=1)
        shutil.rmtree(tmp)
    print("inputs", inp, "runs", list(RUNS))


if __name__ == "__main__":
    main()
