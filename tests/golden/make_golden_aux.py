"""Golden vectors for the callers either side of the path,
made by running the REFERENCE package itself in the build container:

    python tests/golden/make_golden_aux.py

* metrics.npz: blockmend.metrics psnr / psnr_masked / ssim on seeded image
  pairs (u8 and float, identical frames, sizes 11..97);
* masks.npz: blockmend.loss gen_dispersed_mask / gen_random_mask states on
  several grids, rates and seeds, plus the first SplitMix64 draws.
The GPU box never runs this; the tests read the npz files.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from blockmend import metrics as rm  # noqa: E402  (the reference)
from blockmend.image import BlockGrid, ImageBuffer  # noqa: E402
from blockmend.loss import SplitMix64, gen_dispersed_mask, gen_random_mask  # noqa: E402


def metric_cases():
    rng = np.random.default_rng(20260)
    cases = []
    for k, (h, w, kind) in enumerate([(11, 11, "u8"), (17, 23, "u8"), (64, 64, "u8"), (97, 80, "f64"),
                                      (48, 72, "u8"), (33, 41, "f64"), (64, 48, "same")]):
        a = rng.integers(0, 256, size=(h, w)).astype(np.float64)
        if kind == "f64":
            a = a + rng.normal(0, 3.0, size=(h, w))
        b = np.clip(a + rng.normal(0, 6.0, size=(h, w)), -20, 280) if kind != "same" else a.copy()
        if kind == "u8":
            b = np.clip(np.round(b), 0, 255)
        sel = rng.random((h, w)) < 0.3
        cases.append((a, b, sel))
    return cases


def main():
    out = {}
    for i, (a, b, sel) in enumerate(metric_cases()):
        out[f"a{i}"], out[f"b{i}"], out[f"sel{i}"] = a, b, sel
        out[f"psnr{i}"] = rm.psnr(ImageBuffer(a), ImageBuffer(b))
        out[f"psnrm{i}"] = rm.psnr_masked(ImageBuffer(a), ImageBuffer(b), sel)
        out[f"ssim{i}"] = rm.ssim(ImageBuffer(a), ImageBuffer(b))
    np.savez_compressed(os.path.join(HERE, "aux", "metrics.npz"), n=len(metric_cases()), **out)

    masks = {}
    grids = [(256, 256, 16), (512, 512, 16), (1920, 1080, 16), (200, 136, 8), (72, 88, 16), (3840, 2160, 8)]
    k = 0
    for (w, h, bs) in grids:
        g = BlockGrid(w, h, block_size=bs)
        masks[f"disp_{w}x{h}_{bs}"] = gen_dispersed_mask(g).states
        for rate, seed in ((0.2, 1), (0.25, 77), (0.5, 2**63 + 5), (0.0, 3), (1.0, 4)):
            if (w, h) == (3840, 2160) and rate not in (0.2,):
                continue
            masks[f"rand_{w}x{h}_{bs}_{rate}_{seed}"] = np.packbits(gen_random_mask(g, rate, seed).states == 1)
            k += 1
    r = SplitMix64(12345)
    masks["splitmix_12345"] = np.array([r.next_u64() for _ in range(64)], dtype=np.uint64)
    np.savez_compressed(os.path.join(HERE, "aux", "masks.npz"), **masks)
    print("wrote", len(out), "metric arrays,", len(masks), "mask arrays")


if __name__ == "__main__":
    main()
