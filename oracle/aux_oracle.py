"""CPU oracle of the callers either side of the path.

TEST INFRASTRUCTURE ONLY (tests/ import it; the product never does).
Restates, in NumPy/SciPy FP64:
  * psnr / psnr_masked (blockmend/metrics.py:50-73): 10 log10(255^2 / MSE);
  * ssim (metrics.py:76-116): separable 11-tap Gaussian (sigma 1.5,
    normalised) windowed moments, axis 0 then axis 1, K1 0.01, K2 0.03,
    L 255, mean over the windows that lie fully inside the frame;
  * the loss patterns (loss.py:24-77): SplitMix64, modulo Fisher-Yates,
    dispersed odd/odd blocks, exact-count random blocks, and whole
    block-row slices (the BASELINE slice pattern).
Pinned against the reference's own outputs in tests/golden/aux/
(tests/golden/make_golden_aux.py) by tests/test_aux_oracle.py.
"""

from __future__ import annotations

import math

import numpy as np
from scipy.ndimage import correlate1d

M64 = (1 << 64) - 1


def psnr(a, b, select=None) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if select is not None:
        select = np.asarray(select, dtype=bool)
        if not select.any():
            return math.inf
        d = a[select] - b[select]
    else:
        d = a - b
    mse = float(np.mean(d * d))
    return math.inf if mse == 0.0 else 10.0 * math.log10(255.0 * 255.0 / mse)


def gauss11() -> np.ndarray:
    x = np.arange(-5, 6, dtype=np.float64)
    g = np.exp(-(x * x) / (2.0 * 1.5 * 1.5))
    return g / g.sum()


def ssim(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if min(a.shape) < 11:
        raise ValueError("image too small for SSIM")
    g = gauss11()

    def win(x):
        return correlate1d(correlate1d(x, g, axis=0, mode="constant"), g, axis=1, mode="constant")[5:-5, 5:-5]

    ma, mb = win(a), win(b)
    va, vb, cab = win(a * a) - ma * ma, win(b * b) - mb * mb, win(a * b) - ma * mb
    c1, c2 = (0.01 * 255.0) ** 2, (0.03 * 255.0) ** 2
    s = ((2 * ma * mb + c1) * (2 * cab + c2)) / ((ma * ma + mb * mb + c1) * (va + vb + c2))
    return float(s.mean())


def splitmix_draws(seed: int, count: int) -> list[int]:
    out, st = [], seed & M64
    for _ in range(count):
        st = (st + 0x9E3779B97F4A7C15) & M64
        z = st
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        out.append(z ^ (z >> 31))
    return out


def shuffled(count: int, seed: int) -> list[int]:
    order = list(range(count))
    draws = splitmix_draws(seed, max(count - 1, 0))
    for t, i in enumerate(range(count - 1, 0, -1)):
        j = draws[t] % (i + 1)
        order[i], order[j] = order[j], order[i]
    return order


def mask_states(kind: str, h: int, w: int, bs: int = 16, rate: float = 0.25, seed: int = 0) -> np.ndarray:
    rows, cols = h // bs, w // bs
    lost = np.zeros((rows, cols), dtype=bool)
    if kind == "dispersed":
        lost[1::2, 1::2] = True
    elif kind == "random":
        n = int(math.floor(rate * rows * cols + 0.5))
        for idx in shuffled(rows * cols, seed)[:n]:
            lost[idx // cols, idx % cols] = True
    elif kind == "slice":
        n = int(math.floor(rate * rows + 0.5))
        for r in shuffled(rows, seed)[:n]:
            lost[r, :] = True
    else:
        raise ValueError(kind)
    st = np.zeros((h, w), dtype=np.uint8)
    st[: rows * bs, : cols * bs] = np.repeat(np.repeat(lost, bs, axis=0), bs, axis=1).astype(np.uint8)
    return st
