"""CPU: the aux oracle (metrics, loss patterns) against the reference's own
outputs (tests/golden/aux, made by tests/golden/make_golden_aux.py)."""

import math
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import aux_oracle as ao  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden", "aux")


def _close(x, y, tol):
    if math.isinf(x) or math.isinf(y):
        return x == y
    return abs(x - y) <= tol * max(1.0, abs(y))


def test_metrics_oracle_matches_reference():
    g = np.load(os.path.join(GOLD, "metrics.npz"))
    for i in range(int(g["n"])):
        a, b, sel = g[f"a{i}"], g[f"b{i}"], g[f"sel{i}"]
        assert _close(ao.psnr(a, b), float(g[f"psnr{i}"]), 1e-12), i
        assert _close(ao.psnr(a, b, sel), float(g[f"psnrm{i}"]), 1e-12), i
        assert _close(ao.ssim(a, b), float(g[f"ssim{i}"]), 1e-12), i


def test_ssim_rejects_small():
    with pytest.raises(ValueError):
        ao.ssim(np.zeros((10, 40)), np.zeros((10, 40)))


def test_mask_oracle_matches_reference():
    g = np.load(os.path.join(GOLD, "masks.npz"))
    assert [int(x) for x in g["splitmix_12345"]] == ao.splitmix_draws(12345, 64)
    n = 0
    for key in g.files:
        if key.startswith("disp_"):
            w, h = map(int, key.split("_")[1].split("x"))
            bs = int(key.split("_")[2])
            assert np.array_equal(ao.mask_states("dispersed", h, w, bs), g[key]), key
            n += 1
        elif key.startswith("rand_"):
            _, wh, bs, rate, seed = key.split("_")
            w, h = map(int, wh.split("x"))
            st = ao.mask_states("random", h, w, int(bs), float(rate), int(seed))
            assert np.array_equal(np.packbits(st == 1), g[key]), key
            n += 1
    assert n >= 20


def test_slice_oracle_matches_synth():
    from paper_2205_11226_b200.synth import slice_mask_states

    for seed in (3001, 3002, 5):
        assert np.array_equal(ao.mask_states("slice", 1080, 1920, 16, 0.10, seed), slice_mask_states(1080, 1920, 0.10, seed))
