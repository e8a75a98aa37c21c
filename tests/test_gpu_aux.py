"""GPU: device metrics and loss-pattern generation
against the reference's golden outputs and the aux oracle."""

import math
import os

import numpy as np
import pytest

from oracle import aux_oracle as ao

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "aux")


def _close(x, y, tol):
    if math.isinf(x) or math.isinf(y):
        return x == y
    return abs(x - y) <= tol * max(1.0, abs(y))


def test_metrics_vs_reference_golden(native):
    import paper_2205_11226_b200 as bm

    g = np.load(os.path.join(GOLD, "metrics.npz"))
    for i in range(int(g["n"])):
        a, b, sel = g[f"a{i}"], g[f"b{i}"], g[f"sel{i}"]
        assert _close(bm.psnr(bm.ImageBuffer(a), bm.ImageBuffer(b)), float(g[f"psnr{i}"]), 1e-10), i
        assert _close(bm.psnr_masked(a, b, sel), float(g[f"psnrm{i}"]), 1e-10), i
        assert _close(bm.ssim(a, b), float(g[f"ssim{i}"]), 1e-10), i


def test_metrics_batch_u8_frames(native):
    import torch

    import paper_2205_11226_b200 as bm
    from paper_2205_11226_b200.synth import make_config

    px, st = make_config(3, frames=3)
    rng = np.random.default_rng(1)
    test = np.clip(px.astype(np.int32) + rng.integers(-9, 10, size=px.shape), 0, 255).astype(np.uint8)
    tp, tt, ts = torch.from_numpy(px).cuda(), torch.from_numpy(test).cuda(), torch.from_numpy(st).cuda()
    ps = bm.psnr_batch(tp, tt)
    pm = bm.psnr_batch(tp, tt, select=(ts == 1))
    ss = bm.ssim_batch(tp, tt)
    for f in range(3):
        assert _close(ps[f], ao.psnr(px[f], test[f]), 1e-10)
        assert _close(pm[f], ao.psnr(px[f], test[f], st[f] == 1), 1e-10)
        assert _close(ss[f], ao.ssim(px[f], test[f]), 1e-10)


def test_metrics_edge_cases(native):
    import paper_2205_11226_b200 as bm

    a = np.arange(24 * 30, dtype=np.float64).reshape(24, 30) % 251
    assert bm.psnr(a, a) == math.inf
    assert bm.psnr_masked(a, a + 1, np.zeros_like(a, dtype=bool)) == math.inf
    assert _close(bm.ssim(a, a), 1.0, 1e-12)
    with pytest.raises(ValueError):
        bm.ssim(a[:10], a[:10])
    with pytest.raises(bm.DimensionMismatchError):
        bm.psnr(a, a[:, :-1])


@pytest.mark.parametrize("grid", [(256, 256, 16), (1920, 1080, 16), (200, 136, 8), (72, 88, 16), (3840, 2160, 8)])
def test_device_masks_vs_reference_golden(native, grid):
    import paper_2205_11226_b200 as bm

    g = np.load(os.path.join(GOLD, "masks.npz"))
    w, h, bs = grid
    d = bm.gen_masks_device("dispersed", 2, h, w, block_size=bs).cpu().numpy()
    assert np.array_equal(d[0], g[f"disp_{w}x{h}_{bs}"]) and np.array_equal(d[1], d[0])
    keys = [k for k in g.files if k.startswith(f"rand_{w}x{h}_{bs}_")]
    assert keys
    for key in keys:
        rate, seed = float(key.split("_")[3]), int(key.split("_")[4])
        r = bm.gen_masks_device("random", 1, h, w, block_size=bs, rate=rate, seeds=[seed]).cpu().numpy()
        assert np.array_equal(np.packbits(r[0] == 1), g[key]), key


def test_device_slice_masks_match_oracle(native):
    import paper_2205_11226_b200 as bm

    seeds = [3001 + f for f in range(6)] + [2**64 - 1]
    d = bm.gen_masks_device("slice", len(seeds), 1080, 1920, rate=0.10, seeds=seeds).cpu().numpy()
    for f, s in enumerate(seeds):
        assert np.array_equal(d[f], ao.mask_states("slice", 1080, 1920, 16, 0.10, s)), f
