"""Seeded synthetic luma frames and loss masks for BASELINE.json's configs.

The reference measures on Kodak/Tecnick images (absent here);
BASELINE.json replaces them with this generator:
1/f^2 Gaussian-spectrum noise + filled convex polygons with hard edges +
two oriented sinusoid textures, rounded and clipped to uint8.

Masks reuse the reference's own generators (loss.py:55-77, restated in
``loss.py`` of this package) plus the macroblock-row slice pattern of
config 3.  Everything is numpy on the host: it builds inputs, it is not on
the measured path.
"""

from __future__ import annotations

import math

import numpy as np

from .image import BlockGrid, PixelState
from .loss import SplitMix64, fisher_yates, gen_dispersed_mask, gen_random_mask


def synth_frame(h: int, w: int, seed: int, noise_std: float = 14.0, density: float = 1.0) -> np.ndarray:
    """One uint8 [h, w] frame (SURVEY.md §8(d) generator G)."""
    rng = np.random.default_rng(seed)
    # 1/f^2 power spectrum -> amplitude 1/|f|
    fy = np.fft.fftfreq(h)[:, None]
    fx = np.fft.rfftfreq(w)[None, :]
    f = np.sqrt(fx * fx + fy * fy)
    f[0, 0] = 1.0
    spec = (rng.standard_normal(f.shape) + 1j * rng.standard_normal(f.shape)) / f
    spec[0, 0] = 0.0
    noise = np.fft.irfft2(spec, s=(h, w))
    noise = (noise - noise.mean()) / (noise.std() + 1e-12)
    img = noise * noise_std + 128.0

    # filled convex polygons with sharp edges
    n_poly = int(round(6 * density))
    yy, xx = np.mgrid[0:h, 0:w]
    for _ in range(n_poly):
        nv = int(rng.integers(3, 8))
        radius = rng.uniform(0.05, 0.25) * min(h, w)
        cy, cx = rng.uniform(0, h), rng.uniform(0, w)
        ang = np.sort(rng.uniform(0, 2 * math.pi, nv))
        py = cy + radius * np.sin(ang)
        px = cx + radius * np.cos(ang)
        fill = rng.uniform(0, 255)
        r0, r1 = max(0, int(py.min())), min(h, int(py.max()) + 2)
        c0, c1 = max(0, int(px.min())), min(w, int(px.max()) + 2)
        if r0 >= r1 or c0 >= c1:
            continue
        sy = yy[r0:r1, c0:c1]
        sx = xx[r0:r1, c0:c1]
        inside = np.ones(sy.shape, dtype=bool)
        for i in range(nv):  # vertices sorted by angle -> counter-clockwise convex hull
            ay, ax = py[i], px[i]
            by, bx = py[(i + 1) % nv], px[(i + 1) % nv]
            inside &= (bx - ax) * (sy - ay) - (by - ay) * (sx - ax) >= 0
        img[r0:r1, c0:c1][inside] = fill

    # two oriented sinusoid textures inside random rectangles
    for _ in range(2):
        theta = rng.uniform(0, math.pi)
        period = rng.uniform(4, 16)
        amp = rng.uniform(20, 60)
        rh = int(rng.uniform(h / 4, h / 2))
        rw = int(rng.uniform(w / 4, w / 2))
        r0 = int(rng.integers(0, max(1, h - rh)))
        c0 = int(rng.integers(0, max(1, w - rw)))
        sy = yy[r0 : r0 + rh, c0 : c0 + rw]
        sx = xx[r0 : r0 + rh, c0 : c0 + rw]
        phase = (sx * math.cos(theta) + sy * math.sin(theta)) * (2 * math.pi / period)
        img[r0 : r0 + rh, c0 : c0 + rw] += amp * np.sin(phase)

    return np.clip(np.round(img), 0, 255).astype(np.uint8)


def frame_params(cfg: int, frame: int):
    """(seed, noise_std, density) per frame: 'edge/texture density varied per frame by seed'."""
    seed = 1000 * cfg + frame
    if cfg in (1, 2):
        return seed, 14.0, 1.0
    rng = np.random.default_rng(seed + 7919)
    return seed, float(rng.uniform(6, 24)), float(rng.uniform(0.5, 2.0))


def slice_mask_states(h: int, w: int, rate: float, seed: int) -> np.ndarray:
    """Whole macroblock rows lost: round(rate * rows) rows by seeded Fisher-Yates (loss.py:24-44)."""
    grid = BlockGrid(w, h)
    count = int(math.floor(rate * grid.rows + 0.5))
    order = fisher_yates(grid.rows, SplitMix64(seed))
    states = np.zeros((h, w), dtype=np.uint8)
    for r in order[:count]:
        states[r * 16 : (r + 1) * 16, : grid.cols * 16] = PixelState.LOST
    return states


def mask_for(pattern: str, h: int, w: int, seed: int) -> np.ndarray:
    if pattern == "dispersed":
        return gen_dispersed_mask(BlockGrid(w, h)).states
    if pattern == "slice":
        return slice_mask_states(h, w, 0.10, seed)
    if pattern == "random16":
        return gen_random_mask(BlockGrid(w, h), 0.20, seed).states
    if pattern == "random8":
        return gen_random_mask(BlockGrid(w, h, block_size=8), 0.20, seed).states
    raise ValueError(pattern)


CONFIGS = {
    # cfg: (frames, h, w, pattern(s), profile, forced_layer)
    1: (1, 256, 256, ("dispersed",), "sentinel", None),
    2: (1, 512, 512, ("dispersed",), "efficient", None),
    3: (16, 1080, 1920, ("slice",), "efficient", None),
    4: (8, 2160, 3840, ("random8",), "sentinel", "HQL"),
    5: (256, 1080, 1920, ("dispersed", "slice", "random16"), "efficient", None),
}


def make_config(cfg: int, frames: int | None = None, crop: tuple[int, int] | None = None, first: int = 0):
    """Frames [first, first+B) of BASELINE config `cfg`: u8 pixels and states [B,h,w].

    `frames` limits the batch (parity crops / CPU samples); `crop` takes the
    top-left (h, w) crop of every frame with its mask.
    """
    nb, h, w, patterns, _, _ = CONFIGS[cfg]
    nb = nb - first if frames is None else frames
    hh, ww = (h, w) if crop is None else crop
    px = np.empty((nb, hh, ww), dtype=np.uint8)
    st = np.empty((nb, hh, ww), dtype=np.uint8)
    for i in range(nb):
        f = first + i
        seed, noise, dens = frame_params(cfg, f)
        px[i] = synth_frame(h, w, seed, noise, dens)[:hh, :ww]
        st[i] = mask_for(patterns[f % len(patterns)], h, w, seed + 1)[:hh, :ww]
    return px, st
