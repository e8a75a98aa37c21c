"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
Writes tests/golden/<case>.npz with the inputs, the reference's float64
output, and its LayerDecision stream packed as bm_patch_record rows.
The GPU box never runs this (no /root/reference there); tests read the npz.
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import blockmend as ref  # noqa: E402  (the reference)
from blockmend.corpus import small_corpus  # noqa: E402

from oracle.oracle import RECORD_DTYPE, REC_DEFERRED, REC_FALLBACK, REC_HAS_BW, REC_HAS_M, REC_HAS_NU, REC_HAS_PHI  # noqa: E402
from paper_2205_11226_b200.synth import mask_for, synth_frame  # noqa: E402

LAYER = {None: -1, "BRL": 0, "IDL": 1, "HQL": 2}


def pack(decisions, n_y_of, gaps):
    out = np.zeros(len(decisions), dtype=RECORD_DTYPE)
    gi = 0
    for i, d in enumerate(decisions):
        r = out[i]
        r["beta_gap"] = math.nan
        if d.layer is not None and d.layer.value == "HQL" and not d.fallback:
            r["beta_gap"] = gaps[gi]
            gi += 1
        r["row"], r["col"] = d.patch_origin
        r["layer"] = LAYER[d.layer.value if d.layer is not None else None]
        f = 0
        if d.fallback:
            f |= REC_FALLBACK
        if d.deferred_fill:
            f |= REC_DEFERRED
        r["phi"] = d.phi if d.phi is not None else math.nan
        if d.phi is not None:
            f |= REC_HAS_PHI
        r["nu"] = d.nu if d.nu is not None else math.nan
        if d.nu is not None:
            f |= REC_HAS_NU
        r["beta"] = d.beta if d.beta is not None else math.nan
        r["alpha"] = d.alpha if d.alpha is not None else math.nan
        if d.beta is not None:
            f |= REC_HAS_BW
        r["m_candidates"] = d.m_candidates if d.m_candidates is not None else -1
        if d.m_candidates is not None:
            f |= REC_HAS_M
        r["rings_used"] = d.rings_used
        r["n_y"] = n_y_of.get(d.patch_origin, 0) if not d.deferred_fill else 0
        r["flags"] = f
    return out


def run_case(name, pixels, states, profile, forced=None):
    # record N_y per patch via the driver's own extract_target hook (profiles.py:25-36)
    n_y_of = {}
    orig = ref.profiles.extract_target

    def hook(work, st, patch):
        t = orig(work, st, patch)
        n_y_of[tuple(patch)] = t.n_y
        return t

    ref.profiles.extract_target = hook
    # beta_gap: relative epsilon gap of the reference's beta choice (estimators.py:197-206)
    gaps = []
    orig_bs = ref.estimators._beta_search

    def bs_hook(d, y, y0):
        beta = orig_bs(d, y, y0)
        eps = []
        for b in ref.estimators.BETA_GRID:
            w = ref.estimators._weights_from_quadforms(d, b)
            eps.append(float(((y0 - w @ y) ** 2).sum()))
        best = eps[int(np.where(ref.estimators.BETA_GRID == beta)[0][0])]
        dy = 1e-11 * float(np.max(np.abs(y0)))
        noise = 2.0 * np.sqrt(best * len(y0)) * dy + len(y0) * dy * dy + 1e-300
        others = [abs(e - best) / noise for b, e in zip(ref.estimators.BETA_GRID, eps) if b != beta]
        gaps.append(min(others))
        return beta

    ref.estimators._beta_search = bs_hook
    try:
        if profile == "sentinel":
            prof = ref.Profile.sentinel()
        elif isinstance(profile, tuple):
            prof = ref.Profile.custom(*profile)
        else:
            prof = ref.Profile.named(profile)
        layer = None if forced is None else ref.Layer(forced)
        out, rep = ref.conceal_image(ref.ImageBuffer(pixels), ref.LossMask(states), prof, forced_layer=layer)
    finally:
        ref.profiles.extract_target = orig
        ref.estimators._beta_search = orig_bs
    recs = pack(rep.decisions, n_y_of, gaps)
    np.savez_compressed(
        os.path.join(HERE, f"{name}.npz"),
        pixels=np.asarray(pixels, dtype=np.float64),
        states=np.asarray(states, dtype=np.uint8),
        t_phi=prof.t_phi,
        t_nu=prof.t_nu,
        forced=-1 if forced is None else LAYER[forced],
        out=out.pixels,
        records=recs,
    )
    print(f"{name}: {len(recs)} records, counts={rep.layer_counts}, deferred={rep.deferred_fills}", flush=True)


def main():
    img64 = synth_frame(64, 64, 4242, 14.0, 1.0).astype(np.float64)
    disp64 = mask_for("dispersed", 64, 64, 1)
    rnd64 = ref.gen_random_mask(ref.BlockGrid(64, 64), 0.35, 7).states
    for prof in ("sentinel", "efficient", "express", "excellent"):
        run_case(f"synth64_dispersed_{prof}", img64, disp64, prof)
    for prof in ("efficient", "express", "sentinel"):
        run_case(f"synth64_random35_{prof}", img64, rnd64, prof)
    # noisier texture: more HQL under the gate
    img64n = synth_frame(64, 64, 777, 30.0, 2.0).astype(np.float64)
    run_case("synth64n_random35_efficient", img64n, rnd64, "efficient")
    # 8x8 losses inside 16x16 cells (config 4 pattern), forced HQL and forced IDL
    r8 = ref.gen_random_mask(ref.BlockGrid(64, 64, block_size=8), 0.2, 11).states
    run_case("synth64_random8_forcedHQL", img64, r8, "sentinel", "HQL")
    run_case("synth64_random8_forcedIDL", img64, r8, "sentinel", "IDL")
    run_case("synth64_random8_efficient", img64, r8, "efficient")
    # non-integer pixels, one lost block, edge-clipped support
    rng = np.random.default_rng(1)
    fl48 = rng.uniform(0, 255, (48, 48))
    one48 = ref.gen_dispersed_mask(ref.BlockGrid(48, 48)).states
    run_case("float48_one_sentinel", fl48, one48, "sentinel")
    run_case("float48_one_efficient", fl48, one48, "efficient")
    run_case("float48_one_forcedBRL", fl48, one48, "sentinel", "BRL")
    # corpus crops (the reference's own fixtures), random 50% losses
    corp = small_corpus()
    for nm in ("patch_quilt", "stripe_court", "checker_fade"):
        m = ref.gen_random_mask(ref.BlockGrid(48, 48), 0.5, 3).states
        run_case(f"corpus_{nm}_random50_express", corp[nm].pixels, m, "express")
    # total loss: deferral then 128 fill (profiles.py:215-225)
    run_case("flat48_total_express", np.full((48, 48), 50.0), ref.gen_random_mask(ref.BlockGrid(48, 48), 1.0, 0).states, "express")
    # ragged image (72 x 88) with slice loss and pre-reconstructed pixels
    img_r = synth_frame(72, 88, 99, 14.0, 1.0).astype(np.float64)
    st_r = mask_for("slice", 72, 88, 5)
    st_r[st_r == 0] = np.where(np.random.default_rng(5).random((72, 88)) < 0.05, 2, 0)[st_r == 0]
    st_r[(st_r == 0)] = 0
    if not (st_r == 1).any():
        st_r[16:32, 16:48] = 1
    run_case("ragged72x88_slice_efficient", img_r, st_r, "efficient")
    run_case("ragged72x88_slice_custom", img_r, st_r, (5.0, 2.0))
    # period-2 stripes: exact IDL reconstruction
    cols = np.arange(48) % 2
    stripes = np.tile(np.where(cols == 0, 0.0, 200.0), (48, 1))
    run_case("stripes48_one_express", stripes, one48, "express")
    # slice loss on a 96 x 64 synthetic frame (DAG chains)
    img_s = synth_frame(96, 64, 31, 14.0, 1.0).astype(np.float64)
    st_s = np.zeros((96, 64), np.uint8)
    st_s[32:48, :] = 1
    st_s[48:64, 16:48] = 1
    run_case("synth96x64_slice_efficient", img_s, st_s, "efficient")
    run_case("synth96x64_slice_sentinel", img_s, st_s, "sentinel")


if __name__ == "__main__":
    main()
