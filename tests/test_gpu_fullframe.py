"""Full-size parity at the configs' real dependency depth.

Whole BASELINE frames, concealed on the GPU and compared with outputs of the
REFERENCE package itself (tests/golden/fullframe/, made by
tests/golden/make_golden_fullframe.py running blockmend's own per-cell
driver in dependency-level order) and with the CPU oracle (its level-parallel
driver oracle.conceal_dag, same result as the serial order).

What depth does to this algorithm (measured): every lost
cell's HQL estimate is an ill-conditioned fit (alpha, ridge 1e-6 tr/N_y) on
its predecessors' reconstructed pixels, so a rounding-level difference in a
cell's inputs grows ~10x every 3-5 dependency levels.  The plain-C FP64
restatement of the reference and the reference itself agree to 1e-12 at
level 0 and disagree on 61% of the lost pixels of a 392-level forced-HQL 4K
frame; any implementation that is not bit-identical to NumPy/OpenBLAS
does the same.  Parity at depth is therefore checked two ways:
  * free-running frames (the real chains): the tests/parity.py rule - layer
    decisions identical except at the reference's thresholds, beta choices
    identical except the reference's rounding-decided ties, pixel bars on
    every cell not downstream of such a tie - with the tie counts bounded and
    the all-pixel figures printed;
  * teacher-forced cells (cfg4 4K forced HQL): the cells of six dependency
    levels up to 392, each handed the reference's own reconstruction of its
    predecessors (RECONSTRUCTED state, the reference's values), so the GPU's
    per-cell computation is checked against the reference at full depth
    without the chain's chaotic amplification.
"""

import hashlib
import math
import os

import numpy as np
import pytest

import parity
from oracle import oracle
from paper_2205_11226_b200 import Profile, conceal_batch
from paper_2205_11226_b200.synth import make_config

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "fullframe")

# free-running frames vs the reference: (golden name) -> max excused divergences
# (reference beta ties decided at rounding level; threshold-decided layers), measured
FREE = {
    "cfg3_f0_slice_efficient": 0,
    "cfg5_f0_dispersed_efficient": 4,
    "cfg5_f1_slice_efficient": 2,
    "cfg5_f2_random_efficient": 20,
}


def _profile(name):
    return Profile.sentinel() if name == "sentinel" else Profile.named(name)


def _load(name):
    z = np.load(os.path.join(GOLD, f"{name}.npz"))
    cfg, frame = int(z["cfg"]), int(z["frame"])
    px, st = make_config(cfg, frames=1, first=frame)
    px, st = px[0], st[0]
    assert hashlib.sha256(px.tobytes() + st.tobytes()).hexdigest() == str(z["digest"]), "synthetic inputs changed"
    ref = px.astype(np.float64).copy()
    ref[st == 1] = z["lost_values"]
    return z, px, st, ref


def _levels(st):
    gr, gc = st.shape[0] // 16, st.shape[1] // 16
    lost = (st[: gr * 16, : gc * 16] == 1).reshape(gr, 16, gc, 16).any(axis=(1, 3))
    lv = np.full((gr, gc), -1)
    for r in range(gr):
        for c in range(gc):
            if lost[r, c]:
                m = 0
                for dr, dc in ((-1, -1), (-1, 0), (-1, 1), (0, -1)):
                    rr, cc = r + dr, c + dc
                    if rr >= 0 and 0 <= cc < gc and lv[rr, cc] >= 0:
                        m = max(m, lv[rr, cc] + 1)
                lv[r, c] = m
    return lv


@pytest.mark.parametrize("name", sorted(FREE))
def test_full_frame_vs_reference(native, name):
    import torch

    z, px, st, ref = _load(name)
    prof = _profile(str(z["profile"]))
    res = conceal_batch(torch.from_numpy(px[None]).cuda(), torch.from_numpy(st[None]).cuda(), prof,
                        want_f64=True, records=True)
    gout = res.recon_f64[0].cpu().numpy()
    pr = parity.compare(ref, z["records"], gout, res.records, st, prof.t_phi, prof.t_nu)
    o_out, o_rec, _, _ = oracle.conceal_dag(px.astype(np.float64), st, prof.t_phi, prof.t_nu)
    po = parity.compare(ref, z["records"], o_out, o_rec, st, prof.t_phi, prof.t_nu)
    print(f"\n{name}: depth {res.summary['max_level'] + 1} cells {res.summary['lost_cells']}\n"
          f"  GPU    vs reference: {pr.summary()}\n  oracle vs reference: {po.summary()}")
    assert pr.ok, pr.problems[:5]
    assert len(pr.allowed) + len(pr.beta_ties) <= FREE[name], (pr.allowed, pr.beta_ties)


def test_teacher_forced_4k_hql_vs_reference(native):
    """Cells of dependency levels 0..392 of a 3840x2160 forced-HQL frame, each
    given the reference's own predecessors, against the reference."""
    import torch

    z, px, st, ref = _load("cfg4_f0_random8_forcedHQL")
    lv = _levels(st)
    levels = [int(v) for v in z["teacher_levels"]]
    cell_lv = np.repeat(np.repeat(lv, 16, 0), 16, 1)
    h, w = cell_lv.shape
    frames, states = [], []
    for L in levels:
        f = px.astype(np.float64).copy()
        s = st.copy()
        done = np.zeros(st.shape, bool)
        done[:h, :w] = (cell_lv >= 0) & (cell_lv < L)
        done &= st == 1
        f[done] = ref[done]  # the reference's reconstruction of every earlier level
        s[done] = 2  # RECONSTRUCTED
        frames.append(f)
        states.append(s)
    prof = Profile.sentinel()
    res = conceal_batch(torch.from_numpy(np.stack(frames)).cuda(), torch.from_numpy(np.stack(states)).cuda(), prof,
                        forced_layer="HQL", want_f64=True, records=True)
    gout = res.recon_f64.cpu().numpy()
    rrec = z["records"]
    rcell = np.stack([rrec["row"] // 16, rrec["col"] // 16], 1)
    total_ties = 0
    for i, L in enumerate(levels):
        grec = res.records[res.records["frame"] == i].copy()
        gsel = lv[grec["row"] // 16, grec["col"] // 16] == L
        rsel = lv[rcell[:, 0], rcell[:, 1]] == L
        g_l, r_l = grec[gsel], rrec[rsel].copy()
        g_l["frame"] = 0
        st_l = np.zeros_like(st)
        m = np.zeros(st.shape, bool)
        m[:h, :w] = cell_lv == L
        m &= st == 1
        st_l[m] = 1
        ref_l = gout[i].copy()
        ref_l[m] = ref[m]
        pr = parity.compare(ref_l, r_l, gout[i], g_l, st_l, prof.t_phi, prof.t_nu)
        print(f"\nlevel {L}: {int((lv == L).sum())} cells, {len(r_l)} patches: {pr.summary()}")
        assert pr.ok, (L, pr.problems[:5])
        assert len(pr.allowed) == 0
        # the reference decides ~6-11% of these cells' beta at rounding level
        # (measured: 36 of 596 cells at level 0, 5 of 46 at level 40); with its own inputs even those
        # cells stay inside the north_star pixel bar over EVERY lost pixel
        assert len(pr.beta_ties) <= max(2, 0.15 * int((lv == L).sum()))
        assert pr.max_u8_all <= 1 and pr.u8_off_all <= 0.001 * pr.lost_pixels
        total_ties += len(pr.beta_ties)
    print(f"teacher-forced: {total_ties} reference beta ties over {len(levels)} levels")


def test_full_frame_4k_idl_vs_oracle(native):
    """Forced IDL on a whole 4K frame (393 levels) against the oracle: the IDL
    chain is well conditioned, every pixel agrees."""
    import torch

    px, st = make_config(4, frames=1, first=0)
    prof = Profile.sentinel()
    res = conceal_batch(torch.from_numpy(px).cuda(), torch.from_numpy(st).cuda(), prof, forced_layer="IDL",
                        want_f64=True, records=True)
    o_out, o_rec, status, cells = oracle.conceal_dag(px[0].astype(np.float64), st[0], prof.t_phi, prof.t_nu, 10.0, 1)
    assert status == 0 and cells == res.summary["lost_cells"]
    pr = parity.compare(o_out, o_rec, res.recon_f64[0].cpu().numpy(), res.records, st[0], prof.t_phi, prof.t_nu)
    print(f"\ncfg4 4K forced IDL: depth {res.summary['max_level'] + 1} {pr.summary()}")
    assert pr.ok and not pr.beta_ties and pr.max_u8_all == 0


def test_full_frame_4k_hql_free_running(native):
    """The free-running 392-level forced-HQL frame: early levels agree with the
    reference to rounding; the divergence further down is the algorithm's
    amplification (the oracle diverges from the reference the same way)."""
    import torch

    z, px, st, ref = _load("cfg4_f0_random8_forcedHQL")
    res = conceal_batch(torch.from_numpy(px[None]).cuda(), torch.from_numpy(st[None]).cuda(), Profile.sentinel(),
                        forced_layer="HQL", want_f64=True)
    g = res.recon_f64[0].cpu().numpy()
    lv = _levels(st)
    cell_lv = np.repeat(np.repeat(lv, 16, 0), 16, 1)
    h, w = cell_lv.shape
    lost = np.zeros(st.shape, bool)
    lost[:h, :w] = True
    lost &= st == 1
    rel = np.abs(g - ref) / np.maximum(np.abs(ref), 1.0)
    lvl_px = np.full(st.shape, -1)
    lvl_px[:h, :w] = cell_lv
    stats = []
    for L in (0, 5, 10, 20, 40, 80, 160, 320):
        sel = lost & (lvl_px == L)
        if sel.any():
            stats.append((L, float(np.median(rel[sel])), float(rel[sel].max())))
    print("\n4K forced HQL free-running, GPU vs reference, rel diff by level (median, max):",
          ", ".join(f"L{L}: {a:.1e}/{b:.1e}" for L, a, b in stats))
    print(f"  fraction of lost px with rel > 1e-3: {(rel[lost] > 1e-3).mean():.3f} "
          f"(oracle vs reference on the same frame: 0.606, DESIGN.md §5.1)")
    early = lost & (lvl_px >= 0) & (lvl_px <= 10)
    # levels 0-10: agreement to rounding except where a reference beta tie sits
    # (measured: median 4e-15, 2.5% of the pixels > 1e-3)
    assert np.median(rel[early]) <= 1e-12 and (rel[early] > 1e-3).mean() <= 0.05
