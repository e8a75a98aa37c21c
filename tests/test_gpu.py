"""GPU parity and behaviour tests (run on a B200 with -m gpu).

Parity is checked through the public API (conceal_image / conceal_batch /
the C ABI) against (a) the reference's own golden vectors and (b) the CPU
oracle on seeded synthetic inputs at sizes the oracle finishes in seconds,
with the bars of tests/parity.py.  Full-size configs are checked through
size-independent properties (determinism, frame independence, invariants).
"""

import ctypes
import math
from concurrent.futures import ProcessPoolExecutor

import numpy as np
import pytest

import parity
from golden_cases import CASES, load
from oracle import oracle
from paper_2205_11226_b200 import (
    BlockGrid, ImageBuffer, Layer, LossMask, PixelState, Profile, apply_mask, audit_decisions, conceal_batch,
    conceal_image, gen_dispersed_mask, gen_random_mask,
)
from paper_2205_11226_b200 import estimators as est
from paper_2205_11226_b200.records import RECORD_DTYPE
from paper_2205_11226_b200.synth import make_config

pytestmark = pytest.mark.gpu

LAYER_CODE = {None: -1, "BRL": 0, "IDL": 1, "HQL": 2}


def decisions_to_records(decisions):
    recs = np.zeros(len(decisions), dtype=RECORD_DTYPE)
    for i, d in enumerate(decisions):
        r = recs[i]
        r["row"], r["col"] = d.patch_origin
        r["layer"] = LAYER_CODE[None if d.layer is None else d.layer.value]
        r["flags"] = (1 if d.fallback else 0) | (2 if d.deferred_fill else 0)
        r["rings_used"] = d.rings_used
        r["m_candidates"] = -1 if d.m_candidates is None else d.m_candidates
        r["n_y"] = d.n_y
        r["phi"] = math.nan if d.phi is None else d.phi
        r["nu"] = math.nan if d.nu is None else d.nu
        r["beta"] = math.nan if d.beta is None else d.beta
        r["alpha"] = math.nan if d.alpha is None else d.alpha
        r["beta_gap"] = math.nan if d.beta_gap is None else d.beta_gap
    return recs


def profile_from(t_phi, t_nu):
    return Profile("custom", float(t_phi), float(t_nu))


# ------------------------------------------------------------ golden parity


BUILDS = [256, 512, "cluster"]  # the concealment kernel builds (bm_kernels.cuh): CTA widths, 2-CTA clusters


@pytest.mark.parametrize("build", BUILDS)
@pytest.mark.parametrize("name", CASES)
def test_golden_parity(native, name, build):
    z = load(name)
    forced = int(z["forced"])
    layer = None if forced < 0 else ["BRL", "IDL", "HQL"][forced]
    out, rep = conceal_image(ImageBuffer(z["pixels"]), LossMask(z["states"]), profile_from(z["t_phi"], z["t_nu"]),
                             forced_layer=layer, kernel_build=build)
    recs = decisions_to_records(rep.decisions)
    res = parity.compare(z["out"], z["records"], out.pixels, recs, z["states"], float(z["t_phi"]), float(z["t_nu"]))
    assert res.ok, res.problems
    o_out, o_recs, _, _ = oracle.conceal(z["pixels"], z["states"], float(z["t_phi"]), float(z["t_nu"]), 10.0, forced)
    res_o = parity.compare(o_out, o_recs, out.pixels, recs, z["states"], float(z["t_phi"]), float(z["t_nu"]))
    assert res_o.ok, res_o.problems
    assert rep.patches == len(z["records"])


# -------------------------------------------------- configs vs the oracle


def _oracle_frame(args):
    px, st, t_phi, t_nu, forced = args
    return oracle.conceal(px.astype(np.float64), st, t_phi, t_nu, 10.0, forced)


CFG_CASES = [
    # (id, cfg, frames, crop, profile, forced)
    ("cfg1_full", 1, 1, None, "sentinel", None),
    ("cfg2_full", 2, 1, None, "efficient", None),
    ("cfg2_express", 2, 1, (256, 256), "express", None),
    ("cfg2_excellent", 2, 1, (256, 256), "excellent", None),
    ("cfg3_crop", 3, 2, (160, 320), "efficient", None),
    ("cfg4_crop_hql", 4, 2, (96, 128), "sentinel", "HQL"),
    ("cfg4_crop_idl", 4, 2, (128, 128), "sentinel", "IDL"),
    ("cfg5_crop", 5, 3, (128, 256), "efficient", None),
]


# measured excused divergences (threshold decisions + reference beta ties) per case
EXCUSED_MAX = {"cfg1_full": 4, "cfg2_full": 2}


@pytest.mark.parametrize("build", BUILDS)
@pytest.mark.parametrize("case", CFG_CASES, ids=[c[0] for c in CFG_CASES])
def test_config_parity_vs_oracle(native, case, build):
    import torch

    _, cfg, nf, crop, prof_name, forced = case
    prof = Profile.sentinel() if prof_name == "sentinel" else Profile.named(prof_name)
    if cfg == 3:  # crop a band around the first lost macroblock rows of each frame
        fpx, fst = make_config(cfg, frames=nf)
        px = np.empty((nf,) + crop, np.uint8)
        st = np.empty((nf,) + crop, np.uint8)
        for f in range(nf):
            r = int(np.argmax((fst[f] == 1).any(axis=1)))
            r0 = max(0, min(r - 32, fst.shape[1] - crop[0])) // 16 * 16
            px[f], st[f] = fpx[f, r0 : r0 + crop[0], : crop[1]], fst[f, r0 : r0 + crop[0], : crop[1]]
        assert (st == 1).any()
    else:
        px, st = make_config(cfg, frames=nf, crop=crop)
    fcode = -1 if forced is None else LAYER_CODE[forced]
    res = conceal_batch(torch.from_numpy(px).cuda(), torch.from_numpy(st).cuda(), prof, forced_layer=forced,
                        want_f64=True, records=True, kernel_build=build)
    gout = res.recon_f64.cpu().numpy()
    grec = res.records
    with ProcessPoolExecutor(max_workers=min(nf, 8)) as ex:
        outs = list(ex.map(_oracle_frame, [(px[f], st[f], prof.t_phi, prof.t_nu, fcode) for f in range(nf)]))
    o_out = np.stack([o[0] for o in outs])
    o_rec = []
    for f, o in enumerate(outs):
        r = o[1].copy()
        r["frame"] = f
        o_rec.append(r)
    o_rec = np.concatenate(o_rec)
    pr = parity.compare(o_out, o_rec, gout, grec, st, prof.t_phi, prof.t_nu)
    assert pr.ok, pr.problems[:5]
    print(case[0], build, pr.summary())
    # excused divergences per case, bounded by the measured counts (DESIGN.md
    # §5): layer decisions at a threshold and the reference's rounding-decided
    # beta choices; everything else must match exactly
    excused = len(pr.allowed) + len(pr.beta_ties)
    assert excused <= EXCUSED_MAX.get(case[0], 0), (pr.allowed, pr.beta_ties)
    assert res.summary["patches"] == len(o_rec)


# ------------------------------------------------ reference behaviours


def stripes(size=48, period=2):
    cols = np.arange(size) % period
    return ImageBuffer(np.tile(np.where(cols == 0, 0.0, 200.0), (size, 1)))


def one_lost_block(size=48):
    return gen_dispersed_mask(BlockGrid(size, size))


def test_flat_block_all_brl(native):
    img = ImageBuffer(np.full((48, 48), 77.0))
    mask = one_lost_block()
    out, rep = conceal_image(apply_mask(img, mask), mask, Profile.named("express"))
    assert np.array_equal(out.pixels, img.pixels)
    assert rep.layer_counts == {"BRL": 64, "IDL": 0, "HQL": 0}


def test_periodic_texture_exact_idl(native):
    mask = one_lost_block()
    for img in (stripes(), ImageBuffer(stripes().pixels.T)):
        out, rep = conceal_image(apply_mask(img, mask), mask, Profile.named("express"))
        assert np.array_equal(out.quantized(), img.quantized())
        assert rep.layer_counts["IDL"] == 64


def test_total_loss_defers_then_fills(native):
    img = ImageBuffer(np.full((48, 48), 50.0))
    mask = gen_random_mask(BlockGrid(48, 48), 1.0, 0)
    out, rep = conceal_image(apply_mask(img, mask), mask, Profile.named("express"))
    assert rep.deferred_fills > 0
    assert (out.pixels[:16, :16] == 128.0).all()
    assert np.isfinite(out.pixels).all()


def test_inputs_unmodified_and_identity(native):
    img = ImageBuffer(np.arange(48 * 48, dtype=float).reshape(48, 48) % 251)
    out, rep = conceal_image(img, LossMask.all_available(48, 48), Profile.named("efficient"))
    assert np.array_equal(out.pixels, img.pixels) and rep.patches == 0
    mask = one_lost_block()
    corrupted = apply_mask(img, mask)
    before, sb = corrupted.pixels.copy(), mask.states.copy()
    conceal_image(corrupted, mask, Profile.named("express"))
    assert np.array_equal(corrupted.pixels, before) and np.array_equal(mask.states, sb)


def test_sentinel_equals_forced_hql(native):
    px, st = make_config(2, frames=1, crop=(128, 128))
    img, mask = ImageBuffer(px[0].astype(float)), LossMask(st[0])
    a, ra = conceal_image(img, mask, Profile.sentinel())
    b, rb = conceal_image(img, mask, Profile.sentinel(), forced_layer=Layer.HQL)
    assert np.array_equal(a.pixels, b.pixels)
    assert [d.beta for d in ra.decisions] == [d.beta for d in rb.decisions]


def test_forced_layers_and_audit(native):
    px, st = make_config(5, frames=1, crop=(96, 96))
    img, mask = ImageBuffer(px[0].astype(float)), LossMask(st[0])
    for layer in (Layer.BRL, Layer.IDL, Layer.HQL):
        out, rep = conceal_image(img, mask, Profile.sentinel(), forced_layer=layer)
        assert rep.layer_counts[layer.value] + sum(d.fallback for d in rep.decisions) >= rep.patches - rep.deferred_fills
    for name in ("express", "efficient", "excellent"):
        prof = Profile.named(name)
        _, rep = conceal_image(img, mask, prof)
        assert audit_decisions(rep.decisions, prof) == []


def test_lost_left_and_bad_states(native):
    img = ImageBuffer(np.full((20, 20), 5.0))
    st = np.zeros((20, 20), np.uint8)
    st[18, 18] = PixelState.LOST
    with pytest.raises(AssertionError):
        conceal_image(img, LossMask(st), Profile.named("express"))
    import torch

    bad = torch.zeros((1, 32, 32), dtype=torch.uint8, device="cuda")
    bad[0, 3, 3] = 7
    with pytest.raises(ValueError):
        conceal_batch(torch.zeros((1, 32, 32), dtype=torch.uint8, device="cuda"), bad, Profile.named("express"))


@pytest.mark.parametrize("shape", [(10, 10), (12, 40), (40, 15), (1, 1)])
def test_frames_smaller_than_one_cell(native, shape):
    """No full 16x16 cell: the reference returns the image unchanged when no
    pixel is LOST and raises AssertionError otherwise (profiles.py:305); bad
    state values raise ValueError (image.py:69-70) - also without cells."""
    import torch

    img = ImageBuffer(np.arange(shape[0] * shape[1], dtype=np.float64).reshape(shape) % 251)
    out, rep = conceal_image(img, LossMask(np.zeros(shape, np.uint8)), Profile.named("efficient"))
    assert np.array_equal(out.pixels, img.pixels) and rep.patches == 0 and rep.decisions == []
    st = np.zeros(shape, np.uint8)
    st[shape[0] // 2, shape[1] // 2] = PixelState.LOST
    with pytest.raises(AssertionError):
        conceal_image(img, LossMask(st), Profile.named("efficient"))
    bad = torch.zeros((1,) + shape, dtype=torch.uint8, device="cuda")
    bad[0, 0, 0] = 9
    with pytest.raises(ValueError):
        conceal_batch(torch.zeros((1,) + shape, dtype=torch.uint8, device="cuda"), bad, Profile.named("express"))


def test_concurrent_calls_are_independent(native):
    """conceal_image is a pure function, safe to call from several threads at
    once: per-call workspaces, no shared result buffers."""
    from concurrent.futures import ThreadPoolExecutor

    cases = []
    for seed, rate in ((3, 0.3), (4, 0.2), (5, 0.4), (6, 0.25)):
        px, st = make_config(2, frames=1, crop=(96, 128), first=seed)
        cases.append((ImageBuffer(px[0].astype(np.float64)), LossMask(st[0])))
    prof = Profile.named("efficient")
    serial = [conceal_image(img, m, prof) for img, m in cases]

    def run(i):
        img, m = cases[i % len(cases)]
        return i % len(cases), conceal_image(img, m, prof)

    with ThreadPoolExecutor(8) as ex:
        results = list(ex.map(run, range(16)))
    for i, (out, rep) in results:
        s_out, s_rep = serial[i]
        assert np.array_equal(out.pixels, s_out.pixels)
        assert [(d.patch_origin, d.layer, d.beta) for d in rep.decisions] == \
            [(d.patch_origin, d.layer, d.beta) for d in s_rep.decisions]


# --------------------------------------------- full-size properties


def test_full_size_determinism_and_frame_independence(native):
    import torch

    px, st = make_config(5, frames=6)  # 6 full 1080p frames: dispersed, slice, random16 x2
    tp, ts = torch.from_numpy(px).cuda(), torch.from_numpy(st).cuda()
    prof = Profile.named("efficient")
    a = conceal_batch(tp, ts, prof, want_f64=True)
    b = conceal_batch(tp, ts, prof, want_f64=True)
    assert torch.equal(a.recon_f64, b.recon_f64) and torch.equal(a.recon_u8, b.recon_u8)
    assert a.summary["lost_left"] == 0 and a.summary["lost_cells"] > 0
    s = a.summary
    assert s["patches"] == sum(s["layer_counts"].values()) + s["deferred_fills"]
    # frame 4 alone == frame 4 inside the batch (frames are independent) for a
    # fixed kernel build (the default build is chosen from the batch's DAG
    # shape, and the two builds' FP64 reduction orders differ in the last bits)
    for build in BUILDS:
        full = conceal_batch(tp, ts, prof, want_f64=True, kernel_build=build)
        c = conceal_batch(tp[4:5], ts[4:5], prof, want_f64=True, kernel_build=build)
        assert torch.equal(c.recon_f64[0], full.recon_f64[4])
    # non-lost pixels untouched; u8 is the half-up quantization of f64
    lost = ts == PixelState.LOST
    assert torch.equal(a.recon_u8[~lost], tp[~lost])
    q = torch.floor(torch.clamp(a.recon_f64, 0, 255) + 0.5).to(torch.uint8)
    assert torch.equal(q, a.recon_u8)
    assert s["max_level"] >= 100  # the slice frame chains ~120 cells
    # each forced kernel build is deterministic and keeps the same properties
    for build in BUILDS:
        x = conceal_batch(tp, ts, prof, want_f64=True, kernel_build=build)
        y = conceal_batch(tp, ts, prof, want_f64=True, kernel_build=build)
        assert torch.equal(x.recon_f64, y.recon_f64)
        assert x.summary["layer_counts"] == y.summary["layer_counts"]
        assert torch.equal(x.recon_u8[~lost], tp[~lost])


def test_host_abi_matches_device_path(native):
    import torch

    from paper_2205_11226_b200 import _native
    from paper_2205_11226_b200.profiles import make_params

    px, st = make_config(3, frames=1, crop=(128, 256))
    prof = Profile.named("efficient")
    dev = conceal_batch(torch.from_numpy(px).cuda(), torch.from_numpy(st).cuda(), prof)
    out = np.empty_like(px)
    summ = _native.Summary()
    params = make_params(1, 128, 256, 0, prof, 10.0, None)
    rc = native.bm_conceal_host(params, px.ctypes.data, st.ctypes.data, None, out.ctypes.data, None, None,
                                ctypes.byref(summ))
    _native.check(rc)
    assert np.array_equal(out, dev.recon_u8.cpu().numpy())
    assert summ.lost_cells == dev.summary["lost_cells"]


# ------------------------------------------------------------ estimators


def _instances(rng, count, m_range, n_range, spread):
    ts, cs = [], []
    for _ in range(count):
        m, n = int(rng.integers(*m_range)), int(rng.integers(*n_range))
        y0 = rng.uniform(0, spread, n)
        ts.append(est.TargetContext((0, 0), np.ones(32, bool), y0, n))
        cs.append(est.CandidateSet(rng.uniform(0, spread, (m, 4)), rng.uniform(0, spread, (m, n))))
    return ts, cs


def test_hql_estimates_vs_oracle(native):
    rng = np.random.default_rng(5)
    ts, cs = _instances(rng, 24, (2, 400), (1, 33), 255)
    ts2, cs2 = _instances(rng, 4, (1500, 1850), (32, 33), 255)
    ts += ts2
    cs += cs2
    got = est.estimate_batch(Layer.HQL, ts, cs)
    for t, c, g in zip(ts, cs, got):
        vals, info = oracle.hql(t.y0, c.x, c.y)
        assert g.layer.value == ["BRL", "IDL", "HQL"][info["layer"]]
        if g.layer is Layer.HQL:
            if g.diagnostics.bandwidth.beta != info["beta"]:
                assert info["beta_gap"] < parity.BETA_TIE  # rounding-decided grid near-tie
                continue
            assert abs(g.diagnostics.bandwidth.alpha - info["alpha"]) < 1e-7
        assert np.allclose(g.values, vals, rtol=1e-9, atol=1e-9)


def test_idl_brl_estimates(native):
    t = est.TargetContext((0, 0), np.ones(32, bool), np.zeros(4), 4)
    c = est.CandidateSet(np.zeros((1, 4)), np.full((1, 4), math.sqrt(20.0)))
    e = est.idl_estimate(t, c, sigma2=10.0)
    assert abs(e.diagnostics.nu - math.exp(-1.0)) < 1e-12
    rng = np.random.default_rng(3)
    ts, cs = _instances(rng, 16, (1, 300), (1, 33), 255)
    got = est.estimate_batch(Layer.IDL, ts, cs)
    for t, c, g in zip(ts, cs, got):
        vals, raw = oracle.idl(t.y0, c.x, c.y)
        if vals is None:
            assert g.layer is Layer.BRL and g.diagnostics.fallback
        else:
            assert np.allclose(g.values, vals, rtol=1e-12, atol=1e-10)
            assert abs(g.diagnostics.nu - raw) <= 1e-12 * max(raw, 1e-300)
    b = est.brl_estimate(est.TargetContext((0, 0), np.ones(32, bool), np.array([0.0, 255.0]), 2))
    assert b.values.tolist() == [127.5] * 4
    h = est.hql_estimate(est.TargetContext((0, 0), np.ones(32, bool), np.array([10.0, 20.0]), 2),
                         est.CandidateSet(np.zeros((0, 4)), np.zeros((0, 2))))
    assert h.layer is Layer.BRL and h.diagnostics.fallback and np.allclose(h.values, 15.0)
