"""Profiles, layer decisions and the concealment driver (drop-in for
blockmend/profiles.py).

`conceal_image` keeps the reference signature and contract
(profiles.py:263-323): inputs untouched, deterministic, (ImageBuffer,
ConcealmentReport) returned, decisions in (lost cell raster, schedule) order.
Below it the whole driver — cell enumeration, the cross-cell raster
dependency order, the per-cell patch chain, the layer gate and the
estimators — runs on the GPU in one bm_conceal call (csrc/bm_conceal.cu).
`conceal_batch` is the tensor entry for B frames already on the device.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np

from . import _native
from .estimators import CODE_LAYER, DEFAULT_SIGMA2, LAYER_CODE, Layer
from .image import BLOCK_SIZE, ImageBuffer, LossMask, require_same_shape
from .metrics import ConcealmentReport
from .records import RECORD_DTYPE, decode_flags

PROFILE_TABLE = {
    "express": (20.0, 0.01),
    "efficient": (20.0, 0.1),
    "excellent": (20.0, 100.0),
}

DEFERRED_FILL_VALUE = 128.0


@dataclass(frozen=True)
class Profile:
    """Threshold pair controlling layer selection (profiles.py:49-78)."""

    name: str
    t_phi: float
    t_nu: float

    def __post_init__(self):
        if not self.t_nu > 0.0:
            raise ValueError(f"T_nu must be positive, got {self.t_nu}")

    @classmethod
    def named(cls, name: str) -> "Profile":
        try:
            t_phi, t_nu = PROFILE_TABLE[name]
        except KeyError:
            raise ValueError(f"unknown profile {name!r}; choose from {sorted(PROFILE_TABLE)}")
        return cls(name, t_phi, t_nu)

    @classmethod
    def custom(cls, t_phi: float, t_nu: float) -> "Profile":
        if t_phi < 0.0:
            raise ValueError(f"T_phi must be non-negative, got {t_phi}")
        return cls("custom", t_phi, t_nu)

    @classmethod
    def sentinel(cls) -> "Profile":
        """Thresholds that force the full pipeline on every patch."""
        return cls("custom", -1.0, math.inf)


@dataclass
class LayerDecision:
    """Outcome of the layer selection for one patch (profiles.py:81-95)."""

    patch_origin: tuple[int, int]
    layer: Layer | None
    phi: float | None
    nu: float | None
    rings_used: int
    m_candidates: int | None = None
    beta: float | None = None
    alpha: float | None = None
    elapsed_s: float = 0.0
    fallback: bool = False
    deferred_fill: bool = False
    n_y: int = 0
    beta_gap: float | None = None


def flatness(target) -> float:
    """Dynamic range of the usable context (profiles.py:98-102)."""
    from .errors import EmptyContextError

    if target.n_y < 1:
        raise EmptyContextError("flatness needs at least one context sample")
    return float(np.max(target.y0) - np.min(target.y0))


def audit_decisions(decisions, profile: Profile) -> list[str]:
    """Check every recorded decision against its defining predicate (profiles.py:326-340)."""
    problems = []
    for d in decisions:
        if d.deferred_fill or d.fallback:
            continue
        if d.layer is Layer.BRL and not d.phi <= profile.t_phi:
            problems.append(f"{d.patch_origin}: BRL with phi={d.phi} > {profile.t_phi}")
        elif d.layer is Layer.IDL and not d.nu >= profile.t_nu:
            problems.append(f"{d.patch_origin}: IDL with nu={d.nu} < {profile.t_nu}")
        elif d.layer is Layer.HQL and not (d.phi > profile.t_phi and d.nu < profile.t_nu):
            problems.append(f"{d.patch_origin}: HQL with phi={d.phi}, nu={d.nu}")
    return problems


# ------------------------------------------------------------------ batch API


@dataclass
class BatchResult:
    """Outputs of conceal_batch (device tensors unless noted)."""

    recon_u8: object | None  # torch.uint8 [B,H,W]
    recon_f64: object | None  # torch.float64 [B,H,W]
    summary: dict  # host: lost_cells, patches, layer_counts, deferred_fills, lost_left, max_level
    records: np.ndarray | None  # host RECORD_DTYPE array in the reference's decision order


def _workspace(torch, params, device, want_records):
    """Per-call device buffers (workspace, summary, record slots).

    Allocated from torch's caching allocator on the call's stream, so repeated
    calls reuse the same memory without a module-global buffer: concurrent
    calls (threads, streams, devices) never share a workspace, which keeps
    conceal_batch / conceal_image reentrant like the reference's pure
    function.
    """
    lib = _native.lib()
    nbytes = int(lib.bm_workspace_bytes(params))
    buf = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device)
    summary = torch.zeros(_native.SUMMARY_BYTES, dtype=torch.uint8, device=device)
    rec = rec2 = None
    if want_records:
        # at least one record slot: frames smaller than one 16x16 cell have none
        nrec = max(1, int(lib.bm_max_records(params)))
        rec = torch.empty(nrec * RECORD_DTYPE.itemsize, dtype=torch.uint8, device=device)
        rec2 = torch.empty_like(rec)
    return nbytes, buf, summary, rec, rec2


def make_params(frames, height, width, pixel_dtype, profile, sigma2, forced_layer) -> _native.Params:
    p = _native.Params()
    p.frames, p.height, p.width = int(frames), int(height), int(width)
    p.pixel_dtype = pixel_dtype
    p.t_phi = float(profile.t_phi)
    p.t_nu = float(profile.t_nu)
    p.sigma2 = float(sigma2)
    p.forced_layer = -1 if forced_layer is None else LAYER_CODE[Layer(forced_layer)]
    p.flags = 0
    return p


def conceal_batch(
    frames,
    states,
    profile: Profile,
    *,
    sigma2: float = DEFAULT_SIGMA2,
    forced_layer: Layer | None = None,
    want_u8: bool = True,
    want_f64: bool = False,
    records: bool = False,
    out_u8=None,
    sync: bool = True,
    time_kernel: bool = False,
    kernel_build: int | None = None,
) -> BatchResult:
    """Conceal B frames resident on the GPU.

    frames: torch.uint8 or torch.float64 [B,H,W] (cuda); states: torch.uint8
    [B,H,W] (cuda, values in {0,1,2}).  Runs asynchronously on torch's current
    stream; with sync=True the summary is read back (raising the reference's
    errors for leftover LOST pixels / bad states).  kernel_build: None picks
    the build from the dependency DAG's shape; 256, 512 or 'cluster' (2-CTA
    clusters of 512 threads per cell) forces one, 'narrow512' keeps the
    512-thread build for narrow DAGs (all meet the parity bar; their FP64
    reduction orders differ, so results can differ in the last bits).
    """
    torch = _native.require_cuda()
    if frames.dim() == 2:
        frames = frames[None]
    if states.dim() == 2:
        states = states[None]
    if tuple(frames.shape) != tuple(states.shape):
        from .errors import DimensionMismatchError

        raise DimensionMismatchError(f"shape mismatch: {tuple(frames.shape)} vs {tuple(states.shape)}")
    if not frames.is_cuda or not states.is_cuda:
        raise ValueError("conceal_batch expects CUDA tensors (use conceal_image for host arrays)")
    if frames.dtype == torch.uint8:
        pix_dtype = 0
    else:
        if frames.dtype != torch.float64:
            frames = frames.to(torch.float64)
        pix_dtype = 1
    frames = frames.contiguous()
    states = states.to(torch.uint8).contiguous()
    b, h, w = frames.shape
    params = make_params(b, h, w, pix_dtype, profile, sigma2, forced_layer)
    if time_kernel:
        params.flags |= _native.BM_FLAG_TIME_KERNEL
    if kernel_build is not None:
        flag = {256: _native.BM_FLAG_BUILD_256, 512: _native.BM_FLAG_BUILD_512,
                "cluster": _native.BM_FLAG_BUILD_CLUSTER, "narrow512": _native.BM_FLAG_NARROW_512}.get(kernel_build)
        if flag is None:
            raise ValueError("kernel_build must be None, 256, 512, 'cluster' or 'narrow512'")
        params.flags |= flag
    dev = frames.device
    with torch.cuda.device(dev):  # the C ABI works on the current device
        nbytes, ws, summ_buf, rec, rec2 = _workspace(torch, params, dev, records)
        u8 = None
        if want_u8:
            u8 = out_u8 if out_u8 is not None else torch.empty((b, h, w), dtype=torch.uint8, device=dev)
        f64 = torch.empty((b, h, w), dtype=torch.float64, device=dev) if want_f64 else None
        stream = torch.cuda.current_stream(dev).cuda_stream
        lib = _native.lib()
        _native.check(
            lib.bm_conceal(
                params, frames.data_ptr(), states.data_ptr(), f64.data_ptr() if f64 is not None else None,
                u8.data_ptr() if u8 is not None else None, rec.data_ptr() if records else None,
                summ_buf.data_ptr(), ws.data_ptr(), nbytes, stream,
            )
        )
        summary = None
        recs = None
        if sync or records:
            raw = summ_buf.cpu().numpy().tobytes()
            s = _native.Summary.from_buffer_copy(raw)
            summary = {
                "lost_cells": int(s.lost_cells),
                "patches": int(s.patches),
                "layer_counts": {"BRL": int(s.layer_counts[0]), "IDL": int(s.layer_counts[1]),
                                 "HQL": int(s.layer_counts[2])},
                "deferred_fills": int(s.deferred_fills),
                "lost_left": int(s.lost_left),
                "max_level": int(s.max_level),
                "bad_states": int(s.bad_states),
                "flop64": int(s.flop64),
                "flop32": int(s.flop32),
                "hql_patches": int(s.hql_patches),
                "gate_candidates": int(s.gate_candidates),
                "kernel_build": {256: "256", 512: "512", 1024: "cluster"}.get(int(s.kernel_build)),
            }
            if s.bad_states:
                _native.check(_native.BM_ERR_STATES)
            if s.lost_left:
                _native.check(_native.BM_ERR_LOST_LEFT)
            if records:
                import ctypes

                cnt = ctypes.c_int64(0)
                _native.check(lib.bm_compact_records(params, rec.data_ptr(), ws.data_ptr(), rec2.data_ptr(),
                                                     ctypes.byref(cnt), stream))
                n = int(cnt.value)
                recs = rec2[: n * RECORD_DTYPE.itemsize].cpu().numpy().view(RECORD_DTYPE).copy()
    return BatchResult(u8, f64, summary, recs)


def decisions_from_records(recs: np.ndarray, clock_khz: int) -> list[LayerDecision]:
    hz = max(1, clock_khz) * 1e3
    out = []
    for r in recs:
        f = decode_flags(r)
        if f["deferred"]:
            out.append(LayerDecision((int(r["row"]), int(r["col"])), None, None, None, 0, deferred_fill=True))
            continue
        has_bw = f["has_bw"]
        out.append(
            LayerDecision(
                patch_origin=(int(r["row"]), int(r["col"])),
                layer=CODE_LAYER[int(r["layer"])],
                phi=float(r["phi"]) if f["has_phi"] else None,
                nu=float(r["nu"]) if f["has_nu"] else None,
                rings_used=int(r["rings_used"]),
                m_candidates=int(r["m_candidates"]) if f["has_m"] else None,
                beta=float(r["beta"]) if has_bw else None,
                alpha=float(r["alpha"]) if has_bw else None,
                elapsed_s=float(r["cycles"]) / hz,
                fallback=f["fallback"],
                n_y=int(r["n_y"]),
                beta_gap=float(r["beta_gap"]) if has_bw else None,
            )
        )
    return out


def select_and_estimate_batch(img, mask, targets, profile: Profile, sigma2: float = DEFAULT_SIGMA2, *,
                              forced_layer: Layer | None = None) -> list:
    """select_and_estimate (or _forced_estimate with forced_layer) for many
    patches of one working image in one device call (bm_select_and_estimate:
    the fused kernel's patch step, one CTA per patch, no write-back)."""
    from .errors import EmptyContextError
    from .estimators import BandwidthParams, EstimateDiagnostics, PatchEstimate

    if not targets:
        return []
    for t in targets:
        if t.n_y < 1:
            raise EmptyContextError("flatness needs at least one context sample")
    torch = _native.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    pixels = np.asarray(img.pixels if isinstance(img, ImageBuffer) else img, dtype=np.float64)
    states = np.asarray(mask.states if isinstance(mask, LossMask) else mask, dtype=np.uint8)
    require_same_shape(pixels, states)
    n = len(targets)
    origins = np.array([t.patch_origin for t in targets], dtype=np.int32).reshape(n, 2)
    layouts = np.array([t.layout_bits() for t in targets], dtype=np.uint32)
    y0 = np.zeros((n, 32))
    for i, t in enumerate(targets):
        y0[i, : t.n_y] = t.y0
    h, w = pixels.shape
    params = make_params(1, h, w, 1, profile, sigma2, forced_layer)

    def put(a):
        return torch.from_numpy(np.ascontiguousarray(a)).to(dev)

    t_px, t_st, t_o, t_l, t_y = put(pixels), put(states), put(origins), put(layouts.view(np.int32)), put(y0)
    vals = torch.empty((n, 4), dtype=torch.float64, device=dev)
    rec = torch.empty((n, RECORD_DTYPE.itemsize), dtype=torch.uint8, device=dev)
    _native.check(_native.lib().bm_select_and_estimate(
        params, t_px.data_ptr(), t_st.data_ptr(), n, t_o.data_ptr(), t_l.data_ptr(), t_y.data_ptr(),
        vals.data_ptr(), rec.data_ptr(), torch.cuda.current_stream(dev).cuda_stream))
    vals = vals.cpu().numpy()
    recs = rec.cpu().numpy().view(RECORD_DTYPE).reshape(-1)
    hz = max(1, int(_native.lib().bm_device_clock_khz())) * 1e3
    out = []
    for i in range(n):
        r = recs[i]
        f = decode_flags(r)
        layer = CODE_LAYER[int(r["layer"])]
        bw = None
        if f["has_bw"]:
            bw = BandwidthParams(float(r["beta"]), float(r["alpha"]), None)
        elif layer is Layer.IDL:
            bw = BandwidthParams(None, None, sigma2)
        diag = EstimateDiagnostics(
            phi=float(r["phi"]) if f["has_phi"] else None,
            nu=float(r["nu"]) if f["has_nu"] else None,
            m_candidates=int(r["m_candidates"]) if f["has_m"] else None,
            rings_used=int(r["rings_used"]),
            bandwidth=bw,
            elapsed_s=float(r["cycles"]) / hz,
            fallback=f["fallback"],
            beta_gap=float(r["beta_gap"]) if f["has_bw"] else None,
        )
        out.append(PatchEstimate(vals[i].copy(), layer, diag))
    return out


def select_and_estimate(img, mask, target, profile: Profile, sigma2: float = DEFAULT_SIGMA2):
    """Pick and run the cheapest suitable layer for one patch (profiles.py:105-133):
    phi <= T_phi -> BRL; else the ring-by-ring support expansion with the
    cumulative nu; nu >= T_nu -> IDL, else HQL with its ladder."""
    return select_and_estimate_batch(img, mask, [target], profile, sigma2)[0]


def conceal_image(
    img: ImageBuffer,
    mask: LossMask,
    profile: Profile,
    *,
    sigma2: float = DEFAULT_SIGMA2,
    forced_layer: Layer | None = None,
    parallel_blocks: bool = False,
    kernel_build: int | None = None,
) -> tuple[ImageBuffer, ConcealmentReport]:
    """Reconstruct every lost pixel (drop-in for blockmend.conceal_image).

    `parallel_blocks` is accepted for API compatibility; the GPU schedule is
    always concurrent across independent cells and bit-equivalent to the
    serial raster order (profiles.py:285-302).  kernel_build (B200-specific,
    keyword-only): see conceal_batch.
    """
    del parallel_blocks
    pixels = img.pixels if isinstance(img, ImageBuffer) else np.asarray(img, dtype=np.float64)
    states = mask.states if isinstance(mask, LossMask) else np.asarray(mask, dtype=np.uint8)
    require_same_shape(pixels, states)
    torch = _native.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    px = torch.from_numpy(np.array(pixels, dtype=np.float64, copy=True)).to(dev)
    st = torch.from_numpy(np.array(states, dtype=np.uint8, copy=True)).to(dev)
    t0 = time.perf_counter()
    res = conceal_batch(px, st, profile, sigma2=sigma2, forced_layer=forced_layer, want_u8=False,
                        want_f64=True, records=True, kernel_build=kernel_build)
    out = res.recon_f64[0].cpu().numpy()
    total = time.perf_counter() - t0
    decisions = decisions_from_records(res.records, int(_native.lib().bm_device_clock_khz()))
    counts = {layer.value: 0 for layer in Layer}
    deferred = 0
    times = []
    for d in decisions:
        if d.deferred_fill:
            deferred += 1
        else:
            counts[d.layer.value] += 1
            times.append(d.elapsed_s)
    report = ConcealmentReport(counts, times, total, deferred, decisions)
    return ImageBuffer(out), report


__all__ = [
    "PROFILE_TABLE",
    "DEFERRED_FILL_VALUE",
    "BLOCK_SIZE",
    "Profile",
    "LayerDecision",
    "BatchResult",
    "flatness",
    "audit_decisions",
    "conceal_batch",
    "conceal_image",
    "decisions_from_records",
    "make_params",
    "select_and_estimate",
    "select_and_estimate_batch",
]
