"""Estimator layer API on the GPU (reference: blockmend/estimators.py).

Constants and types mirror the reference; brl/idl/hql_estimate run the same
device code the fused concealment kernel uses, through bm_estimate_batch
(dense instances, one CTA per instance).  `estimate_batch` is the batched
entry; the single-instance functions keep the reference signatures
(estimators.py:96-132, 248-286).
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import EmptyContextError, InsufficientCandidatesError, WeightUnderflowError

DEFAULT_SIGMA2 = 10.0
BETA_GRID = 2.0 ** np.arange(-8, 13)
RIDGE_SCALE = 1e-6
ALPHA_MIN = 0.0
ALPHA_MAX = 4.0
MAX_CANDIDATES = 2048


class Layer(str, enum.Enum):
    BRL = "BRL"
    IDL = "IDL"
    HQL = "HQL"


LAYER_CODE = {Layer.BRL: 0, Layer.IDL: 1, Layer.HQL: 2}
CODE_LAYER = {0: Layer.BRL, 1: Layer.IDL, 2: Layer.HQL}


@dataclass
class TargetContext:
    patch_origin: tuple[int, int]
    layout_usable: np.ndarray
    y0: np.ndarray
    n_y: int
    n_x: int = 4


@dataclass
class CandidateSet:
    x: np.ndarray  # (M', 4)
    y: np.ndarray  # (M', N_y)
    ring_index: int = 0
    exhausted: bool = True

    @property
    def m_current(self) -> int:
        return self.x.shape[0]


@dataclass
class BandwidthParams:
    beta: float | None
    alpha: float | None
    sigma2: float | None


@dataclass
class EstimateDiagnostics:
    phi: float | None = None
    nu: float | None = None
    m_candidates: int | None = None
    rings_used: int | None = None
    bandwidth: BandwidthParams | None = None
    elapsed_s: float | None = None
    fallback: bool = False
    beta_gap: float | None = None


@dataclass
class PatchEstimate:
    values: np.ndarray
    layer: Layer
    diagnostics: EstimateDiagnostics = field(default_factory=EstimateDiagnostics)


def _estimate_batch(layer: Layer, targets, csets, sigma2: float) -> list[PatchEstimate]:
    torch = _native.require_cuda()
    from .records import RECORD_DTYPE, decode_flags

    count = len(targets)
    if count == 0:
        return []
    max_m = max(1, max(c.x.shape[0] for c in csets))
    if max_m > MAX_CANDIDATES:
        raise ValueError(f"at most {MAX_CANDIDATES} candidates per instance")
    n_y = np.zeros(count, np.int32)
    m = np.zeros(count, np.int32)
    y0 = np.zeros((count, 32))
    x = np.zeros((count, max_m, 4))
    y = np.zeros((count, max_m, 32))
    for i, (t, c) in enumerate(zip(targets, csets)):
        n = int(t.n_y)
        if not 1 <= n <= 32:
            raise EmptyContextError("estimators need 1..32 context samples")
        n_y[i] = n
        m[i] = c.x.shape[0]
        y0[i, :n] = t.y0
        if m[i]:
            x[i, : m[i]] = c.x
            y[i, : m[i], :n] = c.y
    dev = torch.device("cuda")
    tn = torch.from_numpy(n_y).to(dev)
    tm = torch.from_numpy(m).to(dev)
    ty0 = torch.from_numpy(y0).to(dev)
    tx = torch.from_numpy(x).to(dev)
    ty = torch.from_numpy(y).to(dev)
    out = torch.empty((count, 4), dtype=torch.float64, device=dev)
    info = torch.empty((count, RECORD_DTYPE.itemsize), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream().cuda_stream
    _native.check(
        _native.lib().bm_estimate_batch(
            LAYER_CODE[layer], count, max_m, float(sigma2), tn.data_ptr(), tm.data_ptr(), ty0.data_ptr(),
            tx.data_ptr(), ty.data_ptr(), out.data_ptr(), info.data_ptr(), stream,
        )
    )
    torch.cuda.synchronize()
    vals = out.cpu().numpy()
    recs = info.cpu().numpy().view(RECORD_DTYPE).reshape(-1)
    res = []
    for i in range(count):
        r = recs[i]
        f = decode_flags(r)
        lay = CODE_LAYER[int(r["layer"])]
        bw = None
        if lay is Layer.HQL:
            bw = BandwidthParams(float(r["beta"]), float(r["alpha"]), None)
        elif lay is Layer.IDL:
            bw = BandwidthParams(None, None, sigma2)
        diag = EstimateDiagnostics(
            nu=float(r["nu"]) if f["has_nu"] else None,
            m_candidates=int(r["m_candidates"]),
            bandwidth=bw,
            fallback=f["fallback"],
            beta_gap=float(r["beta_gap"]) if lay is Layer.HQL else None,
        )
        res.append(PatchEstimate(vals[i].copy(), lay, diag))
    return res


def estimate_batch(layer: Layer, targets, csets, sigma2: float = DEFAULT_SIGMA2) -> list[PatchEstimate]:
    """Run one layer (with its degradation ladder) on many instances at once."""
    return _estimate_batch(Layer(layer), targets, csets, sigma2)


def brl_estimate(target) -> PatchEstimate:
    """brl_estimate (estimators.py:96-102) on the GPU."""
    if target.n_y < 1:
        raise EmptyContextError("BRL needs at least one context sample")
    empty = CandidateSet(np.zeros((0, 4)), np.zeros((0, target.n_y)))
    est = _estimate_batch(Layer.BRL, [target], [empty], DEFAULT_SIGMA2)[0]
    est.diagnostics.m_candidates = 0
    est.diagnostics.fallback = False
    return est


def idl_estimate(target, cset, sigma2: float = DEFAULT_SIGMA2) -> PatchEstimate:
    """idl_estimate (estimators.py:122-132) on the GPU (FP32 weights)."""
    if cset.x.shape[0] < 1:
        raise InsufficientCandidatesError("IDL needs at least one candidate")
    est = _estimate_batch(Layer.IDL, [target], [cset], sigma2)[0]
    if est.layer is not Layer.IDL:
        raise WeightUnderflowError("all IDL weights underflowed (nu = 0)")
    return est


def hql_estimate(target, cset, sigma2: float = DEFAULT_SIGMA2) -> PatchEstimate:
    """hql_estimate with its HQL -> IDL -> BRL ladder (estimators.py:248-286)."""
    return _estimate_batch(Layer.HQL, [target], [cset], sigma2)[0]
