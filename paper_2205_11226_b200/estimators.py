"""Estimator layer API on the GPU (drop-in for blockmend/estimators.py).

Constants and types mirror the reference.  Two device back ends:
  * brl/idl/hql_estimate and `estimate_batch` run the same device code the
    fused concealment kernel uses (bm_estimate_batch: the DMMA HQL pipeline
    with its degradation ladder, one CTA per instance);
  * the stage functions a library user composes by hand - sample_covariance,
    kernel_weights, predict_xy, optimize_beta, optimize_alpha, idl_weights,
    raw_idl_weights, CovarianceBlocks.solve_yy - run bm_estimator_stages
    (csrc/bm_api.cu), which takes the caller's CovarianceBlocks as input so a
    hand-built covariance (a diagonal C_YY, a chosen C_XY) means what it
    means in the reference.
Every function accepts one instance like the reference; the *_batch forms
take lists and make one device call.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import EmptyContextError, InsufficientCandidatesError, WeightUnderflowError
from .framework import CandidateSet, TargetContext

DEFAULT_SIGMA2 = 10.0
BETA_GRID = 2.0 ** np.arange(-8, 13)
RIDGE_SCALE = 1e-6
ALPHA_MIN = 0.0
ALPHA_MAX = 4.0
_ALPHA_DENOM_FLOOR = 1e-12
MAX_CANDIDATES = 2048

BM_STAGE_COVARIANCE, BM_STAGE_KERNEL_WEIGHTS, BM_STAGE_OPTIMIZE_BETA, BM_STAGE_OPTIMIZE_ALPHA = 0, 1, 2, 3
BM_STAGE_IDL_WEIGHTS, BM_STAGE_PREDICT, BM_STAGE_SOLVE = 4, 5, 6
COV_DOUBLES = 16 + 128 + 1024 + 1


class Layer(str, enum.Enum):
    BRL = "BRL"
    IDL = "IDL"
    HQL = "HQL"


LAYER_CODE = {Layer.BRL: 0, Layer.IDL: 1, Layer.HQL: 2}
CODE_LAYER = {0: Layer.BRL, 1: Layer.IDL, 2: Layer.HQL}


@dataclass
class KernelWeights:
    """Normalised weights and their unnormalised total nu (estimators.py:45-48)."""

    w: np.ndarray
    raw_sum: float


@dataclass
class CovarianceBlocks:
    """Sample covariance of the stacked (x, y) candidates, C_YY ridge-regularised
    (estimators.py:51-68).  solve_yy runs on the device."""

    c_xx: np.ndarray  # (4, 4)
    c_xy: np.ndarray  # (4, N_y)
    c_yy: np.ndarray  # (N_y, N_y), ridge included
    ridge: float
    _cho: tuple | None = field(default=None, repr=False)

    def solve_yy(self, rhs: np.ndarray) -> np.ndarray:
        """C_YY^-1 @ rhs (cho_solve on the device); rhs (N_y,) or (N_y, k)."""
        rhs = np.asarray(rhs, dtype=np.float64)
        cols = rhs.reshape(rhs.shape[0], -1).T  # (k, N_y)
        n = self.c_yy.shape[0]
        t = TargetContext((0, 0), np.zeros(32, bool), np.zeros(n), n)
        out = []
        for lo in range(0, max(len(cols), 1), MAX_CANDIDATES):
            part = cols[lo : lo + MAX_CANDIDATES]
            cs = CandidateSet(np.zeros((len(part), 4)), part)
            res = _stages(BM_STAGE_SOLVE, [t], [cs], covs=[self], want_mat=True)
            _raise_linalg(res["status"][0])
            out.append(res["mat"][0, : len(part), :n])
        sol = np.concatenate(out, 0).T
        return sol.reshape(rhs.shape)


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


# ------------------------------------------------------------ dense packing


def _pack(targets, csets):
    """Dense device layout of the bm_estimate_batch / bm_estimator_stages ABI."""
    torch = _native.require_cuda()
    count = len(targets)
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
        if not 0 <= n <= 32:
            raise ValueError("estimators take 0..32 context samples")
        n_y[i] = n
        m[i] = c.x.shape[0]
        y0[i, :n] = np.asarray(t.y0, dtype=np.float64)[:n]
        if m[i]:
            x[i, : m[i]] = c.x
            y[i, : m[i], :n] = np.asarray(c.y, dtype=np.float64).reshape(m[i], -1)[:, :n]
    dev = torch.device("cuda", torch.cuda.current_device())

    def put(a):
        return torch.from_numpy(a).to(dev)

    return torch, dev, max_m, put(n_y), put(m), put(y0), put(x), put(y)


def _cov_rows(cov: CovarianceBlocks, n: int) -> np.ndarray:
    row = np.zeros(COV_DOUBLES)
    row[:16] = np.asarray(cov.c_xx, dtype=np.float64).reshape(4, 4).ravel()
    cxy = np.zeros((4, 32))
    cxy[:, :n] = np.asarray(cov.c_xy, dtype=np.float64).reshape(4, n)
    row[16:144] = cxy.ravel()
    cyy = np.zeros((32, 32))
    cyy[:n, :n] = np.asarray(cov.c_yy, dtype=np.float64).reshape(n, n)
    row[144:1168] = cyy.ravel()
    row[1168] = float(cov.ridge)
    return row


def _stages(stage, targets, csets, *, sigma2=DEFAULT_SIGMA2, betas=None, covs=None, weights=None, want_mat=False):
    torch, dev, max_m, n_y, m, y0, x, y = _pack(targets, csets)
    count = len(targets)
    beta = torch.from_numpy(np.asarray(betas if betas is not None else np.ones(count), dtype=np.float64)).to(dev)
    if covs is not None:
        cov = torch.from_numpy(np.stack([_cov_rows(c, int(t.n_y)) for c, t in zip(covs, targets)])).to(dev)
    else:
        cov = torch.zeros((count, COV_DOUBLES), dtype=torch.float64, device=dev)
    w = torch.zeros((count, max_m), dtype=torch.float64, device=dev)
    if weights is not None:
        for i, wi in enumerate(weights):
            w[i, : len(wi)] = torch.from_numpy(np.asarray(wi, dtype=np.float64))
    mat = torch.zeros((count, max_m, 32), dtype=torch.float64, device=dev) if want_mat else None
    sc = torch.zeros((count, 40), dtype=torch.float64, device=dev)
    status = torch.zeros(count, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    _native.check(_native.lib().bm_estimator_stages(
        stage, count, max_m, float(sigma2), n_y.data_ptr(), m.data_ptr(), y0.data_ptr(), x.data_ptr(), y.data_ptr(),
        beta.data_ptr(), cov.data_ptr(), w.data_ptr(), mat.data_ptr() if mat is not None else None, sc.data_ptr(),
        status.data_ptr(), stream))
    return {"cov": cov.cpu().numpy(), "w": w.cpu().numpy(), "mat": mat.cpu().numpy() if mat is not None else None,
            "scalars": sc.cpu().numpy(), "status": status.cpu().numpy()}


def _raise_linalg(status) -> None:
    if int(status) == 2:
        raise np.linalg.LinAlgError("C_YY is not positive definite")  # scipy.linalg.cho_factor (estimators.py:63)


# ------------------------------------------------------------------ layers


def _estimate_batch(layer: Layer, targets, csets, sigma2: float) -> list[PatchEstimate]:
    from .records import RECORD_DTYPE, decode_flags

    count = len(targets)
    if count == 0:
        return []
    for t in targets:
        if not 1 <= int(t.n_y) <= 32:
            raise EmptyContextError("estimators need 1..32 context samples")
    torch, dev, max_m, tn, tm, ty0, tx, ty = _pack(targets, csets)
    out = torch.empty((count, 4), dtype=torch.float64, device=dev)
    info = torch.empty((count, RECORD_DTYPE.itemsize), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    _native.check(
        _native.lib().bm_estimate_batch(
            LAYER_CODE[layer], count, max_m, float(sigma2), tn.data_ptr(), tm.data_ptr(), ty0.data_ptr(),
            tx.data_ptr(), ty.data_ptr(), out.data_ptr(), info.data_ptr(), stream,
        )
    )
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
    """Fill the patch with the context mean (estimators.py:96-102) on the GPU."""
    if target.n_y < 1:
        raise EmptyContextError("BRL needs at least one context sample")
    empty = CandidateSet(np.zeros((0, 4)), np.zeros((0, target.n_y)))
    est = _estimate_batch(Layer.BRL, [target], [empty], DEFAULT_SIGMA2)[0]
    est.diagnostics.m_candidates = 0
    est.diagnostics.fallback = False
    return est


def idl_estimate(target, cset, sigma2: float = DEFAULT_SIGMA2) -> PatchEstimate:
    """idl_estimate (estimators.py:122-132) on the GPU."""
    if cset.x.shape[0] < 1:
        raise InsufficientCandidatesError("IDL needs at least one candidate")
    est = _estimate_batch(Layer.IDL, [target], [cset], sigma2)[0]
    if est.layer is not Layer.IDL:
        raise WeightUnderflowError("all IDL weights underflowed (nu = 0)")
    est.diagnostics.fallback = False
    return est


def hql_estimate(target, cset, sigma2: float = DEFAULT_SIGMA2) -> PatchEstimate:
    """hql_estimate with its HQL -> IDL -> BRL ladder (estimators.py:248-286)."""
    return _estimate_batch(Layer.HQL, [target], [cset], sigma2)[0]


# ------------------------------------------------------------------ stages


def raw_idl_weights(y0: np.ndarray, y: np.ndarray, sigma2: float) -> np.ndarray:
    """Unnormalised weights exp(-||y_j - y0||^2 / (2 sigma2 N_y)) (estimators.py:105-109)."""
    y0 = np.asarray(y0, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64).reshape(-1, y0.shape[0])
    if len(y) == 0:
        return np.zeros(0)
    t = TargetContext((0, 0), np.zeros(32, bool), y0, y0.shape[0])
    out = []
    for lo in range(0, len(y), MAX_CANDIDATES):
        part = y[lo : lo + MAX_CANDIDATES]
        res = _stages(BM_STAGE_IDL_WEIGHTS, [t], [CandidateSet(np.zeros((len(part), 4)), part)], sigma2=sigma2,
                      want_mat=True)
        out.append(res["mat"][0, : len(part), 0])
    return np.concatenate(out)


def idl_weights_batch(targets, csets, sigma2: float = DEFAULT_SIGMA2) -> list[KernelWeights]:
    for c in csets:
        if c.m_current < 1:
            raise InsufficientCandidatesError("IDL needs at least one candidate")
    res = _stages(BM_STAGE_IDL_WEIGHTS, targets, csets, sigma2=sigma2)
    return [KernelWeights(res["w"][i, : c.m_current].copy(), float(res["scalars"][i, 0])) for i, c in enumerate(csets)]


def idl_weights(target: TargetContext, cset: CandidateSet, sigma2: float = DEFAULT_SIGMA2) -> KernelWeights:
    """Scalar-bandwidth Nadaraya-Watson weights (estimators.py:112-119)."""
    return idl_weights_batch([target], [cset], sigma2)[0]


def sample_covariance_batch(csets) -> list[CovarianceBlocks]:
    for c in csets:
        if c.m_current < 2:
            raise InsufficientCandidatesError(f"insufficient candidates for covariance (M'={c.m_current})")
    targets = [TargetContext((0, 0), np.zeros(32, bool), np.zeros(c.y.shape[1]), c.y.shape[1]) for c in csets]
    res = _stages(BM_STAGE_COVARIANCE, targets, csets)
    out = []
    for i, c in enumerate(csets):
        n = c.y.shape[1]
        row = res["cov"][i]
        out.append(CovarianceBlocks(row[:16].reshape(4, 4).copy(), row[16:144].reshape(4, 32)[:, :n].copy(),
                                    row[144:1168].reshape(32, 32)[:n, :n].copy(), float(row[1168])))
    return out


def sample_covariance(cset: CandidateSet) -> CovarianceBlocks:
    """Unbiased covariance blocks of the stacked candidates, divisor M'-1, ridge on C_YY
    (estimators.py:135-151)."""
    return sample_covariance_batch([cset])[0]


def kernel_weights(target: TargetContext, cset: CandidateSet, beta: float, cov: CovarianceBlocks) -> KernelWeights:
    """Gaussian kernel weights with bandwidth beta * C_YY, log-domain shift (estimators.py:167-181)."""
    if beta <= 0.0:
        raise ValueError(f"beta must be positive, got {beta}")
    if cset.m_current < 1:
        raise InsufficientCandidatesError("kernel weights need at least one candidate")
    res = _stages(BM_STAGE_KERNEL_WEIGHTS, [target], [cset], betas=[beta], covs=[cov])
    _raise_linalg(res["status"][0])
    return KernelWeights(res["w"][0, : cset.m_current].copy(), float(res["scalars"][0, 0]))


def predict_xy(target: TargetContext, cset: CandidateSet, weights: KernelWeights):
    """Weighted prototype / context predictions (x0_pred, y0_pred) (estimators.py:184-186)."""
    if cset.m_current == 0:
        return np.zeros(4), np.zeros(cset.y.shape[1] if cset.y.ndim == 2 else 0)
    n = cset.y.shape[1]
    t = TargetContext(target.patch_origin, np.zeros(32, bool), np.zeros(n), n)
    res = _stages(BM_STAGE_PREDICT, [t], [cset], weights=[weights.w])
    s = res["scalars"][0]
    return s[:4].copy(), s[4 : 4 + n].copy()


def optimize_beta(target: TargetContext, cset: CandidateSet, cov: CovarianceBlocks) -> float:
    """Grid argmin of the context prediction error, ties to the smaller beta (estimators.py:189-206)."""
    if cset.m_current < 2:
        raise InsufficientCandidatesError("beta optimization needs at least two candidates")
    res = _stages(BM_STAGE_OPTIMIZE_BETA, [target], [cset], covs=[cov])
    _raise_linalg(res["status"][0])
    return float(res["scalars"][0, 0])


def optimize_alpha(target: TargetContext, cset: CandidateSet, beta: float, cov: CovarianceBlocks) -> float:
    """Closed-form leave-one-out least-squares scale of the correction, clamped
    to [0, 4] (estimators.py:209-245)."""
    if cset.m_current < 2:
        return 0.0
    res = _stages(BM_STAGE_OPTIMIZE_ALPHA, [target], [cset], betas=[beta], covs=[cov])
    _raise_linalg(res["status"][0])
    return float(res["scalars"][0, 0])
