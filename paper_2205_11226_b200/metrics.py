"""Run report and quality metrics (mirrors blockmend/metrics.py).

`ConcealmentReport` / `usage_fractions` are the report types of
conceal_image (metrics.py:21-43, 119-124).  `psnr`, `psnr_masked` and `ssim`
keep the reference signatures (ImageBuffer or array in, float out,
metrics.py:50-116) and run on the GPU through the C ABI (bm_sqdiff_batch,
bm_ssim_batch).  `psnr_batch` / `ssim_batch` take
[B,H,W] CUDA tensors and return one value per frame — the harness's step after
concealment for batch configs.  No CPU fallback.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .errors import DimensionMismatchError

SSIM_WINDOW = 11
SSIM_SIGMA = 1.5
SSIM_K1 = 0.01
SSIM_K2 = 0.03
SSIM_L = 255.0


@dataclass
class ConcealmentReport:
    layer_counts: dict[str, int]
    patch_times: list[float]
    total_time: float
    deferred_fills: int = 0
    decisions: list = field(default_factory=list)
    psnr: float | None = None
    ssim: float | None = None

    @property
    def patches(self) -> int:
        return sum(self.layer_counts.values()) + self.deferred_fills

    def mean_patch_time(self) -> float:
        return sum(self.patch_times) / len(self.patch_times) if self.patch_times else 0.0


def usage_fractions(report: ConcealmentReport) -> dict[str, float]:
    total = sum(report.layer_counts.values())
    if total == 0:
        raise ValueError("empty report: no patches were reconstructed by any layer")
    return {layer: count / total for layer, count in report.layer_counts.items()}


# ----------------------------------------------------------------- device


def _as_device(x, torch, dev):
    """ImageBuffer / array / tensor -> contiguous CUDA tensor (u8 kept, else f64)."""
    if hasattr(x, "pixels"):
        x = x.pixels
    if isinstance(x, torch.Tensor):
        t = x
    else:
        a = np.asarray(x)
        t = torch.from_numpy(np.ascontiguousarray(a if a.dtype == np.uint8 else a.astype(np.float64)))
    if t.dtype not in (torch.uint8, torch.float64):
        t = t.to(torch.float64)
    return t.to(dev).contiguous()


def _pair(ref, test):
    from . import _native

    torch = _native.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    a = _as_device(ref, torch, dev)
    b = _as_device(test, torch, dev)
    if tuple(a.shape) != tuple(b.shape):
        raise DimensionMismatchError(f"shape mismatch: {tuple(a.shape)} vs {tuple(b.shape)}")
    if a.dtype != b.dtype:  # mixed u8 / float: compare in FP64
        a, b = a.to(torch.float64), b.to(torch.float64)
    if a.dim() == 2:
        a, b = a[None], b[None]
    return torch, a.contiguous(), b.contiguous()


def _sqdiff(torch, a, b, sel):
    from . import _native

    B, H, W = a.shape
    out = torch.empty((2, B), dtype=torch.float64, device=a.device)
    dtype = 0 if a.dtype == torch.uint8 else 1
    _native.check(_native.lib().bm_sqdiff_batch(
        a.data_ptr(), b.data_ptr(), dtype, None if sel is None else sel.data_ptr(), B, H, W,
        out[0].data_ptr(), out[1].data_ptr(), torch.cuda.current_stream().cuda_stream))
    return out.cpu().numpy()


def _psnr_from(s: float, n: float) -> float:
    if n == 0:
        return math.inf
    mse = s / n
    if mse == 0.0:
        return math.inf
    return 10.0 * math.log10(255.0**2 / mse)


def psnr_batch(ref, test, select=None) -> list[float]:
    """Per-frame PSNR of [B,H,W] frames (metrics.py:50-58 / 61-73 with select)."""
    torch, a, b = _pair(ref, test)
    sel = None
    if select is not None:
        sel = select.pixels if hasattr(select, "pixels") else select
        sel = _as_device(np.asarray(sel, dtype=np.uint8) if not isinstance(sel, torch.Tensor) else sel.to(torch.uint8),
                         torch, a.device)
        if sel.dim() == 2:
            sel = sel[None]
        if tuple(sel.shape) != tuple(a.shape):
            raise DimensionMismatchError("psnr_masked needs three same-shape arrays")
        sel = (sel != 0).to(torch.uint8).contiguous()
    sums = _sqdiff(torch, a, b, sel)
    return [_psnr_from(float(s), float(n)) for s, n in zip(sums[0], sums[1])]


def psnr(ref, test) -> float:
    """10 log10(255^2 / MSE) over all pixels; identical frames give +inf (metrics.py:50-58)."""
    return psnr_batch(ref, test)[0]


def psnr_masked(ref, test, select) -> float:
    """PSNR restricted to the selected pixels (metrics.py:61-73)."""
    return psnr_batch(ref, test, select)[0]


def ssim_batch(ref, test) -> list[float]:
    """Per-frame mean SSIM of [B,H,W] frames (metrics.py:86-116)."""
    from . import _native

    torch, a, b = _pair(ref, test)
    B, H, W = a.shape
    if min(H, W) < SSIM_WINDOW:
        raise ValueError(f"image too small for SSIM (min side {SSIM_WINDOW})")
    out = torch.empty(B, dtype=torch.float64, device=a.device)
    dtype = 0 if a.dtype == torch.uint8 else 1
    _native.check(_native.lib().bm_ssim_batch(a.data_ptr(), b.data_ptr(), dtype, B, H, W, out.data_ptr(),
                                              torch.cuda.current_stream().cuda_stream))
    return [float(v) for v in out.cpu().numpy()]


def ssim(ref, test) -> float:
    """Mean SSIM, 11x11 Gaussian window (sigma 1.5), windows fully inside (metrics.py:86-116)."""
    return ssim_batch(ref, test)[0]
