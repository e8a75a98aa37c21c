"""ConcealmentReport — the run report returned by conceal_image (mirrors
blockmend/metrics.py:21-43; the quality metrics themselves are out of scope)."""

from __future__ import annotations

from dataclasses import dataclass, field


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
