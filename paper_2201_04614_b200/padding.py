"""Padding-policy outlier census (reference padding.py:145-205).

`outlier_report(data, config, policies=None)` runs the dual-quant path on the
GPU once per padding policy (zero padding first) and reports, per policy, the
total and border outlier counts and the reduction versus zero padding -- the
study the paper's padding section is built on.  Border outliers are counted
on the device (csrc/k_stats.cu).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .model import (
    CompressionConfig,
    PaddingGranularity,
    PaddingPolicy,
    PaddingValue,
)

__all__ = ["PaddingOutlierStats", "outlier_report"]


@dataclass(frozen=True)
class PaddingOutlierStats:
    """Outlier census for one padding policy on one (data, config) pair."""

    policy: PaddingPolicy
    total_outliers: int
    border_outliers: int

    @property
    def border_pct(self) -> float:
        if self.total_outliers == 0:
            return 0.0
        return 100.0 * self.border_outliers / self.total_outliers


def outlier_report(data: np.ndarray, config: CompressionConfig,
                   policies: list[PaddingPolicy] | None = None,
                   ) -> list[tuple[PaddingOutlierStats, float]]:
    """(stats, reduction_vs_zero_pct) per policy, zero padding first
    (padding.py:162-205: same policy order, same lane-width substitution)."""
    from .vector import dualquant_vector

    if policies is None:
        policies = [PaddingPolicy(kind, gran)
                    for kind in (PaddingValue.MINIMUM, PaddingValue.MAXIMUM, PaddingValue.MEAN)
                    for gran in PaddingGranularity]
    zero_policy = PaddingPolicy(PaddingValue.ZERO, PaddingGranularity.GLOBAL)
    ordered = [zero_policy] + [p for p in policies if p.value_kind is not PaddingValue.ZERO]
    rows: list[tuple[PaddingOutlierStats, float]] = []
    zero_total = 0
    for i, pol in enumerate(ordered):
        cfg = CompressionConfig(
            error_bound=config.error_bound, block_edge=config.block_edge,
            lane_width=config.lane_width if config.lane_width != 1 else 8, padding=pol,
            radius=config.radius, thread_count=config.thread_count)
        _, (total, border) = dualquant_vector(data, cfg, collect_border=True)
        report = PaddingOutlierStats(pol, total, border)
        if i == 0:
            zero_total = total
            reduction = 0.0
        elif zero_total == 0:
            reduction = 0.0
        else:
            reduction = 100.0 * (zero_total - total) / zero_total
        rows.append((report, reduction))
    return rows
