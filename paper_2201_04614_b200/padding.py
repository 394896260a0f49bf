"""Padding-policy outlier study (drop-in for reference padding.py:145-205).

`outlier_report(data, config, policies=None)` returns, zero padding first and
then each non-zero policy in the order given (default: min, max, mean, each
at global, block and edge granularity), a `PaddingOutlierStats` row -- total
outliers, border outliers -- with the reduction of the total versus zero
padding in percent; the same rows as the reference.

The reference compresses the array once per policy.  Here the array goes to
the device once and two passes replace the ten:

1. the fused compress kernel with zero padding gives the zero-padding total,
   and the device border census (csrc/k_stats.cu) its border outliers;
2. the policy census (csrc/k_census.cu) gives, for every policy, how many
   block origins are outliers.

By finding 1 a padding policy only changes the prediction at
block origins, and the narrowing check ignores the policy, so away from the
origins every policy has exactly the zero-padding outliers.  An origin is a
border element (all its block-local coordinates are 0).  Hence, with o(P) the
origin outliers of policy P:
    total(P)  = total(zero)  - o(zero) + o(P)
    border(P) = border(zero) - o(zero) + o(P)
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, gpu
from .errors import BoundTooSmallError
from .model import (
    ArrayDescriptor,
    CompressionConfig,
    PaddingGranularity,
    PaddingPolicy,
    PaddingValue,
    build_block_grid,
    resolve_error_bound,
)

__all__ = ["PaddingOutlierStats", "outlier_report", "origin_outlier_census"]

_ZERO = PaddingPolicy(PaddingValue.ZERO, PaddingGranularity.GLOBAL)


@dataclass(frozen=True)
class PaddingOutlierStats:
    """One row of the study: a policy and its outlier counts."""

    policy: PaddingPolicy
    total_outliers: int
    border_outliers: int

    @property
    def border_pct(self) -> float:
        """Share of the outliers that sit on a block border, in percent."""
        t = self.total_outliers
        return 0.0 if t == 0 else 100.0 * self.border_outliers / t


def _census_slot(policy: PaddingPolicy) -> int:
    """Index of a policy in the census output (k_census.cu layout)."""
    if policy.value_kind is PaddingValue.ZERO:
        return 0
    return 3 * policy.kind_code + policy.gran_code


def origin_outlier_census(x: torch.Tensor, grid, eb: float, radius: int) -> np.ndarray:
    """int64[12]: block origins that are outliers under each policy
    (slot 0 zero padding, slot 3*kind + gran otherwise), counted on the
    device in one pass over the CUDA float32 tensor `x`."""
    lib = _lib.load()
    g = _lib.geom(grid.descriptor.dims, grid.block_edge)
    wsb = int(lib.vlz_padding_census_ws_size(ctypes.byref(g)))
    ws = torch.empty(wsb, dtype=torch.uint8, device=x.device)
    out = torch.empty(12, dtype=torch.int64, device=x.device)
    rc = lib.vlz_padding_census(x.data_ptr(), ctypes.byref(g), float(eb), int(radius),
                                out.data_ptr(), ws.data_ptr(), wsb,
                                torch.cuda.current_stream(x.device).cuda_stream)
    if rc != 0:
        raise RuntimeError(f"vlz_padding_census failed ({rc})")
    return out.cpu().numpy()


def outlier_report(data: np.ndarray, config: CompressionConfig,
                   policies: list[PaddingPolicy] | None = None,
                   ) -> list[tuple[PaddingOutlierStats, float]]:
    """[(stats, reduction_vs_zero_pct)] per policy, zero padding first."""
    if policies is None:
        policies = [PaddingPolicy(k, g)
                    for k in (PaddingValue.MINIMUM, PaddingValue.MAXIMUM, PaddingValue.MEAN)
                    for g in PaddingGranularity]
    rows_for = [_ZERO] + [p for p in policies if p.value_kind is not PaddingValue.ZERO]

    # the zero-padding run goes through the vector path's validation (lane
    # width 1 stands in as 8, as in the reference) and raises its errors
    zero_cfg = CompressionConfig(
        error_bound=config.error_bound, block_edge=config.block_edge,
        lane_width=8 if config.lane_width == 1 else config.lane_width, padding=_ZERO,
        radius=config.radius, thread_count=config.thread_count)
    desc = ArrayDescriptor.from_array(data)
    eb = resolve_error_bound(zero_cfg.error_bound, data)
    grid = build_block_grid(desc, zero_cfg.block_edge)
    gpu.check_resolved_eb(eb, data)
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2201_04614_b200 needs a CUDA device (B200); no CPU fallback")
    x = torch.from_numpy(np.ascontiguousarray(data)).cuda()
    dev = gpu.compress_device(x, zero_cfg, eb=eb)
    dev.source = None
    try:
        dev.check()
    except BoundTooSmallError as exc:
        raise BoundTooSmallError(exc.index, float(data.ravel()[exc.index]), eb) from None
    total0 = dev.n_outliers
    border0 = gpu.border_outliers_device(dev.codes[: desc.element_count], grid)
    origins = origin_outlier_census(x, grid, eb, zero_cfg.radius)
    away_total = total0 - int(origins[0])
    away_border = border0 - int(origins[0])

    out: list[tuple[PaddingOutlierStats, float]] = []
    for pol in rows_for:
        o = int(origins[_census_slot(pol)])
        st = PaddingOutlierStats(pol, away_total + o, away_border + o)
        red = 0.0
        if pol is not rows_for[0] and total0:
            red = 100.0 * (total0 - st.total_outliers) / total0
        out.append((st, red))
    return out
