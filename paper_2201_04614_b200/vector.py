"""GPU drop-in for the reference lane kernel (vector.py:205-260).

`dualquant_vector(data, config, collect_border=False)` takes and returns the
same objects as the reference: a C-contiguous float32 numpy array in, a
CodeStream out (uint32 codes, float32 outliers, int64 per-block counts,
int64 padding scalars), byte-identical to the reference's stream.  The work
runs in the fused sm_100a kernels of libvlzgpu.so; `lane_width` and
`thread_count` are validated like the reference but do not change execution
(they never change the reference's output either, test_vector.py:36-93).
"""

from __future__ import annotations

import numpy as np
import torch

from . import gpu
from .errors import ConfigError
from .model import (
    VECTOR_LANE_WIDTHS,
    ArrayDescriptor,
    CodeStream,
    CompressionConfig,
    PaddingScalars,
    build_block_grid,
    resolve_error_bound,
)


def _device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2201_04614_b200 needs a CUDA device (B200); no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def to_codestream(dev: gpu.DeviceCodeStream) -> CodeStream:
    """Copy a device stream back into the reference's CodeStream layout."""
    n_out = dev.n_outliers
    codes = dev.codes.cpu().numpy().view(np.uint16).astype(np.uint32)
    return CodeStream(
        codes=codes,
        outlier_values=dev.outliers[:n_out].cpu().numpy().copy(),
        outlier_counts=dev.counts[: dev.grid.block_count].cpu().numpy().copy(),
        grid=dev.grid,
        resolved_abs=dev.eb,
        radius=dev.radius,
        scalars=PaddingScalars(dev.padding, dev.scalars.cpu().numpy().astype(np.int64)),
    )


def border_outliers(stream: CodeStream) -> int:
    """Outliers whose block-local coordinates include a 0 (vector.py:82-87),
    from a host CodeStream (the GPU path uses gpu.border_outliers_device)."""
    grid = stream.grid
    dims = grid.descriptor.dims
    nd = len(dims)
    b = grid.block_edge
    codes = stream.codes
    # canonical position -> block-local coordinates, vectorised per block shape
    total = 0
    idx = np.arange(grid.block_count)
    per = grid.blocks_per_dim
    coords = np.stack(np.unravel_index(idx, per), axis=1)
    ext = np.minimum(b, np.array(dims)[None, :] - coords * b)
    sizes = np.prod(ext, axis=1)
    starts = np.concatenate([[0], np.cumsum(sizes)[:-1]])
    for shape in {tuple(e) for e in ext.tolist()}:
        sel = np.all(ext == np.array(shape)[None, :], axis=1)
        m = np.zeros(shape, dtype=bool)
        for d in range(nd):
            m[tuple(slice(None) if a != d else 0 for a in range(nd))] = True
        flat = np.flatnonzero(m.ravel())
        pos = starts[sel][:, None] + flat[None, :]
        total += int(np.count_nonzero(codes[pos] == 0))
    return total


def dualquant_vector(data: np.ndarray, config: CompressionConfig, collect_border: bool = False):
    """Fused GPU dual-quantization with the reference's signature and output."""
    if config.lane_width not in VECTOR_LANE_WIDTHS:
        raise ConfigError(
            f"vector kernel needs a lane width in {VECTOR_LANE_WIDTHS}, "
            f"got {config.lane_width} (lane width 1 is the scalar kernel)"
        )
    return dualquant(data, config, collect_border)


def dualquant_scalar(data: np.ndarray, config: CompressionConfig, counters=None):
    """Drop-in for the reference's scalar kernel (kernel.py:124-193): the
    same stream as the vector path, and the scalar error order -- the first
    flat index that is non-finite (ConfigError) or overflows the quantizer
    (BoundTooSmallError) decides, kernel.py:138-145.  `counters` (the
    reference's op tally for the paper's figures) is not supported."""
    if counters is not None:
        raise ConfigError("kernel counters are not collected by the GPU kernels")
    return dualquant(data, config, scalar_order=True)


def dualquant(data: np.ndarray, config: CompressionConfig, collect_border: bool = False,
              scalar_order: bool = False):
    """dualquant_vector without the lane-width restriction (any lane width
    yields the same stream; used by pipeline.compress_detailed)."""
    desc = ArrayDescriptor.from_array(data)
    eb = resolve_error_bound(config.error_bound, data)
    build_block_grid(desc, config.block_edge)
    gpu.check_resolved_eb(eb, data)
    dev = _device()
    x = torch.from_numpy(np.ascontiguousarray(data)).to(dev, non_blocking=False)
    out = gpu.compress_device(x, config, eb=eb)
    out.source = None
    try:
        out.check(scalar_order=scalar_order)
    except Exception as exc:
        from .errors import BoundTooSmallError

        if isinstance(exc, BoundTooSmallError):
            idx = exc.index
            raise BoundTooSmallError(idx, float(data.ravel()[idx]), eb) from None
        raise
    stream = to_codestream(out)
    if collect_border:
        total = int(stream.outlier_counts.sum())
        border = gpu.border_outliers_device(out.codes[: desc.element_count], stream.grid)
        return stream, (total, border)
    return stream
