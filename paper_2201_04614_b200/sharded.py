"""Multi-GPU dual-quantization: block-aligned slab sharding along dim 0.

Blocks never read their neighbours (the halo comes from padding scalars,
reference reconstruct.py:5-7), so a field split into slabs whose dim-0
boundaries are multiples of the block edge compresses shard by shard with no
halo exchange.  Each rank owns a contiguous range of block indices, of code
positions and of outliers; the global stream is the concatenation in rank
order, byte-identical to the single-GPU stream.

Collectives (torch.distributed; NCCL on GPUs, gloo in the CPU tests):
  * relative error bound: all-reduce MIN/MAX of the shard value ranges
    (model.py:104-110) -- before compression, like the reference;
  * *:global padding: one all-gather of the partial statistics (sum,
    count, min, -max per rank, padding.py:62-85) between the fused kernel and
    the origin fix-up; the finish kernel reduces the gathered records;
  * all-gather of the per-shard outlier totals -> each shard's offset into
    the global outlier array (CodeStream.outlier_values).
Bulk data never crosses GPUs.

The compute steps are delegated to a backend with the begin/finish protocol
of the C ABI (vlz_dq_compress_begin / vlz_dq_compress_finish); `GpuBackend`
is the product backend, tests substitute a CPU one to exercise this host
logic on gloo without a GPU.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _lib
from .errors import ConfigError
from .model import (
    ArrayDescriptor,
    BlockGrid,
    CompressionConfig,
    ErrorBoundMode,
    PaddingGranularity,
    PaddingValue,
    build_block_grid,
    resolve_error_bound_from_range,
)


def slab_bounds(d0: int, block_edge: int, world: int, rank: int):
    """Planes [z0, z1) of `rank`: whole dim-0 block layers, balanced."""
    nb0 = -(-d0 // block_edge)
    base, extra = divmod(nb0, world)
    b0 = rank * base + min(rank, extra)
    b1 = b0 + base + (1 if rank < extra else 0)
    return min(d0, b0 * block_edge), min(d0, b1 * block_edge)


@dataclass
class ShardInfo:
    rank: int
    world: int
    z0: int
    z1: int
    full_grid: BlockGrid
    local_grid: BlockGrid
    block_offset: int      # first global block index of the shard
    code_offset: int       # first global code position of the shard
    outlier_offset: int    # first global outlier index of the shard
    total_outliers: int


def _reduce_range(lo: float, hi: float, group, device):
    t = torch.tensor([lo, -hi], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return float(t[0]), -float(t[1])


def gather_stats(stats: torch.Tensor, group=None) -> torch.Tensor:
    """Every rank's 4 statistic words [sum, count, min, -max] in rank order
    (int64 [world * 4]): the one collective of a *:global step (32 B per rank,
    one all-gather instead of a SUM and a MIN all-reduce).  The reduction runs
    inside the finish kernel (vlz_dq_compress_finish_gathered)."""
    world = dist.get_world_size(group)
    allst = torch.empty(world * 4, dtype=stats.dtype, device=stats.device)
    dist.all_gather_into_tensor(allst, stats.contiguous(), group=group)
    return allst


def reduce_gathered(allst: torch.Tensor) -> torch.Tensor:
    """Host-side form of the finish kernel's reduction of gathered records:
    [sum, count] summed (int64 wraps like the reference's np.sum), [min,
    -max] minimised.  For backends without the fused reduction (tests)."""
    a = allst.view(-1, 4)
    return torch.cat([a[:, 0:2].sum(dim=0), a[:, 2:4].min(dim=0).values])


def reduce_stats(stats: torch.Tensor, group=None):
    """In place: the statistics of all ranks reduced (gather_stats +
    reduce_gathered)."""
    stats.copy_(reduce_gathered(gather_stats(stats, group)))
    return stats


class GpuBackend:
    """begin/finish on the device through libvlzgpu.so."""

    def __init__(self):
        self.lib = _lib.load()

    def value_range(self, x):
        from .gpu import value_range

        return value_range(x)

    def begin(self, x, grid, eb, config):
        lib = self.lib
        pol = config.padding
        g = _lib.geom(grid.descriptor.dims, grid.block_edge)
        p = _lib.params(eb, config.radius, pol.kind_code, pol.gran_code)
        dev = x.device
        n = grid.descriptor.element_count
        h = {
            "g": g, "p": p, "x": x,
            "codes": torch.empty(max(n, 1), dtype=torch.int16, device=dev),
            "outliers": torch.empty(max(n, 1), dtype=torch.float32, device=dev),
            "counts": torch.empty(max(grid.block_count, 1), dtype=torch.int64, device=dev),
            "scalars": torch.empty(max(pol.scalar_count(grid), 1), dtype=torch.int64, device=dev),
            "result": torch.empty(8, dtype=torch.int64, device=dev),
            "stats": torch.zeros(4, dtype=torch.int64, device=dev),
        }
        wsb = lib.vlz_workspace_size(ctypes.byref(g))
        h["ws"] = torch.empty(max(wsb, 256), dtype=torch.uint8, device=dev)
        st = torch.cuda.current_stream().cuda_stream
        rc = lib.vlz_dq_compress_begin(
            x.data_ptr(), ctypes.byref(g), ctypes.byref(p), h["codes"].data_ptr(),
            h["counts"].data_ptr(), h["scalars"].data_ptr(), h["result"].data_ptr(),
            h["stats"].data_ptr(), h["ws"].data_ptr(), h["ws"].numel(), st)
        if rc != 0:
            raise RuntimeError(f"vlz_dq_compress_begin failed ({rc})")
        return h

    def finish(self, h, stats):
        """`stats`: one reduced record or the gathered records of all ranks
        (int64 [nranks * 4]); the scan kernel reduces them."""
        st = torch.cuda.current_stream().cuda_stream
        stats = stats.contiguous()
        rc = self.lib.vlz_dq_compress_finish_gathered(
            h["x"].data_ptr(), ctypes.byref(h["g"]), ctypes.byref(h["p"]), stats.data_ptr(),
            stats.numel() // 4, h["codes"].data_ptr(), h["outliers"].data_ptr(),
            h["counts"].data_ptr(), h["scalars"].data_ptr(), h["result"].data_ptr(),
            h["ws"].data_ptr(), h["ws"].numel(), st)
        if rc != 0:
            raise RuntimeError(f"vlz_dq_compress_finish failed ({rc})")
        return h

    def n_outliers(self, h):
        return h["result"][2:3]


def compress_sharded(x_local: torch.Tensor, full_shape, config: CompressionConfig, group=None,
                     backend=None, eb: float | None = None):
    """Compress this rank's slab of a field of `full_shape` (dim-0 sharded).

    Returns (handle, ShardInfo); the handle holds the shard's codes, outliers,
    counts and scalars (device tensors for GpuBackend)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    backend = backend or GpuBackend()
    full = ArrayDescriptor(len(full_shape), tuple(int(d) for d in full_shape))
    full_grid = build_block_grid(full, config.block_edge)
    # decided from the shape alone, so every rank raises together before any
    # collective (a rank that went on would wait for the others forever)
    if -(-full.dims[0] // config.block_edge) < world:
        raise ConfigError("more ranks than dim-0 block layers")
    z0, z1 = slab_bounds(full.dims[0], config.block_edge, world, rank)
    if tuple(x_local.shape) != (z1 - z0,) + tuple(full.dims[1:]):
        raise ConfigError(f"rank {rank} holds {tuple(x_local.shape)}, expected planes [{z0},{z1})")
    local = ArrayDescriptor(full.ndims, (z1 - z0,) + tuple(full.dims[1:]))
    local_grid = build_block_grid(local, config.block_edge)
    dev = x_local.device
    if eb is None:
        if config.error_bound.mode is ErrorBoundMode.ABSOLUTE:
            eb = float(config.error_bound.value)
        else:
            lo, hi = backend.value_range(x_local)
            lo, hi = _reduce_range(lo, hi, group, dev)
            eb = resolve_error_bound_from_range(config.error_bound, lo, hi)
    h = backend.begin(x_local, local_grid, eb, config)
    pol = config.padding
    stats = h["stats"]
    if pol.value_kind is not PaddingValue.ZERO and pol.granularity is PaddingGranularity.GLOBAL:
        stats = gather_stats(stats, group)  # reduced by the finish kernel
    backend.finish(h, stats)
    totals = torch.empty(world, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(totals, backend.n_outliers(h), group=group)
    tot = totals.tolist()
    per_layer = full_grid.blocks_per_dim[1] * full_grid.blocks_per_dim[2] if full.ndims == 3 else (
        full_grid.blocks_per_dim[1] if full.ndims == 2 else 1)
    plane = 1
    for d in full.dims[1:]:
        plane *= d
    info = ShardInfo(
        rank=rank, world=world, z0=z0, z1=z1, full_grid=full_grid, local_grid=local_grid,
        block_offset=(z0 // config.block_edge) * per_layer,
        code_offset=z0 * plane,
        outlier_offset=int(sum(tot[:rank])),
        total_outliers=int(sum(tot)),
    )
    h["eb"] = eb
    return h, info
