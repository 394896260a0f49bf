"""Slab sharding through the CUDA begin/finish protocol on one GPU.

The shards of a field are compressed one after another on the same device
(no kernel waits on another), their partial *:global statistics are reduced
exactly as sharded.reduce_stats does across ranks, and the concatenated
stream must equal the single-shot compression of the whole field.  The
NCCL plumbing itself runs at world size 1 (torchrun --nproc-per-node N on an
N-GPU box exercises N > 1; tests/test_sharded_cpu.py covers N = 2 on gloo)."""

from __future__ import annotations

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402

from paper_2201_04614_b200 import model as M  # noqa: E402
from paper_2201_04614_b200 import workloads  # noqa: E402
from paper_2201_04614_b200.sharded import GpuBackend, compress_sharded, slab_bounds  # noqa: E402
from paper_2201_04614_b200.vector import dualquant  # noqa: E402


def _cfg(eb, b, pol, radius):
    return M.CompressionConfig(M.ErrorBound.absolute(eb), block_edge=b,
                               padding=M.PaddingPolicy.parse(pol), radius=radius)


@pytest.mark.parametrize("pol", ["mean:global", "min:global", "zero", "max:block", "mean:edge"])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_shards_concatenate_to_single_stream(pol, world):
    d = workloads.gen_c3(shape=(72, 50, 64))
    eb = workloads.value_range_eb(d, 1e-4)
    cfg = _cfg(eb, 8, pol, 512)
    ref = dualquant(d, cfg)
    be = GpuBackend()
    hs = []
    grid_full = M.build_block_grid(M.ArrayDescriptor(3, d.shape), 8)
    for r in range(world):
        z0, z1 = slab_bounds(d.shape[0], 8, world, r)
        x = torch.from_numpy(np.ascontiguousarray(d[z0:z1])).cuda()
        g = M.build_block_grid(M.ArrayDescriptor(3, x.shape), 8)
        hs.append(be.begin(x, g, eb, cfg))
    stats = torch.stack([h["stats"] for h in hs])
    red = torch.stack([stats[:, 0].sum(), stats[:, 1].sum(), stats[:, 2].min(), stats[:, 3].min()])
    for i, h in enumerate(hs):
        # odd shards: the gathered records of all ranks, reduced in the finish
        # kernel (vlz_dq_compress_finish_gathered); even: pre-reduced record
        be.finish(h, stats.reshape(-1).clone() if i % 2 else red.clone())
    torch.cuda.synchronize()
    codes, outl, counts, scal = [], [], [], []
    for h in hs:
        n_out = int(h["result"][2])
        n = h["x"].numel()
        codes.append(h["codes"][:n].cpu().numpy().view(np.uint16))
        outl.append(h["outliers"][:n_out].cpu().numpy())
        nb = M.build_block_grid(M.ArrayDescriptor(3, tuple(h["x"].shape)), 8).block_count
        counts.append(h["counts"][:nb].cpu().numpy())
        scal.append(h["scalars"].cpu().numpy())
    assert np.concatenate(codes).astype(np.uint32).tobytes() == ref.codes.tobytes()
    assert np.concatenate(outl).tobytes() == ref.outlier_values.tobytes()
    assert np.concatenate(counts).tobytes() == ref.outlier_counts.tobytes()
    if pol.endswith(":global") and not pol.startswith("zero"):
        assert all(s[:1].tobytes() == ref.scalars.values.tobytes() for s in scal)
    elif pol != "zero":
        assert np.concatenate(scal).tobytes() == ref.scalars.values.tobytes()
    assert grid_full.block_count == ref.outlier_counts.size


def test_compress_sharded_world1_nccl():
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        d = workloads.gen_c3(shape=(40, 48, 64))
        cfg = M.CompressionConfig(M.ErrorBound.relative(1e-4), block_edge=8, radius=512)
        ref = dualquant(d, cfg)
        h, info = compress_sharded(torch.from_numpy(d).cuda(), d.shape, cfg)
        torch.cuda.synchronize()
        assert h["eb"] == ref.resolved_abs
        assert info.total_outliers == ref.outlier_values.size
        assert h["codes"].cpu().numpy().view(np.uint16).astype(np.uint32).tobytes() == \
            ref.codes.tobytes()
    finally:
        dist.destroy_process_group()
