"""Slab-sharded compression on world_size 2 over gloo (CPU, no GPU).

The product's sharding host logic (paper_2201_04614_b200/sharded.py: slab
bounds, relative-bound range all-reduce, *:global statistics all-reduce,
outlier-offset all-gather) runs unchanged; the per-shard compute is the CPU
oracle behind the same begin/finish protocol as the CUDA backend.  The
assembled global stream must equal the single-process oracle stream on the
whole array, byte for byte."""

from __future__ import annotations

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)

CASES = [
    ((37, 20, 19), 8, "mean:global", ("abs", 1e-3), 512),
    ((37, 20, 19), 8, "max:global", ("rel", 1e-4), 32768),
    ((40, 16, 24), 16, "zero", ("abs", 1e-2), 64),
    ((33, 9, 10), 8, "min:block", ("abs", 1e-3), 512),
    ((25, 30), 8, "mean:edge", ("rel", 1e-3), 512),
    ((1001,), 64, "mean:global", ("abs", 1e-3), 512),
]


def _field(shape, seed):
    rng = np.random.default_rng(seed)
    mesh = np.add.reduce(np.meshgrid(*[np.linspace(0, 4, s) for s in shape], indexing="ij"))
    return (50 + 10 * np.sin(mesh) + rng.normal(0, 0.05, shape)).astype(np.float32)


class OracleBackend:
    """CPU stand-in for sharded.GpuBackend (test infrastructure)."""

    def __init__(self, oracle):
        self.o = oracle

    def value_range(self, x):
        return self.o.minmax(x.numpy())

    def begin(self, x, grid, eb, config):
        st = self.o.global_stats(x.numpy(), eb)
        stats = torch.tensor([st[0], st[1], st[2], -st[3]], dtype=torch.int64)
        return {"x": x, "grid": grid, "eb": eb, "config": config, "stats": stats}

    def finish(self, h, stats):
        from paper_2201_04614_b200.sharded import reduce_gathered

        cfg = h["config"]
        pol = str(cfg.padding)
        s0 = None
        if pol.endswith(":global") and not pol.startswith("zero"):
            s = reduce_gathered(stats).tolist()  # the GPU finish kernel's reduction
            s0 = self.o.stat_value(pol.split(":")[0], s[0], s[1], s[2], -s[3])
        h["stream"] = self.o.dualquant(h["x"].numpy(), h["eb"], cfg.block_edge, cfg.radius, pol,
                                       threads=1, global_scalar=s0)
        h["nout"] = torch.tensor([h["stream"]["outlier_values"].size], dtype=torch.int64)
        return h

    def n_outliers(self, h):
        return h["nout"]


def _worker(rank, world, port, results):
    sys.path[:0] = [REPO, os.path.join(REPO, "oracle")]
    import oracle

    from paper_2201_04614_b200 import model as M
    from paper_2201_04614_b200.sharded import compress_sharded, slab_bounds

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = []
        for i, (shape, b, pol, (mode, ebv), radius) in enumerate(CASES):
            data = _field(shape, i)
            z0, z1 = slab_bounds(shape[0], b, world, rank)
            eb = M.ErrorBound.absolute(ebv) if mode == "abs" else M.ErrorBound.relative(ebv)
            cfg = M.CompressionConfig(eb, block_edge=b, padding=M.PaddingPolicy.parse(pol),
                                      radius=radius)
            h, info = compress_sharded(torch.from_numpy(np.ascontiguousarray(data[z0:z1])),
                                       shape, cfg, backend=OracleBackend(oracle))
            out.append(dict(stream=h["stream"], eb=h["eb"], z0=info.z0, z1=info.z1,
                            block_offset=info.block_offset, code_offset=info.code_offset,
                            outlier_offset=info.outlier_offset,
                            total=info.total_outliers))
        results[rank] = out
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2])
def test_sharded_stream_equals_single_process(world, oracle):
    manager = mp.Manager()
    results = manager.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    for i, (shape, b, pol, (mode, ebv), radius) in enumerate(CASES):
        data = _field(shape, i)
        eb = ebv if mode == "abs" else ebv * (float(data.max()) - float(data.min()))
        ref = oracle.dualquant(data, eb, b, radius, pol)
        parts = [results[r][i] for r in range(world)]
        assert all(p["eb"] == eb for p in parts)
        codes = np.concatenate([p["stream"]["codes"] for p in parts])
        ovals = np.concatenate([p["stream"]["outlier_values"] for p in parts])
        counts = np.concatenate([p["stream"]["outlier_counts"] for p in parts])
        if pol.endswith(":global") and not pol.startswith("zero"):
            scal = parts[0]["stream"]["scalars"]
            assert all(np.array_equal(p["stream"]["scalars"], scal) for p in parts)
        else:
            scal = np.concatenate([p["stream"]["scalars"] for p in parts])
        assert codes.tobytes() == ref["codes"].tobytes(), (i, pol)
        assert ovals.tobytes() == ref["outlier_values"].tobytes(), (i, pol)
        assert counts.tobytes() == ref["outlier_counts"].tobytes(), (i, pol)
        assert scal.tobytes() == ref["scalars"].tobytes(), (i, pol)
        # offsets the all-gather produced
        acc_codes = acc_out = acc_blocks = 0
        for p in parts:
            assert p["code_offset"] == acc_codes
            assert p["outlier_offset"] == acc_out
            assert p["block_offset"] == acc_blocks
            assert p["total"] == ref["outlier_values"].size
            acc_codes += p["stream"]["codes"].size
            acc_out += p["stream"]["outlier_values"].size
            acc_blocks += p["stream"]["outlier_counts"].size


def test_slab_bounds_partition():
    from paper_2201_04614_b200.sharded import slab_bounds

    for d0, b, world in ((2048, 8, 8), (100, 8, 3), (37, 8, 2), (9, 8, 2), (1001, 64, 4)):
        prev = 0
        for r in range(world):
            z0, z1 = slab_bounds(d0, b, world, r)
            assert z0 == prev and z0 % b == 0
            prev = z1
        assert prev == d0


def _too_many_ranks_worker(rank, world, port, results):
    sys.path[:0] = [REPO, os.path.join(REPO, "oracle")]
    import oracle

    from paper_2201_04614_b200 import model as M
    from paper_2201_04614_b200.errors import ConfigError
    from paper_2201_04614_b200.sharded import compress_sharded, slab_bounds

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shape = (12, 9, 10)  # 2 block layers of b=8 for 3 ranks
        z0, z1 = slab_bounds(shape[0], 8, world, rank)
        data = _field(shape, 0)
        cfg = M.CompressionConfig(M.ErrorBound.relative(1e-3), block_edge=8)
        try:
            compress_sharded(torch.from_numpy(np.ascontiguousarray(data[z0:z1])), shape, cfg,
                             backend=OracleBackend(oracle))
            results[rank] = "no error"
        except ConfigError as exc:
            results[rank] = str(exc)
    finally:
        dist.destroy_process_group()


def test_more_ranks_than_layers_raises_on_every_rank():
    # only the empty-slab rank used to raise; the others entered
    # the range all-reduce and waited forever
    manager = mp.Manager()
    results = manager.dict()
    ctx = mp.spawn(_too_many_ranks_worker, args=(3, _free_port(), results), nprocs=3,
                   join=False)
    import time

    deadline = time.time() + 120
    while not ctx.join(timeout=5) and time.time() < deadline:
        pass
    alive = [p for p in ctx.processes if p.is_alive()]
    for p in alive:
        p.kill()
    assert not alive, "a rank hung in a collective"
    assert dict(results) == {r: "more ranks than dim-0 block layers" for r in range(3)}
