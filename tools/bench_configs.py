"""Per-configuration device throughput (BASELINE.json configs C1-C4 and an
outlier-stress variant), for DESIGN.md / profiling -- not the driver's bench.

Each case: compress + decompress through the device API, L2 flushed (256 MB
write) before every timed call, median of `reps`; prints one JSON line per
case with input GB/s per phase and the fused-kernel share.
"""

from __future__ import annotations

import ctypes
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2201_04614_b200 import _lib, gpu, workloads  # noqa: E402
from paper_2201_04614_b200 import model as M  # noqa: E402


def timed(fn, flush, reps):
    lib = _lib.load()
    ts, kt = [], []
    kms = (ctypes.c_double * 8)()
    kc = (ctypes.c_int64 * 8)()
    # call time with the library's per-kernel event timing off (as a user
    # calls it); kernel times from separate calls with it on
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    for _ in range(reps):
        flush.zero_()
        torch.cuda.synchronize()
        lib.vlz_timing(1)
        fn()
        torch.cuda.synchronize()
        lib.vlz_timing(0)
        lib.vlz_timing_collect(kms, kc, 8)
        kt.append(dict(init=kms[0], compress=kms[1], scan_c=kms[2], scan_d=kms[3],
                       decompress=kms[4], redo=kms[6], edge=kms[7]))
    kt.sort(key=lambda k: k["compress"] + k["decompress"])
    return statistics.median(ts), kt[len(kt) // 2]


def run(name, data, rel, b, pol, radius, reps=7):
    M.allow_block_256(True)
    x = torch.from_numpy(data).cuda()
    eb = workloads.value_range_eb(data, rel)
    cfg = M.CompressionConfig(M.ErrorBound.absolute(eb), block_edge=b, radius=radius,
                              padding=M.PaddingPolicy.parse(pol))
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    dev = gpu.compress_device(x, cfg, eb=eb).check()
    n_out = dev.n_outliers
    y = torch.empty_like(x)
    res = torch.empty(8, dtype=torch.int64, device="cuda")

    def comp():
        gpu.compress_device(x, cfg, eb=eb, out=dev)

    def decomp():
        gpu.decompress_device(dev.codes, dev.outliers, n_out, dev.counts, dev.scalars, dev.grid,
                              eb, radius, cfg.padding, out=y, result=res, check=False)

    for _ in range(2):
        comp()
        decomp()
    tc, kc = timed(comp, flush, reps)
    td, kd = timed(decomp, flush, reps)
    # the same calls captured once into CUDA graphs (launch overhead removed;
    # SURVEY 8d asks for this on the launch-bound small configs)
    graphs = {}
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        comp()
        decomp()
    torch.cuda.current_stream().wait_stream(side)
    for ph, fn in (("compress", comp), ("decompress", decomp)):
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            fn()
        graphs[ph] = gr
    tg = {}
    for ph, gr in graphs.items():
        ts = []
        for _ in range(reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            gr.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        tg[ph] = statistics.median(ts)
    n = data.size
    alg = 6 * n + 4 * n_out + 8 * dev.grid.block_count
    print(json.dumps(dict(
        case=name, shape=list(data.shape), block=b, padding=pol, radius=radius,
        outliers=n_out, outlier_frac=n_out / n,
        compress_gbs=4 * n / tc / 1e6, decompress_gbs=4 * n / td / 1e6,
        compress_ms=tc, decompress_ms=td,
        graph_compress_ms=tg["compress"], graph_decompress_ms=tg["decompress"],
        graph_compress_gbs=4 * n / tg["compress"] / 1e6,
        graph_decompress_gbs=4 * n / tg["decompress"] / 1e6,
        fused_compress_tbs=alg / (kc["compress"] * 1e-3) / 1e12 if kc["compress"] else None,
        fused_decompress_tbs=alg / (kd["decompress"] * 1e-3) / 1e12 if kd["decompress"] else None,
        kernels_compress=kc, kernels_decompress=kd)), flush=True)


def main():
    which = sys.argv[1:] or ["C1", "C2", "C3", "C4", "stress"]
    if "C1" in which:
        c1 = workloads.gen_c1()
        run("C1 b=256", c1, 1e-4, 256, "zero", 512)
        run("C1 b=64", c1, 1e-4, 64, "zero", 512)
    if "C2" in which:
        c2 = workloads.gen_c2()
        run("C2 zero", c2, 1e-4, 16, "zero", 512)
        run("C2 mean:block", c2, 1e-4, 16, "mean:block", 512)
    if "C3" in which:
        c3 = workloads.gen_c3()
        run("C3 mean:global", c3, 1e-3, 8, "mean:global", 512)
    if "C4" in which:
        c4 = workloads.gen_c4(512)
        run("C4 b=8 R=512", c4, 1e-3, 8, "mean:global", 512)
        run("C4 b=16 R=32768", c4, 1e-3, 16, "mean:global", 32768)
    if "1D" in which:  # large 1-D stream (C1 recipe at 256 M elements)
        rng = np.random.default_rng(5)
        n = 256 * 1024 * 1024
        walk = np.cumsum(rng.normal(0, 1, n).astype(np.float32)) * np.float32(0.01)
        big = (walk + np.sin(np.arange(n, dtype=np.float32) * np.float32(2 * np.pi / 4096)))
        big = big.astype(np.float32)
        run("1D 256M b=256", big, 1e-4, 256, "zero", 512)
        run("1D 256M b=64 mean:global", big, 1e-4, 64, "mean:global", 512)
    if "2D" in which:  # large 2-D field (C2 recipe at 16384 x 16384)
        rng = np.random.default_rng(6)
        y, x = np.meshgrid(np.linspace(0, 1, 16384, dtype=np.float32),
                           np.linspace(0, 1, 16384, dtype=np.float32), indexing="ij")
        f = np.zeros((16384, 16384), np.float32)
        for _ in range(8):
            ky, kx = rng.integers(1, 16, 2)
            f += np.sin(2 * np.pi * (ky * y + kx * x) + rng.uniform(0, 6.28)).astype(np.float32)
        run("2D 16384^2 b=16 mean:block", f, 1e-4, 16, "mean:block", 512)
        run("2D 16384^2 b=8 zero", f, 1e-4, 8, "zero", 512)
    if "big" in which:  # block edges 32 / 64 (tools/bench_bigblocks.py cases)
        c4 = workloads.gen_c4(512)
        for b in (32, 64):
            run(f"C4 512^3 b={b}", c4, 1e-3, b, "mean:global", 512)
        rng = np.random.default_rng(6)
        y, x = np.meshgrid(np.linspace(0, 1, 8192, dtype=np.float32),
                           np.linspace(0, 1, 8192, dtype=np.float32), indexing="ij")
        f = np.zeros((8192, 8192), np.float32)
        for _ in range(8):
            ky, kx = rng.integers(1, 16, 2)
            f += np.sin(2 * np.pi * (ky * y + kx * x) + rng.uniform(0, 6.28)).astype(np.float32)
        for b in (32, 64):
            run(f"2D 8192^2 b={b}", f, 1e-4, b, "mean:block", 512)
    if "stress" in which:
        c4 = workloads.gen_c4(256)
        run("stress b=8 R=512 eb=1e-5", c4, 1e-5, 8, "mean:global", 512)


if __name__ == "__main__":
    main()
