"""One warm 1-D compress + decompress of a 256 M-element random walk on
cuda:0 (workload for ncu captures of the fused 1-D kernels).
usage: python tools/run_1d.py [block_edge] [padding] [n]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2201_04614_b200 import gpu  # noqa: E402
from paper_2201_04614_b200 import model as M  # noqa: E402

b = int(sys.argv[1]) if len(sys.argv) > 1 else 256
pol = sys.argv[2] if len(sys.argv) > 2 else "zero"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 256 * 1024 * 1024
M.allow_block_256(True)
g = torch.Generator(device="cuda").manual_seed(5)
x = (torch.randn(n, device="cuda", generator=g) * 0.01).cumsum(0)
x += torch.sin(torch.arange(n, device="cuda", dtype=torch.float32) * (2 * 3.14159265 / 4096))
x = x.float().contiguous()
eb = 1e-4 * float(x.max() - x.min())
cfg = M.CompressionConfig(M.ErrorBound.absolute(eb), block_edge=b,
                          padding=M.PaddingPolicy.parse(pol), radius=512)
for _ in range(2):
    dev = gpu.compress_device(x, cfg, eb=eb).check()
    y = gpu.decompress_device(dev.codes, dev.outliers, dev.n_outliers, dev.counts, dev.scalars,
                              dev.grid, eb, 512, cfg.padding)
torch.cuda.synchronize()
err = (y - x).abs().max().item()
print(f"1-D n={n} b={b} {pol}: outliers {dev.n_outliers}, max err {err:.3g} (eb {eb:.3g})")
assert err <= eb
