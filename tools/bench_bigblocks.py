"""Large-block (b=32/64) 2-D and 3-D throughput through tools/bench_configs.run."""
import sys, json
sys.path.insert(0, '.')
sys.argv = ['x']
import tools.bench_configs as bc
from paper_2201_04614_b200 import workloads
import numpy as np
c4 = workloads.gen_c4(512)
for b in (32, 64):
    bc.run(f"C4 512^3 b={b}", c4, 1e-3, b, "mean:global", 512)
rng = np.random.default_rng(6)
y, x = np.meshgrid(np.linspace(0, 1, 8192, dtype=np.float32), np.linspace(0, 1, 8192, dtype=np.float32), indexing="ij")
f = np.zeros((8192, 8192), np.float32)
for _ in range(8):
    ky, kx = rng.integers(1, 16, 2)
    f += np.sin(2 * np.pi * (ky * y + kx * x) + rng.uniform(0, 6.28)).astype(np.float32)
for b in (32, 64):
    bc.run(f"2D 8192^2 b={b}", f, 1e-4, b, "mean:block", 512)
