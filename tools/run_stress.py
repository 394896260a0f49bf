"""One compress + decompress of the outlier-stress field (C4 recipe at 256^3,
eb = 1e-5 * range, b=8, R=512, mean:global: ~18 % outliers), for ncu
captures of the sentinel-heavy decompress path."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2201_04614_b200 import gpu, workloads  # noqa: E402
from paper_2201_04614_b200 import model as M  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
data = workloads.gen_c4(n)
eb = workloads.value_range_eb(data, 1e-5)
cfg = M.CompressionConfig(M.ErrorBound.absolute(eb), block_edge=8, radius=512)
x = torch.from_numpy(data).cuda()
for _ in range(reps):
    s = gpu.compress_device(x, cfg, eb=eb).check()
    y = gpu.decompress_device(s.codes, s.outliers, s.n_outliers, s.counts, s.scalars, s.grid, eb,
                              512, cfg.padding)
torch.cuda.synchronize()
assert float((y.double() - x.double()).abs().max()) <= eb
print(f"stress {n}^3: {s.n_outliers} outliers ({s.n_outliers / data.size:.3f})")
