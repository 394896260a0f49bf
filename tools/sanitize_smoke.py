"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck): every kernel family once on small shapes, incl. edge tiles, the
TMA decompress, *:global origins, outliers, the entropy stage and the border
census."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2201_04614_b200 as vlzg  # noqa: E402
from paper_2201_04614_b200 import model as M  # noqa: E402
from paper_2201_04614_b200.padding import outlier_report  # noqa: E402

rng = np.random.default_rng(0)
cases = [((64,), 8), ((1000,), 64), ((24, 40), 8), ((36, 72), 16), ((16, 16, 256), 8),
         ((13, 21, 132), 8), ((16, 32, 64), 16), ((9, 20, 30), 8), ((48, 64, 128), 8)]
for shape, b in cases:
    idx = np.indices(shape).astype(np.float64)
    data = sum(np.sin(0.1 * (k + 1) * idx[k]) * 30 for k in range(len(shape)))
    data = (data + rng.normal(0, 0.2, shape)).astype(np.float32)
    for pol in ("zero", "mean:global", "max:block", "min:edge"):
        cfg = M.CompressionConfig(M.ErrorBound.absolute(1e-2), block_edge=b, radius=64,
                                  padding=M.PaddingPolicy.parse(pol))
        blob = vlzg.compress(data, cfg)
        back, _ = vlzg.decompress(blob)
        assert np.max(np.abs(back.astype(np.float64) - data)) <= 1e-2
    if len(shape) > 1:
        outlier_report(data, M.CompressionConfig(M.ErrorBound.absolute(1e-2), block_edge=b,
                                                 radius=64))
torch.cuda.synchronize()
print("sanitize workload ok")
