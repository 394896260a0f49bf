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
# fused 1-D kernels (bulk-copy ring; >= 4 M elements), b = 32/64 fast kernels,
# the int64 redo path and an outlier-heavy field
M.allow_block_256(True)
x1 = (np.cumsum(rng.normal(0, 1, 1 << 22)) * 0.01).astype(np.float32)
x1[rng.random(x1.size) < 0.01] = 50.0
for b, pol in ((256, "zero"), (64, "mean:global")):
    cfg = M.CompressionConfig(M.ErrorBound.absolute(1e-3), block_edge=b, radius=512,
                              padding=M.PaddingPolicy.parse(pol))
    back, _ = vlzg.decompress(vlzg.compress(x1, cfg))
    assert np.max(np.abs(back.astype(np.float64) - x1)) <= 1e-3
M.allow_block_256(False)
for shape, b in (((64, 64, 128), 64), ((32, 64, 128), 32), ((64, 256), 64)):
    idx = np.indices(shape).astype(np.float64)
    data = (sum(np.sin(0.05 * (k + 1) * idx[k]) for k in range(len(shape))) * 10
            + rng.normal(0, 0.05, shape)).astype(np.float32)
    for eb in (1e-2, 1e-4):  # 1e-4: many outliers at radius 64
        cfg = M.CompressionConfig(M.ErrorBound.absolute(eb), block_edge=b, radius=64,
                                  padding=M.PaddingPolicy.parse("mean:block"))
        back, _ = vlzg.decompress(vlzg.compress(data, cfg))
        assert np.max(np.abs(back.astype(np.float64) - data)) <= eb
big = (rng.uniform(-1, 1, (40, 33, 70)) * 1.0e9).astype(np.float32)  # int64 redo
cfg = M.CompressionConfig(M.ErrorBound.absolute(1.0), block_edge=8, radius=512)
back, _ = vlzg.decompress(vlzg.compress(big, cfg))
assert np.max(np.abs(back.astype(np.float64) - big)) <= 1.0
# crafted containers (over-subscribed codebooks, short padding sections)
import json  # noqa: E402

with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests",
                       "golden", "container_full.json")) as fh:
    for c in json.load(fh):
        try:
            vlzg.decompress(bytes.fromhex(c["blob"]))
        except Exception:  # noqa: BLE001 -- verdicts are checked by the tests
            pass
torch.cuda.synchronize()
print("sanitize workload ok")
