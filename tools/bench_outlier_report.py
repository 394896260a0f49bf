"""outlier_report: one-pass census (paper_2201_04614_b200.padding) vs the
reference's structure restated on the GPU path (one dualquant_vector per
policy, each with its own host->device copy).  Prints one JSON line per
shape; both give the same rows (checked)."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2201_04614_b200 import model as M  # noqa: E402
from paper_2201_04614_b200 import workloads  # noqa: E402
from paper_2201_04614_b200.padding import outlier_report  # noqa: E402
from paper_2201_04614_b200.vector import dualquant_vector  # noqa: E402


def per_policy(data, cfg):
    rows = []
    pols = [M.PaddingPolicy(M.PaddingValue.ZERO)] + [
        M.PaddingPolicy(k, g) for k in (M.PaddingValue.MINIMUM, M.PaddingValue.MAXIMUM,
                                        M.PaddingValue.MEAN) for g in M.PaddingGranularity]
    for pol in pols:
        c = M.CompressionConfig(cfg.error_bound, block_edge=cfg.block_edge, padding=pol,
                                radius=cfg.radius)
        _, (t, b) = dualquant_vector(data, c, collect_border=True)
        rows.append((t, b))
    return rows


for name, data, rel in (("C3", workloads.gen_c3(), 1e-3), ("C4", workloads.gen_c4(512), 1e-3),
                        ("C2", workloads.gen_c2(), 1e-4)):
    eb = workloads.value_range_eb(data, rel)
    b = 16 if data.ndim == 2 else 8
    cfg = M.CompressionConfig(M.ErrorBound.absolute(eb), block_edge=b, radius=512)
    outlier_report(data, cfg)
    per_policy(data, cfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    new = outlier_report(data, cfg)
    t1 = time.perf_counter()
    old = per_policy(data, cfg)
    t2 = time.perf_counter()
    assert [(r.total_outliers, r.border_outliers) for r, _ in new] == old
    print(json.dumps({"case": name, "shape": list(data.shape), "census_ms": (t1 - t0) * 1e3,
                      "per_policy_ms": (t2 - t1) * 1e3, "speedup": (t2 - t1) / (t1 - t0)}),
          flush=True)
