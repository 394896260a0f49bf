"""Golden vectors for the autotune host logic, produced by the REFERENCE
(run in the build container, where /root/reference exists):

    python tests/golden/make_golden_autotune.py

Records TuneSpace.build, sample_blocks picks, narrowed_autotune and
TuneReport.csv_rows of /root/reference/pkg/src/vlz/autotune.py into
tests/golden/autotune.json."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from vlz.autotune import TuneReport, TuneSpace, narrowed_autotune, sample_blocks  # noqa: E402
from vlz.model import ArrayDescriptor, build_block_grid  # noqa: E402

out = {"spaces": [], "samples": [], "narrowed": [], "csv": None}
for edges, lanes in [((8, 16, 32, 64), (4, 8, 16)), ((8, 16, 32), (4, 8)), ((16,), (16,))]:
    out["spaces"].append({"edges": edges, "lanes": lanes,
                          "configs": TuneSpace.build(edges, lanes).configs})
for shape, b, frac, seed in [((1000,), 8, 0.1, 1), ((33, 47), 16, 0.25, 7),
                              ((20, 17, 9), 8, 0.5, 3), ((64, 64, 64), 32, 0.1, 11),
                              ((5,), 64, 1.0, 0)]:
    grid = build_block_grid(ArrayDescriptor(len(shape), tuple(shape)), b)
    out["samples"].append({"shape": shape, "b": b, "fraction": frac, "seed": seed,
                           "picks": sample_blocks(grid, frac, seed).tolist()})
space = TuneSpace.build()
for hist, k in [([(8, 8), (16, 8), (8, 8), (32, 16)], 2), ([(64, 16), (16, 4)], 1),
                ([], 2), ([(8, 16)], 2), ([(32, 4), (32, 8), (16, 16), (16, 16)], 3)]:
    out["narrowed"].append({"history": hist, "k": k,
                            "configs": narrowed_autotune(hist, space, k).configs})
rep = TuneReport(configs=((8, 4), (8, 8), (16, 4)), mean_s=(1e-3, 2.5e-4, 7e-6),
                 std_s=(0.0, 1e-5, 3e-9), chosen=(16, 4), sample_fraction=0.1,
                 iterations=3, seed=1, tuning_seconds=0.5)
out["csv"] = {"report": {k: getattr(rep, k) for k in ("configs", "mean_s", "std_s", "chosen")},
              "rows": rep.csv_rows()}
with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "autotune.json"), "w") as f:
    json.dump(out, f, indent=1)
