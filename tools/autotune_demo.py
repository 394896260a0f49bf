"""GPU autotune on a seeded 3-D field: prints the TuneReport CSV rows
(reference autotune.py TUNE_CSV_FIELDS) and the chosen configuration."""
import json
import sys
import os

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2201_04614_b200.autotune import TUNE_CSV_FIELDS, TuneSpace, autotune  # noqa: E402
from paper_2201_04614_b200.model import CompressionConfig, ErrorBound  # noqa: E402

shape = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "512,512,512").split(","))
g = torch.Generator(device="cuda").manual_seed(0)
z, y, x = torch.meshgrid(*[torch.linspace(0, 6.28, n, device="cuda") for n in shape], indexing="ij")
data = (torch.sin(3 * z) * torch.cos(2 * y) + torch.sin(5 * x)
        + 1e-3 * torch.randn(shape, device="cuda", generator=g)).float().contiguous()
rep = autotune(data, TuneSpace.build(), fraction=0.10, iterations=5,
               base=CompressionConfig(ErrorBound.relative(1e-4), radius=512))
print(",".join(TUNE_CSV_FIELDS))
for r in rep.csv_rows():
    print(",".join(str(v) for v in r))
print(json.dumps({"shape": shape, "chosen": rep.chosen, "tuning_seconds": rep.tuning_seconds}))
