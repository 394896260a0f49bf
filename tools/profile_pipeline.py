"""cProfile of compress()/decompress() on a BASELINE config (stage costs)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2201_04614_b200 as vlzg  # noqa: E402
from paper_2201_04614_b200 import model as M  # noqa: E402
from paper_2201_04614_b200 import workloads  # noqa: E402

data = workloads.gen_c4(512)
eb = workloads.value_range_eb(data, 1e-3)
cfg = M.CompressionConfig(M.ErrorBound.absolute(eb), block_edge=8, radius=512,
                          padding=M.PaddingPolicy.parse("mean:global"))
blob = vlzg.compress(data, cfg)
vlzg.decompress(blob)
torch.cuda.synchronize()
for name, fn in (("compress", lambda: vlzg.compress(data, cfg)),
                 ("decompress", lambda: vlzg.decompress(blob))):
    pr = cProfile.Profile()
    pr.enable()
    fn()
    pr.disable()
    print("=====", name)
    pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
