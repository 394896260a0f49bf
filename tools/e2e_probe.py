"""Concurrency probe of the host entry points: compress_host and
decompress_host of a 2 GiB slab, alone and from two threads at once."""
import ctypes
import os
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2201_04614_b200 import _lib  # noqa: E402
from paper_2201_04614_b200 import model as M  # noqa: E402

shape = (int(sys.argv[1]) if len(sys.argv) > 1 else 256, 2048, 1024)
K = int(sys.argv[2]) if len(sys.argv) > 2 else 6
n = int(np.prod(shape))
x = torch.linspace(0, 50, n, device="cuda").sin_().reshape(shape)
h_in = torch.empty(shape, dtype=torch.float32, pin_memory=True)
h_in.copy_(x)
del x
torch.cuda.empty_cache()
lib = _lib.load()
eb = 1e-4
grid = M.build_block_grid(M.ArrayDescriptor(3, shape), 8)
g = _lib.geom(shape, 8)
p = _lib.params(eb, 512, 3, 0)
bufs = [dict(codes=torch.empty(n, dtype=torch.int16, pin_memory=True),
             out=torch.empty(n, dtype=torch.float32, pin_memory=True),
             cnt=torch.empty(grid.block_count, dtype=torch.int64, pin_memory=True),
             sc=torch.empty(1, dtype=torch.int64, pin_memory=True),
             back=torch.empty(shape, dtype=torch.float32, pin_memory=True),
             r=_lib.Result(), rd=_lib.Result()) for _ in range(2)]


def comp(b):
    assert lib.vlz_dq_compress_host(h_in.data_ptr(), ctypes.byref(g), ctypes.byref(p),
                                    b["codes"].data_ptr(), b["out"].data_ptr(), b["cnt"].data_ptr(),
                                    b["sc"].data_ptr(), ctypes.byref(b["r"]), 0) == 0


def decomp(b):
    assert lib.vlz_dq_decompress_host(b["codes"].data_ptr(), b["out"].data_ptr(), b["r"].n_outliers,
                                      b["cnt"].data_ptr(), b["sc"].data_ptr(), ctypes.byref(g),
                                      ctypes.byref(p), b["back"].data_ptr(), ctypes.byref(b["rd"]),
                                      0) == 0


comp(bufs[0])
comp(bufs[1])
decomp(bufs[0])
decomp(bufs[1])


def loop(fn, b):
    for _ in range(K):
        fn(b)


for name, jobs in [("compress alone", [(comp, bufs[0])]), ("decompress alone", [(decomp, bufs[1])]),
                   ("compress || decompress", [(comp, bufs[0]), (decomp, bufs[1])]),
                   ("compress || compress", [(comp, bufs[0]), (comp, bufs[1])])]:
    th = [threading.Thread(target=loop, args=j) for j in jobs]
    t = time.perf_counter()
    for x_ in th:
        x_.start()
    for x_ in th:
        x_.join()
    dt = (time.perf_counter() - t) / K
    print(f"{shape[0]} planes chunk {os.environ.get('VLZ_CHUNK_MB', '64')} MB: {name:26s} "
          f"{dt * 1e3:7.1f} ms per iteration ({len(jobs)} calls)", flush=True)
