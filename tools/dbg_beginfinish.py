import ctypes, torch, numpy as np, sys
sys.path.insert(0, '.')
from paper_2201_04614_b200 import _lib, workloads, model as M
lib = _lib.load()
dev = torch.device('cuda', 0)
x = workloads.gen_c5_slab((0, 64), dev, shape=(64, 2048, 1024))
eb = 1e-4 * (x.max().item() - x.min().item())
g = _lib.geom(x.shape, 8); p = _lib.params(eb, 512, 3, 0)
n = x.numel(); nb = lib.vlz_block_count(ctypes.byref(g))
codes = torch.empty(n, dtype=torch.int16, device=dev); outl = torch.empty(n, device=dev)
counts = torch.empty(nb, dtype=torch.int64, device=dev); sc = torch.empty(1, dtype=torch.int64, device=dev)
res = torch.full((8,), -7, dtype=torch.int64, device=dev); stats = torch.empty(4, dtype=torch.int64, device=dev)
wsb = lib.vlz_workspace_size(ctypes.byref(g)); ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
sp = torch.cuda.current_stream().cuda_stream
print('begin', lib.vlz_dq_compress_begin(x.data_ptr(), ctypes.byref(g), ctypes.byref(p), codes.data_ptr(), counts.data_ptr(), sc.data_ptr(), res.data_ptr(), stats.data_ptr(), ws.data_ptr(), wsb, sp))
torch.cuda.synchronize(); print('after begin res', res.tolist(), 'stats', stats.tolist())
print('finish', lib.vlz_dq_compress_finish(x.data_ptr(), ctypes.byref(g), ctypes.byref(p), stats.data_ptr(), codes.data_ptr(), outl.data_ptr(), counts.data_ptr(), sc.data_ptr(), res.data_ptr(), ws.data_ptr(), wsb, sp))
torch.cuda.synchronize(); print('after finish res', res.tolist(), 'sc', sc.tolist(), 'counts sum', counts.sum().item())
