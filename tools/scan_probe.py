import ctypes, sys, os, torch
sys.path.insert(0, os.getcwd())
from paper_2201_04614_b200 import _lib, gpu, workloads
from paper_2201_04614_b200 import model as M
dev = torch.device("cuda", 0)
x = workloads.gen_c5_slab(z_range=(0, 1024), device=dev, shape=(1024, 2048, 1024))
lib = _lib.load()
mm = torch.empty(2, dtype=torch.float64, device=dev)
lib.vlz_minmax(x.data_ptr(), x.numel(), mm.data_ptr(), None)
lo, hi = mm.tolist(); eb = 1e-4 * (hi - lo)
cfg = M.CompressionConfig(M.ErrorBound.absolute(eb), block_edge=8, radius=512, padding=M.PaddingPolicy.parse("mean:global"))
out = gpu.compress_device(x, cfg, eb=eb)
torch.cuda.synchronize()
kms = (ctypes.c_double * 8)(); kc = (ctypes.c_int64 * 8)()
for i in range(3):
    lib.vlz_timing(1); gpu.compress_device(x, cfg, eb=eb, out=out); torch.cuda.synchronize(); lib.vlz_timing(0)
    lib.vlz_timing_collect(kms, kc, 8)
    print("scan_c", kms[2], "compress", kms[1], "n_out", out.n_outliers)
