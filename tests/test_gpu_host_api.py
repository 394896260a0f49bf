"""The host-buffer C entry points (chunked H2D/compute/D2H pipeline) give
exactly the device entry points' results, including *:global padding with a
non-zero scalar (origin patches) and corrupt-stream verdicts."""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2201_04614_b200 import _lib, gpu, workloads  # noqa: E402
from paper_2201_04614_b200 import model as M  # noqa: E402
from paper_2201_04614_b200.errors import CorruptStreamError  # noqa: E402
from paper_2201_04614_b200.reconstruct import reconstruct_arrays  # noqa: E402


def _host_compress(data, eb, b, pol, radius):
    lib = _lib.load()
    p = M.PaddingPolicy.parse(pol)
    grid = M.build_block_grid(M.ArrayDescriptor(data.ndim, data.shape), b)
    g = _lib.geom(data.shape, b)
    pr = _lib.params(eb, radius, p.kind_code, p.gran_code)
    n = data.size
    codes = np.empty(n, np.uint16)
    outl = np.empty(n, np.float32)
    counts = np.empty(grid.block_count, np.int64)
    scal = np.empty(max(p.scalar_count(grid), 1), np.int64)
    r = _lib.Result()
    rc = lib.vlz_dq_compress_host(np.ascontiguousarray(data).ctypes.data, ctypes.byref(g),
                                  ctypes.byref(pr), codes.ctypes.data, outl.ctypes.data,
                                  counts.ctypes.data, scal.ctypes.data, ctypes.byref(r), 0)
    assert rc == 0
    return codes, outl[: r.n_outliers], counts, scal[: p.scalar_count(grid)], r


def _device_compress(data, eb, b, pol, radius):
    cfg = M.CompressionConfig(M.ErrorBound.absolute(eb), block_edge=b,
                              padding=M.PaddingPolicy.parse(pol), radius=radius)
    d = gpu.compress_device(torch.from_numpy(data).cuda(), cfg, eb=eb).check()
    n = d.n_outliers
    return (d.codes.cpu().numpy().view(np.uint16), d.outliers[:n].cpu().numpy(),
            d.counts.cpu().numpy(), d.scalars.cpu().numpy())


@pytest.mark.parametrize("pol", ["mean:global", "max:global", "zero", "min:block", "mean:edge"])
def test_host_pipeline_equals_device(pol):
    # 200 x 256 x 512 float32 = 105 MB -> several 64 MB chunks; offset data so
    # the global mean (s0) is far from 0 and origins need patching
    d = workloads.gen_c3(shape=(200, 64, 128))
    d = np.tile(d, (1, 4, 4)) + np.float32(37.25)
    eb = workloads.value_range_eb(d, 1e-4)
    hc, ho, hn, hs, r = _host_compress(d, eb, 8, pol, 512)
    dc, do, dn, ds = _device_compress(d, eb, 8, pol, 512)
    assert r.status == 0
    assert hc.tobytes() == dc.tobytes()
    assert ho.tobytes() == do.tobytes()
    assert hn.tobytes() == dn.tobytes()
    assert hs.tobytes() == ds.tobytes()
    # decompress through the host pipeline == device reconstruct
    lib = _lib.load()
    p = M.PaddingPolicy.parse(pol)
    g = _lib.geom(d.shape, 8)
    pr = _lib.params(eb, 512, p.kind_code, p.gran_code)
    out = np.empty(d.shape, np.float32)
    rd = _lib.Result()
    rc = lib.vlz_dq_decompress_host(hc.ctypes.data, ho.ctypes.data, ho.size, hn.ctypes.data,
                                    hs.ctypes.data if hs.size else None, ctypes.byref(g),
                                    ctypes.byref(pr), out.ctypes.data, ctypes.byref(rd), 0)
    assert rc == 0 and rd.status == 0
    grid = M.build_block_grid(M.ArrayDescriptor(3, d.shape), 8)
    ref = reconstruct_arrays(dc, do, dn, ds, grid, eb, 512, p)
    assert out.tobytes() == ref.tobytes()
    assert np.abs(out.astype(np.float64) - d.astype(np.float64)).max() <= eb


def test_host_decompress_reports_first_failing_block():
    d = (workloads.gen_c3(shape=(150, 64, 128)) * 3).astype(np.float32)
    eb = workloads.value_range_eb(d, 1e-4)
    hc, ho, hn, hs, _ = _host_compress(d, eb, 8, "mean:block", 512)
    nz = np.flatnonzero(hn)
    assert nz.size >= 2
    bad = hn.copy()
    bad[nz[-1]] += 1  # leftover / exhaustion in a late block (later chunk)
    bad[nz[-2]] -= 1
    lib = _lib.load()
    g = _lib.geom(d.shape, 8)
    pr = _lib.params(eb, 512, 3, 1)
    out = np.empty(d.shape, np.float32)
    rd = _lib.Result()
    rc = lib.vlz_dq_decompress_host(hc.ctypes.data, ho.ctypes.data, ho.size, bad.ctypes.data,
                                    hs.ctypes.data, ctypes.byref(g), ctypes.byref(pr),
                                    out.ctypes.data, ctypes.byref(rd), 0)
    assert rc == 0
    assert rd.status in (5, 6) and rd.index == nz[-2]
    grid = M.build_block_grid(M.ArrayDescriptor(3, d.shape), 8)
    with pytest.raises(CorruptStreamError):
        reconstruct_arrays(hc, ho, bad, hs, grid, eb, 512, M.PaddingPolicy.parse("mean:block"))


def test_host_calls_from_concurrent_threads():
    """Compress and decompress issued from several host threads at once (each
    on its own pooled context) give exactly the serial results."""
    import threading

    d = workloads.gen_c3(shape=(96, 64, 128)) + np.float32(11.5)
    eb = workloads.value_range_eb(d, 1e-4)
    hc, ho, hn, hs, _ = _host_compress(d, eb, 8, "mean:global", 512)
    lib = _lib.load()
    g = _lib.geom(d.shape, 8)
    pr = _lib.params(eb, 512, 3, 0)
    want = np.empty(d.shape, np.float32)
    rd = _lib.Result()
    assert lib.vlz_dq_decompress_host(hc.ctypes.data, ho.ctypes.data, ho.size, hn.ctypes.data,
                                      hs.ctypes.data, ctypes.byref(g), ctypes.byref(pr),
                                      want.ctypes.data, ctypes.byref(rd), 0) == 0
    errs = []

    def worker(k):
        try:
            for _ in range(3):
                if k % 2 == 0:
                    c2, o2, n2, s2, r2 = _host_compress(d, eb, 8, "mean:global", 512)
                    assert r2.status == 0
                    assert c2.tobytes() == hc.tobytes() and o2.tobytes() == ho.tobytes()
                    assert n2.tobytes() == hn.tobytes() and s2.tobytes() == hs.tobytes()
                else:
                    out = np.empty(d.shape, np.float32)
                    r3 = _lib.Result()
                    rc = lib.vlz_dq_decompress_host(hc.ctypes.data, ho.ctypes.data, ho.size,
                                                    hn.ctypes.data, hs.ctypes.data,
                                                    ctypes.byref(g), ctypes.byref(pr),
                                                    out.ctypes.data, ctypes.byref(r3), 0)
                    assert rc == 0 and r3.status == 0
                    assert out.tobytes() == want.tobytes()
        except BaseException as e:  # reported below
            errs.append(e)

    th = [threading.Thread(target=worker, args=(k,)) for k in range(6)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    lib.vlz_host_release()
    assert not errs, errs[0]
