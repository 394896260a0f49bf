"""Parity of the CUDA path (libvlzgpu.so) with the reference.

* golden corpus: byte equality with streams and decompressed arrays produced
  by the reference itself (tests/golden/make_golden.py);
* full size (BASELINE.json C1-C4): equality with the reference's sha256 (C1,
  C2) or with the pinned CPU oracle (C3, C4, outlier stress), plus the
  size-independent properties: error bound, exact round trip, idempotent
  recompression.
All calls go through the C ABI (ctypes), no CPU fallback exists."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import load_json

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2201_04614_b200 import gpu, workloads  # noqa: E402
from paper_2201_04614_b200 import model as M  # noqa: E402
from paper_2201_04614_b200.errors import (  # noqa: E402
    BoundTooSmallError,
    ConfigError,
    CorruptStreamError,
    DegenerateRangeError,
)
from paper_2201_04614_b200.reconstruct import reconstruct_arrays, reconstruct_stream  # noqa: E402
from paper_2201_04614_b200.vector import dualquant, dualquant_vector  # noqa: E402



@pytest.fixture(autouse=True)
def _allow_256():
    # the golden generator allowed block 256 (BASELINE config 1); per test,
    # so other modules' settings cannot leak in
    prev = M.valid_block_edges()
    M.allow_block_256(True)
    yield
    M.allow_block_256(256 in prev)


def _cfg(eb, b, pol, radius, lanes=8):
    return M.CompressionConfig(M.ErrorBound.absolute(eb), block_edge=b, lane_width=lanes,
                               padding=M.PaddingPolicy.parse(pol), radius=radius)


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_corpus_compress_matches_reference(corpus_cases):
    for c in corpus_cases:
        s = dualquant_vector(c["data"], _cfg(c["eb"], c["block_edge"], c["padding"], c["radius"]))
        tag = c["tag"]
        assert s.codes.dtype == np.uint32
        assert np.array_equal(s.codes, c["codes"].astype(np.uint32)), tag
        assert s.outlier_values.tobytes() == c["outlier_values"].tobytes(), tag
        assert np.array_equal(s.outlier_counts, c["outlier_counts"]), tag
        assert np.array_equal(s.scalars.values, c["scalars"]), tag


def test_corpus_decompress_matches_reference(corpus_cases):
    n = 0
    for c in corpus_cases:
        if "decompressed" not in c:
            continue
        grid = M.build_block_grid(M.ArrayDescriptor(len(c["shape"]), tuple(c["shape"])),
                                  c["block_edge"])
        for codes in (c["codes"], c["codes"].astype(np.uint32)):  # u16 and u32 kernels
            out = reconstruct_arrays(codes, c["outlier_values"], c["outlier_counts"],
                                     c["scalars"], grid, c["eb"], c["radius"],
                                     M.PaddingPolicy.parse(c["padding"]))
            assert out.tobytes() == c["decompressed"].tobytes(), c["tag"]
        n += 1
    assert n > 50


def test_corpus_round_trip_matches_oracle(oracle, corpus_cases):
    for c in corpus_cases:
        grid = M.build_block_grid(M.ArrayDescriptor(len(c["shape"]), tuple(c["shape"])),
                                  c["block_edge"])
        out = reconstruct_arrays(c["codes"], c["outlier_values"], c["outlier_counts"],
                                 c["scalars"], grid, c["eb"], c["radius"],
                                 M.PaddingPolicy.parse(c["padding"]))
        ref = oracle.reconstruct(c["codes"].astype(np.uint32), c["outlier_values"],
                                 c["outlier_counts"], c["scalars"], tuple(c["shape"]),
                                 c["block_edge"], c["eb"], c["radius"], c["padding"])
        assert out.tobytes() == ref.tobytes(), c["tag"]
        err = np.abs(out.astype(np.float64) - c["data"].astype(np.float64))
        assert err.max(initial=0.0) <= c["eb"], c["tag"]


def test_error_cases():
    # vector-path cases go through dualquant_vector; lane-width-1 cases
    # (scalar kernel order, kernel.py:138-145) through compress() at lane 1
    # -- the reference's pipeline.py:28-31 dispatch -- and dualquant_scalar
    import paper_2201_04614_b200 as vlzg
    from paper_2201_04614_b200.vector import dualquant_scalar

    n_lane1 = 0
    for c in load_json("errors.json"):
        data = np.array(c["data"], dtype=np.float32).reshape(c["shape"])
        exp = c["expect"]
        lane = c.get("lane", 8)
        if c["eb"] is None:
            cfg = M.CompressionConfig(M.ErrorBound.relative(c["rel"]), block_edge=c["block_edge"],
                                      lane_width=lane)
        else:
            cfg = M.CompressionConfig(M.ErrorBound.absolute(c["eb"]), block_edge=c["block_edge"],
                                      lane_width=lane, padding=M.PaddingPolicy.parse(c["padding"]),
                                      radius=32768)
        calls = [dualquant_vector] if lane != 1 else [vlzg.compress, dualquant_scalar]
        n_lane1 += lane == 1
        for fn in calls:
            if exp is None:
                fn(data, cfg)
                continue
            cls = {"ConfigError": ConfigError, "BoundTooSmallError": BoundTooSmallError,
                   "DegenerateRangeError": DegenerateRangeError}[exp["type"]]
            with pytest.raises(cls) as err:
                fn(data, cfg)
            assert str(err.value) == exp["message"], (c["tag"], fn.__name__)
            assert type(err.value) is cls
            if cls is BoundTooSmallError:
                assert (err.value.index, err.value.value, err.value.bound) == (
                    exp["index"], exp["value"], exp["bound"]), c["tag"]
    assert n_lane1 >= 5


def test_corrupt_streams(corrupt_cases):
    for c in corrupt_cases:
        grid = M.build_block_grid(M.ArrayDescriptor(len(c["shape"]), tuple(c["shape"])),
                                  c["block_edge"])
        with pytest.raises(CorruptStreamError) as err:
            reconstruct_arrays(c["codes"], c["outlier_values"], c["outlier_counts"], c["scalars"],
                               grid, c["eb"], c["radius"], M.PaddingPolicy.parse(c["padding"]))
        assert str(err.value) == c["expect"]["message"], c["tag"]


def test_lane_width_rules():
    data = np.zeros(8, dtype=np.float32)
    with pytest.raises(ConfigError):
        dualquant_vector(data, M.CompressionConfig(M.ErrorBound.absolute(1e-4), lane_width=1))
    d = np.random.default_rng(0).uniform(-10, 10, (20, 12)).astype(np.float32)
    ref = dualquant(d, _cfg(1e-4, 8, "mean:global", 32768, lanes=1))
    for lanes in (4, 8, 16):
        assert dualquant_vector(d, _cfg(1e-4, 8, "mean:global", 32768, lanes)).same_bytes(ref)


def test_border_stats_constant_field():
    data = np.full((16, 16), 100.0, dtype=np.float32)
    _, (total, border) = dualquant_vector(data, _cfg(1e-4, 8, "zero", 32768), collect_border=True)
    assert total == 4 and border == 4


# ---------------------------------------------------------------- full size


def _check_full(oracle, data, eb, b, pol, radius, ref_hashes=None):
    cfg = _cfg(eb, b, pol, radius)
    s = dualquant(data, cfg)
    if ref_hashes is not None:
        assert _sha(s.codes.astype(np.uint16)) == ref_hashes["codes_u16_sha"]
        assert _sha(s.outlier_values) == ref_hashes["outliers_sha"]
        assert _sha(s.outlier_counts) == ref_hashes["counts_sha"]
        assert _sha(s.scalars.values) == ref_hashes["scalars_sha"]
    else:
        o = oracle.dualquant(data, eb, b, radius, pol)
        assert np.array_equal(s.codes, o["codes"])
        assert s.outlier_values.tobytes() == o["outlier_values"].tobytes()
        assert np.array_equal(s.outlier_counts, o["outlier_counts"])
        assert np.array_equal(s.scalars.values, o["scalars"])
    back = reconstruct_stream(s)
    # size-independent properties: bound, exact inverse, idempotence
    err = np.abs(back.astype(np.float64) - data.astype(np.float64))
    assert err.max() <= eb
    # closed form of the exact inverse (DESIGN.md finding 2): verbatim value
    # at outliers, float32((2 d) eb) with d the prequantized value elsewhere
    qd = oracle.prequantize(data, eb)
    recon = ((2.0 * qd.astype(np.float64)) * eb).astype(np.float32).ravel()
    mask = _outlier_mask_rowmajor(s, data.shape)
    assert int(mask.sum()) == s.outlier_values.size
    expected = np.where(mask, data.ravel(), recon)
    assert back.ravel().tobytes() == expected.tobytes()
    again = dualquant(back, cfg)
    assert again.same_bytes(s)
    return s


def _outlier_mask_rowmajor(s, shape):
    """Row-major mask of outlier positions from the canonical code stream."""
    grid = s.grid
    m = np.zeros(shape, dtype=bool)
    nd = len(shape)
    pos = 0
    codes = s.codes
    # walk blocks; vectorised per block
    for bi in range(grid.block_count):
        org = grid.block_origin(bi)
        ext = grid.block_extents(bi)
        size = int(np.prod(ext))
        if s.outlier_counts[bi]:
            blk = codes[pos:pos + size].reshape(ext) == 0
            m[tuple(slice(o, o + e) for o, e in zip(org, ext))] = blk
        pos += size
    assert nd in (1, 2, 3)
    return m.ravel()


def test_fullsize_c1_c2_match_reference_hashes(oracle):
    data = {"C1": workloads.gen_c1(), "C2": workloads.gen_c2()}
    for c in load_json("fullsize.json"):
        d = data[c["config"]]
        # the generator is seeded numpy on the same image: a different data
        # hash means the pin cannot run, which must fail, not fall back
        assert _sha(d) == c["data_sha"], f"{c['config']} data differs from the pinned field"
        _check_full(oracle, d, c["eb"], c["block_edge"], c["padding"], c["radius"], ref_hashes=c)


def test_fullsize_c3_matches_oracle(oracle):
    d = workloads.gen_c3()
    eb = workloads.value_range_eb(d, 1e-3)
    _check_full(oracle, d, eb, 8, "mean:global", 512)
    _check_full(oracle, d, eb, 8, "mean:block", 512)


def test_fullsize_c4_matches_oracle(oracle):
    d = workloads.gen_c4(512)
    eb = workloads.value_range_eb(d, 1e-3)
    for b, r in ((8, 512), (16, 32768)):
        _check_full(oracle, d, eb, b, "mean:global", r)


def test_outlier_stress_matches_oracle(oracle, scratch_layout):
    # C4 field at eb = 1e-5 * range: ~18% outliers at R=512
    d = workloads.gen_c4(128)
    eb = workloads.value_range_eb(d, 1e-5)
    for pol in ("zero", "max:edge", "min:block"):
        s = _check_full(oracle, d, eb, 8, pol, 512)
        assert s.outlier_values.size > 0.05 * d.size


def test_int64_redo_path(oracle):
    # |d| >= 2^28 forces the int64 stencil redo (dq_compress.cuh)
    rng = np.random.default_rng(3)
    d = (rng.uniform(-1, 1, (40, 33, 70)) * 1.0e9).astype(np.float32)
    for pol in ("mean:global", "zero", "max:block", "min:edge"):
        _check_full(oracle, d, 0.9, 8, pol, 32768)


@pytest.mark.parametrize("shape,b", [((24, 40, 256), 8), ((33, 50, 260), 8), ((32, 48, 256), 16),
                                     ((64, 64, 128), 32), ((70, 130, 136), 64), ((128, 128, 64), 64),
                                     ((96, 512), 8), ((100, 516), 16), ((128, 512), 32),
                                     ((130, 260), 64)])
def test_fused_kernels_int64_tails(oracle, shape, b):
    # 16-byte aligned rows keep the fused 2-D / 3-D kernels eligible; a slab of
    # values near 1e9 at eb 0.9 pushes |d| past 2^24 (compress) and 2^27
    # (decompress) in SOME tiles, so the warps that meet them redo them in
    # int64 after their loops (compress_redo_tail / decompress_redo_tail; the
    # b >= 32 3-D shapes take turns on the CTA's shared memory) while the rest
    # of the grid stays on the int32 path
    rng = np.random.default_rng(sum(shape) * 7 + b)
    idx = np.indices(shape).astype(np.float64)
    data = sum(np.sin(0.06 * (k + 1) * idx[k]) * 300.0 for k in range(len(shape)))
    data = (data + rng.normal(0, 2.0, shape)).astype(np.float32)
    data[..., -5:] *= np.float32(3.0e6)  # a few wide columns in the last window
    lo, n = shape[0] // 3, max(3, shape[0] // 4)
    data[lo:lo + n] = (rng.uniform(-1, 1, data[lo:lo + n].shape) * 1.0e9).astype(np.float32)
    for pol in ("mean:global", "zero", "max:block", "min:edge"):
        s = _check_full(oracle, data, 0.9, b, pol, 32768)
        assert s.outlier_values.size > 0


@pytest.mark.parametrize("shape,b", [((21, 44, 260), 8), ((19, 44, 196), 16),
                                     ((45, 300), 8), ((37, 196), 16), ((9, 12, 132), 8)])
def test_fast_kernel_edge_tiles(oracle, shape, b):
    # D2 % 4 == 0 keeps the fast decompress kernel eligible; the last window
    # of every block row (W = 128 or 64 columns) and the last block row are
    # partial, so dq_decompress_edge_kernel runs, with outliers and sentinels
    rng = np.random.default_rng(sum(shape) + b)
    idx = np.indices(shape).astype(np.float64)
    smooth = sum(np.sin(0.07 * (k + 1) * idx[k]) * 40.0 for k in range(len(shape)))
    data = (smooth + rng.normal(0, 0.05, shape)).astype(np.float32)
    data.ravel()[rng.integers(0, data.size, 50)] *= 7.0  # spikes -> outliers
    for eb, pol in ((1e-3, "mean:global"), (1e-4, "zero"), (1e-3, "max:block")):
        s = _check_full(oracle, data, eb, b, pol, 512)
        assert s.outlier_values.size > 0


def test_outlier_report_matches_reference():
    # padding.py:162-205 on the GPU (border census: csrc/k_stats.cu)
    from conftest import load_border
    from paper_2201_04614_b200.padding import outlier_report

    for c in load_border():
        cfg = _cfg(c["eb"], c["block_edge"], "zero", c["radius"])
        rows = outlier_report(c["data"], cfg)
        got = [dict(kind=r.policy.value_kind.value, gran=r.policy.granularity.value,
                    total=r.total_outliers, border=r.border_outliers, reduction=red)
               for r, red in rows]
        assert got == c["rows"], c["tag"]


@pytest.mark.parametrize("shape,b,radius", [((37, 45, 29), 8, 16), ((300, 170), 16, 32),
                                             ((5000,), 64, 8), ((20, 70, 130), 32, 64)])
def test_outlier_report_matches_per_policy_oracle(oracle, shape, b, radius):
    # the one-pass census (k_census.cu) against ten full oracle compressions,
    # one per policy, with the border outliers counted from each stream
    from paper_2201_04614_b200.padding import outlier_report
    from paper_2201_04614_b200.vector import border_outliers

    rng = np.random.default_rng(sum(shape))
    idx = np.indices(shape).astype(np.float64)
    data = sum(np.sin(0.07 * (k + 2) * idx[k]) * 20 for k in range(len(shape)))
    data = (data + rng.normal(0, 0.4, shape) + 100).astype(np.float32)
    eb = 1e-2
    rows = outlier_report(data, _cfg(eb, b, "zero", radius))
    assert len(rows) == 10
    zero_total = None
    for st, red in rows:
        pol = str(st.policy)
        o = oracle.dualquant(data, eb, b, radius, pol)
        grid = M.build_block_grid(M.ArrayDescriptor(len(shape), shape), b)
        cs = M.CodeStream(o["codes"], o["outlier_values"], o["outlier_counts"], grid, eb, radius,
                          M.PaddingScalars(st.policy, o["scalars"]))
        total = int(o["outlier_counts"].sum())
        assert (st.total_outliers, st.border_outliers) == (total, border_outliers(cs)), pol
        zero_total = total if zero_total is None else zero_total
        if zero_total:
            assert red == 100.0 * (zero_total - total) / zero_total


@pytest.mark.parametrize("b", [8, 16, 32, 64, 256])
def test_fused_1d_kernels(oracle, b):
    # dq_1d.cuh: full tiles through the bulk-copy ring plus a
    # partial tail tile with a partial last block; random walk + spikes give
    # outliers in most blocks, near-ties exercise the exact fp64 path
    rng = np.random.default_rng(b)
    n = (1 << 22) + 2048 * 37 + 3 * 256 + 13  # >= 4 M: the fused path (k_1d.cu D1_MIN_N)
    walk = np.cumsum(rng.normal(0, 1, n)) * 0.01 + np.sin(np.arange(n) * (2 * np.pi / 4096))
    data = walk.astype(np.float32)
    data[rng.integers(0, n, 400)] *= 9.0
    eb = float(np.float32(1e-4 * (data.max() - data.min())))
    for pol in ("zero", "mean:global", "max:global", "min:block", "mean:block", "mean:edge",
                "max:edge"):
        s = _check_full(oracle, data, eb, b, pol, 512)
        assert s.outlier_values.size > 0


def test_fused_1d_int64_rows(oracle):
    # |q| >= 2^30 in some rows: those rows go to the int64 generic kernels
    # through the redo list (compress and decompress)
    rng = np.random.default_rng(11)
    data = (rng.uniform(-1, 1, (1 << 22) + 2048 * 9 + 100) * 2.0e9).astype(np.float32)
    for b in (8, 64, 256):
        for pol in ("zero", "mean:global", "max:block"):
            _check_full(oracle, data, 0.9, b, pol, 32768)


def test_fused_1d_kernels_many_tiles_per_warp(oracle):
    # ~20 M elements: every warp of the persistent grid streams several tiles,
    # so the bulk-copy ring is refilled and reused (stage / phase bookkeeping)
    rng = np.random.default_rng(21)
    n = 20 * 1024 * 1024 + 1000
    data = (np.cumsum(rng.normal(0, 1, n)) * 0.01).astype(np.float32)
    eb = float(np.float32(1e-4 * (data.max() - data.min())))
    for b, pol in ((64, "mean:global"), (256, "zero"), (8, "max:block")):
        _check_full(oracle, data, eb, b, pol, 512)


@pytest.mark.parametrize("shape,b", [((70, 96, 200), 32), ((64, 64, 128), 32),
                                     ((130, 140, 136), 64), ((300, 520), 32),
                                     ((260, 600), 64), ((256, 512), 64)])
def test_fast_kernels_large_blocks(oracle, shape, b):
    # b = 32 / 64 through the fused kernels (8-row ring stages): interior
    # tiles and partial windows / block rows, outliers and every policy family
    rng = np.random.default_rng(sum(shape) * b)
    idx = np.indices(shape).astype(np.float64)
    smooth = sum(np.sin(0.05 * (k + 1) * idx[k]) * 30.0 for k in range(len(shape)))
    data = (smooth + rng.normal(0, 0.05, shape)).astype(np.float32)
    data.ravel()[rng.integers(0, data.size, 200)] *= 6.0
    for eb, pol in ((1e-3, "mean:global"), (1e-4, "zero"), (1e-3, "max:block"),
                    (1e-3, "mean:edge"), (1e-3, "min:global")):
        s = _check_full(oracle, data, eb, b, pol, 512)
        assert s.outlier_values.size > 0


def test_decompress_with_device_outlier_count():
    # vlz_dq_decompress_dn reads the stored outlier count from the compressor's
    # device result block: same output and same corrupt-stream verdict as the
    # host-count entry point, with no host round trip between the two calls
    import ctypes

    from paper_2201_04614_b200 import _lib

    lib = _lib.load()
    cases = [(workloads.gen_c3(shape=(64, 96, 128)), 8, "mean:global"),
             (workloads.gen_c3(shape=(48, 80, 200)), 16, "max:block"),
             ((np.cumsum(np.random.default_rng(2).normal(0, 1, (1 << 22) + 777)) * 0.01)
              .astype(np.float32), 64, "zero")]
    for data, b, pol in cases:
        eb = workloads.value_range_eb(data, 1e-4)
        cfg = _cfg(eb, b, pol, 512)
        x = torch.from_numpy(data).cuda()
        dev = gpu.compress_device(x, cfg, eb=eb).check()
        ref = gpu.decompress_device(dev.codes, dev.outliers, dev.n_outliers, dev.counts,
                                    dev.scalars, dev.grid, eb, 512, cfg.padding)
        g = _lib.geom(dev.grid.descriptor.dims, b)
        p = _lib.params(eb, 512, cfg.padding.kind_code, cfg.padding.gran_code)
        wsb = lib.vlz_workspace_size(ctypes.byref(g))
        ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
        out = torch.empty_like(x)
        res = torch.empty(8, dtype=torch.int64, device="cuda")
        sc = dev.scalars.data_ptr() if dev.scalars.numel() else None
        stream = torch.cuda.current_stream().cuda_stream
        rc = lib.vlz_dq_decompress_dn(dev.codes.data_ptr(), dev.outliers.data_ptr(),
                                      dev.result[2:3].data_ptr(), dev.counts.data_ptr(), sc,
                                      ctypes.byref(g), ctypes.byref(p), out.data_ptr(),
                                      res.data_ptr(), ws.data_ptr(), wsb, stream)
        assert rc == 0
        assert int(res[0].item()) == 0
        assert torch.equal(out, ref)
        # a stored count one short: the sentinel-total verdict, as with a host count
        short = dev.result.clone()
        short[2] -= 1
        rc = lib.vlz_dq_decompress_dn(dev.codes.data_ptr(), dev.outliers.data_ptr(),
                                      short[2:3].data_ptr(), dev.counts.data_ptr(), sc,
                                      ctypes.byref(g), ctypes.byref(p), out.data_ptr(),
                                      res.data_ptr(), ws.data_ptr(), wsb, stream)
        assert rc == 0 and int(res[0].item()) == _lib.ST_SENTINEL_TOTAL


@pytest.mark.parametrize("shape,b", [(((1 << 22) + 5000,), 64), (((1 << 22) + 5000,), 256),
                                     ((40, 64, 256), 32), ((96, 96, 128), 64), ((300, 512), 64)])
def test_fused_kernels_error_precedence(shape, b):
    # quantize.py:58-72 through the fused 1-D / large-block kernels: the first
    # non-finite value wins over an earlier overflow; else the first overflow
    rng = np.random.default_rng(7)
    base = rng.uniform(-1, 1, shape).astype(np.float32)
    flat = base.reshape(-1)
    n = flat.size
    ovf_at, nan_at = n // 3, (2 * n) // 3
    eb = 1e-6
    d = flat.copy()
    d[ovf_at] = 1.0e5  # |v / 2eb| = 5e10 >= 2^31 - 1
    d[nan_at] = np.nan
    with pytest.raises(ConfigError) as err:
        dualquant_vector(d.reshape(shape), _cfg(eb, b, "mean:global", 512))
    assert str(nan_at) in str(err.value)
    d2 = flat.copy()
    d2[ovf_at] = 1.0e5
    d2[n - 1] = -2.0e5
    with pytest.raises(BoundTooSmallError) as err:
        dualquant_vector(d2.reshape(shape), _cfg(eb, b, "zero", 512))
    assert err.value.index == ovf_at


@pytest.fixture(params=["compact", "dense"])
def scratch_layout(request, monkeypatch):
    # compress_device gives arrays up to gpu.DENSE_SCRATCH_MAX elements the
    # dense outlier scratch (one slot per element; dense blocks are copied) and
    # larger ones the compact one (8 slots per block; dense blocks regenerated
    # from codes + input): force either for the arrays of a test
    monkeypatch.setattr(gpu, "DENSE_SCRATCH_MAX", 0 if request.param == "compact" else 1 << 40)
    return request.param


@pytest.mark.parametrize("shape,b", [((5000,), 8), ((70001,), 64), ((1 << 20,), 256),
                                     ((4_500_000,), 256), ((45, 300), 8), ((37, 196), 16),
                                     ((100, 516), 32), ((130, 260), 64), ((21, 44, 260), 8),
                                     ((19, 44, 196), 16), ((40, 70, 136), 32), ((70, 130, 136), 64)])
def test_dense_blocks_regenerated_from_codes(oracle, shape, b, scratch_layout):
    # the outlier scratch holds 8 slots per block; blocks with more outliers
    # keep only their count and the scan kernel regenerates the values from the
    # codes and the input (regen_block).  Noise far above radius * 2eb makes
    # most elements outliers -- full and partial blocks, outlier and in-range
    # origins, every policy family, fused and generic kernels, 1-D to 3-D.
    prev = M.valid_block_edges()
    M.allow_block_256(True)
    try:
        rng = np.random.default_rng(sum(shape) + 31 * b)
        idx = np.indices(shape).astype(np.float64)
        data = sum(np.sin(0.05 * (k + 1) * idx[k]) * 3.0 for k in range(len(shape)))
        noise = rng.normal(0, 1.0, shape)
        quiet = rng.random(shape) < 0.35  # some elements stay predictable
        data = (data + np.where(quiet, 0.0, noise)).astype(np.float32)
        for eb, pol, radius in ((1e-3, "zero", 16), (1e-3, "mean:global", 16),
                                (2e-3, "max:block", 8), (1e-3, "min:edge", 32)):
            s = _check_full(oracle, data, eb, b, pol, radius)
            assert s.outlier_values.size > 0.3 * data.size
            assert int(s.outlier_counts.max()) >= min(8, b - 1)
    finally:
        M.allow_block_256(256 in prev)


@pytest.mark.parametrize("shape,b,pol", [((40, 72, 256), 8, "mean:global"), ((300, 516), 16, "zero"),
                                         ((1 << 20,), 64, "max:block")])
def test_capped_outlier_array(oracle, shape, b, pol, scratch_layout):
    # vlz_dq_compress_capped: an outlier array sized to the stream (not to the
    # worst case).  Enough capacity: the same stream as the oracle's.  Too
    # little: codes / counts / scalars complete, the first `capacity` outliers
    # written, nothing past the array touched, status -> OutlierCapacityError
    # carrying the true count; a retry with that count succeeds.
    import torch
    from paper_2201_04614_b200.errors import OutlierCapacityError

    rng = np.random.default_rng(sum(shape) + b)
    idx = np.indices(shape).astype(np.float64)
    data = sum(np.sin(0.05 * (k + 1) * idx[k]) * 20.0 for k in range(len(shape)))
    data = (data + rng.normal(0, 0.02, shape)).astype(np.float32)
    data.ravel()[rng.integers(0, data.size, 4000)] *= 5.0  # spikes -> outliers, some blocks dense
    eb, radius = 1e-3, 64
    cfg = _cfg(eb, b, pol, radius)
    o = oracle.dualquant(data, eb, b, radius, pol)
    n_true = int(o["outlier_values"].size)
    assert n_true > 100
    x = torch.from_numpy(data).cuda()
    # exact fit
    dev = gpu.compress_device(x, cfg, eb=eb, outlier_capacity=n_true).check()
    assert dev.outliers.numel() == n_true and dev.n_outliers == n_true
    assert dev.outliers.cpu().numpy().tobytes() == o["outlier_values"].tobytes()
    assert np.array_equal(dev.codes.cpu().numpy().view(np.uint16).astype(np.uint32), o["codes"])
    # too small: guard words behind the array stay intact
    cap = n_true // 3
    small = gpu.compress_device(x, cfg, eb=eb, outlier_capacity=cap)
    guard = torch.full((cap + 64,), float("nan"), dtype=torch.float32, device="cuda")
    small.outliers = guard[:cap]
    small = gpu.compress_device(x, cfg, eb=eb, out=small, outlier_capacity=cap)
    with pytest.raises(OutlierCapacityError) as ei:
        small.check()
    assert ei.value.needed == n_true and ei.value.capacity == cap
    assert bool(torch.isnan(guard[cap:]).all())
    assert small.outliers.cpu().numpy().tobytes() == o["outlier_values"][:cap].tobytes()
    assert np.array_equal(small.codes.cpu().numpy().view(np.uint16).astype(np.uint32), o["codes"])
    assert np.array_equal(small.counts.cpu().numpy(), o["outlier_counts"])
    assert np.array_equal(small.scalars.cpu().numpy(), o["scalars"])
    # retry with the reported count
    again = gpu.compress_device(x, cfg, eb=eb, outlier_capacity=ei.value.needed).check()
    assert again.outliers.cpu().numpy().tobytes() == o["outlier_values"].tobytes()
    # zero capacity is legal
    none = gpu.compress_device(x, cfg, eb=eb, outlier_capacity=0)
    with pytest.raises(OutlierCapacityError):
        none.check()


def test_cuda_graph_replay_resets_per_call_state(oracle):
    # the per-call reset lives in the first kernel of each call, guarded by a
    # nonce baked into the launch: a captured graph replays the same nonce, so
    # the call's last kernel must leave the flag cleared.  Replays over new
    # input contents (global statistics, error minima, look-back words and the
    # result block are all per-call state) must match the oracle every time.
    import torch
    from paper_2201_04614_b200 import gpu

    shape, b, radius, pol = (40, 72, 256), 8, 512, "mean:global"
    cfg = _cfg(1e-3, b, pol, radius)
    rng = np.random.default_rng(5)
    idx = np.indices(shape).astype(np.float64)

    def field(k):
        d = sum(np.sin(0.05 * (j + 1 + k) * idx[j]) * (3.0 + k) for j in range(3)) + 10.0 * k
        return (d + rng.normal(0, 0.01, shape)).astype(np.float32)

    x = torch.from_numpy(field(0)).cuda()
    dev = gpu.compress_device(x, cfg, eb=1e-3).check()
    y = torch.empty_like(x)
    res = torch.empty(8, dtype=torch.int64, device="cuda")

    import ctypes

    from paper_2201_04614_b200 import _lib

    lib = _lib.load()
    g = _lib.geom(dev.grid.descriptor.dims, b)
    p = _lib.params(1e-3, radius, cfg.padding.kind_code, cfg.padding.gran_code)
    wsb = lib.vlz_workspace_size(ctypes.byref(g))
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")  # same workspace for both directions

    def step():
        st = torch.cuda.current_stream().cuda_stream
        gpu.compress_device(x, cfg, eb=1e-3, out=dev, workspace=ws)
        rc = lib.vlz_dq_decompress_dn(dev.codes.data_ptr(), dev.outliers.data_ptr(),
                                      dev.result[2:3].data_ptr(), dev.counts.data_ptr(),
                                      dev.scalars.data_ptr(), ctypes.byref(g), ctypes.byref(p),
                                      y.data_ptr(), res.data_ptr(), ws.data_ptr(), wsb, st)
        assert rc == 0

    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        step()
    torch.cuda.current_stream().wait_stream(side)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        step()
    for k in range(1, 5):
        data = field(k)
        x.copy_(torch.from_numpy(data))
        gr.replay()
        torch.cuda.synchronize()
        o = oracle.dualquant(data, 1e-3, b, radius, pol)
        assert np.array_equal(dev.codes.cpu().numpy().view(np.uint16).astype(np.uint32), o["codes"]), k
        n = int(dev.result.cpu()[2])
        assert n == o["outlier_values"].size
        assert dev.outliers[:n].cpu().numpy().tobytes() == o["outlier_values"].tobytes()
        assert np.array_equal(dev.scalars.cpu().numpy(), o["scalars"])
        back = oracle.reconstruct(o["codes"], o["outlier_values"], o["outlier_counts"], o["scalars"],
                                  shape, b, 1e-3, radius, pol)
        assert y.cpu().numpy().tobytes() == back.tobytes(), k
        assert int(res.cpu()[0]) == 0
