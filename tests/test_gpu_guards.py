"""Out-of-bounds write guards for the CUDA path (compute-sanitizer is not
available on the GPU pool): every output the kernels write -- codes, outlier
values, counts, padding scalars, result block, workspace, decompressed array,
Huffman payload and decoded symbols -- is a slice of a larger buffer whose
head and tail guards hold a known pattern, checked after each call.  Ragged
shapes exercise edge tiles, partial blocks, the TMA and cp.async decompress
producers and the *:global origin fix-up."""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2201_04614_b200 import _lib, gpu  # noqa: E402
from paper_2201_04614_b200 import model as M  # noqa: E402
from paper_2201_04614_b200.huffman import build_codebook_from_freqs  # noqa: E402

GUARD = 256  # bytes on each side (keeps 16-byte alignment)


class Guarded:
    def __init__(self, nbytes: int, fill: int = 0xA5):
        self.n = max(int(nbytes), 1)
        self.buf = torch.full((self.n + 2 * GUARD,), fill, dtype=torch.uint8, device="cuda")
        self.fill = fill

    def ptr(self) -> int:
        return self.buf.data_ptr() + GUARD

    def view(self, dtype) -> torch.Tensor:
        return self.buf[GUARD:GUARD + self.n].view(dtype)

    def check(self, what):
        head = self.buf[:GUARD]
        tail = self.buf[GUARD + self.n:]
        assert bool((head == self.fill).all()), f"{what}: write before the buffer"
        assert bool((tail == self.fill).all()), f"{what}: write past the buffer"


SHAPES = [((1000,), 64), ((777,), 8), ((24, 40), 8), ((37, 70), 16), ((16, 16, 256), 8),
          ((13, 21, 132), 8), ((16, 32, 64), 16), ((9, 20, 30), 8), ((8, 64, 128), 8)]


@pytest.mark.parametrize("shape,b", SHAPES)
@pytest.mark.parametrize("pol", ["zero", "mean:global", "max:block", "min:edge"])
def test_no_out_of_bounds_writes(shape, b, pol):
    rng = np.random.default_rng(len(shape) * 100 + b)
    idx = np.indices(shape).astype(np.float64)
    data = sum(np.sin(0.1 * (k + 1) * idx[k]) * 30 for k in range(len(shape)))
    data = (data + rng.normal(0, 0.3, shape)).astype(np.float32)
    _run_guarded(data, b, pol, 1e-2, 64)


def _field(kind, shape, seed):
    rng = np.random.default_rng(seed)
    if kind == "walk":  # 1-D random walk with spikes (fused 1-D kernels)
        d = np.cumsum(rng.normal(0, 1, shape)) * 0.01
        d[rng.random(shape) < 0.01] = 50.0
        return d.astype(np.float32)
    if kind == "huge":  # |d| >= 2^24: the int64 redo tiles
        return (rng.uniform(-1, 1, shape) * 1.0e9).astype(np.float32)
    idx = np.indices(shape).astype(np.float64)
    d = sum(np.sin(0.05 * (k + 1) * idx[k]) for k in range(len(shape))) * 10
    return (d + rng.normal(0, 0.05, shape)).astype(np.float32)


# paths the small shapes above do not reach (round 2): the fused 1-D kernels
# (bulk-copy ring, >= 4 M elements), 8-row staged b = 32 / 64 fast kernels,
# outlier-heavy blocks (eb 1e-4 at radius 64) and the int64 redo list
LARGE = [
    ("walk", (1 << 22,), 256, "zero", 1e-3, 512),
    ("walk", (1 << 22,) , 64, "mean:global", 1e-3, 512),
    ("waves", (64, 64, 128), 64, "mean:block", 1e-4, 64),
    ("waves", (32, 64, 128), 32, "max:edge", 1e-2, 64),
    ("waves", (64, 256), 64, "mean:global", 1e-4, 64),
    ("huge", (40, 33, 70), 8, "mean:global", 1.0, 512),
    ("huge", (24, 40, 64), 16, "zero", 1.0, 512),
]


@pytest.mark.parametrize("dense_ws", [False, True])
@pytest.mark.parametrize("kind,shape,b,pol,eb,radius", LARGE)
def test_no_out_of_bounds_writes_large_paths(kind, shape, b, pol, eb, radius, dense_ws):
    prev = M.valid_block_edges()
    M.allow_block_256(True)
    try:
        _run_guarded(_field(kind, shape, b), b, pol, eb, radius, dense_ws)
    finally:
        M.allow_block_256(256 in prev)


def _run_guarded(data, b, pol, eb, radius, dense_ws=False):
    lib = _lib.load()
    shape = data.shape
    n = data.size
    grid = M.build_block_grid(M.ArrayDescriptor(len(shape), shape), b)
    policy = M.PaddingPolicy.parse(pol)
    g = _lib.geom(shape, b)
    p = _lib.params(eb, radius, policy.kind_code, policy.gran_code)
    ns = policy.scalar_count(grid)
    x = Guarded(4 * n)
    x.view(torch.float32).copy_(torch.from_numpy(data.ravel()).cuda())
    codes, outl = Guarded(2 * n), Guarded(4 * n)
    counts, scal = Guarded(8 * grid.block_count), Guarded(8 * max(ns, 1))
    res = Guarded(64)
    # the workspace guards cover both scratch layouts: 8 slots per block
    # (compact) and one slot per element (dense, chosen by the size passed)
    wsb = int((lib.vlz_workspace_size_dense if dense_ws else lib.vlz_workspace_size)(ctypes.byref(g)))
    ws = Guarded(wsb, fill=0)
    rc = lib.vlz_dq_compress(x.ptr(), ctypes.byref(g), ctypes.byref(p), codes.ptr(), outl.ptr(),
                             counts.ptr(), scal.ptr() if ns else None, res.ptr(), ws.ptr(), wsb,
                             None)
    assert rc == 0
    torch.cuda.synchronize()
    for name, gbuf in (("input", x), ("codes", codes), ("outliers", outl), ("counts", counts),
                       ("scalars", scal), ("result", res), ("workspace", ws)):
        gbuf.check(f"compress {name}")
    r = res.view(torch.int64).cpu().numpy()
    assert r[0] & 0xffffffff == 0
    n_out = int(r[2])
    # decompress into a guarded output
    out, dres = Guarded(4 * n), Guarded(64)
    ws.buf.fill_(0)
    rc = lib.vlz_dq_decompress(codes.ptr(), outl.ptr() if n_out else None, n_out, counts.ptr(),
                               scal.ptr() if ns else None, ctypes.byref(g), ctypes.byref(p),
                               out.ptr(), dres.ptr(), ws.ptr(), wsb, None)
    assert rc == 0
    torch.cuda.synchronize()
    for name, gbuf in (("codes", codes), ("outliers", outl), ("counts", counts),
                       ("output", out), ("result", dres), ("workspace", ws)):
        gbuf.check(f"decompress {name}")
    back = out.view(torch.float32).cpu().numpy()
    assert np.max(np.abs(back.astype(np.float64) - data.ravel())) <= eb
    # entropy stage: exact-size payload (whole 32-bit words) and decoded symbols
    c16 = codes.view(torch.int16)
    freqs = gpu.histogram_device(c16, radius)
    cb = build_codebook_from_freqs(freqs)
    nbits = int((freqs[cb.symbols] * cb.lengths.astype(np.uint64)).sum())
    tab = Guarded(int(lib.vlz_huff_table_bytes()))
    syms = np.ascontiguousarray(cb.symbols, dtype=np.uint16)
    lens = np.ascontiguousarray(cb.lengths, dtype=np.uint8)
    assert lib.vlz_huff_table(syms.ctypes.data, lens.ctypes.data, len(syms), tab.ptr(), None) == 0
    cap = (nbits + 31) // 32 * 4
    pay = Guarded(cap)
    hws = Guarded(int(lib.vlz_huff_encode_ws_size(n)), fill=0)
    info = Guarded(32)
    rc = lib.vlz_huff_encode_device(codes.ptr(), n, tab.ptr(), int(syms.max()) + 1,
                                    int(lens.max()), pay.ptr(), cap, info.ptr(), hws.ptr(),
                                    hws.n, None)
    assert rc == 0
    torch.cuda.synchronize()
    for name, gbuf in (("table", tab), ("payload", pay), ("workspace", hws), ("info", info)):
        gbuf.check(f"encode {name}")
    inf = info.view(torch.int64).cpu().numpy()
    assert int(inf[0]) == nbits and int(inf[2]) == 0
    nbytes = (nbits + 7) // 8
    dpay = Guarded((nbytes + 3) // 4 * 4 + 16, fill=0)
    dpay.view(torch.uint8)[:nbytes].copy_(pay.view(torch.uint8)[:nbytes])
    dec = Guarded(2 * n)
    dws = Guarded(int(lib.vlz_huff_decode_ws_size(nbytes)), fill=0)
    consumed = ctypes.c_int64(0)
    rc = lib.vlz_huff_decode_device(dpay.ptr(), nbytes, nbits, syms.ctypes.data,
                                    lens.ctypes.data, len(syms), n, dec.ptr(),
                                    ctypes.byref(consumed), dws.ptr(), dws.n, None)
    assert rc == 0 and consumed.value == nbits
    for name, gbuf in (("decoded", dec), ("workspace", dws), ("payload", dpay)):
        gbuf.check(f"decode {name}")
    assert torch.equal(dec.view(torch.int16), c16)


def test_crafted_books_device_decode_guards():
    """Over-subscribed codebooks from crafted containers: the
    device decoder's table builder and decode passes stay inside their
    buffers (the verdicts themselves are pinned in test_container_full)."""
    from conftest import load_json
    from paper_2201_04614_b200.container import deserialize

    lib = _lib.load()
    n_books = 0
    for c in load_json("container_full.json"):
        p = deserialize(bytes.fromhex(c["blob"]))
        cb = p.codebook
        if not len(cb.lengths) or int(cb.lengths.max()) > 58:
            continue
        pay = bytes(p.code_bits)
        nbytes = len(pay)
        count = p.descriptor.element_count
        dpay = Guarded((nbytes + 3) // 4 * 4 + 16, fill=0)
        if nbytes:
            dpay.view(torch.uint8)[:nbytes].copy_(torch.frombuffer(bytearray(pay),
                                                                   dtype=torch.uint8).cuda())
        dec = Guarded(2 * count)
        dws = Guarded(int(lib.vlz_huff_decode_ws_size(nbytes)), fill=0)
        syms = np.ascontiguousarray(cb.symbols, dtype=np.uint16)
        lens = np.ascontiguousarray(cb.lengths, dtype=np.uint8)
        consumed = ctypes.c_int64(0)
        rc = lib.vlz_huff_decode_device(dpay.ptr(), nbytes, p.code_bit_length, syms.ctypes.data,
                                        lens.ctypes.data, len(syms), count, dec.ptr(),
                                        ctypes.byref(consumed), dws.ptr(), dws.n, None)
        assert rc >= 0, c["tag"]
        torch.cuda.synchronize()
        for name, gbuf in (("decoded", dec), ("workspace", dws), ("payload", dpay)):
            gbuf.check(f"{c['tag']} decode {name}")
        n_books += 1
    assert n_books >= 20
