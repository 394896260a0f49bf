"""Generate the golden parity fixtures by running the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package `vlz` read-only from /root/reference/pkg/src
and records its outputs for seeded inputs into tests/golden/*.npz (+ .json).
Nothing at test time reads /root/reference; the fixtures are self-contained
(inputs are stored, or regenerated from seeded generators for the full-size
hash pins).

Fixture groups
  corpus.npz      dualquant_vector streams for ~90 seeded arrays x configs
                  (1D/2D/3D, b 8..64, all 10 padding policies, radius 2..32768,
                  eb 1e-2..1e-5, partial blocks, tiny shapes, tie-rich and
                  narrowing-heavy data) + compress() container bytes + the
                  reference decompress() output for the small ones.
  errors.json     error precedence/index cases (non-finite, overflow, eb<=0).
  corrupt.npz     decompression stream-corruption cases + expected exception.
  known.json      hand known-answer cases lifted from the reference tests.
  fullsize.json   sha256 of the reference streams for C1/C2 at full size
                  (regenerated data via paper_2201_04614_b200.workloads).
  border.npz      outlier_report rows (total / border outliers per padding
                  policy, reduction vs zero padding) for seeded arrays.
"""

from __future__ import annotations

import hashlib
import io
import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import vlz  # noqa: E402  (the reference, read-only)
import vlz.model as vmodel  # noqa: E402
from vlz import errors as verr  # noqa: E402
from vlz.container import deserialize  # noqa: E402
from vlz.kernel import dualquant_scalar  # noqa: E402
from vlz.model import CompressionConfig, ErrorBound, PaddingPolicy  # noqa: E402
from vlz.pipeline import compress, decompress  # noqa: E402
from vlz.reconstruct import decompress_parsed, reconstruct_block  # noqa: E402
from vlz.vector import dualquant_vector  # noqa: E402

from paper_2201_04614_b200 import workloads  # noqa: E402

POLICIES = [
    "zero",
    "min:global", "max:global", "mean:global",
    "min:block", "max:block", "mean:block",
    "min:edge", "max:edge", "mean:edge",
]

# allow block edge 256 (BASELINE config 1); the reference reads this module
# global at call time (model.py:149,212)
vmodel.VALID_BLOCK_EDGES = (8, 16, 32, 64, 256)


def _smooth(rng, shape):
    offset = rng.uniform(-700, 700)
    amp = rng.uniform(1.0, 40.0)
    axes = [np.linspace(0.0, rng.uniform(1, 8), s) for s in shape]
    mesh = np.add.reduce(np.meshgrid(*axes, indexing="ij"))
    field = offset + amp * np.sin(mesh) + 0.05 * amp * np.cos(3.0 * mesh)
    return np.clip(field, -1e3, 1e3).astype(np.float32)


def _noise(rng, shape):
    return rng.uniform(-1e3, 1e3, shape).astype(np.float32)


def _ties(rng, shape, eb):
    # values exactly on quantization half-points (k + 0.5) * 2eb where
    # representable, plus exact grid points: stresses round-half-away
    k = rng.integers(-2000, 2000, size=shape).astype(np.float64)
    half = rng.random(shape) < 0.5
    return ((k + np.where(half, 0.5, 0.0)) * (2.0 * eb)).astype(np.float32)


def _narrow(rng, shape):
    # |v| ~ 1e3..4e3 with eb 1e-5: ulp32(v) > eb, so the float32-narrowing
    # bound check fires often and |q| is ~1e8 (exact fp64 path)
    return rng.uniform(1000.0, 4000.0, shape).astype(np.float32) * np.where(
        rng.random(shape) < 0.5, -1, 1
    ).astype(np.float32)


def _big_q(rng, shape, eb):
    # |q| just below the 2^31-1 overflow guard
    lim = (2**31 - 2) * 2.0 * eb
    return (rng.uniform(-1.0, 1.0, shape) * lim).astype(np.float32)


def _cfg(eb, b, pol, radius, lanes=8):
    return CompressionConfig(
        ErrorBound.absolute(eb), block_edge=b, lane_width=lanes,
        padding=PaddingPolicy.parse(pol), radius=radius,
    )


class Store:
    def __init__(self):
        self.arrays = {}
        self.meta = []

    def add(self, meta: dict, **arrays):
        i = len(self.meta)
        meta = dict(meta)
        meta["id"] = i
        self.meta.append(meta)
        for k, v in arrays.items():
            self.arrays[f"{i}.{k}"] = v

    def save(self, name):
        self.arrays["meta"] = np.frombuffer(json.dumps(self.meta).encode(), dtype=np.uint8)
        np.savez_compressed(os.path.join(HERE, name), **self.arrays)
        print(f"wrote {name}: {len(self.meta)} cases")


def stream_case(store, data, eb, b, pol, radius, tag, with_blob):
    cfg = _cfg(eb, b, pol, radius)
    try:
        s = dualquant_vector(data, cfg)
    except verr.VlzError as exc:  # pragma: no cover - corpus avoids errors
        raise RuntimeError(f"unexpected reference error {exc!r} for {tag}")
    arrays = dict(
        data=data,
        codes=s.codes.astype(np.uint16),
        outlier_values=s.outlier_values,
        outlier_counts=s.outlier_counts,
        scalars=s.scalars.values,
    )
    meta = dict(tag=tag, shape=list(data.shape), eb=eb, block_edge=b, padding=pol,
                radius=radius, n_out=int(s.outlier_values.size))
    if with_blob:
        blob = compress(data, cfg)
        back, _ = decompress(blob)
        arrays["blob"] = np.frombuffer(blob, dtype=np.uint8)
        arrays["decompressed"] = back
        # lane-1 scalar kernel must agree (criterion 2) -- recorded, not stored
        ref = dualquant_scalar(data, _cfg(eb, b, pol, radius, lanes=1))
        assert ref.same_bytes(s)
    store.add(meta, **arrays)


def make_corpus():
    store = Store()
    rng = np.random.default_rng(20261020)
    caps = {1: 3000, 2: 70, 3: 18}
    ebs = (1e-2, 1e-4, 1e-5)
    radii = (2, 16, 512, 32768)
    # 1) random small arrays x random configs (all decompressed by reference)
    for i in range(60):
        nd = i % 3 + 1
        shape = tuple(int(round(math.exp(rng.uniform(0, math.log(caps[nd]))))) for _ in range(nd))
        data = (_noise if i % 2 else _smooth)(rng, shape)
        b = (8, 16, 32, 64)[int(rng.integers(0, 4))]
        pol = POLICIES[i % len(POLICIES)]
        eb = ebs[int(rng.integers(0, 3))]
        radius = radii[int(rng.integers(0, 4))]
        stream_case(store, data, eb, b, pol, radius, f"rand{i}", with_blob=data.size <= 3000)
    # 2) edge shapes
    edges = [(1,), (2,), (8,), (9,), (65,), (1, 1), (1, 129), (5, 1, 7), (63, 65, 9),
             (17, 1), (1, 1, 1), (9, 9, 9), (8, 8, 8), (33, 31)]
    for j, shape in enumerate(edges):
        data = (_smooth if j % 2 else _noise)(rng, shape)
        for b in (8, 64):
            pol = POLICIES[(j + b) % len(POLICIES)]
            stream_case(store, data, 1e-4, b, pol, 32768, f"edge{j}_b{b}",
                        with_blob=data.size <= 3000)
    # 3) every policy on a 3D and a 2D array with partial blocks
    d3 = _smooth(rng, (19, 21, 23))
    d2 = _smooth(rng, (45, 37))
    d1 = _smooth(rng, (1000,))
    for pol in POLICIES:
        for b in (8, 16):
            stream_case(store, d3, 1e-3, b, pol, 512, f"pol3d_{pol}_b{b}", with_blob=False)
        stream_case(store, d2, 1e-4, 16, pol, 512, f"pol2d_{pol}", with_blob=True)
        stream_case(store, d1, 1e-4, 32, pol, 64, f"pol1d_{pol}", with_blob=True)
    # 4) larger blocks in 3D (b=32, 64) incl. outlier-heavy noise
    stream_case(store, _smooth(rng, (64, 64, 64)), 1e-4, 32, "mean:block", 512, "big32", False)
    stream_case(store, _noise(rng, (40, 70, 66)), 1e-4, 64, "max:edge", 32768, "big64", False)
    stream_case(store, _noise(rng, (30, 33, 40)), 1e-5, 8, "mean:global", 512, "noise8", False)
    stream_case(store, _noise(rng, (60, 50)), 1e-2, 32, "zero", 2, "r2", True)
    # 5) tie-rich, narrowing-heavy and near-overflow data
    for eb in (0.5, 2.0**-10, 1e-3):
        stream_case(store, _ties(rng, (20, 24, 16), eb), eb, 8, "mean:global", 512,
                    f"ties{eb}", False)
    stream_case(store, _ties(rng, (3000,), 0.25), 0.25, 16, "zero", 32768, "ties1d", True)
    stream_case(store, _narrow(rng, (24, 24, 24)), 1e-5, 8, "mean:global", 32768, "narrow3d", False)
    stream_case(store, _narrow(rng, (2000,)), 1e-5, 64, "min:block", 512, "narrow1d", True)
    stream_case(store, _big_q(rng, (16, 16, 16), 1e-3), 1e-3, 8, "zero", 32768, "bigq_zero", False)
    stream_case(store, _big_q(rng, (16, 16, 16), 1e-3), 1e-3, 8, "mean:block", 32768, "bigq_mean", False)
    stream_case(store, _big_q(rng, (40, 40), 1e-3), 1e-3, 16, "max:edge", 512, "bigq2d", False)
    # 6) constant fields (acceptance criterion 4)
    for dims in ((64,), (24, 16), (8, 8, 16)):
        for b in (8, 16, 32, 64):
            for pol in ("zero", "mean:global"):
                stream_case(store, np.full(dims, 100.0, np.float32), 1e-4, b, pol, 32768,
                            f"const{len(dims)}d_b{b}_{pol}", True)
    # 7) BASELINE config 1 at block 256 (patched valid edges), reduced size
    c1 = workloads.gen_c1(20000, seed=11)
    eb1 = workloads.value_range_eb(c1, 1e-4)
    stream_case(store, c1, eb1, 256, "zero", 512, "c1small_b256", True)
    stream_case(store, c1, eb1, 64, "zero", 512, "c1small_b64", True)
    store.save("corpus.npz")


def _exc(fn):
    try:
        fn()
    except verr.VlzError as exc:
        d = {"type": type(exc).__name__, "message": str(exc)}
        if isinstance(exc, verr.BoundTooSmallError):
            d.update(index=exc.index, value=exc.value, bound=exc.bound)
        return d
    return None


def make_errors():
    cases = []

    def add(tag, data, eb, b=8, pol="mean:global"):
        res = _exc(lambda: dualquant_vector(data, _cfg(eb, b, pol, 32768)))
        cases.append(dict(tag=tag, data=data.tolist(), shape=list(data.shape), eb=eb,
                          block_edge=b, padding=pol, expect=res))

    add("overflow_index", np.array([1.0, 3e5, 1.0], np.float32), 1e-5)
    add("nan", np.array([1.0, np.nan], np.float32), 1e-4)
    add("inf_after_overflow", np.array([3e5, 1.0, np.inf, 2.0], np.float32), 1e-5)
    add("overflow_2d", np.array([[0.0, 1.0], [5e9, -5e9]], np.float32), 1.0)
    add("overflow_exact_limit", np.array([0.0, float(np.float32(2**31 - 1))], np.float32), 0.5)
    add("below_limit", np.array([0.0, float(np.float32(2**31 - 256))], np.float32), 0.5)
    add("neg_inf_3d", np.full((2, 3, 4), 1.0, np.float32) * np.array([1, 1, 1, -np.inf], np.float32), 0.1)
    add("ok_tiny", np.array([1e-38, -1e-45, 0.0], np.float32), 1e-4)
    # relative bound on constant data -> DegenerateRangeError
    const = np.full((10,), 3.0, np.float32)
    res = _exc(lambda: dualquant_vector(const, CompressionConfig(ErrorBound.relative(1e-3))))
    cases.append(dict(tag="degenerate_rel", data=const.tolist(), shape=[10], eb=None, rel=1e-3,
                      block_edge=16, padding="mean:global", expect=res))
    # relative bounds over non-finite data: the resolved bound is NaN (or
    # inf) and the non-finite scan names the index
    for tag, vals in (("rel_nan", [1.0, 2.0, np.nan, 3.0]), ("rel_both_inf", [1.0, np.inf, -np.inf]),
                      ("rel_inf", [1.0, 2.0, np.inf, 2.0])):
        arr = np.array(vals, np.float32)
        res = _exc(lambda: dualquant_vector(arr, CompressionConfig(ErrorBound.relative(1e-3))))
        cases.append(dict(tag=tag, data=[float(v) for v in arr], shape=[arr.size], eb=None,
                          rel=1e-3, block_edge=16, padding="mean:global", expect=res))
    # lane width 1: compress() runs the scalar kernel, whose per-element
    # check order differs from the vector path (kernel.py:138-145)
    for tag, vals, eb in (("lane1_overflow_before_inf", [3e5, 1.0, np.inf, 2.0], 1e-5),
                          ("lane1_nan_before_overflow", [1.0, np.nan, 3e5], 1e-5),
                          ("lane1_overflow_2d", [[0.0, 1.0], [5e9, -np.inf]], 1.0),
                          ("lane1_inf_first", [np.inf, 3e5], 1e-5),
                          ("lane1_ok", [1.0, 2.0, 3.0], 1e-3)):
        arr = np.array(vals, np.float32)
        cfg = CompressionConfig(ErrorBound.absolute(eb), block_edge=8, lane_width=1,
                                padding=PaddingPolicy.parse("mean:global"), radius=32768)
        res = _exc(lambda: compress(arr, cfg))
        cases.append(dict(tag=tag, data=arr.ravel().tolist(), shape=list(arr.shape), eb=eb,
                          block_edge=8, padding="mean:global", lane=1, expect=res))
    for tag, vals in (("lane1_rel_nan", [1.0, 3e5, np.nan]),):
        arr = np.array(vals, np.float32)
        cfg = CompressionConfig(ErrorBound.relative(1e-3), lane_width=1)
        res = _exc(lambda: compress(arr, cfg))
        cases.append(dict(tag=tag, data=arr.ravel().tolist(), shape=list(arr.shape), eb=None,
                          rel=1e-3, block_edge=16, padding="mean:global", lane=1, expect=res))
    with open(os.path.join(HERE, "errors.json"), "w") as fh:
        json.dump(cases, fh, indent=1)
    print(f"wrote errors.json: {len(cases)} cases")


def make_corrupt():
    """reconstruct_block / decompress_parsed error cases on tampered streams."""
    store = Store()
    rng = np.random.default_rng(5)
    data = _smooth(rng, (20, 13))
    data[rng.random(data.shape) < 0.08] = 500.0  # spikes -> a few outliers per block
    cfg = _cfg(1e-4, 8, "mean:block", 32768)
    blob = compress(data, cfg)
    parsed = deserialize(blob)
    from vlz.huffman import decode

    codes = decode(parsed.code_bits, parsed.code_bit_length, parsed.codebook,
                   parsed.descriptor.element_count)
    from vlz.model import build_block_grid
    from vlz.padding import apply_padding

    grid = build_block_grid(parsed.descriptor, 8)

    def run_blocks(codes, ovals, counts):
        # decompress_parsed semantics minus Huffman (reconstruct.py:87-124)
        n_sentinel = int(np.count_nonzero(codes == 0))
        if n_sentinel != len(ovals):
            raise verr.CorruptStreamError(f"{n_sentinel} sentinel codes but {len(ovals)} outliers")
        sizes = np.array([int(np.prod(grid.block_extents(b))) for b in range(grid.block_count)])
        cs = np.concatenate([[0], np.cumsum(sizes)])
        os_ = np.concatenate([[0], np.cumsum(counts)])
        for bi in range(grid.block_count):
            reconstruct_block(codes[cs[bi]:cs[bi + 1]], ovals[os_[bi]:os_[bi + 1]],
                              apply_padding(parsed.scalars, grid, bi), grid.block_extents(bi),
                              parsed.resolved_abs, parsed.radius)

    variants = []
    c = codes.copy(); c[np.flatnonzero(c != 0)[3]] = 2 * parsed.radius  # code out of range
    variants.append(("code_range", c, parsed.outlier_values, parsed.outlier_counts))
    c = codes.copy(); idx = np.flatnonzero(c != 0)[70]; c[idx] = 0  # extra sentinel
    variants.append(("sentinel_total", c, parsed.outlier_values, parsed.outlier_counts))
    cnt = parsed.outlier_counts.copy()
    nz = np.flatnonzero(cnt)
    cnt[nz[0]] -= 1; cnt[nz[1]] += 1  # per-block partition wrong
    variants.append(("partition", codes, parsed.outlier_values, cnt))
    cnt = parsed.outlier_counts.copy(); cnt[nz[0]] += 1; cnt[nz[-1]] -= 1
    variants.append(("partition_rev", codes, parsed.outlier_values, cnt))
    for tag, c, ov, cnt in variants:
        res = _exc(lambda: run_blocks(c, ov, cnt))
        store.add(dict(tag=tag, shape=list(data.shape), eb=parsed.resolved_abs, block_edge=8,
                       padding="mean:block", radius=parsed.radius, expect=res),
                  codes=c.astype(np.uint32), outlier_values=ov, outlier_counts=cnt,
                  scalars=parsed.padding_values)
    store.save("corrupt.npz")


def make_known():
    from vlz.quantize import prequantize

    cases = []
    for v, eb in ((3.2, 0.5), (-0.00015, 1e-4), (2.5, 0.5), (-2.5, 0.5), (0.0, 1.0),
                  (-0.0, 1.0), (1e-45, 1e-3), (1.5, 0.5), (0.49999997, 0.5)):
        arr = np.array([v], np.float32)
        cases.append(dict(kind="prequant", v=float(arr[0]), eb=eb,
                          d=int(prequantize(arr, eb).values[0])))
    # random prequant known answers incl. ties
    rng = np.random.default_rng(17)
    vals = np.concatenate([rng.uniform(-1e3, 1e3, 500), (np.arange(-50, 50) + 0.5) * 0.002])
    vals = vals.astype(np.float32)
    for eb in (1e-2, 1e-3, 1e-4, 1e-5):
        q = prequantize(vals, eb).values
        cases.append(dict(kind="prequant_vec", eb=eb, v=vals.tolist(), d=q.tolist()))
    with open(os.path.join(HERE, "known.json"), "w") as fh:
        json.dump(cases, fh)
    print(f"wrote known.json: {len(cases)} cases")


def make_container():
    """Reference deserialize/decode verdicts on mutated containers
    (container.py:166-298, huffman.py:125-207; test_container.py:118-131)."""
    from vlz.huffman import decode as hdecode

    rng = np.random.default_rng(77)
    blobs = []
    d = _smooth(rng, (13, 11))
    blobs.append(compress(d, _cfg(1e-4, 8, "mean:block", 32768)))
    d2 = _noise(rng, (9, 10, 7))
    blobs.append(compress(d2, _cfg(1e-3, 8, "zero", 512)))
    cases = []

    def verdict(blob):
        try:
            parsed = deserialize(blob)
            hdecode(parsed.code_bits, parsed.code_bit_length, parsed.codebook,
                    parsed.descriptor.element_count)
        except verr.VlzError as exc:
            return {"type": type(exc).__name__, "message": str(exc)}
        return None

    import struct
    import zlib

    H = struct.Struct("<4sHHBBBB3QddHHIQ5QI")

    def fix_crc(b: bytes) -> bytes:
        f = list(H.unpack_from(b, 0))
        total = f[20]
        body = b[H.size: len(b) - 4]
        hdr = H.pack(*f[:-1], 0)
        hdr = H.pack(*f[:-1], zlib.crc32(hdr))
        return hdr + body + struct.pack("<I", zlib.crc32(body)) if total == len(b) else \
            hdr + b[H.size:]

    def set_field(b: bytes, idx: int, val) -> bytes:
        f = list(H.unpack_from(b, 0))
        f[idx] = val
        return fix_crc(H.pack(*f) + b[H.size:])

    def patch(b: bytes, off: int, new: bytes) -> bytes:
        return fix_crc(b[:off] + new + b[off + len(new):])

    for bi, blob in enumerate(blobs):
        f = H.unpack_from(blob, 0)
        off_pad, off_cb, off_codes, off_out = f[16:20]
        muts = [("truncate_half", blob[: len(blob) // 2]), ("truncate_small", blob[:50]),
                ("bad_magic", b"XLZ1" + blob[4:]),
                ("version", blob[:4] + (2).to_bytes(2, "little") + blob[6:]),
                ("header_flip", blob[:40] + bytes([blob[40] ^ 1]) + blob[41:]),
                ("payload_flip", blob[:-10] + bytes([blob[-10] ^ 0x10]) + blob[-9:]),
                ("extra_byte", blob + b"\x00"),
                # structured edits with both CRCs recomputed: deeper validation
                ("ndims4", set_field(blob, 3, 4)),
                ("eb_mode", set_field(blob, 4, 7)),
                ("pad_kind", set_field(blob, 5, 9)),
                ("block12", set_field(blob, 12, 12)),
                ("elemcount", set_field(blob, 15, f[15] + 1)),
                ("dim0", set_field(blob, 7, f[7] + 1)),
                ("offsets_swap", set_field(set_field(blob, 17, f[18]), 18, f[17])),
                ("off_pad", set_field(blob, 16, f[16] + 8)),
                ("radius_small", set_field(blob, 14, 2)),
                ("sym_big", patch(blob, off_cb + 4, struct.pack("<H", 65535))),
                ("len_zero", patch(blob, off_cb + 6, b"\x00")),
                ("nbits_plus", patch(blob, off_codes, struct.pack("<Q",
                                   struct.unpack_from("<Q", blob, off_codes)[0] + 1))),
                ("nbits_minus", patch(blob, off_codes, struct.pack("<Q",
                                    struct.unpack_from("<Q", blob, off_codes)[0] - 3))),
                ("nbits_huge", patch(blob, off_codes, struct.pack("<Q", 1 << 40))),
                ("nout_plus", patch(blob, off_out, struct.pack("<Q",
                                  struct.unpack_from("<Q", blob, off_out)[0] + 1))),
                ("nz_huge", patch(blob, off_out + 8, struct.pack("<Q", 1 << 30))),
                ("padcount_huge", patch(blob, off_pad, struct.pack("<Q", 1 << 30)))]
        nz = struct.unpack_from("<Q", blob, off_out + 8)[0]
        if nz:
            muts.append(("pair_block_oob", patch(blob, off_out + 16, struct.pack("<I", 1 << 20))))
            muts.append(("pair_count", patch(blob, off_out + 20, struct.pack("<I", 999))))
        nbytes = (struct.unpack_from("<Q", blob, off_codes)[0] + 7) // 8
        for k in range(12):  # flips inside the Huffman payload, CRCs fixed
            pos = off_codes + 8 + int(rng.integers(0, nbytes))
            muts.append((f"bits{k}", patch(blob, pos, bytes([blob[pos] ^ int(rng.integers(1, 256))]))))
        for k in range(25):
            b = bytearray(blob)
            pos = int(rng.integers(0, len(b)))
            b[pos] ^= int(rng.integers(1, 256))
            muts.append((f"fuzz{k}", bytes(b)))
        for tag, m in muts:
            cases.append(dict(tag=f"b{bi}_{tag}", blob=m.hex(), expect=verdict(m)))
    with open(os.path.join(HERE, "container.json"), "w") as fh:
        json.dump(cases, fh)
    print(f"wrote container.json: {len(cases)} cases")


def make_container_full():
    """Reference decompress(blob) verdicts (any exception class, or the output
    sha256) on crafted containers that pass the CRCs: over-subscribed
    codebooks (Kraft sum > 1) and padding sections shorter than the policy
    needs.  container_full.json."""
    import struct
    import zlib

    H = struct.Struct("<4sHHBBBB3QddHHIQ5QI")

    def rebuild(blob, new_sections):
        """Re-lay the four sections with fresh offsets and both CRCs."""
        f = list(H.unpack_from(blob, 0))
        offs = [H.size]
        for sec in new_sections[:-1]:
            offs.append(offs[-1] + len(sec))
        payload = b"".join(new_sections)
        total = H.size + len(payload) + 4
        f[16:20] = offs
        f[20] = total
        f[21] = 0
        hdr = H.pack(*f)
        f[21] = zlib.crc32(hdr)
        return H.pack(*f) + payload + struct.pack("<I", zlib.crc32(payload))

    def sections(blob):
        f = H.unpack_from(blob, 0)
        o = list(f[16:20]) + [len(blob) - 4]
        return [blob[o[i]:o[i + 1]] for i in range(4)]

    def verdict(blob):
        try:
            arr, _ = decompress(blob)
        except Exception as exc:  # noqa: BLE001 -- any class the reference raises
            return {"type": type(exc).__name__, "message": str(exc)}
        return {"sha256": hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()}

    rng = np.random.default_rng(91)
    cases = []
    srcs = []
    d = _smooth(rng, (21, 17))
    d[rng.random(d.shape) < 0.03] = 300.0
    srcs.append(("mb2d", compress(d, _cfg(1e-4, 8, "mean:block", 512))))
    d3 = _smooth(rng, (10, 12, 9))
    srcs.append(("me3d", compress(d3, _cfg(1e-3, 8, "max:edge", 512))))
    srcs.append(("mg3d", compress(d3, _cfg(1e-3, 8, "mean:global", 512))))
    d1 = _smooth(rng, (300,))
    srcs.append(("z1d", compress(d1, _cfg(1e-3, 16, "zero", 64))))
    for name, blob in srcs:
        pad, cb, codes, outl = sections(blob)
        nsym = struct.unpack_from("<I", cb, 0)[0]
        ent = [struct.unpack_from("<HB", cb, 4 + 3 * i) for i in range(nsym)]
        nbits = struct.unpack_from("<Q", codes, 0)[0]
        f = H.unpack_from(blob, 0)
        count = f[15]

        def book(lens):
            return struct.pack("<I", len(lens)) + b"".join(
                struct.pack("<HB", s, l) for (s, _), l in zip(ent, lens))

        def with_nbits(nb):
            return struct.pack("<Q", nb) + codes[8:]

        muts = []
        if nsym >= 3:
            ones = [1] * nsym
            muts.append(("all_len1", [pad, book(ones), codes, outl]))
            # all length 1 and exactly `count` bits: decode succeeds with a
            # two-symbol stream and the verdict comes from reconstruction
            if count <= (len(codes) - 8) * 8:
                muts.append(("all_len1_fit", [pad, book(ones), with_nbits(count), outl]))
            short = [max(1, l - 1) for _, l in ent]
            muts.append(("lens_minus1", [pad, book(short), codes, outl]))
            three = [1, 1, 1] + [l for _, l in ent[3:]]
            muts.append(("three_len1", [pad, book(three), codes, outl]))
            longtail = [1] + [l for _, l in ent[1:-1]] + [40]
            muts.append(("len1_long40", [pad, book(longtail), codes, outl]))
        # padding section shorter / longer than the policy's scalar count
        pc = struct.unpack_from("<Q", pad, 0)[0]
        vals = pad[8:]
        for k in sorted({0, 1, pc // 2, max(pc - 1, 0), pc + 3}):
            if k == pc:
                continue
            body = (vals + b"\x07" * 8 * 8)[: 8 * k] if k > pc else vals[: 8 * k]
            muts.append((f"padcount_{k}_of_{pc}", [struct.pack("<Q", k) + body, cb, codes, outl]))
        # a corrupt block before / after the first short-padding block: the
        # earlier failure wins (blocks run in order, reconstruct.py:120-122)
        n_out, nz = struct.unpack_from("<QQ", outl, 0)
        if nz >= 2 and pc >= 4:
            pairs = [list(struct.unpack_from("<II", outl, 16 + 8 * i)) for i in range(nz)]
            pairs[0][1] += 1
            pairs[-1][1] -= 1
            moved = outl[:16] + b"".join(struct.pack("<II", *q) for q in pairs) + outl[16 + 8 * nz:]
            b0 = pairs[0][0]
            nd = f[3]
            per = 1 if name.startswith("mb") else nd
            for k in (max(0, b0 * per - per), (b0 + 2) * per):
                if k < pc:
                    muts.append((f"partition_padcount_{k}",
                                 [struct.pack("<Q", k) + vals[: 8 * k], cb, codes, moved]))
            muts.append(("partition_only", [pad, cb, codes, moved]))
        for tag, secs in muts:
            m = rebuild(blob, secs)
            cases.append(dict(tag=f"{name}_{tag}", blob=m.hex(), expect=verdict(m)))
    with open(os.path.join(HERE, "container_full.json"), "w") as fh:
        json.dump(cases, fh)
    print(f"wrote container_full.json: {len(cases)} cases")
    for c in cases:
        print("  ", c["tag"], c["expect"])


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def make_fullsize():
    out = []
    c1 = workloads.gen_c1()
    eb1 = workloads.value_range_eb(c1, 1e-4)
    c2 = workloads.gen_c2()
    eb2 = workloads.value_range_eb(c2, 1e-4)
    runs = [("C1", c1, eb1, 256, "zero"), ("C1", c1, eb1, 64, "zero"),
            ("C2", c2, eb2, 16, "zero"), ("C2", c2, eb2, 16, "mean:block")]
    for name, data, eb, b, pol in runs:
        s = dualquant_vector(data, _cfg(eb, b, pol, 512, lanes=16))
        out.append(dict(config=name, eb=eb, block_edge=b, padding=pol, radius=512,
                        data_sha=_sha(data),
                        codes_u16_sha=_sha(s.codes.astype(np.uint16)),
                        outliers_sha=_sha(s.outlier_values), counts_sha=_sha(s.outlier_counts),
                        scalars_sha=_sha(s.scalars.values), n_out=int(s.outlier_values.size)))
        print(name, b, pol, "outliers", out[-1]["n_out"])
    with open(os.path.join(HERE, "fullsize.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print("wrote fullsize.json")


def make_border():
    """outlier_report (padding.py:162-205): per-policy total / border outlier
    counts and the reduction versus zero padding, from the reference."""
    from vlz.padding import outlier_report

    cases = []
    rng = np.random.default_rng(23)
    shapes = [(200,), (37, 41), (19, 23, 29), (16, 16, 16), (9, 40, 33)]
    for k, shape in enumerate(shapes):
        for b in (8, 16):
            if len(shape) == 1 and b == 16:
                continue
            data = (_smooth(rng, shape) + 0.003 * _noise(rng, shape)).astype(np.float32)
            eb = float(0.002 * (float(data.max()) - float(data.min())))
            for radius in (8, 512):
                cfg = _cfg(eb, b, "zero", radius)
                rows = outlier_report(data, cfg)
                cases.append(dict(
                    tag=f"border{k}_b{b}_r{radius}", shape=list(shape),
                    data=data.tobytes().hex(), eb=eb, block_edge=b, radius=radius,
                    rows=[dict(kind=r.policy.value_kind.value, gran=r.policy.granularity.value,
                               total=r.total_outliers, border=r.border_outliers,
                               reduction=red) for r, red in rows]))
    blob = json.dumps(cases).encode()
    np.savez_compressed(os.path.join(HERE, "border.npz"),
                        meta=np.frombuffer(blob, dtype=np.uint8))
    print(f"wrote border.npz: {len(cases)} cases")


if __name__ == "__main__":
    what = sys.argv[1:] or ["corpus", "errors", "corrupt", "known", "fullsize", "container",
                            "border"]
    for w in what:
        globals()[f"make_{w}"]()
