"""GPU Huffman encoder (csrc/k_huffenc.cu) against the native host packer,
which is pinned to the reference by tests/test_container.py (byte-identical
containers and codebooks).  Covers chunk boundaries (4096 symbols per CTA),
ragged tails, one-symbol books, deep codewords that span three 32-bit words,
and the reference's error precedence (huffman.py:102-104)."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2201_04614_b200 import gpu  # noqa: E402
from paper_2201_04614_b200.errors import CorruptStreamError  # noqa: E402
from paper_2201_04614_b200.huffman import build_codebook, encode  # noqa: E402


def _dev(codes):
    return torch.from_numpy(codes.view(np.int16).copy()).cuda()


def _check(codes):
    cb = build_codebook(codes)
    want = encode(codes, cb)
    got = gpu.huffman_encode_device(_dev(codes), cb.symbols, cb.lengths)
    assert got[1] == want[1]
    assert got[0] == want[0]
    return cb


@pytest.mark.parametrize("n", [1, 2, 15, 16, 17, 4095, 4096, 4097, 8192 + 33, 100_003])
def test_sizes_around_chunk_boundaries(n):
    rng = np.random.default_rng(n)
    codes = (512 + np.round(rng.normal(0, 3, n))).astype(np.uint16)
    codes[rng.integers(0, n, max(1, n // 50))] = 0  # outlier sentinels
    _check(codes)


def test_single_symbol_book():
    _check(np.full(10_000, 512, np.uint16))


def test_deep_codewords_cross_words():
    # Fibonacci-like frequencies give codeword lengths far beyond 32 bits
    fib = [1, 1]
    while len(fib) < 45:
        fib.append(fib[-1] + fib[-2])
    parts = [np.full(f, 100 + k, np.uint16) for k, f in enumerate(fib[:30])]
    codes = np.concatenate(parts)
    rng = np.random.default_rng(0)
    rng.shuffle(codes)
    cb = _check(codes[:300_000])
    assert int(cb.lengths.max()) > 20


def test_random_books_and_skews():
    rng = np.random.default_rng(7)
    for trial in range(6):
        n = int(rng.integers(1000, 300_000))
        k = int(rng.integers(2, 3000))
        p = rng.dirichlet(np.full(k, 0.3))
        codes = rng.choice(np.arange(1, k + 1, dtype=np.uint16) * 7, size=n, p=p).astype(np.uint16)
        _check(codes)


def test_large_stream():
    rng = np.random.default_rng(11)
    codes = (512 + np.round(rng.laplace(0, 2, 20_000_000))).clip(1, 1023).astype(np.uint16)
    _check(codes)


def test_error_precedence():
    cb = build_codebook(np.array([3, 3, 7], np.uint16))
    for stream, bad in (([5, 9], 9), ([9, 5], 9), ([5, 3], 5), ([3, 4], 4)):
        s = np.array(stream * 3000, np.uint16)
        with pytest.raises(CorruptStreamError, match=f"symbol {bad} not in the codebook"):
            gpu.huffman_encode_device(_dev(s), cb.symbols, cb.lengths)


# ---- decoder (csrc/k_huffdec.cu) -------------------------------------------

from conftest import load_json  # noqa: E402

from paper_2201_04614_b200 import errors as E  # noqa: E402
from paper_2201_04614_b200.container import deserialize  # noqa: E402
from paper_2201_04614_b200.huffman import HuffmanCodebook, decode, decode_device  # noqa: E402


def _verdict(fn):
    try:
        r = fn()
        return ("ok", r if isinstance(r, np.ndarray) else r.cpu().numpy().view(np.uint16))
    except E.VlzError as exc:
        return (type(exc).__name__, str(exc))


def _same_verdict(payload, nbits, cb, count):
    h = _verdict(lambda: decode(payload, nbits, cb, count))
    d = _verdict(lambda: decode_device(payload, nbits, cb, count))
    assert h[0] == d[0]
    if h[0] == "ok":
        assert np.array_equal(h[1], d[1])
    else:
        assert h[1] == d[1]
    return h


@pytest.mark.parametrize("n", [1, 2, 31, 280, 281, 4096, 100_003, 3_000_000])
def test_decode_round_trip(n):
    rng = np.random.default_rng(n + 1)
    codes = (512 + np.round(rng.normal(0, 4, n))).astype(np.uint16)
    codes[rng.integers(0, n, max(1, n // 40))] = 0
    cb = build_codebook(codes)
    payload, nbits = encode(codes, cb)
    got = decode_device(payload, nbits, cb, n).cpu().numpy().view(np.uint16)
    assert np.array_equal(got, codes)


def test_decode_deep_and_skewed_books():
    rng = np.random.default_rng(5)
    fib = [1, 1]
    while len(fib) < 32:
        fib.append(fib[-1] + fib[-2])
    codes = np.concatenate([np.full(f, 40 + k, np.uint16) for k, f in enumerate(fib)])
    rng.shuffle(codes)
    for c in (codes[:500_000], np.full(5000, 9, np.uint16),
              rng.choice(np.arange(1, 2001, dtype=np.uint16), 400_000,
                         p=rng.dirichlet(np.full(2000, 0.2))).astype(np.uint16)):
        cb = build_codebook(c)
        payload, nbits = encode(c, cb)
        got = decode_device(payload, nbits, cb, c.size).cpu().numpy().view(np.uint16)
        assert np.array_equal(got, c)


def test_decode_verdicts_match_host():
    rng = np.random.default_rng(9)
    codes = (300 + np.round(rng.normal(0, 3, 50_000))).astype(np.uint16)
    cb = build_codebook(codes)
    payload, nbits = encode(codes, cb)
    n = codes.size
    cases = [
        (payload, nbits, n - 1),            # fewer symbols than the stream holds -> 5
        (payload, nbits, n + 7),            # more symbols than the stream holds -> 3
        (payload, nbits + 3, n),            # declared length too long -> 5 or 2
        (payload, nbits - 1, n),            # declared length too short -> 5
        (payload[: len(payload) // 2], nbits // 2, n),  # truncated -> 3
        (payload, 0, 0),                    # empty stream, zero bits -> ok
        (payload, 5, 0),                    # empty stream, nonzero bits -> 1
        (payload[:10], nbits, n),           # shorter than declared -> 2
        (b"", 0, 3),                        # nothing to read -> 3
    ]
    for pl, nb, cnt in cases:
        _same_verdict(pl, nb, cb, cnt)
    # incomplete book (one symbol, code "0"): any 1 bit is an invalid prefix
    one = HuffmanCodebook.from_lengths(np.array([7], np.uint32), np.array([1], np.uint8))
    for pl, nb, cnt in ((b"\x00\x10", 16, 16), (b"\x00" * 300 + b"\x80", 2408, 2408),
                        (b"\x00" * 300, 2400, 2400)):
        _same_verdict(pl, nb, one, cnt)
    # random corruption of a valid payload
    for t in range(20):
        pl = bytearray(payload)
        for _ in range(1 + t % 4):
            i = int(rng.integers(0, len(pl)))
            pl[i] ^= 1 << int(rng.integers(0, 8))
        _same_verdict(bytes(pl), nbits, cb, n)


def test_decode_reference_mutated_containers():
    cases = load_json("container.json")
    n = 0
    for c in cases:
        try:
            p = deserialize(bytes.fromhex(c["blob"]))
        except E.VlzError:
            continue
        if not len(p.codebook.lengths) or int(p.codebook.lengths.max()) > 58:
            continue
        got = _verdict(lambda: decode_device(p.code_bits, p.code_bit_length, p.codebook,
                                             p.descriptor.element_count))
        exp = c["expect"]
        if exp is None:
            assert got[0] == "ok", c["tag"]
        else:
            assert got == (exp["type"], exp["message"]), c["tag"]
        n += 1
    assert n > 20
