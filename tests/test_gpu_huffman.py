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
