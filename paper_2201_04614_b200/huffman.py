"""Canonical Huffman coding of the code stream (entropy stage after the path).

Same codebook, bit order and error verdicts as the reference
(/root/reference/pkg/src/vlz/huffman.py): lengths from a Huffman merge whose
ties are broken by the smallest symbol of each subtree (huffman.py:56-88),
canonical codewords sorted by (length, symbol) (huffman.py:33-45), MSB-first
packing with a zero-padded last byte (huffman.py:91-122), and a decoder that
reads exactly `count` symbols (huffman.py:125-207).  The work is done natively
in libvlzgpu.so (csrc/huffman.cpp); the histogram runs on the GPU when the
codes are device resident.
"""

from __future__ import annotations

import ctypes
import warnings
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ConfigError, CorruptStreamError


@dataclass(frozen=True)
class HuffmanCodebook:
    symbols: np.ndarray   # uint32, sorted by (length, symbol)
    lengths: np.ndarray   # uint8, same order
    codewords: np.ndarray  # uint64, canonical codes

    @classmethod
    def from_lengths(cls, symbols: np.ndarray, lengths: np.ndarray) -> "HuffmanCodebook":
        order = np.lexsort((symbols, lengths))
        symbols = np.asarray(symbols)[order].astype(np.uint32)
        lengths = np.asarray(lengths)[order].astype(np.uint8)
        cw = np.zeros(len(symbols), dtype=np.uint64)
        code = 0
        for i in range(len(symbols)):
            cw[i] = code
            code += 1
            if i + 1 < len(symbols):
                code <<= int(lengths[i + 1]) - int(lengths[i])
        return cls(symbols, lengths, cw)

    def kraft_sum(self) -> float:
        return float(np.sum(2.0 ** (-self.lengths.astype(np.float64))))


def histogram(codes) -> np.ndarray:
    """uint64[65536] symbol frequencies of a uint16/uint32 code array (numpy
    array on the host, or a CUDA tensor -> counted on the device)."""
    if hasattr(codes, "is_cuda") and codes.is_cuda:
        from .gpu import histogram_device

        return histogram_device(codes)
    c = np.ascontiguousarray(codes).ravel()
    if c.dtype != np.uint16:
        if c.size and int(c.max()) > 0xFFFF:
            raise CorruptStreamError(f"symbol {int(c.max())} not in the codebook")
        c = c.astype(np.uint16)
    freqs = np.empty(65536, dtype=np.uint64)
    _lib.load().vlz_histogram_host(c.ctypes.data, c.size, freqs.ctypes.data)
    return freqs


def build_codebook_from_freqs(freqs: np.ndarray) -> HuffmanCodebook:
    lib = _lib.load()
    freqs = np.ascontiguousarray(freqs, dtype=np.uint64)
    syms = np.empty(65536, dtype=np.uint16)
    lens = np.empty(65536, dtype=np.uint8)
    n = ctypes.c_int32(0)
    rc = lib.vlz_huff_build(freqs.ctypes.data, syms.ctypes.data, lens.ctypes.data,
                            ctypes.byref(n))
    if rc == -1:
        raise ConfigError("cannot build a codebook for an empty code stream")
    if rc != 0:
        raise ConfigError("Huffman code lengths exceed 64 bits")
    k = n.value
    return HuffmanCodebook.from_lengths(syms[:k].astype(np.uint32), lens[:k])


def build_codebook(codes) -> HuffmanCodebook:
    """Optimal prefix-code lengths for the symbols of `codes` (huffman.py:56)."""
    if getattr(codes, "size", None) == 0 or (hasattr(codes, "numel") and codes.numel() == 0):
        raise ConfigError("cannot build a codebook for an empty code stream")
    return build_codebook_from_freqs(histogram(codes))


def encode(codes, codebook: HuffmanCodebook):
    """Pack a symbol stream into bits; returns (payload bytes, bit_length).
    A CUDA tensor of uint16 codes is packed on the GPU (csrc/k_huffenc.cu)."""
    if hasattr(codes, "is_cuda") and codes.is_cuda:
        from .gpu import huffman_encode_device

        return huffman_encode_device(codes, codebook.symbols, codebook.lengths)
    lib = _lib.load()
    c = np.ascontiguousarray(codes).ravel()
    if c.size == 0:
        return b"", 0
    if c.dtype != np.uint16:
        if int(c.max()) > 0xFFFF:
            raise CorruptStreamError(f"symbol {int(c.max())} not in the codebook")
        c = c.astype(np.uint16)
    syms = codebook.symbols.astype(np.uint16)
    lens = np.ascontiguousarray(codebook.lengths, dtype=np.uint8)
    max_bits = int(c.size) * int(lens.max())
    out = np.empty(max_bits // 8 + 1, dtype=np.uint8)
    nbits = ctypes.c_int64(0)
    bad = ctypes.c_int64(-1)
    rc = lib.vlz_huff_encode(c.ctypes.data, c.size, syms.ctypes.data, lens.ctypes.data,
                             len(syms), out.ctypes.data, out.size, ctypes.byref(nbits),
                             ctypes.byref(bad))
    if rc == -1:
        raise CorruptStreamError(f"symbol {bad.value} not in the codebook")
    if rc != 0:
        raise RuntimeError(f"vlz_huff_encode failed ({rc})")
    nb = nbits.value
    return out[: (nb + 7) // 8].tobytes(), nb


def raise_decode_verdict(rc: int, consumed: int, bit_length: int) -> None:
    """The reference's decode errors (huffman.py:135-207), by verdict code."""
    if rc == 1:
        raise CorruptStreamError("nonzero bit length for an empty stream")
    if rc == 2:
        raise CorruptStreamError("bit payload shorter than its declared length")
    if rc == 3:
        raise CorruptStreamError("bit stream underrun mid-symbol")
    if rc == 4:
        raise CorruptStreamError("invalid prefix in bit stream")
    if rc == 5:
        raise CorruptStreamError(f"decoded {consumed} bits but the stream declares {bit_length}")
    if rc != 0:
        raise RuntimeError(f"Huffman decode failed ({rc})")


def decode(payload: bytes, bit_length: int, codebook: HuffmanCodebook, count: int) -> np.ndarray:
    """Decode exactly `count` symbols consuming exactly `bit_length` bits
    (native host decoder; decode_device runs on the GPU)."""
    lib = _lib.load()
    out = np.empty(max(int(count), 1), dtype=np.uint16)
    buf = np.frombuffer(payload, dtype=np.uint8) if len(payload) else np.zeros(1, np.uint8)
    syms = codebook.symbols.astype(np.uint16)
    lens = np.ascontiguousarray(codebook.lengths, dtype=np.uint8)
    consumed = ctypes.c_int64(0)
    rc = lib.vlz_huff_decode(buf.ctypes.data, len(payload), int(bit_length), syms.ctypes.data,
                             lens.ctypes.data, len(syms), int(count), out.ctypes.data,
                             ctypes.byref(consumed))
    raise_decode_verdict(rc, consumed.value, bit_length)
    return out[: int(count)]


def decode_device(payload: bytes, bit_length: int, codebook: HuffmanCodebook, count: int,
                  device=None, device_src=None):
    """decode() on the GPU (csrc/k_huffdec.cu, self-synchronising parallel
    decode); returns an int16-storage CUDA tensor of `count` uint16 symbols.
    `device_src` = (CUDA uint8 tensor, offset): the payload bytes are already
    on the device there (deserialize(blob, device=...)), no host copy."""
    import torch

    from .gpu import _stream

    lib = _lib.load()
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    nbytes = len(payload)
    dpay = torch.empty((nbytes + 3) // 4 * 4 + 16, dtype=torch.uint8, device=dev)
    dpay[nbytes:].zero_()  # the decoder reads up to 16 bytes past the payload
    if nbytes and device_src is not None:
        src, off = device_src
        dpay[:nbytes].copy_(src[off: off + nbytes])
    elif nbytes:
        with warnings.catch_warnings():  # read-only view: only ever read (H2D source)
            warnings.simplefilter("ignore", UserWarning)
            host = torch.frombuffer(payload, dtype=torch.uint8, count=nbytes)
        dpay[:nbytes].copy_(host)
    out = torch.empty(max(int(count), 1), dtype=torch.int16, device=dev)
    ws = torch.empty(int(lib.vlz_huff_decode_ws_size(nbytes)), dtype=torch.uint8, device=dev)
    syms = np.ascontiguousarray(codebook.symbols, dtype=np.uint16)
    lens = np.ascontiguousarray(codebook.lengths, dtype=np.uint8)
    consumed = ctypes.c_int64(0)
    rc = lib.vlz_huff_decode_device(dpay.data_ptr(), nbytes, int(bit_length), syms.ctypes.data,
                                    lens.ctypes.data, len(syms), int(count), out.data_ptr(),
                                    ctypes.byref(consumed), ws.data_ptr(), ws.numel(),
                                    _stream(None))
    raise_decode_verdict(rc, consumed.value, bit_length)
    return out[: int(count)]
