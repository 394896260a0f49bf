"""End-to-end entry points of the drop-in (reference pipeline.py:16-32,
reconstruct.py:74-129).

    blob = compress(data, config)          # float32 ndarray -> VLZ1 bytes
    arr, desc = decompress(blob)           # VLZ1 bytes -> float32 ndarray

Both run the dual-quant path on the GPU (libvlzgpu.so); the entropy stage
(histogram on the GPU, canonical Huffman codebook + MSB-first coding natively
on the host) and the container framing produce the reference's exact bytes.
`lane_width` 1 and the vector lane widths give the same bytes, as in the
reference (its scalar and vector kernels are byte-identical); lane width 1
keeps the scalar kernel's error order (first offending index wins,
kernel.py:138-145) where the vector path reports non-finite values first.
"""

from __future__ import annotations

import numpy as np
import torch

from . import gpu
from .container import ParsedContainer, deserialize, serialize_parts
from .errors import BoundTooSmallError, ConfigError
from .huffman import build_codebook_from_freqs, decode, decode_device, encode
from .model import (
    ArrayDescriptor,
    CodeStream,
    CompressionConfig,
    PaddingScalars,
    build_block_grid,
    resolve_error_bound,
)
from .reconstruct import reconstruct_arrays

__all__ = ["compress", "compress_detailed", "decompress", "decompress_parsed"]


def _device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2201_04614_b200 needs a CUDA device (B200); no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


_H2D_CHUNK = 1 << 24  # float32 elements (64 MB) per pinned staging buffer


def _to_device(data: np.ndarray, device) -> torch.Tensor:
    """Host array -> device tensor through two pinned staging buffers: the
    (multi-threaded) copy of chunk i into one overlaps the DMA of chunk i-1
    from the other (a pageable .to() runs at ~11 GB/s)."""
    src = torch.from_numpy(np.ascontiguousarray(data)).reshape(-1)
    n = src.numel()
    x = torch.empty(n, dtype=src.dtype, device=device)
    if n <= _H2D_CHUNK // 4:
        x.copy_(src)
        return x.view(data.shape)
    stream = torch.cuda.current_stream(device)
    bufs = [torch.empty(_H2D_CHUNK, dtype=src.dtype, pin_memory=True) for _ in range(2)]
    done = [None, None]
    for i, s0 in enumerate(range(0, n, _H2D_CHUNK)):
        k = i & 1
        m = min(_H2D_CHUNK, n - s0)
        if done[k] is not None:
            done[k].synchronize()  # the DMA out of this buffer has finished
        bufs[k][:m].copy_(src[s0:s0 + m])
        x[s0:s0 + m].copy_(bufs[k][:m], non_blocking=True)
        done[k] = torch.cuda.Event()
        done[k].record(stream)
    for e in done:
        if e is not None:
            e.synchronize()  # staging buffers return to the caching host allocator
    return x.view(data.shape)


def _compress(data: np.ndarray, config: CompressionConfig, want_stream: bool):
    desc = ArrayDescriptor.from_array(data)
    eb = resolve_error_bound(config.error_bound, data)
    grid = build_block_grid(desc, config.block_edge)
    gpu.check_resolved_eb(eb, data)
    x = _to_device(data, _device())
    dev = gpu.compress_device(x, config, eb=eb)
    try:
        dev.check(scalar_order=config.lane_width == 1)  # pipeline.py:28-31
    except BoundTooSmallError as exc:
        raise BoundTooSmallError(exc.index, float(data.ravel()[exc.index]), eb) from None
    n_out = dev.n_outliers
    dcodes = dev.codes[: desc.element_count]
    freqs = gpu.histogram_device(dcodes, config.radius)
    codebook = build_codebook_from_freqs(freqs)
    # exact payload size: sum of frequency x codeword length
    nbits_hint = int((freqs[codebook.symbols] * codebook.lengths.astype(np.uint64)).sum())
    if int(codebook.lengths.max()) <= 58:
        bits, nbits = gpu.huffman_encode_device(dcodes, codebook.symbols, codebook.lengths,
                                                nbits_hint=nbits_hint, keep_on_device=True)
    else:  # pathological book (> 10^12 symbols): native host packer
        bits, nbits = encode(dcodes.cpu().numpy().view(np.uint16), codebook)
    outliers = dev.outliers[:n_out].cpu().numpy()
    counts = dev.counts[: grid.block_count].cpu().numpy()
    scalars = dev.scalars.cpu().numpy().astype(np.int64)
    blob = serialize_parts(desc, config, eb, config.radius, codebook, bits, nbits, scalars,
                           counts, outliers, grid.block_count)
    stream = None
    if want_stream:
        codes16 = dcodes.cpu().numpy().view(np.uint16)
        stream = CodeStream(codes=codes16.astype(np.uint32), outlier_values=outliers,
                            outlier_counts=counts, grid=grid, resolved_abs=eb,
                            radius=config.radius,
                            scalars=PaddingScalars(config.padding, scalars))
    return blob, stream


def compress(data: np.ndarray, config: CompressionConfig) -> bytes:
    """pipeline.py:16-23: float32 array -> container bytes."""
    return _compress(data, config, want_stream=False)[0]


def compress_detailed(data: np.ndarray, config: CompressionConfig):
    """pipeline.py:26-32: (container bytes, CodeStream)."""
    return _compress(data, config, want_stream=True)


def decompress_parsed(parsed: ParsedContainer, thread_count: int = 1):
    """reconstruct.py:74-124: Huffman decode and block reconstruction, both on
    the GPU (thread_count is accepted for compatibility and ignored)."""
    desc = parsed.descriptor
    grid = build_block_grid(desc, parsed.block_edge)
    cb = parsed.codebook
    if len(cb.lengths) and int(cb.lengths.max()) <= 58:
        src = None
        if parsed.device_payload is not None:
            src = (parsed.device_payload, parsed.device_code_offset)
        codes = decode_device(parsed.code_bits, parsed.code_bit_length, cb, desc.element_count,
                              device=_device(), device_src=src)
    else:  # empty or pathological book: verdicts from the native host decoder
        codes = decode(parsed.code_bits, parsed.code_bit_length, cb, desc.element_count)
    out = reconstruct_arrays(codes, parsed.outlier_values, parsed.outlier_counts,
                             parsed.padding_values, grid, parsed.resolved_abs, parsed.radius,
                             parsed.padding_policy)
    return out, desc


def decompress(blob: bytes, thread_count: int = 1):
    """reconstruct.py:127-129: container bytes -> (float32 array, descriptor).
    The payload goes to the GPU once: its CRC and the Huffman decode run there."""
    return decompress_parsed(deserialize(blob, device=_device()), thread_count=thread_count)
