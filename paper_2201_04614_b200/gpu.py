"""Device-level API: run the dual-quant kernels on CUDA tensors.

PyTorch is only the tensor/stream plumbing here: every computation happens
in libvlzgpu.so (paper_2201_04614_b200/csrc).  Results stay on the device;
`check()` reads back the 64-byte status block and raises the reference's
exception for it (errors.py; reference quantize.py:58-72, reconstruct.py:
43-66,87-91).

    dev = compress_device(x, config)            # x: cuda float32 tensor
    dev.check()                                  # raises on bad input
    y = decompress_device(dev)                   # cuda float32 tensor
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import BoundTooSmallError, ConfigError, CorruptStreamError, OutlierCapacityError
from .model import (
    ArrayDescriptor,
    BlockGrid,
    CompressionConfig,
    ErrorBound,
    ErrorBoundMode,
    PaddingGranularity,
    PaddingPolicy,
    PaddingValue,
    build_block_grid,
    resolve_error_bound_from_range,
)


def _ptr(t) -> int:
    return 0 if t is None else t.data_ptr()


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def value_range(x: torch.Tensor, stream=None):
    """(float(min), float(max)) of a float32 CUDA tensor, NaN-propagating like
    numpy (model.py:104-107).  Synchronises."""
    lib = _lib.load()
    out = torch.empty(2, dtype=torch.float64, device=x.device)
    rc = lib.vlz_minmax(_ptr(x), x.numel(), _ptr(out), _stream(stream))
    if rc != 0:
        raise RuntimeError(f"vlz_minmax failed ({rc})")
    lo, hi = out.tolist()
    return lo, hi


def check_resolved_eb(eb: float, data) -> None:
    """quantize.py:58-64 on a resolved bound.  A NaN bound comes from a
    value-range-relative bound over data holding NaN (or both infinities):
    the reference's `eb <= 0` test lets it through and its non-finite scan
    names the first such element, so the same ConfigError is raised here
    (the scan runs on the device for a CUDA tensor)."""
    if eb > 0.0:
        return
    if eb != eb:
        if isinstance(data, torch.Tensor):
            bad = ~torch.isfinite(data.reshape(-1))
            idx = int(torch.argmax(bad.to(torch.uint8)).item())
        else:
            idx = int(np.argmin(np.isfinite(np.asarray(data).ravel())))
        raise ConfigError(f"data contains a non-finite value at flat index {idx}")
    raise ConfigError(f"resolved error bound must be > 0, got {eb}")


def resolve_eb_device(eb: ErrorBound, x: torch.Tensor) -> float:
    if x.numel() == 0:
        raise ConfigError("cannot resolve an error bound for empty data")
    if eb.mode is ErrorBoundMode.ABSOLUTE:
        return float(eb.value)
    lo, hi = value_range(x)
    return resolve_error_bound_from_range(eb, lo, hi)


@dataclass
class DeviceCodeStream:
    """CodeStream fields as CUDA tensors (codes uint16 as int16 storage)."""

    codes: torch.Tensor            # int16 [N], reinterpret as uint16
    outliers: torch.Tensor         # float32 [N] capacity, first n_outliers valid
    counts: torch.Tensor           # int64 [nblocks]
    scalars: torch.Tensor          # int64 [scalar_count]
    result: torch.Tensor           # int64 [8] = vlz_result
    grid: BlockGrid
    eb: float
    radius: int
    padding: PaddingPolicy
    source: torch.Tensor = None    # input (kept for error reporting)
    _host_result: object = None

    @property
    def shape(self):
        return self.grid.descriptor.dims

    def read_result(self) -> _lib.Result:
        if self._host_result is None:
            r = _lib.Result()
            buf = self.result.cpu().numpy()
            ctypes.memmove(ctypes.byref(r), buf.ctypes.data, 64)
            self._host_result = r
        return self._host_result

    @property
    def n_outliers(self) -> int:
        return int(self.read_result().n_outliers)

    def check(self, scalar_order: bool = False) -> "DeviceCodeStream":
        """Raise the reference's exception for a failed compress.  The vector
        path (quantize.py:60-72) reports any non-finite value before any
        overflow; the scalar kernel at lane width 1 (kernel.py:138-145) checks
        element by element, so the smaller flat index decides
        (`scalar_order=True`).  first_overflow counts non-finite values too."""
        r = self.read_result()
        if scalar_order and r.status in (_lib.ST_NONFINITE, _lib.ST_OVERFLOW):
            first = min(int(r.first_nonfinite), int(r.first_overflow))
            if first == int(r.first_nonfinite):
                raise ConfigError(f"data contains a non-finite value at flat index {first}")
            v = float(self.source.reshape(-1)[first].item()) if self.source is not None else float("nan")
            raise BoundTooSmallError(first, v, self.eb)
        if r.status == _lib.ST_NONFINITE:
            raise ConfigError(f"data contains a non-finite value at flat index {r.index}")
        if r.status == _lib.ST_OVERFLOW:
            v = float(self.source.reshape(-1)[r.index].item()) if self.source is not None else float("nan")
            raise BoundTooSmallError(int(r.index), v, self.eb)
        if r.status == _lib.ST_OUTLIER_CAPACITY:
            raise OutlierCapacityError(int(r.n_outliers), int(self.outliers.numel()))
        if r.status != _lib.ST_OK:
            raise RuntimeError(f"unexpected compress status {r.status}")
        return self

    def outlier_values(self) -> torch.Tensor:
        return self.outliers[: self.n_outliers]


def _alloc_like(n, dtype, device):
    return torch.empty(max(int(n), 1), dtype=dtype, device=device)


DENSE_SCRATCH_MAX = 1 << 26  # elements (256 MB of scratch)


class Workspace:
    """Grow-only device workspace cache (one per device)."""

    _cache = {}

    @classmethod
    def get(cls, nbytes: int, device) -> torch.Tensor:
        key = (device.type, device.index)
        ws = cls._cache.get(key)
        if ws is None or ws.numel() < nbytes:
            ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
            cls._cache[key] = ws
        return ws


def compress_device(x: torch.Tensor, config: CompressionConfig, eb: float = None,
                    stream=None, workspace: torch.Tensor = None,
                    out: DeviceCodeStream = None,
                    outlier_capacity: int = None) -> DeviceCodeStream:
    """Fused dual-quant compress of a CUDA float32 tensor (no host sync unless
    the bound is value-range relative).  `outlier_capacity` bounds the outlier
    array (default: the worst case, one slot per element); a stream with more
    outliers makes check() raise OutlierCapacityError carrying the count to
    retry with."""
    if not x.is_cuda:
        raise ConfigError("compress_device needs a CUDA tensor")
    desc = ArrayDescriptor.from_array(x)
    grid = build_block_grid(desc, config.block_edge)
    if desc.ndims != 1 and config.block_edge == 256:
        raise ConfigError("block edge 256 is supported for 1-D arrays only")
    if eb is None:
        eb = resolve_eb_device(config.error_bound, x)
    check_resolved_eb(eb, x)
    x = x.contiguous()
    lib = _lib.load()
    g = _lib.geom(desc.dims, config.block_edge)
    pol = config.padding
    p = _lib.params(eb, config.radius, pol.kind_code, pol.gran_code)
    n = desc.element_count
    ns = pol.scalar_count(grid)
    dev = x.device
    if out is None:
        out = DeviceCodeStream(
            codes=_alloc_like(n, torch.int16, dev),
            outliers=_alloc_like(n if outlier_capacity is None else min(n, int(outlier_capacity)),
                                 torch.float32, dev),
            counts=_alloc_like(grid.block_count, torch.int64, dev),
            scalars=torch.empty(ns, dtype=torch.int64, device=dev),
            result=torch.empty(8, dtype=torch.int64, device=dev),
            grid=grid, eb=eb, radius=config.radius, padding=pol, source=x,
        )
    else:
        out.grid, out.eb, out.radius, out.padding, out.source = grid, eb, config.radius, pol, x
        out._host_result = None
    # arrays up to DENSE_SCRATCH_MAX elements get the dense scratch layout (one
    # slot per element: outlier-dense blocks are copied, not regenerated); for
    # larger ones the 4 bytes per element are not worth it (8 slots per block)
    wsb = (lib.vlz_workspace_size_dense(ctypes.byref(g)) if n <= DENSE_SCRATCH_MAX
           else lib.vlz_workspace_size(ctypes.byref(g)))
    ws = workspace if workspace is not None else Workspace.get(wsb, dev)
    # (the library picks the scratch layout from the size it is told: a cached
    # workspace grown by an earlier, larger call must not switch it)
    ws_bytes = ws.numel() if workspace is not None else wsb
    if outlier_capacity is not None and int(outlier_capacity) < 0:
        raise ConfigError("outlier_capacity must be >= 0")
    cap = min(n, int(out.outliers.numel())) if (outlier_capacity is not None or
                                                out.outliers.numel() < n) else None
    if cap is None:
        rc = lib.vlz_dq_compress(
            _ptr(x), ctypes.byref(g), ctypes.byref(p), _ptr(out.codes), _ptr(out.outliers),
            _ptr(out.counts), _ptr(out.scalars) if ns else None, _ptr(out.result), _ptr(ws),
            ws_bytes, _stream(stream),
        )
    else:
        if outlier_capacity is not None:
            cap = min(cap, int(outlier_capacity))
        rc = lib.vlz_dq_compress_capped(
            _ptr(x), ctypes.byref(g), ctypes.byref(p), _ptr(out.codes), _ptr(out.outliers), cap,
            _ptr(out.counts), _ptr(out.scalars) if ns else None, _ptr(out.result), _ptr(ws),
            ws_bytes, _stream(stream),
        )
    if rc != 0:
        raise RuntimeError(f"vlz_dq_compress failed ({rc})")
    return out


def block_span(grid: BlockGrid, bi: int):
    """(start, size) of block bi in the canonical code stream."""
    dims = grid.descriptor.dims
    nd = len(dims)
    org = grid.block_origin(bi)
    ext = grid.block_extents(bi)
    if nd == 1:
        start = org[0]
    elif nd == 2:
        start = org[0] * dims[1] + ext[0] * org[1]
    else:
        start = org[0] * dims[1] * dims[2] + ext[0] * org[1] * dims[2] + ext[0] * ext[1] * org[2]
    return start, int(np.prod(ext))


def decompress_device(codes: torch.Tensor, outliers: torch.Tensor, n_outliers: int,
                      counts: torch.Tensor, scalars: torch.Tensor, grid: BlockGrid, eb: float,
                      radius: int, padding: PaddingPolicy, out: torch.Tensor = None,
                      result: torch.Tensor = None, stream=None, workspace=None,
                      check: bool = True) -> torch.Tensor:
    """Fused reconstruction (reconstruct.py:74-124 minus Huffman decode).
    codes: int16 (uint16 storage) or int32 (uint32 storage) CUDA tensor."""
    lib = _lib.load()
    desc = grid.descriptor
    g = _lib.geom(desc.dims, grid.block_edge)
    p = _lib.params(eb, radius, padding.kind_code, padding.gran_code)
    dev = codes.device
    short = padding_shortfall(padding, grid, 0 if scalars is None else scalars.numel())
    if short is not None:
        # a padding section shorter than the policy needs (crafted container):
        # the kernels never read past the caller's scalars, and the verdict is
        # the reference's IndexError unless an earlier block fails first
        need = padding.scalar_count(grid)
        full = torch.zeros(need, dtype=torch.int64, device=dev)
        if scalars is not None and scalars.numel():
            full[: scalars.numel()] = scalars.reshape(-1)
        scalars = full
    if out is None:
        out = torch.empty(desc.dims, dtype=torch.float32, device=dev)
    if result is None:
        result = torch.empty(8, dtype=torch.int64, device=dev)
    wsb = lib.vlz_workspace_size(ctypes.byref(g))
    ws = workspace if workspace is not None else Workspace.get(wsb, dev)
    fn = lib.vlz_dq_decompress if codes.element_size() == 2 else lib.vlz_dq_decompress_u32
    rc = fn(_ptr(codes), _ptr(outliers) if n_outliers else None, int(n_outliers), _ptr(counts),
            _ptr(scalars) if scalars is not None and scalars.numel() else None, ctypes.byref(g),
            ctypes.byref(p), _ptr(out), _ptr(result), _ptr(ws), ws.numel(), _stream(stream))
    if rc != 0:
        raise RuntimeError(f"vlz_dq_decompress failed ({rc})")
    if check or short is not None:
        check_decompress(result, codes, counts, n_outliers, grid, radius, short)
    return out


def padding_shortfall(padding: PaddingPolicy, grid: BlockGrid, n_scalars: int):
    """(first block, scalar index) at which the reference's halo lookup
    (padding.py:113-129, apply_padding, run block by block in
    reconstruct.py:104-124) indexes past a padding section of `n_scalars`
    values, or None when the section is long enough."""
    need = padding.scalar_count(grid)
    if n_scalars >= need:
        return None
    if padding.granularity is PaddingGranularity.GLOBAL:
        return 0, n_scalars
    if padding.granularity is PaddingGranularity.BLOCK:
        return n_scalars, n_scalars
    return n_scalars // grid.descriptor.ndims, n_scalars  # edge: values[b*nd + d]


def check_decompress(result: torch.Tensor, codes, counts, n_outliers, grid, radius, short=None):
    r = _lib.Result()
    buf = result.cpu().numpy()
    ctypes.memmove(ctypes.byref(r), buf.ctypes.data, 64)
    if r.status == _lib.ST_SENTINEL_TOTAL:  # checked before the block loop
        raise CorruptStreamError(f"{r.n_outliers} sentinel codes but {n_outliers} outliers")
    if short is not None and (r.status == _lib.ST_OK or int(r.index) >= short[0]):
        n = short[1]  # numpy's message for values[n] on a length-n array
        raise IndexError(f"index {n} is out of bounds for axis 0 with size {n}")
    if r.status == _lib.ST_OK:
        return
    bi = int(r.index)
    start, size = block_span(grid, bi)
    blk = codes[start:start + size].cpu().numpy()
    blk = blk.view(np.uint16) if blk.dtype == np.int16 else blk.view(np.uint32)
    if r.status == _lib.ST_CORRUPT_CODE:
        raise CorruptStreamError(f"code {int(blk.max())} out of range for radius {radius}")
    if r.status == _lib.ST_EXHAUSTED:
        raise CorruptStreamError("outlier list exhausted before sentinels")
    if r.status == _lib.ST_LEFTOVER:
        cnt = counts.cpu().numpy()
        off = int(cnt[:bi].sum())
        avail = max(0, min(int(cnt[bi]), int(n_outliers) - off))
        raise CorruptStreamError(
            f"block consumed {int((blk == 0).sum())} outliers but {avail} were stored"
        )
    raise RuntimeError(f"unexpected decompress status {r.status}")


def histogram_device(codes: torch.Tensor, radius: int = 512, stream=None) -> np.ndarray:
    """uint64[65536] frequencies of a uint16 (int16 storage) CUDA code tensor."""
    lib = _lib.load()
    freqs = torch.empty(65536, dtype=torch.int64, device=codes.device)
    c = codes.contiguous()
    rc = lib.vlz_histogram(_ptr(c), c.numel(), int(radius), _ptr(freqs), _stream(stream))
    if rc != 0:
        raise RuntimeError(f"vlz_histogram failed ({rc})")
    return freqs.cpu().numpy().view(np.uint64)


def huffman_encode_device(codes: torch.Tensor, symbols: np.ndarray, lengths: np.ndarray,
                          nbits_hint: int | None = None, stream=None,
                          keep_on_device: bool = False):
    """MSB-first canonical Huffman packing of a uint16 (int16 storage) CUDA
    code tensor on the GPU (csrc/k_huffenc.cu); returns (payload bytes,
    bit_length) exactly as huffman.encode.  `nbits_hint` (sum of frequency x
    length, known once the book is built) sizes the output exactly."""
    from .errors import CorruptStreamError

    lib = _lib.load()
    c = codes.contiguous()
    n = c.numel()
    if n == 0:
        return b"", 0
    syms = np.ascontiguousarray(symbols, dtype=np.uint16)
    lens = np.ascontiguousarray(lengths, dtype=np.uint8)
    maxlen = int(lens.max())
    if maxlen > 58:
        raise ValueError("codeword longer than 58 bits")
    dev = c.device
    st = _stream(stream)
    tab = torch.empty(int(lib.vlz_huff_table_bytes()), dtype=torch.uint8, device=dev)
    rc = lib.vlz_huff_table(syms.ctypes.data, lens.ctypes.data, len(syms), _ptr(tab), st)
    if rc != 0:
        raise RuntimeError(f"vlz_huff_table failed ({rc})")
    bits_cap = int(nbits_hint) if nbits_hint is not None else n * maxlen
    cap = (bits_cap + 31) // 32 * 4 + 4
    out = torch.empty(cap, dtype=torch.uint8, device=dev)
    ws = torch.empty(int(lib.vlz_huff_encode_ws_size(n)), dtype=torch.uint8, device=dev)
    info = torch.empty(4, dtype=torch.int64, device=dev)
    rc = lib.vlz_huff_encode_device(_ptr(c), n, _ptr(tab), int(syms.max()) + 1, maxlen,
                                    _ptr(out), cap,
                                    _ptr(info), _ptr(ws), ws.numel(), st)
    if rc != 0:
        raise RuntimeError(f"vlz_huff_encode_device failed ({rc})")
    inf = info.cpu().tolist()
    none = (1 << 63) - 1
    bad = inf[1] if inf[1] != none else inf[3]
    if bad != none:
        raise CorruptStreamError(f"symbol {bad & 0xFFFF} not in the codebook")
    if inf[2]:
        raise RuntimeError("vlz_huff_encode_device: output capacity too small")
    nb = int(inf[0])
    if keep_on_device:  # (CUDA uint8 tensor, bits): serialize_parts copies it once
        return out, nb
    return out[: (nb + 7) // 8].cpu().numpy().tobytes(), nb


def border_outliers_device(codes: torch.Tensor, grid, stream=None) -> int:
    """Outliers whose block-local coordinates include a 0 (vector.py:82-87),
    counted on the device over a canonical uint16 (int16 storage) stream."""
    lib = _lib.load()
    c = codes.contiguous()
    g = _lib.geom(grid.descriptor.dims, grid.block_edge)
    total = torch.empty(1, dtype=torch.int64, device=c.device)
    rc = lib.vlz_border_outliers(_ptr(c), ctypes.byref(g), _ptr(total), _stream(stream))
    if rc != 0:
        raise RuntimeError(f"vlz_border_outliers failed ({rc})")
    return int(total.item())


def crc32_device(data: torch.Tensor, nbytes: int | None = None, stream=None) -> int:
    """zlib.crc32 of the first `nbytes` bytes of a CUDA tensor (any dtype),
    computed on the device (csrc/k_crc.cu)."""
    return int(crc32_device_async(data, nbytes, stream).item()) & 0xFFFFFFFF


def crc32_device_async(data: torch.Tensor, nbytes: int | None = None, stream=None):
    """crc32_device without the host synchronisation: returns the int32[1]
    CUDA tensor the CRC lands in (stream-ordered)."""
    lib = _lib.load()
    flat = data.reshape(-1).view(torch.uint8)
    n = flat.numel() if nbytes is None else int(nbytes)
    if n > flat.numel():
        raise ValueError("crc32_device: range past the tensor")
    ws = torch.empty(int(lib.vlz_crc32_ws_size(n)), dtype=torch.uint8, device=flat.device)
    out = torch.empty(1, dtype=torch.int32, device=flat.device)
    rc = lib.vlz_crc32_device(_ptr(flat) if n else None, n, _ptr(out), _ptr(ws), ws.numel(),
                              _stream(stream))
    if rc != 0:
        raise RuntimeError(f"vlz_crc32_device failed ({rc})")
    return out


def launch_count() -> int:
    return int(_lib.load().vlz_launch_count())
