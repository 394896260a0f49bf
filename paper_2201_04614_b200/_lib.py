"""ctypes binding of libvlzgpu.so (include/vlz_gpu.h).

The library is built in-tree by __graft_entry__.build() / `make -C
paper_2201_04614_b200/csrc`.  There is deliberately no fallback: if the
shared object is missing or cannot be loaded the import fails loudly.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VLZ_LIB") or os.path.join(_HERE, "libvlzgpu.so")  # VLZ_LIB: A/B runs of two builds


class Geom(ctypes.Structure):
    _fields_ = [("nd", ctypes.c_int32), ("block_edge", ctypes.c_int32),
                ("dims", ctypes.c_int64 * 3)]


class Params(ctypes.Structure):
    _fields_ = [("eb", ctypes.c_double), ("radius", ctypes.c_int32),
                ("pad_kind", ctypes.c_int32), ("pad_gran", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class Result(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("index", ctypes.c_int64), ("n_outliers", ctypes.c_int64),
                ("first_nonfinite", ctypes.c_int64), ("first_overflow", ctypes.c_int64),
                ("first_bad_block", ctypes.c_int64), ("sentinels", ctypes.c_int64),
                ("pad0", ctypes.c_int64)]


assert ctypes.sizeof(Result) == 64

# status codes (VLZ_ST_*)
ST_OK, ST_NONFINITE, ST_OVERFLOW = 0, 1, 2
ST_CORRUPT_CODE, ST_EXHAUSTED, ST_LEFTOVER, ST_SENTINEL_TOTAL = 4, 5, 6, 7
ST_OUTLIER_CAPACITY = 8

# exported symbols and their prototypes (must match include/vlz_gpu.h)
_P = ctypes.POINTER
_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
PROTOTYPES = {
    "vlz_block_count": (_i64, [_P(Geom)]),
    "vlz_scalar_count": (_i64, [_P(Geom), ctypes.c_int32, ctypes.c_int32]),
    "vlz_workspace_size": (ctypes.c_size_t, [_P(Geom)]),
    "vlz_workspace_size_dense": (ctypes.c_size_t, [_P(Geom)]),
    "vlz_dq_compress": (ctypes.c_int, [_vp, _P(Geom), _P(Params), _vp, _vp, _vp, _vp, _vp, _vp,
                                       ctypes.c_size_t, _vp]),
    "vlz_dq_compress_capped": (ctypes.c_int, [_vp, _P(Geom), _P(Params), _vp, _vp, _i64, _vp, _vp,
                                              _vp, _vp, ctypes.c_size_t, _vp]),
    "vlz_dq_compress_begin": (ctypes.c_int, [_vp, _P(Geom), _P(Params), _vp, _vp, _vp, _vp, _vp,
                                             _vp, ctypes.c_size_t, _vp]),
    "vlz_dq_compress_finish": (ctypes.c_int, [_vp, _P(Geom), _P(Params), _vp, _vp, _vp, _vp, _vp,
                                              _vp, _vp, ctypes.c_size_t, _vp]),
    "vlz_dq_compress_finish_gathered": (ctypes.c_int, [_vp, _P(Geom), _P(Params), _vp,
                                                       ctypes.c_int32, _vp, _vp, _vp, _vp, _vp,
                                                       _vp, ctypes.c_size_t, _vp]),
    "vlz_dq_decompress": (ctypes.c_int, [_vp, _vp, _i64, _vp, _vp, _P(Geom), _P(Params), _vp, _vp,
                                         _vp, ctypes.c_size_t, _vp]),
    "vlz_dq_decompress_u32": (ctypes.c_int, [_vp, _vp, _i64, _vp, _vp, _P(Geom), _P(Params), _vp,
                                             _vp, _vp, ctypes.c_size_t, _vp]),
    "vlz_dq_decompress_dn": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _P(Geom), _P(Params), _vp,
                                            _vp, _vp, ctypes.c_size_t, _vp]),
    "vlz_minmax": (ctypes.c_int, [_vp, _i64, _vp, _vp]),
    "vlz_dq_compress_host": (ctypes.c_int, [_vp, _P(Geom), _P(Params), _vp, _vp, _vp, _vp,
                                            _P(Result), ctypes.c_int]),
    "vlz_dq_decompress_host": (ctypes.c_int, [_vp, _vp, _i64, _vp, _vp, _P(Geom), _P(Params), _vp,
                                              _P(Result), ctypes.c_int]),
    "vlz_host_release": (None, []),
    "vlz_histogram": (ctypes.c_int, [_vp, _i64, ctypes.c_int32, _vp, _vp]),
    "vlz_histogram_host": (None, [_vp, _i64, _vp]),
    "vlz_huff_build": (ctypes.c_int, [_vp, _vp, _vp, _P(ctypes.c_int32)]),
    "vlz_huff_encode": (ctypes.c_int, [_vp, _i64, _vp, _vp, ctypes.c_int32, _vp, _i64, _P(_i64),
                                       _P(_i64)]),
    "vlz_border_outliers": (ctypes.c_int, [_vp, _P(Geom), _vp, _vp]),
    "vlz_huff_table_bytes": (ctypes.c_size_t, []),
    "vlz_huff_table": (ctypes.c_int, [_vp, _vp, ctypes.c_int32, _vp, _vp]),
    "vlz_huff_encode_ws_size": (ctypes.c_size_t, [_i64]),
    "vlz_huff_encode_device": (ctypes.c_int, [_vp, _i64, _vp, ctypes.c_int32, ctypes.c_int32,
                                              _vp, _i64, _vp, _vp,
                                              ctypes.c_size_t, _vp]),
    "vlz_huff_decode_ws_size": (ctypes.c_size_t, [_i64]),
    "vlz_huff_decode_device": (ctypes.c_int, [_vp, _i64, _i64, _vp, _vp, ctypes.c_int32, _i64,
                                              _vp, _P(_i64), _vp, ctypes.c_size_t, _vp]),
    "vlz_huff_decode": (ctypes.c_int, [_vp, _i64, _i64, _vp, _vp, ctypes.c_int32, _i64, _vp,
                                       _P(_i64)]),
    "vlz_padding_census_ws_size": (ctypes.c_size_t, [_P(Geom)]),
    "vlz_padding_census": (ctypes.c_int, [_vp, _P(Geom), ctypes.c_double, ctypes.c_int32, _vp,
                                          _vp, ctypes.c_size_t, _vp]),
    "vlz_crc32_ws_size": (ctypes.c_size_t, [_i64]),
    "vlz_crc32_device": (ctypes.c_int, [_vp, _i64, _vp, _vp, ctypes.c_size_t, _vp]),
    "vlz_launch_count": (_i64, []),
    "vlz_timing": (None, [ctypes.c_int]),
    "vlz_timing_collect": (ctypes.c_int, [_P(ctypes.c_double), _P(_i64), ctypes.c_int]),
    "vlz_version": (ctypes.c_char_p, []),
    "vlz_test_prequant_sweep": (ctypes.c_int, [ctypes.c_double, _vp, _vp]),
    "vlz_test_fast_enabled": (ctypes.c_int, [ctypes.c_double]),
    "vlz_bench_stream": (ctypes.c_int, [ctypes.c_int32, _vp, _vp, _i64, ctypes.c_int32, _vp]),
}

_lib = None


def load():
    """Load libvlzgpu.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the CUDA extension first "
                "(python -c 'import __graft_entry__ as g; g.build()')"
            )
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in PROTOTYPES.items():
            if os.environ.get("VLZ_LIB") and not hasattr(lib, name) and \
                    name.startswith(("vlz_test_", "vlz_bench_", "vlz_workspace_size_dense",
                                     "vlz_dq_compress_capped")):
                continue  # an older build under A/B comparison (tools/ab_lib.sh)
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def geom(shape, block_edge) -> Geom:
    g = Geom()
    g.nd = len(shape)
    g.block_edge = int(block_edge)
    for i in range(3):
        g.dims[i] = int(shape[i]) if i < len(shape) else 1
    return g


def params(eb, radius, kind_code, gran_code) -> Params:
    p = Params()
    p.eb = float(eb)
    p.radius = int(radius)
    p.pad_kind = int(kind_code)
    p.pad_gran = int(gran_code)
    p.reserved = 0
    return p
