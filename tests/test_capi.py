"""The C-ABI library: it loads without a GPU and exports exactly the entry
points include/vlz_gpu.h declares; host-side geometry helpers agree with the
data model.  No kernel is launched here (CPU container)."""

from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import REPO

HEADER = os.path.join(REPO, "include", "vlz_gpu.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(vlz_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2201_04614_b200 import _lib

    if not os.path.exists(_lib.LIB_PATH):
        pytest.fail("libvlzgpu.so not built (run __graft_entry__.build())")
    return _lib.load()


def test_library_exports_every_declared_symbol(lib):
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in include/vlz_gpu.h but not exported"


def test_python_prototypes_cover_the_header(lib):
    from paper_2201_04614_b200 import _lib

    assert set(declared_symbols()) == set(_lib.PROTOTYPES)


def test_struct_sizes_match_header(lib):
    from paper_2201_04614_b200 import _lib

    assert ctypes.sizeof(_lib.Geom) == 32
    assert ctypes.sizeof(_lib.Params) == 24
    assert ctypes.sizeof(_lib.Result) == 64


@pytest.mark.parametrize("shape,b", [((1000,), 8), ((1_048_576,), 256), ((45, 37), 16),
                                     ((19, 21, 23), 8), ((100, 500, 500), 8), ((64, 64, 64), 64)])
def test_block_and_scalar_counts_match_model(lib, shape, b):
    from paper_2201_04614_b200 import _lib
    from paper_2201_04614_b200 import model as M

    M.allow_block_256(True)
    try:
        grid = M.build_block_grid(M.ArrayDescriptor(len(shape), shape), b)
        g = _lib.geom(shape, b)
        assert lib.vlz_block_count(ctypes.byref(g)) == grid.block_count
        for pol in ("zero", "mean:global", "min:block", "max:edge"):
            p = M.PaddingPolicy.parse(pol)
            assert lib.vlz_scalar_count(ctypes.byref(g), p.kind_code, p.gran_code) == \
                p.scalar_count(grid)
        # the outlier scratch is 8 float32 slots per block (dense blocks are
        # regenerated from the codes), not one per element
        ws = lib.vlz_workspace_size(ctypes.byref(g))
        assert ws >= 32 * grid.block_count
        assert ws < 64 * grid.block_count + 8 * grid.descriptor.element_count // 32 + (2 << 20)
    finally:
        M.allow_block_256(False)


def test_invalid_geometry_rejected(lib):
    from paper_2201_04614_b200 import _lib

    assert lib.vlz_block_count(ctypes.byref(_lib.geom((10, 10), 256))) == -1  # 256 is 1-D only
    assert lib.vlz_block_count(ctypes.byref(_lib.geom((10,), 12))) == -1
    assert lib.vlz_block_count(ctypes.byref(_lib.geom((0, 4), 8))) == -1
    assert lib.vlz_workspace_size(ctypes.byref(_lib.geom((4,), 7))) == 0


def test_device_entry_points_reject_bad_arguments_before_launch(lib):
    """Argument validation happens on the host: null pointers / bad params
    return VLZ_E_ARG without touching CUDA (works on a CPU-only box)."""
    from paper_2201_04614_b200 import _lib

    g = _lib.geom((64,), 8)
    p = _lib.params(1e-3, 1, 0, 0)  # radius 1 is invalid
    rc = lib.vlz_dq_compress(None, ctypes.byref(g), ctypes.byref(p), None, None, None, None,
                             None, None, 0, None)
    assert rc == 1
    p = _lib.params(1e-3, 512, 0, 0)
    rc = lib.vlz_dq_decompress(None, None, 0, None, None, ctypes.byref(g), ctypes.byref(p), None,
                               None, None, 0, None)
    assert rc == 1


def test_geometry_block_span_matches_canonical_order():
    """gpu.block_span (closed form used by error reporting) equals the
    reference's cumulative block sizes (reconstruct.py:93-100)."""
    from paper_2201_04614_b200 import model as M

    pytest.importorskip("torch")
    from paper_2201_04614_b200.gpu import block_span

    for shape, b in (((45, 37), 16), ((19, 21, 23), 8), ((77,), 8), ((9, 10, 11), 8)):
        grid = M.build_block_grid(M.ArrayDescriptor(len(shape), shape), b)
        sizes = [int(np.prod(grid.block_extents(i))) for i in range(grid.block_count)]
        starts = np.concatenate([[0], np.cumsum(sizes)[:-1]])
        for i in range(grid.block_count):
            assert block_span(grid, i) == (int(starts[i]), sizes[i])
