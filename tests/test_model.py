"""Host-side data model: same validation rules and messages as the reference
(pkg/src/vlz/model.py:48-269, errors.py:8-62); reference-generated error
cases from tests/golden/errors.json for the checks that run on the host."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import load_json
from paper_2201_04614_b200 import model as M
from paper_2201_04614_b200.errors import (
    BoundTooSmallError,
    ConfigError,
    CorruptStreamError,
    DegenerateRangeError,
    VlzError,
)


def test_error_taxonomy():
    assert issubclass(ConfigError, VlzError)
    assert issubclass(CorruptStreamError, VlzError)
    e = BoundTooSmallError(1, 300000.0, 1e-05)
    assert (e.index, e.value, e.bound) == (1, 300000.0, 1e-05)
    exp = [c for c in load_json("errors.json") if c["tag"] == "overflow_index"][0]["expect"]
    assert str(e) == exp["message"]


def test_config_validation():
    eb = M.ErrorBound.absolute(1e-3)
    with pytest.raises(ConfigError, match="block edge must be one of"):
        M.CompressionConfig(eb, block_edge=12)
    with pytest.raises(ConfigError, match="lane width"):
        M.CompressionConfig(eb, lane_width=3)
    with pytest.raises(ConfigError, match="quantizer radius"):
        M.CompressionConfig(eb, radius=1)
    with pytest.raises(ConfigError, match="quantizer radius"):
        M.CompressionConfig(eb, radius=32769)
    with pytest.raises(ConfigError, match="thread count"):
        M.CompressionConfig(eb, thread_count=0)
    with pytest.raises(ConfigError, match="error bound value must be > 0"):
        M.ErrorBound.absolute(0.0)
    assert M.CompressionConfig(eb, block_edge=8, lane_width=16).effective_lanes == 8


def test_block_256_is_opt_in():
    eb = M.ErrorBound.absolute(1e-3)
    with pytest.raises(ConfigError):
        M.CompressionConfig(eb, block_edge=256)
    M.allow_block_256(True)
    try:
        assert M.CompressionConfig(eb, block_edge=256).block_edge == 256
    finally:
        M.allow_block_256(False)


def test_padding_policy_parse():
    p = M.PaddingPolicy.parse("min:edge")
    assert (p.kind_code, p.gran_code) == (1, 2)
    assert str(M.PaddingPolicy.parse("mean")) == "mean:global"
    for bad in ("foo", "mean:bar", "a:b:c"):
        with pytest.raises(ConfigError):
            M.PaddingPolicy.parse(bad)


def test_descriptor_and_grid():
    with pytest.raises(ConfigError, match="only float32"):
        M.ArrayDescriptor.from_array(np.zeros(4, np.float64))
    with pytest.raises(ConfigError, match="every extent"):
        M.ArrayDescriptor.from_array(np.zeros((0, 3), np.float32))
    with pytest.raises(ConfigError, match="ndims"):
        M.ArrayDescriptor.from_array(np.zeros((1, 1, 1, 1), np.float32))
    d = M.ArrayDescriptor.from_array(np.zeros((19, 21, 23), np.float32))
    g = M.build_block_grid(d, 8)
    assert g.blocks_per_dim == (3, 3, 3) and g.block_count == 27
    assert g.block_extents(26) == (3, 5, 7)
    assert g.block_origin(5) == (0, 8, 16)


def test_relative_bound_resolution():
    data = np.array([1.0, 3.0, 2.0], np.float32)
    assert M.resolve_error_bound(M.ErrorBound.relative(0.5), data) == 1.0
    with pytest.raises(DegenerateRangeError) as err:
        M.resolve_error_bound(M.ErrorBound.relative(1e-3), np.full(10, 3.0, np.float32))
    exp = [c for c in load_json("errors.json") if c["tag"] == "degenerate_rel"][0]["expect"]
    assert str(err.value) == exp["message"]


def test_codestream_same_bytes():
    d = M.ArrayDescriptor(1, (8,))
    g = M.build_block_grid(d, 8)
    s = M.PaddingScalars(M.PaddingPolicy(), np.array([3], np.int64))
    a = M.CodeStream(np.arange(8, dtype=np.uint32), np.zeros(0, np.float32),
                     np.zeros(1, np.int64), g, 1e-3, 512, s)
    b = M.CodeStream(np.arange(8, dtype=np.uint32), np.zeros(0, np.float32),
                     np.zeros(1, np.int64), g, 1e-3, 512, s)
    assert a.same_bytes(b)
    with pytest.raises(ConfigError):
        M.PaddingScalars(M.PaddingPolicy(), np.array([3], np.int32))


def test_nan_relative_bound_names_first_nonfinite():
    # a relative bound over NaN data resolves to NaN; the reference
    # lets it past `eb <= 0` and reports the first non-finite index
    from paper_2201_04614_b200.gpu import check_resolved_eb

    n = 0
    for c in load_json("errors.json"):
        if not c["tag"].startswith("rel_"):
            continue
        data = np.array(c["data"], dtype=np.float32)
        eb = M.resolve_error_bound(M.ErrorBound.relative(c["rel"]), data)
        if eb == float("inf"):  # passes; the kernel's non-finite scan reports (GPU tests)
            check_resolved_eb(eb, data)
            continue
        with pytest.raises(ConfigError) as err:
            check_resolved_eb(eb, data)
        assert str(err.value) == c["expect"]["message"], c["tag"]
        n += 1
    assert n == 1
    with pytest.raises(ConfigError, match="must be > 0"):
        check_resolved_eb(0.0, np.zeros(3, np.float32))
