"""Autotune host logic against the reference's own outputs
(tests/golden/autotune.json, made by tests/golden/make_golden_autotune.py
from /root/reference/pkg/src/vlz/autotune.py), plus the sampled-block
column the GPU tuner times (built with torch on CPU here; no launches)."""

from __future__ import annotations

import json
import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from paper_2201_04614_b200 import ConfigError
from paper_2201_04614_b200.autotune import (
    TuneReport,
    TuneSpace,
    apply_chosen,
    gather_block_column,
    narrowed_autotune,
    sample_blocks,
)
from paper_2201_04614_b200.model import (
    ArrayDescriptor,
    CompressionConfig,
    ErrorBound,
    build_block_grid,
)

G = json.load(open(os.path.join(GOLDEN, "autotune.json")))


def _t(x):
    return tuple(tuple(c) for c in x)


def test_space_build_matches_reference():
    for s in G["spaces"]:
        assert TuneSpace.build(s["edges"], s["lanes"]).configs == _t(s["configs"])


def test_space_rejects_bad_entries():
    with pytest.raises(ConfigError):
        TuneSpace(())
    with pytest.raises(ConfigError):
        TuneSpace(((12, 8),))
    with pytest.raises(ConfigError):
        TuneSpace(((8, 1),))


def test_sample_blocks_matches_reference():
    for s in G["samples"]:
        grid = build_block_grid(ArrayDescriptor(len(s["shape"]), tuple(s["shape"])), s["b"])
        assert sample_blocks(grid, s["fraction"], s["seed"]).tolist() == s["picks"]
    grid = build_block_grid(ArrayDescriptor(1, (100,)), 8)
    for bad in (0.0, -0.1, 1.5):
        with pytest.raises(ConfigError):
            sample_blocks(grid, bad, 1)


def test_narrowed_matches_reference():
    space = TuneSpace.build()
    for s in G["narrowed"]:
        got = narrowed_autotune([tuple(h) for h in s["history"]], space, s["k"])
        assert got.configs == _t(s["configs"])


def test_csv_rows_and_apply_chosen():
    r = G["csv"]["report"]
    rep = TuneReport(configs=_t(r["configs"]), mean_s=tuple(r["mean_s"]),
                     std_s=tuple(r["std_s"]), chosen=tuple(r["chosen"]),
                     sample_fraction=0.1, iterations=3, seed=1, tuning_seconds=0.5)
    assert rep.csv_rows() == G["csv"]["rows"]
    cfg = apply_chosen(CompressionConfig(ErrorBound.absolute(1e-3)), rep)
    assert (cfg.block_edge, cfg.lane_width) == (16, 4)


@pytest.mark.parametrize("shape,b", [((1000,), 64), ((33, 47), 16), ((20, 17, 9), 8), ((9, 40, 70), 8), ((70, 9, 33), 16)])
def test_gather_block_column(shape, b):
    rng = np.random.default_rng(5)
    x = torch.from_numpy(rng.standard_normal(shape).astype(np.float32))
    grid = build_block_grid(ArrayDescriptor.from_array(x), b)
    picks = sample_blocks(grid, 0.5, 2)
    col = gather_block_column(x, grid, picks)
    k, nd = len(picks), len(shape)
    c = k if nd == 1 else min(k, grid.blocks_per_dim[-1])
    r = -(-k // c)
    want = (k * b,) if nd == 1 else (r * b,) + (b,) * (nd - 2) + (c * b,)
    assert col.shape == want
    cgrid = build_block_grid(ArrayDescriptor.from_array(col), b)
    assert cgrid.block_count == (k if nd == 1 else r * c)
    for i in range(cgrid.block_count):
        bi = int(picks[i % k])
        ext = grid.block_extents(bi)
        src = x[tuple(slice(o, o + e) for o, e in zip(grid.block_origin(bi), ext))]
        blk = col[tuple(slice(o, o + b) for o in cgrid.block_origin(i))]
        assert torch.equal(blk[tuple(slice(0, e) for e in ext)], src)
        assert float(blk.abs().sum()) == pytest.approx(float(src.abs().sum()), rel=1e-5)


def test_iterations_checked_before_any_gpu_work():
    from paper_2201_04614_b200.autotune import autotune

    with pytest.raises(ConfigError):
        autotune(np.zeros((8, 8), np.float32), TuneSpace.build(), iterations=0)
