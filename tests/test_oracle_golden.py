"""Pin the CPU oracle (oracle/vlz_oracle.c) against vectors produced by the
reference implementation (tests/golden/make_golden.py).  No GPU needed.

An oracle that agrees with the reference on every golden case is then used
as the checker for the CUDA kernels at sizes where reference outputs are not
stored (tests/test_gpu_parity.py)."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import load_json


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_oracle_matches_reference_corpus(oracle, corpus_cases):
    assert len(corpus_cases) > 100
    for c in corpus_cases:
        got = oracle.dualquant(c["data"], c["eb"], c["block_edge"], c["radius"], c["padding"])
        tag = c["tag"]
        assert np.array_equal(got["codes"].astype(np.uint16), c["codes"]), tag
        assert got["codes"].max(initial=0) < 65536
        assert got["outlier_values"].tobytes() == c["outlier_values"].tobytes(), tag
        assert np.array_equal(got["outlier_counts"], c["outlier_counts"]), tag
        assert np.array_equal(got["scalars"], c["scalars"]), tag


def test_oracle_reconstruct_matches_reference_decompress(oracle, corpus_cases):
    checked = 0
    for c in corpus_cases:
        if "decompressed" not in c:
            continue
        out = oracle.reconstruct(
            c["codes"].astype(np.uint32), c["outlier_values"], c["outlier_counts"], c["scalars"],
            tuple(c["shape"]), c["block_edge"], c["eb"], c["radius"], c["padding"],
        )
        assert out.tobytes() == c["decompressed"].tobytes(), c["tag"]
        checked += 1
    assert checked > 50


def test_oracle_thread_count_determinism(oracle, corpus_cases):
    for c in corpus_cases[:40]:
        a = oracle.dualquant(c["data"], c["eb"], c["block_edge"], c["radius"], c["padding"], threads=1)
        b = oracle.dualquant(c["data"], c["eb"], c["block_edge"], c["radius"], c["padding"], threads=4)
        for k in a:
            assert a[k].tobytes() == b[k].tobytes()


def test_oracle_error_cases(oracle):
    for c in load_json("errors.json"):
        data = np.array(c["data"], dtype=np.float32).reshape(c["shape"])
        exp = c["expect"]
        if c["eb"] is None or c.get("lane", 8) == 1:
            continue  # relative-bound resolution and the lane-1 order are host logic
        if exp is None:
            oracle.dualquant(data, c["eb"], c["block_edge"], 32768, c["padding"])
            continue
        with pytest.raises(oracle.OracleError) as err:
            oracle.dualquant(data, c["eb"], c["block_edge"], 32768, c["padding"])
        status = {"ConfigError": oracle.NONFINITE, "BoundTooSmallError": oracle.OVERFLOW}[exp["type"]]
        assert err.value.status == status, c["tag"]
        idx = exp.get("index")
        if idx is None:
            idx = int(exp["message"].rsplit(" ", 1)[1])
        assert err.value.index == idx, c["tag"]


def test_oracle_corrupt_streams(oracle, corrupt_cases):
    kinds = {
        "code_range": oracle.CORRUPT_CODE,
        "sentinel_total": oracle.SENTINEL_TOTAL,
        "partition": oracle.EXHAUSTED,
        "partition_rev": oracle.LEFTOVER,
    }
    for c in corrupt_cases:
        with pytest.raises(oracle.OracleError) as err:
            oracle.reconstruct(c["codes"], c["outlier_values"], c["outlier_counts"], c["scalars"],
                               tuple(c["shape"]), c["block_edge"], c["eb"], c["radius"],
                               c["padding"])
        assert err.value.status == kinds[c["tag"]], c["tag"]


def test_oracle_prequant_known_answers(oracle):
    for c in load_json("known.json"):
        if c["kind"] == "prequant":
            d = oracle.prequantize(np.array([c["v"]], np.float32), c["eb"])
            assert int(d[0]) == c["d"], c
        else:
            d = oracle.prequantize(np.array(c["v"], np.float32), c["eb"])
            assert d.tolist() == c["d"]


def test_oracle_fullsize_reference_hashes(oracle):
    """C1 (1D, b=256 and 64) and C2 (1800x3600, zero and mean:block) at
    BASELINE.json's full size, against sha256 of the reference's streams."""
    from paper_2201_04614_b200 import workloads

    data = {"C1": workloads.gen_c1(), "C2": workloads.gen_c2()}
    for c in load_json("fullsize.json"):
        d = data[c["config"]]
        assert _sha(d) == c["data_sha"], "generator drifted"
        got = oracle.dualquant(d, c["eb"], c["block_edge"], c["radius"], c["padding"])
        assert _sha(got["codes"].astype(np.uint16)) == c["codes_u16_sha"]
        assert _sha(got["outlier_values"]) == c["outliers_sha"]
        assert _sha(got["outlier_counts"]) == c["counts_sha"]
        assert _sha(got["scalars"]) == c["scalars_sha"]


def test_oracle_border_census_matches_reference_outlier_report(oracle):
    # padding.py:162-205 / vector.py:82-87: total and border outliers per
    # policy, from the pinned oracle's stream through the host census
    from types import SimpleNamespace

    from conftest import load_border
    from paper_2201_04614_b200 import model as M
    from paper_2201_04614_b200.vector import border_outliers

    n = 0
    for c in load_border():
        grid = M.build_block_grid(M.ArrayDescriptor(len(c["shape"]), tuple(c["shape"])),
                                  c["block_edge"])
        for row in c["rows"]:
            pol = f"{row['kind']}:{row['gran']}" if row["kind"] != "zero" else "zero"
            o = oracle.dualquant(c["data"], c["eb"], c["block_edge"], c["radius"], pol)
            assert int(o["outlier_counts"].sum()) == row["total"], (c["tag"], pol)
            s = SimpleNamespace(grid=grid, codes=o["codes"])
            assert border_outliers(s) == row["border"], (c["tag"], pol)
            n += 1
    assert n >= 150
