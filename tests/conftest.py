"""Shared test fixtures.

Markers: `gpu` tests need a B200 (run on the GPU box with `-m gpu`); every
other test runs on the CPU build container.  The golden fixtures under
tests/golden/ were produced by the reference implementation itself
(tests/golden/make_golden.py) and are the parity pin for the CPU oracle
(oracle/), which in turn is the checker for the CUDA path at sizes where
storing reference outputs is impractical.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
for p in (REPO, os.path.join(REPO, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def load_cases(name: str):
    """Load a golden npz written by make_golden.Store as a list of dicts."""
    z = np.load(os.path.join(GOLDEN, name))
    meta = json.loads(bytes(z["meta"]))
    cases = []
    for m in meta:
        c = dict(m)
        prefix = f"{m['id']}."
        for k in z.files:
            if k.startswith(prefix):
                c[k[len(prefix):]] = z[k]
        cases.append(c)
    return cases


def load_json(name: str):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def load_border():
    """border.npz: outlier_report rows from the reference (make_golden.make_border)."""
    z = np.load(os.path.join(GOLDEN, "border.npz"))
    cases = json.loads(bytes(z["meta"]))
    for c in cases:
        c["data"] = np.frombuffer(bytes.fromhex(c["data"]), dtype=np.float32).reshape(c["shape"])
    return cases


@pytest.fixture(scope="session")
def corpus_cases():
    return load_cases("corpus.npz")


@pytest.fixture(scope="session")
def corrupt_cases():
    return load_cases("corrupt.npz")


@pytest.fixture(scope="session")
def oracle():
    import oracle as _oracle  # oracle/oracle.py (test infrastructure)

    _oracle.lib()
    return _oracle
