"""Exhaustive sweep of the float32 exact-fast prequantizer.

For each bound below, all 2^32 float32 bit patterns go through both forms of
quant_fast the compress kernels use (scalar, and the paired-FP32 form of
dq_compress_fast.cuh) and, where the fast path accepts a pattern, through the
exact float64 quant_exact (the reference's quantize.py:31-42,66-78 and the
narrowing check vector.py:72-77).  Zero accepted-but-wrong patterns and zero
form disagreements are required.  The per-bound fallback rate (finite
patterns sent to the exact path) is written to gpurun_out/prequant_sweep.json
when that directory exists (committed copy: profiles/r02/)."""

from __future__ import annotations

import json
import os

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2201_04614_b200 import _lib  # noqa: E402

EBS = {
    "C5 1e-4*range": 0.00042740070819854737,
    "C1 1e-4*range": 0.0014935896039009096,
    "C2 1e-4*range": 0.0004225547552108765,
    "C3 1e-3*range": 0.002361815094947815,
    "C4 1e-3*range": 0.2068639584570192,
    "stress 1e-5*range": 0.0017146239634929226,
    "0.5 (2eb = 1)": 0.5,
    "2^-10": 2.0 ** -10,
    "0.1": 0.1,
    "1/3": 1.0 / 3.0,
    "1e-30": 1e-30,
    "3.7e+20": 3.7e20,
    "inv32 just below 2^100": 2.0 ** -101 * (1 + 2.0 ** -20),
    "inv32 just above 2^-100": 2.0 ** 99 * (1 - 2.0 ** -20),
}


def test_prequant_fast_path_exhaustive():
    lib = _lib.load()
    cnt = torch.zeros(6, dtype=torch.int64, device="cuda")
    rows = {}
    for name, eb in EBS.items():
        assert lib.vlz_test_fast_enabled(eb) == 1, name
        rc = lib.vlz_test_prequant_sweep(eb, cnt.data_ptr(),
                                         torch.cuda.current_stream().cuda_stream)
        assert rc == 0
        acc, fb, nf, bad, form, first = [int(v) for v in cnt.cpu().tolist()]
        first &= (1 << 64) - 1
        assert acc + fb + nf == 1 << 32, name
        assert nf == 2 * ((1 << 23) - 1) + 2  # NaNs and the two infinities
        assert bad == 0, f"{name}: {bad} accepted patterns disagree (first 0x{first:08x})"
        assert form == 0, f"{name}: scalar and paired forms disagree (first 0x{first:08x})"
        rows[name] = {"eb": eb, "accepted": acc, "exact_path": fb,
                      "exact_path_frac_of_finite": fb / (acc + fb)}
    # outside the enable window the fast path is off (every element exact)
    assert lib.vlz_test_fast_enabled(2.0 ** -102) == 0
    assert lib.vlz_test_fast_enabled(2.0 ** 100) == 0
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
    if os.path.isdir(out):
        with open(os.path.join(out, "prequant_sweep.json"), "w") as fh:
            json.dump(rows, fh, indent=1)
