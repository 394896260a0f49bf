"""bench.py's N-rank GPU arm on a one-GPU box: `--gpus 2` re-launches the
bench as two ranks (torch.distributed.run), both placed on cuda:0 with gloo
collectives (VLZ_BENCH_ONE_DEVICE=1; the ranks' kernels never wait on one
another, only the timing is meaningless).  The two-rank stream -- slab-
sharded compress with the statistics all-gathered and reduced in the finish
kernel, per-rank outlier offsets, the piece hashes gathered on rank 0 -- must
have the digest of the one-rank stream of the same field."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(gpus: int, planes: int):
    env = dict(os.environ, VLZ_BENCH_ONE_DEVICE="1")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", str(gpus),
                        "--planes", str(planes), "--steps", "2", "--warmup", "1", "--no-e2e",
                        "--no-cpu-baseline"], capture_output=True, text=True, timeout=900,
                       env=env, cwd=REPO)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_two_ranks_give_the_one_rank_stream():
    one = _bench(1, 256)
    two = _bench(2, 256)
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert one["stream_digest"] and two["stream_digest"] == one["stream_digest"]
    assert two["n_outliers"] == one["n_outliers"]
    assert two["config"]["eb"] == one["config"]["eb"]
