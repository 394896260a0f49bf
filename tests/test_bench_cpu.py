"""bench.py's multi-rank plumbing on CPU (no GPU): `--gpus N` without
torchrun's environment re-launches bench.py under torch.distributed.run with
N ranks; `--cpu-check` runs the GPU arm's orchestration (range all-reduce,
mean:global statistics all-gather, per-shard compress, piece hashes gathered
on rank 0) with gloo and the CPU oracle per shard.  The stream digest must be
the same at 1, 2 and 4 ranks and equal the single-process oracle stream's."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--cpu-check", *args],
                       capture_output=True, text=True, timeout=600, env=env, cwd=REPO)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0]), r.stderr


def test_spawned_ranks_give_the_single_process_stream(oracle):
    sys.path.insert(0, REPO)
    import bench
    from paper_2201_04614_b200 import workloads

    shape = (64, 48, 40)
    x = workloads.gen_c5_slab_numpy((0, shape[0]), shape=shape)
    eb = bench.REL_EB * (float(x.max()) - float(x.min()))
    o = oracle.dualquant(x, eb, 8, 512, "mean:global")
    per_layer = 6 * 5
    want = bench.combine_digest(
        [bench.piece_hashes(o["codes"].astype(np.uint16), o["outlier_counts"],
                            o["outlier_values"], 0, shape[0], shape[0], shape[1] * shape[2],
                            per_layer, 8)], o["scalars"])
    one, _ = _run("--gpus", "1")
    assert one["n_ranks"] == 1 and one["stream_digest"] == want
    for n in (2, 4):
        got, err = _run("--gpus", str(n))
        assert "spawning" in err and got["n_ranks"] == n
        assert got["eb"] == one["eb"] and got["stream_digest"] == want, n


def test_generator_slabs_tile_the_field():
    # any block-aligned z-slab of the C5 generator is the same slice of the
    # whole field (noise seeded per 8-plane group), so sharded runs compress
    # exactly the 1-GPU field
    from paper_2201_04614_b200 import workloads

    shape = (48, 20, 24)
    full = workloads.gen_c5_slab_numpy((0, 48), shape=shape)
    for z0, z1 in ((0, 16), (16, 40), (40, 48), (8, 24)):
        part = workloads.gen_c5_slab_numpy((z0, z1), shape=shape)
        assert part.tobytes() == full[z0:z1].tobytes(), (z0, z1)
