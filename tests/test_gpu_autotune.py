"""GPU autotune: the tuner times real fused-compress launches over the
sampled block column; a scripted timer (the reference's test device,
/root/reference/pkg/tests/test_autotune.py:23-46) checks the argmin and tie
rules through the real launch sequence."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2201_04614_b200 import gpu  # noqa: E402
from paper_2201_04614_b200.autotune import TuneSpace, apply_chosen, autotune  # noqa: E402
from paper_2201_04614_b200.model import CompressionConfig, ErrorBound  # noqa: E402


class Script:
    """One timestamp per timer() call: start, (t0, t1) per launch, end."""

    def __init__(self, costs):
        self.stamps, now = [0.0], 0.0
        for c in costs:
            self.stamps += [now, now + c]
            now += c
        self.stamps.append(now)
        self.calls = 0

    def __call__(self):
        self.calls += 1
        return self.stamps[self.calls - 1]


@pytest.mark.parametrize("winner", [8, 16, 32, 64])
def test_scripted_argmin(winner):
    data = np.random.default_rng(3).uniform(-10, 10, (70, 65, 66)).astype(np.float32)
    space = TuneSpace.build()
    edges = sorted({b for b, _ in space.configs})
    iters = 2
    costs = [(0.5 if b == winner else 10.0 + b) for _ in range(iters) for b in edges]
    before = gpu.launch_count()
    timer = Script(costs)
    rep = autotune(data, space, 0.2, iters, seed=4, timer=timer,
                   base=CompressionConfig(ErrorBound.absolute(1e-3)))
    assert timer.calls == len(timer.stamps)
    assert gpu.launch_count() > before
    lanes = max(l for b, l in space.configs if b == winner)
    assert rep.chosen == (winner, lanes)  # ties inside one edge -> largest lane
    assert rep.mean_s[space.configs.index(rep.chosen)] == pytest.approx(0.5)


def test_event_timed_tuner_runs_and_applies():
    data = np.random.default_rng(8).standard_normal((128, 96, 80)).astype(np.float32)
    space = TuneSpace.build((8, 16, 32))
    rep = autotune(data, space, fraction=0.25, iterations=3,
                   base=CompressionConfig(ErrorBound.relative(1e-4)))
    assert rep.chosen in space.configs
    assert all(m > 0 for m in rep.mean_s) and rep.tuning_seconds > 0
    cfg = apply_chosen(CompressionConfig(ErrorBound.relative(1e-4)), rep)
    x = torch.from_numpy(data).cuda()
    dev = gpu.compress_device(x, cfg).check()
    y = gpu.decompress_device(dev.codes, dev.outliers, dev.n_outliers, dev.counts,
                              dev.scalars, dev.grid, dev.eb, cfg.radius, cfg.padding)
    assert float((y - x).abs().max()) <= dev.eb
