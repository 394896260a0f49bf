"""Bit-exact parity at the benchmark configuration (BASELINE.json config 5).

C5 = 2048x2048x1024 float32 (2^32 elements, 16 GiB), Lorenzo-3D b=8, eb =
1e-4 * value range, R=512, mean:global.  It is the only case where element
offsets exceed 2^31, the grid has 8.4 M blocks and the mean:global sum runs
over 4.3e9 prequantized values.  The whole field is compressed and
decompressed on one B200 through the C ABI; then

* the value range (relative bound) and the mean:global statistics are checked
  against the pinned CPU oracle summed slab by slab on the host (reference
  padding.py:53-110, wrapping int64 sum like np.sum);
* codes, outlier values, per-block counts and decompressed bytes of the
  first, middle and last 8-plane block layers plus two seeded random ones are
  compared with oracle.dualquant(slab, global_scalar=s0) at their
  closed-form stream offsets (reference vector.py:205-260: blocks are
  independent, so a block-aligned slab with the full-field scalar is exactly
  that slice of the full stream);
* every reconstructed value is within eb of the input (whole field, on the
  device).
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2201_04614_b200 import gpu, workloads  # noqa: E402
from paper_2201_04614_b200 import model as M  # noqa: E402

SHAPE = (2048, 2048, 1024)
B, R = 8, 512
SLAB = 64  # planes per host round trip of the statistics pass


def _wrap64(v: int) -> int:
    return ((v + (1 << 63)) % (1 << 64)) - (1 << 63)


def test_c5_full_field_bit_exact(oracle):
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    free, _ = torch.cuda.mem_get_info(dev)
    if free < 90 << 30:
        pytest.skip(f"C5 needs ~80 GB of device memory, {free >> 30} GB free")
    x = workloads.gen_c5_slab((0, SHAPE[0]), dev, shape=SHAPE)
    assert x.numel() == 1 << 32
    cfg = M.CompressionConfig(M.ErrorBound.relative(1e-4), block_edge=B, radius=R,
                              padding=M.PaddingPolicy.parse("mean:global"))
    lo, hi = gpu.value_range(x)

    # host passes (64 planes = 1 GiB at a time): value range, then the
    # mean:global statistics, from the oracle
    h_lo, h_hi = np.inf, -np.inf
    for z0 in range(0, SHAPE[0], SLAB):
        a, b = oracle.minmax(x[z0:z0 + SLAB].cpu().numpy())
        h_lo, h_hi = min(h_lo, a), max(h_hi, b)
    assert (lo, hi) == (h_lo, h_hi)
    eb = M.resolve_error_bound_from_range(cfg.error_bound, lo, hi)
    tot = cnt = 0
    mn, mx = None, None
    for z0 in range(0, SHAPE[0], SLAB):
        st = oracle.global_stats(x[z0:z0 + SLAB].cpu().numpy(), eb)
        tot += int(st[0])
        cnt += int(st[1])
        mn = int(st[2]) if mn is None else min(mn, int(st[2]))
        mx = int(st[3]) if mx is None else max(mx, int(st[3]))
    assert cnt == 1 << 32
    s0 = oracle.stat_value("mean", _wrap64(tot), cnt, mn, mx)

    ds = gpu.compress_device(x, cfg, eb=eb).check()
    grid = ds.grid
    assert grid.block_count == 256 * 256 * 128
    assert int(ds.scalars[0].item()) == s0
    n_out = ds.n_outliers
    counts = ds.counts[: grid.block_count]
    assert int(counts.sum().item()) == n_out
    per_layer = grid.blocks_per_dim[1] * grid.blocks_per_dim[2]
    plane = SHAPE[1] * SHAPE[2]
    y = gpu.decompress_device(ds.codes, ds.outliers, n_out, ds.counts, ds.scalars, grid, eb, R,
                              cfg.padding)

    rng = np.random.default_rng(2026)
    layers = [0, SHAPE[0] // B // 2, SHAPE[0] // B - 1] + [int(v) for v in
                                                           rng.integers(1, SHAPE[0] // B - 1, 2)]
    starts = torch.cumsum(counts, 0) - counts  # exclusive outlier offsets per block
    for L in layers:
        z0 = L * B
        slab = x[z0:z0 + B].cpu().numpy()
        o = oracle.dualquant(slab, eb, B, R, "mean:global", global_scalar=s0)
        c0, c1 = z0 * plane, (z0 + B) * plane
        codes = ds.codes[c0:c1].cpu().numpy().view(np.uint16)
        assert np.array_equal(codes.astype(np.uint32), o["codes"]), f"codes, layer {L}"
        b0 = L * per_layer
        assert np.array_equal(counts[b0:b0 + per_layer].cpu().numpy(), o["outlier_counts"]), L
        k0 = int(starts[b0].item())
        k = o["outlier_values"].size
        got = ds.outliers[k0:k0 + k].cpu().numpy()
        assert got.tobytes() == o["outlier_values"].tobytes(), f"outliers, layer {L}"
        assert np.array_equal(o["scalars"], np.array([s0], np.int64))
        back = oracle.reconstruct(o["codes"], o["outlier_values"], o["outlier_counts"],
                                  o["scalars"], slab.shape, B, eb, R, "mean:global")
        assert y[z0:z0 + B].cpu().numpy().tobytes() == back.tobytes(), f"decompress, layer {L}"
        # the last layer holds element offsets up to 2^32 - 1
        if L == SHAPE[0] // B - 1:
            assert c1 == 1 << 32

    # error bound over the whole field, on the device, 64 planes at a time
    worst = 0.0
    for z0 in range(0, SHAPE[0], SLAB):
        d = (y[z0:z0 + SLAB].double() - x[z0:z0 + SLAB].double()).abs().max().item()
        worst = max(worst, d)
    assert worst <= eb
