"""Seeded synthetic stand-ins for the BASELINE.json configurations.

The paper measures on SDRBench fields (CESM 1800x3600, Hurricane 100x500x500,
NYX 512^3) which are not available offline.  These
generators reproduce the shapes, sizes and value character that BASELINE.json
names (see SURVEY.md section 8d for the exact recipes):

  C1  1D  N=1,048,576   x = cumsum(N(0,1))*0.01 + sin(2*pi*i/4096)
  C2  2D  1800x3600     64 sinusoidal modes, k in [1,16]^2, amp 1/|k|, + N(0,1e-3)
  C3  3D  100x500x500   128 modes, k in [1,12]^3, amp |k|^-1.5, + N(0,1e-3)
  C4  3D  512^3         exp(g), g a Gaussian random field with P(k) ~ k^-3
  C5  3D  2048x2048x1024 64 modes as C2 (k in [1,16]^3, amp 1/|k|), built on device

Coordinates are normalised to [0,1) per axis; generation is float64 and the
result is cast to float32.  Seed = config index.  C1-C4 are numpy (bit-stable
for the golden hashes); C5 and the bench's large fields are generated on the
GPU with torch (`*_torch` variants), slab by slab.
"""

from __future__ import annotations

import math

import numpy as np

CONFIGS = {
    "C1": dict(shape=(1_048_576,), block_edge=256, radius=512, padding="zero", rel_eb=1e-4),
    "C2": dict(shape=(1800, 3600), block_edge=16, radius=512, padding="zero", rel_eb=1e-4),
    "C3": dict(shape=(100, 500, 500), block_edge=8, radius=512, padding="mean:global", rel_eb=1e-3),
    "C4": dict(shape=(512, 512, 512), block_edge=8, radius=512, padding="mean:global", rel_eb=1e-3),
    "C5": dict(shape=(2048, 2048, 1024), block_edge=8, radius=512, padding="mean:global", rel_eb=1e-4),
}


def gen_c1(n: int = 1_048_576, seed: int = 1) -> np.ndarray:
    rng = np.random.default_rng(seed)
    i = np.arange(n, dtype=np.float64)
    x = np.cumsum(rng.standard_normal(n)) * 0.01 + np.sin(2.0 * math.pi * i / 4096.0)
    return x.astype(np.float32)


def _modes(rng, nd, count, kmax, power):
    ks = rng.integers(1, kmax + 1, size=(count, nd)).astype(np.float64)
    phase = rng.uniform(0.0, 2.0 * math.pi, size=count)
    amp = np.linalg.norm(ks, axis=1) ** (-power)
    return ks, phase, amp


def gen_modes(shape, count, kmax, power, noise, seed) -> np.ndarray:
    """Sum of `count` random sinusoidal modes on [0,1)^nd plus N(0, noise).

    sin(a+b+c) is evaluated as Im(e^{ia} e^{i(b+c)}): one 2D complex
    exponential per mode, then exact elementwise float64 products, so the
    cost is two multiply-adds per element per mode.
    """
    rng = np.random.default_rng(seed)
    nd = len(shape)
    if nd not in (2, 3):
        raise ValueError("gen_modes builds 2D/3D fields")
    ks, phase, amp = _modes(rng, nd, count, kmax, power)
    axes = [np.arange(s, dtype=np.float64) / s for s in shape]
    acc = np.zeros(shape, dtype=np.float64)
    for m in range(count):
        a = 2.0 * math.pi * ks[m, 0] * axes[0] + phase[m]
        if nd == 2:
            inner = 2.0 * math.pi * ks[m, 1] * axes[1]
            re, im = np.cos(inner), np.sin(inner)
            acc += (amp[m] * np.sin(a))[:, None] * re[None, :]
            acc += (amp[m] * np.cos(a))[:, None] * im[None, :]
        else:
            inner = (2.0 * math.pi * ks[m, 1] * axes[1])[:, None] + (
                2.0 * math.pi * ks[m, 2] * axes[2]
            )[None, :]
            re, im = np.cos(inner), np.sin(inner)
            sa, ca = amp[m] * np.sin(a), amp[m] * np.cos(a)
            for p in range(shape[0]):
                acc[p] += sa[p] * re
                acc[p] += ca[p] * im
    out = acc.astype(np.float32)
    del acc
    out += rng.normal(0.0, noise, size=shape).astype(np.float32)
    return out


def gen_c2(shape=(1800, 3600), seed: int = 2) -> np.ndarray:
    return gen_modes(shape, 64, 16, 1.0, 1e-3, seed)


def gen_c3(shape=(100, 500, 500), seed: int = 3) -> np.ndarray:
    return gen_modes(shape, 128, 12, 1.5, 1e-3, seed)


def gen_c4(n: int = 512, seed: int = 4) -> np.ndarray:
    """exp(g), g a unit-variance Gaussian random field with P(k) ~ k^-3."""
    rng = np.random.default_rng(seed)
    white = rng.standard_normal((n, n, n))
    f = np.fft.rfftn(white)
    k0 = np.fft.fftfreq(n) * n
    k2 = np.fft.rfftfreq(n) * n
    kk = np.sqrt(k0[:, None, None] ** 2 + k0[None, :, None] ** 2 + k2[None, None, :] ** 2)
    kk[0, 0, 0] = 1.0
    f *= kk ** (-1.5)
    f[0, 0, 0] = 0.0
    g = np.fft.irfftn(f, s=(n, n, n), axes=(0, 1, 2))
    g /= g.std()
    return np.exp(g).astype(np.float32)


def value_range_eb(data: np.ndarray, rel: float) -> float:
    """The reference's relative-bound resolution (model.py:104-110)."""
    return float(rel) * (float(data.max()) - float(data.min()))


NOISE_GROUP = 8  # planes per noise seed in the C5 generators (one b=8 block layer)

# --------------------------------------------------------------------------
# device-side generators (bench only; no parity pin needed, these just have
# to be the same field on every run)
# --------------------------------------------------------------------------


def gen_modes_torch(shape, count, kmax, power, noise, seed, device, z_range=None):
    """3-D mode-sum field (C5 recipe) for planes z_range of `shape`, built on
    the GPU: per mode one 2-D float64 phase plane, then float32 broadcast
    multiply-adds over the slab.  Deterministic for a given (seed, z_range)."""
    import torch

    rng = np.random.default_rng(seed)
    ks, phase, amp = _modes(rng, 3, count, kmax, power)
    D0, D1, D2 = shape
    z0, z1 = z_range if z_range is not None else (0, D0)
    out = torch.zeros((z1 - z0, D1, D2), dtype=torch.float32, device=device)
    zz = torch.arange(z0, z1, dtype=torch.float64, device=device) / D0
    yy = torch.arange(D1, dtype=torch.float64, device=device) / D1
    xx = torch.arange(D2, dtype=torch.float64, device=device) / D2
    for m in range(count):
        a = 2.0 * math.pi * float(ks[m, 0]) * zz + float(phase[m])
        inner = (2.0 * math.pi * float(ks[m, 1]) * yy)[:, None] + (
            2.0 * math.pi * float(ks[m, 2]) * xx
        )[None, :]
        cb, sb = torch.cos(inner).float(), torch.sin(inner).float()
        sa = (float(amp[m]) * torch.sin(a)).float()
        ca = (float(amp[m]) * torch.cos(a)).float()
        out.addcmul_(sa[:, None, None], cb[None])
        out.addcmul_(ca[:, None, None], sb[None])
    # noise per group of NOISE_GROUP planes, each from its own seed: any
    # block-aligned slab of the field is the same slice of the whole field
    # (z-sharded runs then see exactly the 1-GPU field)
    gen = torch.Generator(device=device)
    for g0 in range(z0 - z0 % NOISE_GROUP, z1, NOISE_GROUP):
        gen.manual_seed(seed * 1_000_003 + g0 // NOISE_GROUP)
        nz = torch.randn((NOISE_GROUP, D1, D2), generator=gen, device=device,
                         dtype=torch.float32)
        a, b = max(g0, z0), min(g0 + NOISE_GROUP, z1)
        out[a - z0:b - z0].add_(nz[a - g0:b - g0], alpha=noise)
    return out


def gen_c5_slab(z_range, device, shape=(2048, 2048, 1024), seed: int = 5):
    """BASELINE config 5 (64 modes, k in [1,16]^3, amp 1/|k|, + N(0,1e-3))."""
    return gen_modes_torch(shape, 64, 16, 1.0, 1e-3, seed, device, z_range)


def gen_c5_slab_numpy(z_range, shape=(2048, 2048, 1024), seed: int = 5) -> np.ndarray:
    """CPU (float64) build of the C5 recipe for a slab -- used by the
    reference arm of bench.py, which must not touch the GPU path.  The 2-D
    phase plane e^{i(b+c)} is the outer product of two 1-D exponentials."""
    rng = np.random.default_rng(seed)
    ks, phase, amp = _modes(rng, 3, 64, 16, 1.0)
    D0, D1, D2 = shape
    z0, z1 = z_range
    zz, yy, xx = np.arange(z0, z1) / D0, np.arange(D1) / D1, np.arange(D2) / D2
    acc = np.zeros((z1 - z0, D1, D2), dtype=np.float64)
    t2 = np.empty((D1, D2), dtype=np.float64)
    for m in range(64):
        a = 2.0 * math.pi * ks[m, 0] * zz + phase[m]
        b = 2.0 * math.pi * ks[m, 1] * yy
        c = 2.0 * math.pi * ks[m, 2] * xx
        re = np.outer(np.cos(b), np.cos(c)) - np.outer(np.sin(b), np.sin(c))
        im = np.outer(np.sin(b), np.cos(c)) + np.outer(np.cos(b), np.sin(c))
        sa, ca = amp[m] * np.sin(a), amp[m] * np.cos(a)
        for p in range(z1 - z0):
            np.multiply(re, sa[p], out=t2)
            acc[p] += t2
            np.multiply(im, ca[p], out=t2)
            acc[p] += t2
    out = acc.astype(np.float32)
    for g0 in range(z0 - z0 % NOISE_GROUP, z1, NOISE_GROUP):  # as gen_modes_torch
        nz = np.random.default_rng(seed * 1_000_003 + g0 // NOISE_GROUP).normal(
            0.0, 1e-3, (NOISE_GROUP, D1, D2)).astype(np.float32)
        a, b = max(g0, z0), min(g0 + NOISE_GROUP, z1)
        out[a - z0:b - z0] += nz[a - g0:b - g0]
    return out
