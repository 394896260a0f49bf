"""Host<->device copy bandwidth on this box (pinned buffers): H2D alone, D2H
alone, and both directions at once on two streams -- the ceiling of the e2e
(host-buffer) numbers in bench.py."""
import time

import torch

n = 1 << 29  # 2 GiB of float32
h_a = torch.empty(n, dtype=torch.float32, pin_memory=True)
h_b = torch.empty(n, dtype=torch.float32, pin_memory=True)
d_a = torch.empty(n, dtype=torch.float32, device="cuda")
d_b = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def bw(fn, nbytes, reps=5):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return nbytes * reps / (time.perf_counter() - t) / 1e9


def h2d():
    with torch.cuda.stream(s1):
        d_a.copy_(h_a, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_b.copy_(d_b, non_blocking=True)


def both():
    h2d()
    d2h()


print(f"H2D {bw(h2d, 4 * n):.1f} GB/s  D2H {bw(d2h, 4 * n):.1f} GB/s  "
      f"both directions {bw(both, 8 * n):.1f} GB/s total")
