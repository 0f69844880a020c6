"""PCIe roofline for the end-to-end (host-buffer) metric: H2D and D2H of the metric step's bytes
(285 MB in, 268 MB out at N = 2^24) from/to pinned memory, alone and concurrently."""
import time

import torch

N = 2 ** 24
h_in = torch.empty(17 * N, dtype=torch.uint8).pin_memory()
h_out = torch.empty(16 * N, dtype=torch.uint8).pin_memory()
d_in = torch.empty(17 * N, dtype=torch.uint8, device="cuda")
d_out = torch.empty(16 * N, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d(); d2h()


a, b, c = t(h2d), t(d2h), t(both)
print(f"H2D {17 * N / a / 1e6:.1f} GB/s ({a:.2f} ms), D2H {16 * N / b / 1e6:.1f} GB/s ({b:.2f} ms), "
      f"concurrent {c:.2f} ms per (285 MB in + 268 MB out)")
