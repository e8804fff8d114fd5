"""Host<->device copy bandwidth probe (pinned buffers): H2D alone, D2H
alone, and both concurrently on two streams -- the ceiling of the e2e
(host-buffer) pipeline, whose per-step traffic is 1 GiB in / 1.27 GB out at C2 (end ticks + statistics).
"""
import time

import torch

GB = 1e9
n_in, n_out = 1 << 30, 1275068416
h_in = torch.empty(n_in, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(n_out, dtype=torch.uint8, pin_memory=True)
d_in = torch.empty(n_in, dtype=torch.uint8, device="cuda")
d_out = torch.empty(n_out, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timeit(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


t_h2d = timeit(lambda: d_in.copy_(h_in, non_blocking=True))
t_d2h = timeit(lambda: h_out.copy_(d_out, non_blocking=True))


def both():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


t_both = timeit(both)
print(f"H2D {n_in / t_h2d / GB:.1f} GB/s ({t_h2d * 1e3:.1f} ms)  D2H {n_out / t_d2h / GB:.1f} GB/s "
      f"({t_d2h * 1e3:.1f} ms)  both {t_both * 1e3:.1f} ms")
