#!/usr/bin/env python3
"""Host<->device copy bandwidth of this box (pinned memory, copy engines), alone and
both directions at once: the ceiling of bench.py's e2e number (5 B per voxel each way:
float32 image + uint8 label in, the same out)."""
import torch

n = 256 << 20
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e-3


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)


def both():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
print(f"H2D {n / t1 / 1e9:.1f} GB/s  D2H {n / t2 / 1e9:.1f} GB/s  "
      f"both at once {n / t3 / 1e9:.1f} GB/s each way")
print(f"e2e ceiling at 5 B/voxel each way: {n / t3 / 1e9 / 5:.2f} GVoxel/s")
