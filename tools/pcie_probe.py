#!/usr/bin/env python3
"""Host<->device copy bandwidth on this box (pinned memory, copy engines): H2D alone,
D2H alone, and both at once on two streams -- the ceiling of bench.py's `e2e` leg,
which moves the same bytes each way per step.  Prints one JSON line."""
import json

import torch


def timed(fn, reps=10):
    torch.cuda.synchronize()
    best = None
    for _ in range(reps):
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        fn()
        t1.record()
        torch.cuda.synchronize()
        ms = t0.elapsed_time(t1)
        best = ms if best is None else min(best, ms)
    return best * 1e-3


n = 209715200  # bytes per direction of one C3 e2e step
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def h2d():
    d_in.copy_(h_in, non_blocking=True)


def d2h():
    h_out.copy_(d_out, non_blocking=True)


def both():
    cur = torch.cuda.current_stream()
    for s in (s1, s2):
        s.wait_stream(cur)
    with torch.cuda.stream(s1):
        h2d()
    with torch.cuda.stream(s2):
        d2h()
    cur.wait_stream(s1)
    cur.wait_stream(s2)


th, td, tb = timed(h2d), timed(d2h), timed(both)
print(json.dumps({"bytes_per_direction": n, "h2d_gbs": n / th / 1e9, "d2h_gbs": n / td / 1e9,
                  "bidir_gbs_per_direction": n / tb / 1e9,
                  "c3_e2e_ceiling_gvox_s": 41943040 / tb / 1e9}))


# the e2e leg's copy pattern: per volume an image (4 B/voxel) and a label (1 B/voxel)
# copy each way, 16 volumes per step, vs the same bytes in groups of k volumes
nv, vox = 16, 2621440
def chunked(k):
    img_b, lbl_b = 4 * vox * k, vox * k
    def f():
        cur = torch.cuda.current_stream()
        for s in (s1, s2):
            s.wait_stream(cur)
        for g in range(0, nv, k):
            o = (img_b + lbl_b) * (g // k)
            with torch.cuda.stream(s1):
                d_in[o:o + img_b].copy_(h_in[o:o + img_b], non_blocking=True)
                d_in[o + img_b:o + img_b + lbl_b].copy_(h_in[o + img_b:o + img_b + lbl_b],
                                                        non_blocking=True)
            with torch.cuda.stream(s2):
                h_out[o:o + img_b].copy_(d_out[o:o + img_b], non_blocking=True)
                h_out[o + img_b:o + img_b + lbl_b].copy_(d_out[o + img_b:o + img_b + lbl_b],
                                                         non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)
    return f
print(json.dumps({f"vols_per_copy_{k}_gbs_per_direction": n / timed(chunked(k)) / 1e9
                  for k in (1, 2, 4, 8, 16)}))
