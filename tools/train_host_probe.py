#!/usr/bin/env python3
"""Host time of one C3 training step with new parameters: the numpy draws, the batched
parameter build, set_params and the launch call, each timed alone (GPU kept busy)."""
import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_11226_b200 as W  # noqa: E402
from paper_1811_11226_b200.augment import FULL, params_from_arrays  # noqa: E402

shape, B = (160, 128, 128), 16
img = torch.randn((B, *shape), device="cuda") * 100
lbl = torch.randint(0, 6, (B, *shape), dtype=torch.uint8, device="cuda")
rng = np.random.default_rng(1)
d = math.pi / 12


def draws():
    return (rng.uniform(-d, d, (B, 3)), rng.uniform(0.9, 1.1, (B, 3)), rng.uniform(-0.1, 0.1, (B, 3)),
            rng.random((B, 3)) < 0.5, rng.uniform(-8, 8, (B, 3)),
            np.stack([rng.uniform(-1000, -150, B), rng.uniform(230, 1500, B)], 1),
            rng.uniform(0.7, 1.5, B), rng.uniform(0, 20, B))


def build(dr, k):
    r, s, sh, f, dp, win, g, sg = dr
    return params_from_arrays(shape, r, s, sh, f, dp, flags=FULL, window=win, gamma=g, sigma=sg,
                              seed=7, volume_ids=np.arange(B) + B * k)


batch = W.AugmentBatch(img, lbl, build(draws(), 0), fill=-1000.0)
batch.run()
torch.cuda.synchronize()
N = 50
t = {"draws": 0.0, "params": 0.0, "set": 0.0, "run_new": 0.0, "run_same": 0.0}
for k in range(N):
    t0 = time.perf_counter(); dr = draws(); t1 = time.perf_counter()
    p = build(dr, k + 1); t2 = time.perf_counter()
    batch.set_params(p); t3 = time.perf_counter()
    batch.run(); t4 = time.perf_counter()
    batch.run(); t5 = time.perf_counter()
    torch.cuda.synchronize()
    t["draws"] += t1 - t0; t["params"] += t2 - t1; t["set"] += t3 - t2
    t["run_new"] += t4 - t3; t["run_same"] += t5 - t4
print({k: round(v / N * 1e6, 1) for k, v in t.items()}, "us per step")
