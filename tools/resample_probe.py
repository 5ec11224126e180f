"""Time the pieces of warp3d_resample on the 512^3 -> 171^3 workload (diagnostic)."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import build; build.build_cuda()
import paper_1811_11226_b200 as W, synth
shape, u = (512, 512, 512), (1.0, 1.0, 1.0)
img, lbl = synth.phantom(shape)
ti, tl = torch.from_numpy(img).cuda(), torch.from_numpy(lbl).cuda()
out_shape = W.warp3d_resample_dims(shape, u, 3.0)
A = W.warp3d_resample_affine(shape, out_shape, u, 3.0)
def t(f, n=5):
    f(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(n): f()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / n
sig = W.warp3d_resample_sigma(u, 3.0)
print("smooth3d ms", t(lambda: W.warp3d_smooth3d(ti, sig)))
p = [W.volume_params(A)]
for v, name in ((0, "auto"), (1, "gather")):
    print("warp", name, "ms", t(lambda: W.warp3d_affine_batched(ti[None], tl[None], p, fill=-1000.0, out_shape=out_shape, variant=v)))
print("resample ms", t(lambda: W.warp3d_resample(ti, tl, u, 3.0)))
print("tiles", W.warp3d_tile_stats())
