import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.getcwd() + "/tests")
import build; build.build_cuda()
import paper_1811_11226_b200 as W, synth, oracle as O
shape = tuple(int(v) for v in sys.argv[1].split(",")) if len(sys.argv) > 1 else (160, 128, 128)
variant = int(sys.argv[2]) if len(sys.argv) > 2 else 0
B = 3
imgs, lbls, params = [], [], []
for i in range(B):
    im, lb = synth.phantom(shape, seed=300 + i)
    imgs.append(np.round(im).astype(np.int16)); lbls.append(lb)
    d = synth.draw(synth.TRAIN, 500 + i)
    A = O.compose_affine(O.make_geom(d.rot_rad, d.scale, d.shear, d.flip, d.generic, d.disp), shape, shape)[1]
    params.append(W.volume_params(A, W.photometric(0xF, window=d.window, gamma=d.gamma, sigma=d.sigma, seed=1, volume_id=i)))
i16 = torch.from_numpy(np.stack(imgs)).cuda(); lb = torch.from_numpy(np.stack(lbls)).cuda()
for labels in ((True,) if os.environ.get("LBL_ONLY") else (False, True)):
    o, ol = W.warp3d_affine_batched(i16, lb if labels else None, params, fill=-1000.0, variant=variant)
    torch.cuda.synchronize()
    print("labels", labels, "ok", W.warp3d_tile_stats(), flush=True)
