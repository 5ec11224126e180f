import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.getcwd()+"/tests")
import build; build.build_cuda()
import paper_1811_11226_b200 as W, synth, oracle as O
def run(shape, B, ranges, fill=-1000.0, lf=0, flags=0xF, ident=False):
    imgs=[]; lbls=[]; params=[]
    for i in range(B):
        im, lb = synth.phantom(shape, seed=100+i) if min(shape)>=8 else synth.random_volume(shape, i)
        d = synth.draw(ranges, i)
        A = O.compose_affine(O.make_geom(d.rot_rad, d.scale, d.shear, d.flip, d.generic, d.disp), shape, shape)[1]
        if ident: A = np.eye(3,4,dtype=np.float32)
        params.append(W.volume_params(A, W.photometric(flags, window=d.window, gamma=d.gamma, sigma=d.sigma, seed=1, volume_id=i)))
        imgs.append(im); lbls.append(lb)
    o, ol = W.warp3d_affine_batched(torch.from_numpy(np.stack(imgs)).cuda(), torch.from_numpy(np.stack(lbls)).cuda(), params, fill=fill, label_fill=lf)
    torch.cuda.synchronize()
    return o
for name, args in [("smoke-like", ((44,36,40), 2, synth.TRAIN)), ("16^3 ident", ((16,16,16), 1, synth.TRAIN, -5.0, 9, 0, True)), ("c3-like", ((160,128,128), 16, synth.TRAIN)), ("c3 1 vol", ((160,128,128), 1, synth.TRAIN))]:
    try:
        run(*args); print(name, "OK", W.warp3d_tile_stats(), flush=True)
    except Exception as e:
        print(name, "FAIL", str(e)[:200], flush=True); break
