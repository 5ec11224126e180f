import os, sys, subprocess, numpy as np, torch
sys.path.insert(0, os.getcwd())
import build
sys.argv = [sys.argv[0]]
subprocess.run([build.NVCC, *build.ARCH, "-O3", "-std=c++17", "-shared", "-Xcompiler", "-fPIC", "-fmad=false",
                "-DW3D_DEBUG_TMA", "-I", "include", "-o", "paper_1811_11226_b200/libwarp3d.so",
                *build.CUDA_SOURCES], check=True)
import paper_1811_11226_b200 as W, synth, oracle as O
shape=(160,128,128)
for B in (1,):
    imgs=[]; lbls=[]; params=[]
    for i in range(B):
        im, lb = synth.phantom(shape, seed=100+i)
        d = synth.draw(synth.TRAIN, i)
        A = O.compose_affine(O.make_geom(d.rot_rad, d.scale, d.shear, d.flip, d.generic, d.disp), shape, shape)[1]
        params.append(W.volume_params(A, W.photometric(0xF, window=d.window, gamma=d.gamma, sigma=d.sigma, seed=1, volume_id=i)))
        imgs.append(im); lbls.append(lb)
    for lab in (False, True):
        o, ol = W.warp3d_affine_batched(torch.from_numpy(np.stack(imgs)).cuda(), torch.from_numpy(np.stack(lbls)).cuda() if lab else None, params, fill=-1000.0)
        torch.cuda.synchronize()
        print("B", B, "labels", lab, "done", W.warp3d_tile_stats(), flush=True)
