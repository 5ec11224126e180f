#!/bin/bash
# ncu --set full of one launch of the warp kernel, built with W3D_NVCC_EXTRA (diagnostic variants)
mkdir -p gpurun_out
TAG=${TAG:-var}
python build.py cuda > gpurun_out/build_$TAG.log 2>&1 || { tail -3 gpurun_out/build_$TAG.log; exit 1; }
export W3D_NVCC_EXTRA
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline ${NCU_BENCH_ARGS}"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && tail -1 gpurun_out/plain_$TAG.log | cut -c1-120
ncu --set full --clock-control none --import-source on -k regex:warp3d_cube -s 3 -c 1 -o gpurun_out/prof_$TAG -f $CMD > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?"
