#!/bin/bash
# Secondary workloads of SURVEY Sec. 8.d on one GPU: C2 (latency), C4 (512^3, large
# rotations), C5 (256 volumes on one GPU), staged vs gather on C3 and C4, int16 input,
# plus one ncu --set full capture of the C4 warp launch.  Output: gpurun_out/sweep_*.log
mkdir -p gpurun_out
python build.py all > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
run() {  # name, bench args
  timeout 600 python bench.py --no-e2e --no-cpu-baseline "${@:2}" > gpurun_out/sweep_$1.log 2>&1
  echo "$1 rc=$?"; tail -1 gpurun_out/sweep_$1.log | cut -c1-200
}
run c2 --workload c2 --steps 200
run c3_gather --workload c3 --variant gather --steps 100
run c3_i16 --workload c3 --input i16 --steps 200
run c4 --workload c4 --steps 30 --warmup 5
run c4_gather --workload c4 --variant gather --steps 30 --warmup 5
run c5 --workload c5 --steps 20 --warmup 3
if [ "${NCU:-0}" == "1" ]; then
  ncu --set full --clock-control none --import-source on -k regex:warp3d_cube -s 3 -c 1 \
      -o gpurun_out/prof_c4 -f python bench.py --workload c4 --steps 3 --warmup 3 --no-e2e \
      --no-cpu-baseline > gpurun_out/ncu_c4.log 2>&1; echo "ncu c4 rc=$?"
fi
