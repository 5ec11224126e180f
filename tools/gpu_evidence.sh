#!/bin/bash
# Round evidence on one B200: build, gpu suite, smoke, every workload's bench line (no
# ncu), the reference arm, the ncu launch list of the default bench command and
# ncu --set full of the C3 and C4 warp launches and of the resample lowpass.  Output: gpurun_out/ev_<TAG>_*
mkdir -p gpurun_out
TAG=${TAG:-r}
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/ev_${TAG}_gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/ev_${TAG}_gpu_tests.log
  timeout 300 python __graft_entry__.py smoke > gpurun_out/ev_${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
fi
python tools/pcie_probe.py > gpurun_out/ev_${TAG}_pcie.json 2>&1; echo "pcie rc=$?"; head -1 gpurun_out/ev_${TAG}_pcie.json | cut -c1-160
b() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/ev_${TAG}_bench_${name}.log 2>&1; echo "bench $name rc=$?"; tail -1 gpurun_out/ev_${TAG}_bench_${name}.log | cut -c1-140; }
b c3
b c1 --workload c1 --no-e2e
b c2 --workload c2 --no-e2e
b c4 --workload c4 --no-e2e --steps 30 --warmup 5
b c5 --workload c5 --no-e2e --steps 20 --warmup 3
b c3_occ --occlusion --no-e2e --no-cpu-baseline --no-c5
b c3_i16 --input i16 --no-e2e --no-cpu-baseline --no-c5
b c3_gather --variant gather --no-e2e --no-cpu-baseline --no-c5 --steps 50
b c4_gather --workload c4 --variant gather --no-e2e --no-cpu-baseline --steps 20 --warmup 3
b resample --workload resample --steps 50
b ref --impl reference --steps 20 --warmup 2
if [ "${NCU:-1}" == "1" ]; then
  CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-c5"
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_${TAG}_launches_c3.csv $CMD > /dev/null 2>&1; echo "ncu launches rc=$?"
  ncu --set full --clock-control none --import-source on -k regex:warp3d_cube -s 3 -c 1 -o gpurun_out/ev_${TAG}_c3 -f $CMD > /dev/null 2>&1; echo "ncu c3 rc=$?"
  ncu --set full --clock-control none --import-source on -k regex:warp3d_cube -s 3 -c 1 -o gpurun_out/ev_${TAG}_c4 -f $CMD --workload c4 > /dev/null 2>&1; echo "ncu c4 rc=$?"
  # -s 6: skip the resample steps' (masked) lowpass launches, capture the first dense one (warp3d_smooth3d, what the roofline times)
  ncu --set full --clock-control none --import-source on -k regex:smooth_fused -s 6 -c 1 -o gpurun_out/ev_${TAG}_resample -f $CMD --workload resample > /dev/null 2>&1; echo "ncu resample rc=$?"
fi
