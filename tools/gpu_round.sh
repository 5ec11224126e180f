#!/bin/bash
# One GPU round: build, gpu tests, smoke, bench (both variants), ncu launch list + full capture.
mkdir -p gpurun_out
TAG=${TAG:-r}
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout ${TEST_TIMEOUT:-1200} python -m pytest tests -m gpu -x -q ${TEST_K:+-k "$TEST_K"} > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
  tail -15 gpurun_out/gpu_tests.log
  timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
fi
timeout 600 python bench.py ${BENCH_ARGS} > gpurun_out/bench_${TAG}.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_${TAG}.log
if [ -n "${BENCH_GATHER}" ]; then
  timeout 600 python bench.py --variant gather --no-e2e --no-cpu-baseline > gpurun_out/bench_${TAG}_gather.log 2>&1; tail -1 gpurun_out/bench_${TAG}_gather.log
fi
if [ "${NCU:-0}" == "1" ]; then
  CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline ${NCU_BENCH_ARGS}"
  $CMD > gpurun_out/ncu_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launches.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:warp3d_cube -s 3 -c 1 -o gpurun_out/prof_${TAG} -f $CMD > gpurun_out/ncu_full.log 2>&1
  echo "ncu rc=$?"; tail -3 gpurun_out/ncu_full.log
fi
