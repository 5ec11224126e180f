#!/bin/bash
# Build + gpu tests + smoke + the bench lines of every workload (no ncu).
mkdir -p gpurun_out
TAG=${TAG:-r}
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q ${TEST_K:+-k "$TEST_K"} > gpurun_out/gpu_tests_${TAG}.log 2>&1; echo "tests rc=$?"
  tail -5 gpurun_out/gpu_tests_${TAG}.log
  timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
fi
b() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/bench_${TAG}_${name}.log 2>&1; echo "bench $name rc=$?"; tail -1 gpurun_out/bench_${TAG}_${name}.log | cut -c1-160; }
b c3
for w in ${WORKLOADS:-c1 c2 c4}; do b $w --workload $w --no-e2e --no-cpu-baseline --steps 50 --warmup 5; done
b c3occ --occlusion --no-e2e --no-cpu-baseline
b ref --impl reference --steps 20 --warmup 2
