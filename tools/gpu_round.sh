mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "not c4 and not c5" > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/gpu_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench1.log 2>&1; echo "bench rc=$?"
tail -3 gpurun_out/bench1.log
timeout 600 python bench.py --steps 50 --warmup 5 --variant gather --no-e2e --no-cpu-baseline > gpurun_out/bench_gather.log 2>&1; tail -1 gpurun_out/bench_gather.log
nproc; free -g | head -2
