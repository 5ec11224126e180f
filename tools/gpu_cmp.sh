#!/bin/bash
# Compare kernel variants on the default workload (no tests).
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for v in ${VARIANTS:-auto staged gather}; do
  timeout 300 python bench.py --variant $v --no-e2e --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/cmp_$v.log 2>&1
  python - "$v" <<'PY'
import json,sys
l=open(f"gpurun_out/cmp_{sys.argv[1]}.log").read().strip().splitlines()[-1]
try:
    d=json.loads(l); print(sys.argv[1], "GVox/s %.1f"%d["value"], "frac %.3f"%d["roofline"]["frac"], "ms %.4f"%d["ms_per_step"], d.get("tiles"), d["clocks"]["sm_mhz"])
except Exception as e: print(sys.argv[1], "FAILED", l[-300:])
PY
done
