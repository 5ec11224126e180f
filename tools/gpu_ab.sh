#!/bin/bash
# A/B of build knobs on the default workload: CONFIGS="name:nvcc_extra:env ..." (no tests)
mkdir -p gpurun_out
for cfg in ${CONFIGS:-"tz20::" "tz16:-DW3D_TZ=16:"}; do
  name=${cfg%%:*}; rest=${cfg#*:}; extra=${rest%%:*}; extra=${extra//_-D/ -D}; envs=${rest#*:}
  W3D_NVCC_EXTRA="$extra" python build.py cuda > gpurun_out/build_$name.log 2>&1 || { echo "$name build failed"; tail -3 gpurun_out/build_$name.log; continue; }
  W3D_NVCC_EXTRA="$extra" env $envs timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 100 ${BENCH_ARGS} > gpurun_out/ab_$name.log 2>&1
  python - "$name" <<'PY'
import json,sys
l=open(f"gpurun_out/ab_{sys.argv[1]}.log").read().strip().splitlines()[-1]
try:
    d=json.loads(l); print(sys.argv[1], "GVox/s %.1f"%d["value"], "frac %.3f"%d["roofline"]["frac"], "ms %.4f"%d["ms_per_step"], d.get("tiles"), d["clocks"]["sm_mhz"])
except Exception as e: print(sys.argv[1], "FAILED", l[-300:])
PY
done
