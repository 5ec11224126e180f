#!/bin/bash
# A/B of a source patch against the tree it applies to, alternating builds on one box:
# PATCH=<diff applied in the tree> ROUNDS=n BENCH_ARGS=... (the tree holds the patched code)
mkdir -p gpurun_out
for r in $(seq 1 ${ROUNDS:-2}); do
  for side in new old; do
    [ $side = old ] && patch -s -R -p1 < "$PATCH"
    python build.py cuda > gpurun_out/build_$side.log 2>&1 || { echo "$side build failed"; tail -3 gpurun_out/build_$side.log; }
    timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 100 ${BENCH_ARGS} > gpurun_out/ab_$side.log 2>&1
    [ $side = old ] && patch -s -p1 < "$PATCH"
    python - "$side" <<'PY'
import json,sys
l=open(f"gpurun_out/ab_{sys.argv[1]}.log").read().strip().splitlines()[-1]
try:
    d=json.loads(l); print(sys.argv[1], "GVox/s %.1f"%d["value"], "frac %.3f"%d["roofline"]["frac"], "ms %.4f"%d["ms_per_step"], d["clocks"]["sm_mhz"])
except Exception as e: print(sys.argv[1], "FAILED", l[-300:])
PY
  done
done
