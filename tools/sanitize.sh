#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over tools/sanitize_cases.py,
# and the GPU parity suite on a W3D_CHECK_BOX build (every staged shared-memory access
# asserted inside its box).  Logs: gpurun_out/sanitizer_<tool>.txt, gpurun_out/checkbox_tests.txt
mkdir -p gpurun_out
python build.py all > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck initcheck racecheck; do
  extra=""; args=""
  [ $tool == memcheck ] && extra="--leak-check full"
  [ $tool == racecheck ] && { extra="--racecheck-report all"; args="--quick"; }
  [ $tool == initcheck ] && extra="--track-unused-memory no"
  timeout 1500 $CS --tool $tool $extra --error-exitcode 97 --target-processes all \
     python tools/sanitize_cases.py $args > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/sanitizer_$tool.txt
done
W3D_NVCC_EXTRA=-DW3D_CHECK_BOX timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider \
   > gpurun_out/checkbox_tests.txt 2>&1
echo "checkbox tests rc=$?"; tail -3 gpurun_out/checkbox_tests.txt
python build.py cuda > /dev/null 2>&1  # back to the product build
