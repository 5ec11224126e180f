#!/bin/bash
# Summaries of one gpu_evidence.sh run (TAG) into profiles/round2/ (bench lines, gpu suite,
# launch list, ncu --set full summaries with the dispatch model and stall counters).
TAG=$1; OUT=profiles/round2; G=gpurun_out
for n in c3 c1 c2 c4 c5 c3_occ c3_i16 c3_gather c4_gather resample ref; do
  tail -1 $G/ev_${TAG}_bench_$n.log > $OUT/bench_${n}_${TAG}.json
done
cp $G/ev_${TAG}_gpu_tests.log $OUT/gpu_tests_${TAG}.txt
cp $G/ev_${TAG}_launches_c3.csv $OUT/launches_c3_${TAG}.csv
python3 tools/launches_summary.py $G/ev_${TAG}_launches_c3.csv --json $OUT/launches_c3_${TAG}.json > $OUT/launches_c3_${TAG}.txt
for w in c3 c4; do
  vox=$([ $w = c3 ] && echo 41943040 || echo 134217728)
  f=$OUT/ncu_full_${w}_${TAG}.txt
  python3 tools/ncu_summary.py $G/ev_${TAG}_$w.ncu-rep $vox > $f 2>&1
  python3 tools/rf_model.py $G/ev_${TAG}_$w.ncu-rep $vox >> $f 2>&1
  ncu -i $G/ev_${TAG}_$w.ncu-rep --page raw --csv 2>/dev/null > /tmp/raw_$w.csv
  python3 - /tmp/raw_$w.csv $vox >> $f <<'PY'
import csv, sys
r = list(csv.reader(open(sys.argv[1])))
h, u, v = r[0], r[1], r[2]
wv = float(sys.argv[2]) / 32 / 592
g = lambda n: float(v[h.index(n)].replace(',', ''))
print(f"smsp__cycles_active.avg per warp-voxel ({sys.argv[2]} voxels / 32 / 592 SMSPs)     {g('smsp__cycles_active.avg') / wv:.1f}")
for n in ['lts__throughput.avg.pct_of_peak_sustained_elapsed', 'l1tex__throughput.avg.pct_of_peak_sustained_active',
          'smsp__pcsamp_warps_issue_stalled_selected', 'smsp__pcsamp_warps_issue_stalled_not_selected',
          'smsp__pcsamp_warps_issue_stalled_math_pipe_throttle', 'smsp__pcsamp_warps_issue_stalled_dispatch_stall',
          'smsp__pcsamp_warps_issue_stalled_wait', 'smsp__pcsamp_warps_issue_stalled_short_scoreboard',
          'smsp__pcsamp_warps_issue_stalled_long_scoreboard', 'smsp__pcsamp_warps_issue_stalled_mio_throttle',
          'smsp__pcsamp_warps_issue_stalled_barrier']:
    if n in h:
        print(f"{n:70s} {v[h.index(n)]:>16s} {u[h.index(n)]}")
PY
done
if [ -f $G/ev_${TAG}_resample.ncu-rep ]; then
  python3 tools/ncu_summary.py $G/ev_${TAG}_resample.ncu-rep 134217728 > $OUT/ncu_full_resample_${TAG}.txt 2>&1
fi
python3 tools/ncu_traffic.py $TAG > /dev/null
[ -f $G/ev_${TAG}_pcie.json ] && cp $G/ev_${TAG}_pcie.json $OUT/pcie_probe_${TAG}.json
