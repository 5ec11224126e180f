#!/usr/bin/env python3
"""Summarise an ncu --set full report of the warp kernel: key metrics, opcode mix
per output voxel, and the hottest SASS regions.  Usage: ncu_summary.py REP VOXELS"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep, vox = sys.argv[1], float(sys.argv[2])


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h, u, v = raw[0], raw[1], raw[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"]
for w in want:
    if w in h:
        i = h.index(w)
        print(f"{w:70s} {v[i]:>16s} {u[i]}")
src = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
hdr = src[1]
ix, isrc = hdr.index("Instructions Executed"), hdr.index("Source")
data = src[2:]
tot = sum(int(r[ix]) for r in data)
print(f"warp instr {tot}  thread-instr/voxel {tot * 32 / vox:.1f}")
c = Counter()
for r in data:
    t = r[isrc].split()
    if not t:
        continue
    op = t[1] if t[0].startswith("@") else t[0]
    c[op.split(".")[0]] += int(r[ix])
print("  ".join(f"{op}:{n * 32 / vox:.1f}" for op, n in c.most_common(30)))
