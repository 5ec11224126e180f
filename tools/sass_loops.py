#!/usr/bin/env python3
"""List the loops (backward branches) of one kernel's SASS with their instruction mix.
usage: sass_loops.py <all.sass> <function-substring>"""
import collections, re, sys

text = open(sys.argv[1]).read().split("Function : ")
fn = [t for t in text if t.startswith(sys.argv[2]) or sys.argv[2] in t.split("\n")[0]]
body = fn[0]
ins = []
for line in body.splitlines():
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr = {a: i for i, (a, _) in enumerate(ins)}
loops = []
for i, (a, s) in enumerate(ins):
    m = re.search(r"BRA (?:\w+, )?0x([0-9a-f]+)", s)
    if m:
        t = int(m.group(1), 16)
        if t <= a and t in addr:
            loops.append((addr[t], i))
print("total instructions", len(ins))
for lo, hi in loops:
    mix = collections.Counter()
    for _, s in ins[lo:hi + 1]:
        op = re.sub(r"^@!?U?P\w+\s+", "", s).split()[0]
        mix[op.split(".")[0]] += 1
    print(f"loop [{ins[lo][0]:#x}, {ins[hi][0]:#x}] {hi - lo + 1} instr:",
          " ".join(f"{k}:{v}" for k, v in mix.most_common()))
