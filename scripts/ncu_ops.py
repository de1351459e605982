"""Executed warp instructions of an ncu --set full capture, by SASS opcode (and the hottest
straight-line blocks), to see where a kernel's issue slots go.

usage: python scripts/ncu_ops.py REPORT.ncu-rep [N]
"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, data = rows[1], rows[2:]
iS, iE = hdr.index("Source"), hdr.index("Instructions Executed")
tot = sum(int(r[iE]) for r in data)
ops = collections.Counter()
for r in data:
    src = r[iS].strip()
    toks = src.split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    ops[op.split(".")[0]] += int(r[iE])
print(f"total warp instructions {tot / 1e6:.1f}M")
for op, n in ops.most_common(N):
    print(f"{op:12s} {n / 1e6:9.1f}M {100 * n / tot:5.1f}%")
