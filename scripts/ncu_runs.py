"""Group the SASS of an ncu capture into runs of equal execution count (loop bodies) and
print each run's share of the executed instructions and its opcode mix.

usage: python scripts/ncu_runs.py REPORT.ncu-rep [min_total_M] [--dump a-b]
"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
thr = float(sys.argv[2]) * 1e6 if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else 1e7
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, data = rows[1], rows[2:]
iS, iE = hdr.index("Source"), hdr.index("Instructions Executed")
if "--dump" in sys.argv:
    a, b = map(int, sys.argv[sys.argv.index("--dump") + 1].split("-"))
    for n in range(a, b + 1):
        print(n, data[n][iE], data[n][iS].strip()[:100])
    sys.exit()
runs, cur = [], None
for n, r in enumerate(data):
    e = int(r[iE])
    op = r[iS].strip().split()[0] if r[iS].strip() else ""
    key = round(e / 5e4)
    if cur and cur[0] == key:
        cur[2] += 1
        cur[3] += e
        cur[4].append(op)
    else:
        if cur:
            runs.append(cur)
        cur = [key, n, 1, e, [op]]
runs.append(cur)
tot = sum(int(r[iE]) for r in data)
print(f"total {tot / 1e6:.1f}M warp instructions")
for key, start, cnt, e, ops in runs:
    if e > thr:
        c = collections.Counter(o.split(".")[0] for o in ops)
        print(f"{start:5d}-{start + cnt - 1:5d} n={cnt:4d} exec={key * 0.05:6.2f}M total={e / 1e6:7.1f}M "
              f"{100 * e / tot:5.1f}%  {dict(c.most_common(7))}")
