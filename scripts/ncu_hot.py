"""Top stall sites of an ncu --set full capture (SASS source page).

usage: python scripts/ncu_hot.py REPORT.ncu-rep [N]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, data = rows[1], rows[2:]
iS, iE = hdr.index("Source"), hdr.index("Instructions Executed")
iW = hdr.index("Warp Stall Sampling (All Samples)")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
idx = [hdr.index(h) for h in reasons]
tot = sum(int(r[iW]) for r in data)
print("samples", tot, "warp instructions", sum(int(r[iE]) for r in data))
T = {h[6:]: sum(int(r[i]) for r in data) for h, i in zip(reasons, idx)}
print({k: round(100 * v / tot, 1) for k, v in sorted(T.items(), key=lambda x: -x[1]) if v > 0})
top = sorted(range(len(data)), key=lambda n: -int(data[n][iW]))[:N]
for n in sorted(top):
    r = data[n]
    rs = sorted(((int(r[i]), h[6:]) for h, i in zip(reasons, idx)), reverse=True)[:2]
    print(f"{n:5d} {int(r[iE]) / 1e6:6.2f}M {100 * int(r[iW]) / tot:5.1f}% {r[iS].strip()[:60]:60s} {rs}")
