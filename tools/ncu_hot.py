"""Top SASS instructions by warp-stall samples from `ncu -i X --page source --csv`.

usage: ncu -i rep --page source --csv > f.csv; python tools/ncu_hot.py f.csv [N]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
si, ni = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, k in enumerate(h) if k.startswith("stall_") and "Not Issued" not in k]
body = [r for r in rows[2:] if len(r) > ni]
tot = sum(int(r[ni]) for r in body) or 1
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
order = sorted(range(len(body)), key=lambda i: -int(body[i][ni]))[:N]
for i in sorted(order):
    r = body[i]
    top = sorted(((int(r[c]), h[c][6:]) for c in stall_cols), reverse=True)[:2]
    print(f"{i:5d} {100 * int(r[ni]) / tot:5.1f}%  {r[si].strip():60s} {top}")
