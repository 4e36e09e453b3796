"""Warp-stall samples per CUDA source line from `ncu -i rep --page source --csv --print-source cuda,sass`.

usage: ncu -i r.ncu-rep --page source --csv --print-source cuda,sass > f.csv; python tools/ncu_lines.py f.csv [N]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
agg = collections.defaultdict(lambda: [0, collections.Counter(), ""])
fname, hdr, cur = None, None, None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        si = hdr.index("Warp Stall Sampling (All Samples)")
        stall_cols = [(i, k) for i, k in enumerate(hdr) if k.startswith("stall_") and "Not Issued" not in k]
        continue
    if hdr is None or len(r) <= si:
        continue
    if r[0].strip():
        cur = (fname, int(r[0]))
        agg[cur][2] = r[1].strip()[:70]
    if cur is None:
        continue
    try:
        n = int(r[si])
    except ValueError:
        continue
    agg[cur][0] += n
    for i, k in stall_cols:
        try:
            agg[cur][1][k[6:]] += int(r[i])
        except (ValueError, IndexError):
            pass
tot = sum(v[0] for v in agg.values()) or 1
for (f, ln), (n, c, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:N]:
    top = ", ".join(f"{k} {100 * x / max(1, n):.0f}%" for k, x in c.most_common(2))
    print(f"{100 * n / tot:5.1f}%  {f}:{ln:<5d} {src:70s} [{top}]")
