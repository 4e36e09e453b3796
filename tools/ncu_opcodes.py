"""Executed warp-instructions per SASS opcode from
`ncu -i rep --page source --csv --print-source sass` (the issue mix of a
kernel: how much of it is FP64 arithmetic and how much is data movement).

usage: python tools/ncu_opcodes.py f.csv [N]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = None
cnt = collections.Counter()
for r in rows:
    if not r:
        continue
    if "Source" in r and any(k.startswith("Instructions Executed") or k == "Warp Instructions Executed" for k in r):
        hdr = r
        si = hdr.index("Source")
        ei = next(i for i, k in enumerate(hdr) if k.startswith("Instructions Executed") or k == "Warp Instructions Executed")
        continue
    if hdr is None or len(r) <= max(si, ei):
        continue
    src = r[si].strip()
    if not src:
        continue
    tok = src.split()
    op = tok[1] if tok[0].startswith("@") and len(tok) > 1 else tok[0]
    try:
        cnt[op.split(".")[0]] += int(float(r[ei]))
    except ValueError:
        pass
if hdr is None:
    sys.exit("no SASS table with an 'Instructions Executed' column found")
tot = sum(cnt.values())
print(f"{'opcode':10s} {'warp-instr':>14s} {'share':>7s}")
for op, n in cnt.most_common(N):
    print(f"{op:10s} {n:14d} {100 * n / tot:6.1f}%")
fp64 = sum(n for op, n in cnt.items() if op in ("DADD", "DMUL", "DFMA"))
print(f"{'total':10s} {tot:14d}   FP64 arithmetic {100 * fp64 / tot:.1f}%")
