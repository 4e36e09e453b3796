"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv`).

usage: python tools/summarize_launches.py launches.csv [--steps K] > summary.md

Groups launches by kernel name and prints count, total and mean duration and
share of the total. ncu serialises launches and runs them cold-cache, so only
the shares are comparable with bench.py's live CUDA-event profile.
"""
import collections
import csv
import re
import sys


def short(name):
    name = re.sub(r"\(.*", "", name) if not name.startswith("void ") else re.sub(r"\(.*", "", name[5:])
    return name.replace("docp_dev::", "")


def main():
    path = sys.argv[1]
    steps = int(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else None
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    ki, vi, ui, bi, gi = (h.index(k) for k in ("Kernel Name", "Metric Value", "Metric Unit", "Block Size", "Grid Size"))
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        ns = v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "ns": 1, "us": 1e3, "ms": 1e6}.get(unit, 1)
        k = short(r[ki])
        a = agg.setdefault(k, {"n": 0, "ns": 0.0, "block": r[bi], "grid": set()})
        a["n"] += 1
        a["ns"] += ns
        a["grid"].add(r[gi])
    tot = sum(a["ns"] for a in agg.values())
    print(f"# ncu launch list summary: {path}\n")
    print(f"total launches {sum(a['n'] for a in agg.values())}, total kernel time {tot / 1e6:.3f} ms"
          + (f" ({tot / 1e6 / steps:.3f} ms per listed step)" if steps else "") + "\n")
    print("| kernel | launches | total ms | mean us | share | block | grids |")
    print("|---|---|---|---|---|---|---|")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["ns"]):
        grids = sorted(a["grid"])
        g = ", ".join(grids[:3]) + (" …" if len(grids) > 3 else "")
        print(f"| `{k}` | {a['n']} | {a['ns'] / 1e6:.3f} | {a['ns'] / a['n'] / 1e3:.1f} | {a['ns'] / tot:.3f} | {a['block']} | {g} |")


if __name__ == "__main__":
    main()
