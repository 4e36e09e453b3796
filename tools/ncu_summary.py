"""Key counters of one or more `ncu --set full` reports, as a markdown table.

usage: python tools/ncu_summary.py rep1.ncu-rep [rep2 ...] > profiles/<round>_ncu_summary.md
       python tools/ncu_summary.py --traffic pcg.ncu-rep > profiles/pcg_traffic.json
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "SMEM wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "SMEM bank conflicts"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__block_size", "block"),
    ("launch__grid_size", "grid"),
    ("launch__shared_mem_per_block_dynamic", "dyn SMEM/CTA"),
]
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
              "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for k, u, v in zip(h, units, vals):
        try:
            x = float(v.replace(",", ""))
        except ValueError:
            d[k] = (v, u)
            continue
        d[k] = (x * UNIT_SCALE.get(u, 1.0), u)
    d["Kernel Name"] = (vals[h.index("Kernel Name")], "")
    return d


def stalls(d, n=3):
    s = [(v[0], k.replace("smsp__pcsamp_warps_issue_stalled_", "")) for k, v in d.items()
         if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")
         and isinstance(v[0], float)]
    tot = sum(x for x, _ in s) or 1
    return ", ".join(f"{name} {100 * x / tot:.0f}%" for x, name in sorted(s, reverse=True)[:n])


def fmt(key, v):
    x, u = v
    if not isinstance(x, float):
        return str(x)
    if key == "gpu__time_duration.sum":
        return f"{x * 1e6:.1f} us"
    if u in ("byte", "Kbyte", "Mbyte", "Gbyte"):
        return f"{x / 1e6:.2f} MB"
    if "pct" in key:
        return f"{x:.1f}"
    return f"{x:,.0f}"


def main():
    args = sys.argv[1:]
    if args and args[0] == "--traffic":
        d = raw(args[1])
        rd = d["dram__bytes_read.sum"][0]
        wr = d["dram__bytes_write.sum"][0]
        print(json.dumps({"report": args[1], "kernel": d["Kernel Name"][0], "dram_bytes_read": rd,
                          "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
                          "duration_s": d["gpu__time_duration.sum"][0]}, indent=1))
        return
    print("| counter | " + " | ".join(a.split("/")[-1].replace(".ncu-rep", "") for a in args) + " |")
    print("|---|" + "---|" * len(args))
    ds = [raw(a) for a in args]
    print("| kernel | " + " | ".join(f"`{d['Kernel Name'][0].split('(')[0]}`" for d in ds) + " |")
    for key, label in KEYS:
        print(f"| {label} | " + " | ".join(fmt(key, d[key]) if key in d else "–" for d in ds) + " |")
    print("| top stalls | " + " | ".join(stalls(d) for d in ds) + " |")


if __name__ == "__main__":
    main()
