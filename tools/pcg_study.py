"""Warm-vs-cold PCG study on the GPU (bench::pcg_study, study.hpp:56-145):
iteration reduction and wall-time speedup of warm starts at three exit
tolerances, forward and backward, over `--sequences` drifting instance
sequences solved as one batch. The paper reports 4% (fwd) / 4% (bwd) at
eps = 1e-12 and 11% / 9% at eps = 1e-4 for its JAX implementation
(BASELINE.md §2).

usage: python tools/pcg_study.py [--sequences 1184] [--steps 50] [--md out.md]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2510_06179_b200.study import pcg_study, summarize  # noqa: E402

PAPER = {(1e-12, "forward"): 0.04, (1e-12, "backward"): 0.04, (1e-4, "forward"): 0.11, (1e-4, "backward"): 0.09}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sequences", type=int, default=1184)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--md", default=None)
    a = ap.parse_args()
    tols = [1e-4, 1e-8, 1e-12]
    res = pcg_study(tols, a.steps, seed=0, sequences=a.sequences, mode="fast")
    rows = summarize(tols, *res)
    for r in rows:
        print(json.dumps(r))
    if a.md:
        with open(a.md, "w") as fh:
            fh.write("# Warm-vs-cold PCG study on one B200 (bench::pcg_study protocol)\n\n")
            fh.write(f"{a.sequences} drifting sequences (random_convex_instance(8, 4, 30), <= 1% coefficient drift per "
                     f"step, seeds 0..{a.sequences - 1}) x {a.steps} steps, solved as one batch; FAST PCG. Cold = zero "
                     "initial guess, warm = the previous step's solution; backward = adjoint solve with cotangent 2z. "
                     "Summaries skip step 0 (study.hpp:133). The seed-0 sequence's iteration counts equal the "
                     "reference's own pcg_study (tests/test_gpu_parity.py::test_pcg_study_matches_reference).\n\n")
            fh.write("| eps | pass | warm not worse | mean iteration reduction | iteration reduction | wall-time "
                     "speedup (batch) | paper (JAX, RTX 3090) |\n|---|---|---|---|---|---|---|\n")
            for r in rows:
                paper = PAPER.get((r["tol"], r["pass"]))
                fh.write(f"| {r['tol']:g} | {r['pass']} | {r['frac_warm_not_worse']:.3f} | "
                         f"{r['mean_iter_reduction']:.2f} | {100 * r['iter_reduction_frac']:.1f}% | "
                         f"{100 * r['speedup']:.1f}% | {'' if paper is None else f'{100 * paper:.0f}%'} |\n")


if __name__ == "__main__":
    main()
