"""RL rollout timing in the paper's protocol (PAPER.md:606-607,
1229-1233): B environments x H = 50 sequential MPC steps, one QP iteration
per step with alpha = {1} and PCG eps = 1e-12 (make_linear_rl_task,
train.hpp:218-235), forward (rollout) and forward + backward
(rollout + rollout_backward), for the paper's problem shapes P1-P6.

GPU: docp_rollout / docp_rollout_backward (CUDA events, median of --reps).
CPU: the reference's rollout + rollout_backward per instance
(oracle/_ref, parallel_for over every host thread).
Reported next to the paper's own RTX 3090 / 64-core CPU timings of its JAX
implementation (context only: other implementation, other hardware).

usage: python tools/rl_bench.py [--reps 5] [--no-cpu] [--md out.md]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

H = 50
# name: (n_x, n_u, T, B, paper GPU fwd s, fwd+bwd s, paper CPU fwd s, fwd+bwd s)
SHAPES = {
    "P1": (8, 4, 40, 64, 0.22, 0.32, 1.33, 2.70),
    "P2": (8, 4, 30, 16, 0.11, 0.18, 0.16, 0.35),
    "P3": (8, 4, 30, 64, 0.18, 0.27, 0.71, 1.49),
    "P4": (8, 4, 30, 256, 0.49, 0.69, 5.09, 10.00),
    "P5": (16, 8, 30, 16, 0.20, 0.32, 0.74, 1.58),
    "P6": (16, 8, 30, 64, 0.45, 0.73, 5.49, 10.96),
}


def gpu(nx, nu, T, B, reps):
    import torch

    import paper_2510_06179_b200 as D
    from paper_2510_06179_b200 import _lib as L
    th = D.generate_affine_quadratic(nx, nu, 0, B, convex=False)  # random_linear_instance draws
    x0 = torch.tensor(th[:, -nx:].copy(), device="cuda")            # x_inits = inst.x_s
    b = D.Batch(D.affine_quadratic(nx, nu, T), B)
    b.upload(L.F_THETA, th)
    cfg = D.SqpConfig(max_sqp_iters=1, step_candidates=[1.0], pcg=D.PcgConfig(epsilon=1e-12, mode="fast"))
    stream = torch.cuda.Stream()  # a stream of its own: rollouts replay as CUDA graphs
    b.set_stream(stream.cuda_stream)
    fwd, both = [], []
    for rep in range(reps + 1):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(stream)
        b.rollout(cfg, x0.data_ptr(), H)
        e1.record(stream)
        b.rollout_backward(cfg.pcg)
        e2.record(stream)
        torch.cuda.synchronize()
        if rep:
            fwd.append(e0.elapsed_time(e1) / 1e3)
            both.append(e0.elapsed_time(e2) / 1e3)
    errs = sum(e is not None for e in b.rollout_errors())
    return float(np.median(fwd)), float(np.median(both)), errs


def cpu(nx, nu, T, B):
    import pyoracle as po
    try:
        cores = len(os.sched_getaffinity(0))
    except AttributeError:
        cores = os.cpu_count() or 1
    os.environ["DOCP_WORKERS"] = str(cores)
    th = po.gen_aq(nx, nu, T, 0, B, convex=False)
    x0 = th[:, -nx:].copy()
    cfg = po.sqp_config(max_sqp_iters=1, alphas=(1.0,))
    t0 = time.perf_counter()
    r, g, ok, msgs = po.rollout_affine(nx, nu, T, th, x0, H, cfg)
    return time.perf_counter() - t0, cores


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--md", default=None)
    a = ap.parse_args()
    rows = []
    for name, (nx, nu, T, B, pg_f, pg_fb, pc_f, pc_fb) in SHAPES.items():
        f, fb, errs = gpu(nx, nu, T, B, a.reps)
        row = {"shape": name, "n_x": nx, "n_u": nu, "T": T, "H": H, "B": B, "gpu_fwd_s": f, "gpu_fwd_bwd_s": fb,
               "truncated": errs, "paper_gpu_fwd_s": pg_f, "paper_gpu_fwd_bwd_s": pg_fb,
               "paper_cpu_fwd_s": pc_f, "paper_cpu_fwd_bwd_s": pc_fb}
        if not a.no_cpu:
            row["ref_cpu_fwd_bwd_s"], row["cpu_cores"] = cpu(nx, nu, T, B)
        rows.append(row)
        print(json.dumps(row), flush=True)
    if a.md:
        with open(a.md, "w") as fh:
            fh.write("# RL rollouts in the paper's timing protocol (H = 50 steps, 1 QP iteration, alpha = {1}, "
                     "eps 1e-12)\n\n")
            fh.write("B200 (this repo, FAST PCG, median of %d) next to the reference C++ on the host cores and the "
                     "paper's JAX numbers on an RTX 3090 / 64-core CPU (BASELINE.md §2, context only).\n\n" % a.reps)
            fh.write("| shape (n_x, n_u, T, B) | B200 fwd s | B200 fwd+bwd s | ref CPU fwd+bwd s | "
                     "paper GPU fwd / fwd+bwd s | paper CPU fwd / fwd+bwd s |\n|---|---|---|---|---|---|\n")
            for r in rows:
                cpu_s = f"{r['ref_cpu_fwd_bwd_s']:.3f} ({r['cpu_cores']} thr)" if "ref_cpu_fwd_bwd_s" in r else "-"
                fh.write(f"| {r['shape']} ({r['n_x']}, {r['n_u']}, {r['T']}, {r['B']}) | {r['gpu_fwd_s']:.4f} | "
                         f"{r['gpu_fwd_bwd_s']:.4f} | {cpu_s} | {r['paper_gpu_fwd_s']} / {r['paper_gpu_fwd_bwd_s']} | "
                         f"{r['paper_cpu_fwd_s']} / {r['paper_cpu_fwd_bwd_s']} |\n")


if __name__ == "__main__":
    main()
