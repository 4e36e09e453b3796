"""C2 (BASELINE.json configs[1]): the cart-pole imitation-learning epoch.

CartpoleParams{horizon = 50} (n_x = 4, n_u = 1), gen_cartpole initial states
(generators.hpp:134-168, seed 0), experts at w* = (1, 2, 1.5, 1), w_u = 0.05
solved with cartpole_expert_config (100 SQP iterations, tol 1e-9), learned
w_x ~ U[0,1]^4 (train.hpp:61-64), epochs of the train_il body
(train.hpp:82-131: solve from the demonstration with the warm lambda cache,
MSE loss on u, backward with the warm lambda~ cache, fixed-order sums, GD
step lr 1e-2), max_sqp_iters = 5.

GPU: docp_il_epoch over B problems (CUDA events, median of the timed epochs
after 3 warm-up epochs). CPU: the reference build (oracle/_ref, its own
gen_cartpole expert solves) running the same epoch body through
parallel_for on every host thread, on a bounded sample.

usage: python tools/c2_bench.py [--B 1024,4096,16384] [--epochs 10] [--cpu-seconds 10] [--md out.md]
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

T = 50
EXPERT = np.array([1.0, 2.0, 1.5, 1.0])
W_U = 0.05
LR = 1e-2


def gpu_epochs(B, epochs, warmup=3):
    import torch

    import paper_2510_06179_b200 as D
    from paper_2510_06179_b200 import _lib as L
    prob = D.cartpole(T)
    nz, nl = D.sizes(prob)
    x0 = D.generate_cartpole_x0(0, B)
    th = np.concatenate([np.tile(EXPERT, (B, 1)), np.full((B, 1), W_U), x0], axis=1)
    z0 = np.zeros((B, nz))
    for t in range(T + 1):
        z0[:, D.flat_offset(4, 1, t, True):D.flat_offset(4, 1, t, True) + 4] = x0
    b = D.Batch(prob, B)
    b.upload(L.F_THETA, th)
    b.upload(L.F_Z, z0)
    b.upload(L.F_LAMBDA, np.zeros((B, nl)))
    b.sqp_solve(D.SqpConfig(max_sqp_iters=100, convergence_tol=1e-9, pcg=D.PcgConfig(mode="fast")))
    failed = sum(e is not None for e in b.errors())
    demos = torch.tensor(b.download(L.F_Z), device="cuda")
    b.upload(L.F_LAMBDA, np.zeros((B, nl)))
    b.upload(L.F_LAMBDA_TILDE, np.zeros((B, nl)))
    w = torch.tensor(D.generate_uniform(0, 4), device="cuda")
    out = torch.zeros(5, dtype=torch.float64, device="cuda")
    cfg = D.SqpConfig(max_sqp_iters=5, pcg=D.PcgConfig(epsilon=1e-12, mode="fast"))
    stream = torch.cuda.current_stream()
    b.set_stream(stream.cuda_stream)

    def epoch():
        b.il_epoch(cfg, w.data_ptr(), 0, 4, demos.data_ptr(), float(B), out.data_ptr(), out.data_ptr() + 8)
        w.sub_(LR * out[1:])

    for _ in range(warmup):
        epoch()
    ms = []
    for _ in range(epochs):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        epoch()
        e1.record(stream)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    med = float(np.median(ms))
    return {"B": B, "ms_per_epoch": med, "problems_per_s": B / (med / 1e3), "expert_failures": failed,
            "loss": float(out[0].item()), "pcg_kernel": D.describe(prob)}


def cpu_epochs(target_s):
    import pyoracle as po
    try:
        cores = len(os.sched_getaffinity(0))
    except AttributeError:
        cores = os.cpu_count() or 1
    os.environ["DOCP_WORKERS"] = str(cores)
    prob = po.cartpole_problem(T)
    nz, nl = po.sizes(prob)

    def sample(n):
        x0, demos = po.gen_cartpole(0, T, n)
        return x0, demos

    def run(n, epochs):
        x0, demos = sample(n)
        lam, lt = np.zeros((n, nl)), np.zeros((n, nl))
        w = np.random.default_rng(0).uniform(0, 1, 4)
        times = []
        for _ in range(epochs):
            th = np.concatenate([np.tile(w, (n, 1)), np.full((n, 1), W_U), x0], axis=1)
            t0 = time.perf_counter()
            loss, grad, *_ = po.il_epoch("ref", prob, th, demos, lam, lt, po.sqp_config(max_sqp_iters=5), 0, 4)
            times.append(time.perf_counter() - t0)
            w = w - LR * grad
        return times

    t1 = run(cores, 2)[1]
    n = int(max(cores, cores * round(target_s / 2 / max(t1, 1e-3))))
    times = run(n, 2)
    return {"value": n / times[1], "unit": "problems/s", "cores": cores, "kind": "reference",
            "sample": f"{n} cart-pole demonstrations (gen_cartpole seed 0, T = 50), second of two IL epochs, "
                      f"parallel_for with {cores} workers: {times[1]:.2f} s"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--B", default="1024,4096,16384")
    ap.add_argument("--epochs", type=int, default=10)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--md", default=None)
    a = ap.parse_args()
    rows = [gpu_epochs(int(B), a.epochs) for B in a.B.split(",")]
    for r in rows:
        print(json.dumps(r), flush=True)
    cpu = None if a.no_cpu else cpu_epochs(a.cpu_seconds)
    if cpu:
        print(json.dumps({"cpu_baseline": cpu}), flush=True)
    if a.md:
        with open(a.md, "w") as fh:
            fh.write("# C2 — cart-pole imitation-learning epoch (n_x = 4, n_u = 1, T = 50), one B200\n\n")
            fh.write("train_il body per problem: SQP solve (5 iterations max) from the demonstration with the warm "
                     "lambda cache, MSE loss, backward with the warm lambda~ cache, fixed-order sums, GD step. "
                     "Median of %d epochs after 3 warm-up epochs; FAST PCG.\n\n" % a.epochs)
            fh.write("| B | problems/s | ms/epoch | PCG kernel |\n|---|---|---|---|\n")
            for r in rows:
                fh.write(f"| {r['B']} | {r['problems_per_s']:,.0f} | {r['ms_per_epoch']:.2f} | "
                         f"{r['pcg_kernel'].split('fast=')[1]} |\n")
            if cpu:
                fh.write(f"\nReference CPU (`oracle/_ref`, {cpu['cores']} threads): **{cpu['value']:,.0f} "
                         f"problems/s** — {cpu['sample']}.\n")


if __name__ == "__main__":
    main()
