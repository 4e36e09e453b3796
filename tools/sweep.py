"""C5 scaling sweep (BASELINE.json configs[4]): batch x horizon on one GPU.

For every (T, B): random_linear_instance(8, 4, T) draws (generators.hpp:52-79,
mt19937_64 seed 0; batches above the 65,536 pool tile it), one warm-up
solve + gradient, then `--reps` timed repetitions of
    sqp_solve(max_sqp_iters = 5, eps = 1e-12, FAST)  +  backward_vjp
from cold caches (lambda = lambda~ = 0, z = 0), CUDA events on the batch
stream. Reports problems/s, PCG iterations per solve and the PCG kernel's
algorithmic GB/s (SURVEY.md §8(d) bytes) against the measured HBM peak.

Batches larger than --chunk (default 65,536) run in chunks through one
device batch of the chunk size: every chunk's thetas are copied in from a
device-resident array of all B (its own uploads inside the timed region), so
B = 1M runs in bounded memory (the blocks of 1M problems at T = 256 would
need 525 GB).

usage: python tools/sweep.py [--T 16,32,64,100,128,256] [--B 1024,4096,16384,65536]
                             [--reps 3] [--chunk 65536] [--md profiles/r1_sweep.md]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2510_06179_b200 as D  # noqa: E402
from paper_2510_06179_b200 import _lib as L  # noqa: E402

POOL = 65536
CONVEX = False
MODE = "fast"


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            j = json.load(fh)
        return float(j["hbm_gbs"])
    except Exception:
        pass
    return 6540.8


NU = 4
NX = 8


def run(T, B, reps, pool_cache, chunk=65536):
    prob = D.affine_quadratic(NX, NU, T)
    nz, nl = D.sizes(prob)
    if T not in pool_cache:
        pool_cache.clear()
        pool_cache[T] = D.generate_affine_quadratic(NX, NU, 0, min(B, POOL), convex=CONVEX)
    pool = pool_cache[T]
    if len(pool) < min(B, POOL):
        pool = pool_cache[T] = D.generate_affine_quadratic(NX, NU, 0, min(B, POOL), convex=CONVEX)
    th = np.resize(pool, (B, pool.shape[1])) if B > len(pool) else pool[:B]
    C = min(B, chunk)
    assert B % C == 0, "the chunk size must divide the batch"
    b = D.Batch(prob, C)
    b.set_stream(torch.cuda.current_stream().cuda_stream)
    th_dev = torch.tensor(th, device="cuda")
    g = torch.tensor(np.random.default_rng(0).standard_normal((C, nz)) * 1e-2, device="cuda")
    b.upload(L.F_LOSS_GRAD_Z, g)
    cfg = D.SqpConfig(max_sqp_iters=5, pcg=D.PcgConfig(epsilon=1e-12, mode=MODE))
    zeros_z = torch.zeros((C, nz), dtype=torch.float64, device="cuda")
    zeros_l = torch.zeros((C, nl), dtype=torch.float64, device="cuda")

    def step():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for c0 in range(0, B, C):
            b.upload(L.F_THETA, th_dev[c0:c0 + C])
            b.upload(L.F_Z, zeros_z)
            b.upload(L.F_LAMBDA, zeros_l)
            b.upload(L.F_LAMBDA_TILDE, zeros_l)
            b.sqp_solve(cfg)
            b.backward_vjp(cfg.pcg)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    step()  # warm-up
    b.profile_begin()
    ms = [step() for _ in range(reps)]
    prof = b.profile_end()
    errs = sum(e is not None for e in b.errors())
    pcg_ms = prof["kernels"]["pcg"]["ms"]
    total_kernel = sum(k["ms"] for k in prof["kernels"].values())
    gbs = prof["pcg_algorithmic_bytes"] / (pcg_ms / 1e3) / 1e9 if pcg_ms else 0.0
    med = float(np.median(ms))
    return {"T": T, "B": B, "ms_per_step": med, "problems_per_s": B / (med / 1e3),
            "pcg_iters_per_solve": prof["pcg_iterations"] / max(1, prof["pcg_solves"]),
            "pcg_share": pcg_ms / total_kernel if total_kernel else None, "pcg_algorithmic_GBps": gbs,
            "pcg_frac_hbm": gbs / hbm_peak(), "pcg_kernel": D.describe(prob), "failed_instances": errs,
            "block_record_MB": B * 16 * NX * NX * (2 * T + 1) / 1e6, "chunks": B // C}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", default="16,32,64,100,128,256")
    ap.add_argument("--B", default="1024,4096,16384,65536")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--md", default=None)
    ap.add_argument("--chunk", type=int, default=65536)
    ap.add_argument("--nu", type=int, default=4)
    ap.add_argument("--nx", type=int, default=8)
    ap.add_argument("--convex", action="store_true", help="random_convex_instance draws (domain-randomised weights)")
    ap.add_argument("--mode", default="fast", choices=["fast", "parity", "fp32"], help="PCG arithmetic")
    a = ap.parse_args()
    global NU, NX, CONVEX, MODE
    NU, NX, CONVEX, MODE = a.nu, a.nx, a.convex, a.mode
    rows = []
    cache = {}
    for T in [int(x) for x in a.T.split(",")]:
        for B in [int(x) for x in a.B.split(",")]:
            r = run(T, B, a.reps, cache, a.chunk)
            rows.append(r)
            print(json.dumps(r), flush=True)
            torch.cuda.empty_cache()
    if a.md:
        with open(a.md, "w") as fh:
            fh.write("# Sweep — solve + gradient on one B200 (%s, cold caches, median of %d)\n\n" % (MODE.upper(), a.reps))
            fh.write(f"Workload: `{'random_convex_instance' if CONVEX else 'random_linear_instance'}({NX}, {NU}, T)` "
                     "draws, `sqp_solve` (5 SQP iterations max, "
                     "eps 1e-12) + `backward_vjp` per problem. PCG GB/s = algorithmic bytes "
                     "(SURVEY.md §8(d)) / PCG kernel time; HBM peak %.1f GB/s (MEASURED_PEAKS.json).\n\n" % hbm_peak())
            fh.write("| T | B | problems/s | ms/step | PCG it/solve | PCG share | PCG GB/s | x HBM | PCG kernel |\n")
            fh.write("|---|---|---|---|---|---|---|---|---|\n")
            for r in rows:
                kern = (r["pcg_kernel"].split("parity=")[1].split(";")[0].split(" fast=")[0] if MODE == "parity"
                        else r["pcg_kernel"].split("fast=")[1].split(" ")[0])
                fh.write(f"| {r['T']} | {r['B']} | {r['problems_per_s']:,.0f} | {r['ms_per_step']:.2f} | "
                         f"{r['pcg_iters_per_solve']:.1f} | {r['pcg_share']:.2f} | {r['pcg_algorithmic_GBps']:,.0f} | "
                         f"{r['pcg_frac_hbm']:.2f} | {kern} |\n")


if __name__ == "__main__":
    main()
