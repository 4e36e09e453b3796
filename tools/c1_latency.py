"""C1 latency: the double integrator (n_x=4, n_u=2, T=20,
dt=0.1), B=1, one SQP step as the reference CLI and tests run it
({max_sqp_iters=1, alpha={1}, eps=1e-12}, test_support.hpp:13-19), loss |z|^2
(test_backward.cpp:9-16): solve + adjoint gradient, end to end through the
public API (host inputs in, gradient out), against the reference build
(oracle/_ref) on one host thread. Reports medians in microseconds.

usage: python tools/c1_latency.py [--reps 300] [--json out.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]


def c1_theta(dt=0.1):
    A = np.block([[np.eye(2), dt * np.eye(2)], [np.zeros((2, 2)), np.eye(2)]])
    B = np.vstack([0.5 * dt * dt * np.eye(2), dt * np.eye(2)])
    return np.concatenate([[1, 1, 0.1, 0.1], [0.1, 0.1], A.flatten(order="F"), B.flatten(order="F"),
                           np.zeros(4), [1.0, -1.0, 0.0, 0.0]])


def median_us(fn, reps, warm=20):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts) * 1e6), float(np.percentile(ts, 90) * 1e6)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=300)
    ap.add_argument("--json", default=None)
    ap.add_argument("--profile", action="store_true", help="per-kernel device times of one call (no-graph runs)")
    args = ap.parse_args()
    import paper_2510_06179_b200 as D
    import pyoracle as po

    T = 20
    th = c1_theta()
    prob = D.affine_quadratic(4, 2, T)
    nz, nl = D.sizes(prob)
    out = {"workload": "C1 double integrator (n_x=4, n_u=2, T=20), B=1, one-shot SQP + adjoint gradient of |z|^2"}
    ref_grad = None
    if po.available("ref"):
        o = po.Oracle("ref", po.aq_problem(4, 2, T))
        cfg = po.sqp_config(max_sqp_iters=1, alphas=(1.0,))

        def cpu():
            s = o.sqp_solve(th, np.zeros(nz), np.zeros(nl), cfg)
            return o.backward(th, 2.0 * s.z, np.zeros(nl))[0]
        ref_grad = cpu()
        out["reference_cpu_us"], out["reference_cpu_p90_us"] = median_us(cpu, args.reps)
    import torch
    for mode, graphs in (("parity", True), ("fast", True), ("parity", False), ("fast", False)):
        cfg = D.one_shot_config(mode=mode)
        b = D.Batch(prob, 1)
        if graphs:  # a batch stream: sqp_solve (one SQP step) and backward_vjp replay cached CUDA graphs
            stream = torch.cuda.Stream()
            b.set_stream(stream.cuda_stream)
        tag = mode if graphs else mode + "_nograph"
        z0, l0 = np.zeros((1, nz)), np.zeros((1, nl))

        def gpu():
            b.upload(D._lib.F_THETA, th[None])
            b.upload(D._lib.F_Z, z0)
            b.upload(D._lib.F_LAMBDA, l0)
            b.sqp_solve(cfg)
            z = b.download(D._lib.F_Z)
            b.upload(D._lib.F_LOSS_GRAD_Z, 2.0 * z)
            b.upload(D._lib.F_LAMBDA_TILDE, l0)
            b.backward_vjp(cfg.pcg)
            return b.download(D._lib.F_GRAD_THETA)[0]
        g = gpu()
        if ref_grad is not None:
            rel = float(np.linalg.norm(g - ref_grad) / np.linalg.norm(ref_grad))
            out[f"gpu_{tag}_rel_err_vs_reference"] = rel
        l0_ = D.kernel_launches()
        gpu()
        out[f"gpu_{tag}_kernels_per_call"] = D.kernel_launches() - l0_
        out[f"gpu_{tag}_us"], out[f"gpu_{tag}_p90_us"] = median_us(gpu, args.reps)
        if args.profile and not graphs:  # where one call's device time goes
            b.profile_begin()
            gpu()
            p = b.profile_end()
            out[f"gpu_{tag}_profile"] = {"kernels": {k: v for k, v in p["kernels"].items() if v["launches"]},
                                          "pcg_iterations": p["pcg_iterations"], "pcg_solves": p["pcg_solves"],
                                          "span_ms": p["span_ms"], "gap_ms": p["gap_ms"]}
    print(json.dumps(out))
    if args.json:
        with open(args.json, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
