"""Warm-vs-cold PCG study on the GPU — bench::pcg_study (study.hpp:56-145).

For every exit tolerance, a sequence of slowly drifting convex instances
(random_convex_instance, coefficients of A, B, b, x_s perturbed by <= 1% per
step) is solved cold (zero initial guess) and warm (the previous step's
solution), for the forward Schur solve and for the backward solve with the
RL-style cotangent 2 z. `sequences` independent sequences (seeds seed,
seed+1, ...) run as one batch; the solves within a step are timed with CUDA
events on the batch stream.
"""
from __future__ import annotations

import numpy as np

from . import _lib as L
from .api import Batch, PcgConfig, affine_quadratic, generate_drift_sequence


def pcg_study(tols, steps: int = 50, seed: int = 0, n_x: int = 8, n_u: int = 4, horizon: int = 30,
              sequences: int = 1, mode: str = "fast"):
    """Returns (cold_iters, warm_iters, cold_ms, warm_ms): iteration arrays
    [tol][step][pass][sequence] (pass 0 = forward, 1 = backward) and the
    batch's solve times [tol][step][pass] in ms."""
    import torch

    prob = affine_quadratic(n_x, n_u, horizon)
    nz = n_x * (horizon + 1) + n_u * horizon
    nl = n_x * (horizon + 1)
    seqs = np.stack([generate_drift_sequence(n_x, n_u, seed + s, steps, 0.01) for s in range(sequences)], axis=1)
    b = Batch(prob, sequences)
    stream = torch.cuda.current_stream()
    b.set_stream(stream.cuda_stream)
    shape = (len(tols), steps, 2, sequences)
    cold_it, warm_it = np.zeros(shape, np.int32), np.zeros(shape, np.int32)
    cold_ms, warm_ms = np.zeros(shape[:3]), np.zeros(shape[:3])
    zeros_z, zeros_l = np.zeros((sequences, nz)), np.zeros((sequences, nl))

    def timed(fn):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    for ti, tol in enumerate(tols):
        cfg = PcgConfig(epsilon=tol, mode=mode)
        warm_l, warm_lt = zeros_l.copy(), zeros_l.copy()
        for k in range(steps):
            b.upload(L.F_THETA, seqs[k])
            b.upload(L.F_Z, zeros_z)
            b.linearize()
            b.assemble_schur()
            b.assemble_gamma(L.RHS_FORWARD)
            for p, field in ((0, L.F_LAMBDA), (1, L.F_LAMBDA_TILDE)):
                if p == 1:  # the RL reward cotangent at the step's solution (study.hpp:96-101)
                    b.upload(L.F_LAMBDA, warm_l)
                    b.recover_primal(L.F_LAMBDA, L.RHS_FORWARD)
                    b.upload(L.F_LOSS_GRAD_Z, 2.0 * b.download(L.F_Z_QP))
                    b.assemble_gamma(L.RHS_ADJOINT)
                b.upload(field, zeros_l)
                cold_ms[ti, k, p] = timed(lambda: b.pcg_solve(cfg, field))
                cold_it[ti, k, p] = b.download(L.F_PCG_ITERS)[:, 0]
                b.upload(field, warm_l if p == 0 else warm_lt)
                warm_ms[ti, k, p] = timed(lambda: b.pcg_solve(cfg, field))
                warm_it[ti, k, p] = b.download(L.F_PCG_ITERS)[:, 0]
                if p == 0:
                    warm_l = b.download(L.F_LAMBDA)
                else:
                    warm_lt = b.download(L.F_LAMBDA_TILDE)
    return cold_it, warm_it, cold_ms, warm_ms


def summarize(tols, cold_it, warm_it, cold_ms, warm_ms):
    """WarmColdSummary (study.hpp:125-144) per (tol, pass), steps >= 1."""
    out = []
    for ti, tol in enumerate(tols):
        for p, name in ((0, "forward"), (1, "backward")):
            c, w = cold_it[ti, 1:, p], warm_it[ti, 1:, p]
            ct, wt = cold_ms[ti, 1:, p].sum(), warm_ms[ti, 1:, p].sum()
            out.append({"tol": tol, "pass": name, "frac_warm_not_worse": float((w <= c).mean()),
                        "mean_iter_reduction": float((c - w).mean()),
                        "iter_reduction_frac": float((c - w).sum() / max(1, c.sum())),
                        "speedup": float((ct - wt) / ct) if ct > 0 else 0.0})
    return out
