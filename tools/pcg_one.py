"""One batched PCG launch with a fixed iteration count on blocks assembled from
random_convex_instance draws (for ncu and clock studies of K2 alone).

  python tools/pcg_one.py [--nx 8 --nu 4 --T 100 --B 1184 --iters 41 --mode fast|parity]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2510_06179_b200 as D  # noqa: E402
from paper_2510_06179_b200 import _lib as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nx", type=int, default=8)
ap.add_argument("--nu", type=int, default=4)
ap.add_argument("--T", type=int, default=100)
ap.add_argument("--B", type=int, default=1184)
ap.add_argument("--iters", type=int, default=41)
ap.add_argument("--mode", default="fast")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
prob = D.affine_quadratic(a.nx, a.nu, a.T)
nz, nl = D.sizes(prob)
b = D.Batch(prob, a.B)
b.upload(L.F_THETA, D.generate_affine_quadratic(a.nx, a.nu, 0, a.B))
b.upload(L.F_Z, np.zeros((a.B, nz)))
b.linearize()
b.assemble_schur()
b.assemble_gamma()
b.profile_begin()
for rep in range(a.reps):
    b.upload(L.F_LAMBDA, np.zeros((a.B, nl)))
    b.pcg_solve(D.PcgConfig(epsilon=1e-300, max_iters=a.iters, mode=a.mode))
prof = b.profile_end()
ms = prof["kernels"]["pcg"]["ms"] / a.reps
print(f"{D.describe(prob)} B={a.B} mode={a.mode}: {ms:.3f} ms per launch of {a.iters} iterations, "
      f"{ms * 1e6 / a.iters / max(1, -(-a.B // 148)):.0f} ns per iteration per problem wave")
for fn in ("docp_h8p_clock", "docp_h8s_clock"):  # A/B builds with -DDOCP_H8P_CLOCK / -DDOCP_H8S_CLOCK
    if not hasattr(L.lib(), fn):
        continue
    import ctypes as C
    buf = (C.c_ulonglong * 16)()
    getattr(L.lib(), fn)(buf)
    if not sum(buf):
        continue
    its = a.iters * a.reps * -(-a.B // 148)  # iterations seen by CTA 0's thread 0 (approx.)
    names = (["S phase1", "barrier", "S phase2", "P phase2", "P phase1", "-", "dot partial", "dot barrier",
              "chain+bcast", "alpha/beta/updates", "loop exit", "setup"] if fn == "docp_h8p_clock" else
             ["S phase1: eta partial", "barriers", "S phase2", "P phase1", "P phase 1b (U)", "P phase2",
              "dot partial", "dot barrier", "dot total", "alpha + updates", "beta + updates", "setup",
              "S phase1: gather + put", "S phase1: sym_times", "S phase1: L x + put", "-"])
    if fn == "docp_h8p_clock" and buf[13]:
        print(f"  chain warp fold: {buf[12] / buf[13]:.0f} cycles per fold (warp 7 lane 0, {buf[13]} folds)")
        buf[12] = buf[13] = 0
    tot = sum(buf)
    for k in range(len(buf)):
        if buf[k] and k < len(names):
            print(f"  {names[k]:24s} {buf[k] / 148 / its:8.0f} cycles/iter  {100 * buf[k] / tot:5.1f}%")
