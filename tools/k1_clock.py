"""K1 (assemble_kernel_t) phase split from an A/B build with -DDOCP_K1_CLOCK:
linearize + Schur / Phi^-1 assembly of the C3 batch, thread 0's clock64
phases summed over its problems.

  python -c "import build; build.build_cuda(force=True, lib='_exp/k1/libdocp_cuda.so', extra_flags=['-DDOCP_K1_CLOCK'])"
  DOCP_LIB_PATH=_exp/k1/libdocp_cuda.so python tools/k1_clock.py [--B 4096 --T 100]
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2510_06179_b200 as D  # noqa: E402
from paper_2510_06179_b200 import _lib as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=4096)
ap.add_argument("--T", type=int, default=100)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
prob = D.affine_quadratic(8, 4, a.T)
nz, nl = D.sizes(prob)
b = D.Batch(prob, a.B)
b.upload(L.F_THETA, D.generate_affine_quadratic(8, 4, 0, a.B))
b.upload(L.F_Z, np.zeros((a.B, nz)))
b.linearize()
b.assemble_schur()
fn = getattr(L.lib(), "docp_k1_clock", None)
if fn is not None:
    buf = (C.c_ulonglong * 16)()
    fn(buf)  # reset
b.profile_begin()
for _ in range(a.reps):
    b.assemble_schur()
prof = b.profile_end()
print(f"assemble_schur: {prof['kernels']['assemble']['ms'] / a.reps:.3f} ms per launch (B={a.B}, T={a.T})")
if fn is not None:
    buf = (C.c_ulonglong * 16)()
    fn(buf)
    names = ["phase A (linearize)", "B: stage A_t, B_t", "B: M1, M2 (divisions)", "B: chi_t", "B: flush S blocks",
             "B: Cholesky", "B: chi^-1 solves", "B: flush Phi^-1 diag", "B: barrier", "C: stair off-diagonal",
             "C: barrier", "problem loop / skip"]
    tot = sum(buf[:12])
    for k in range(12):
        print(f"  {names[k]:24s} {buf[k] / max(1, tot) * 100:5.1f}%  {buf[k] / 148 / 4 / a.reps:10.0f} cycles per CTA-slot")
