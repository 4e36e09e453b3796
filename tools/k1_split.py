"""K1 phase split at C3 (B=4096): docp_linearize (phase A only) against
docp_assemble_schur (phases A+B+C, reference arithmetic), CUDA-event timed."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2510_06179_b200 as D
from paper_2510_06179_b200 import _lib as L

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
prob = D.affine_quadratic(8, 4, 100)
nz, nl = D.sizes(prob)
b = D.Batch(prob, B)
b.upload(L.F_THETA, D.generate_affine_quadratic(8, 4, 0, B))
b.upload(L.F_Z, np.random.default_rng(0).standard_normal((B, nz)))
def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
print(f"linearize (phase A) {t(b.linearize):.3f} ms; assemble_schur (A+B+C, parity) {t(b.assemble_schur):.3f} ms")
