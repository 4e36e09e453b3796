"""Small C3-shaped workload for ncu: one SQP solve + backward of B problems."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2510_06179_b200 as D
from paper_2510_06179_b200 import _lib as L
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1184
mode = sys.argv[2] if len(sys.argv) > 2 else "fast"
prob = D.affine_quadratic(8, 4, 100)
nz, nl = D.sizes(prob)
b = D.Batch(prob, B)
b.upload(L.F_THETA, D.generate_affine_quadratic(8, 4, 0, B))
b.upload(L.F_Z, np.zeros((B, nz)))
b.upload(L.F_LAMBDA, np.zeros((B, nl)))
cfg = D.SqpConfig(max_sqp_iters=5, pcg=D.PcgConfig(mode=mode))
b.sqp_solve(cfg)
b.upload(L.F_LOSS_GRAD_Z, np.random.default_rng(0).standard_normal((B, nz)))
b.upload(L.F_LAMBDA_TILDE, np.zeros((B, nl)))
b.backward_vjp(cfg.pcg)
b.sync()
assert all(e is None for e in b.errors())
print("ok", D.kernel_launches())
