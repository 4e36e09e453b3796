"""One PCG launch at the C2 shape (n_x = 4, n_u = 1, T = 50) with a fixed iteration cap (for ncu)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2510_06179_b200 as D
from paper_2510_06179_b200 import _lib as L
B, T = 4096, 50
prob = D.affine_quadratic(4, 1, T)
nz, nl = D.sizes(prob)
b = D.Batch(prob, B)
b.upload(L.F_THETA, D.generate_affine_quadratic(4, 1, 0, B))
b.upload(L.F_Z, np.zeros((B, nz)))
b.linearize(); b.assemble_schur(); b.assemble_gamma()
for rep in range(3):
    b.upload(L.F_LAMBDA, np.zeros((B, nl)))
    b.pcg_solve(D.PcgConfig(epsilon=1e-300, max_iters=41, mode="fast"))
b.sync()
print("ok")
