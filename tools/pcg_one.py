"""One PCG launch at C3 shape with a fixed iteration cap (for ncu)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2510_06179_b200 as D
from paper_2510_06179_b200 import _lib as L
B, T, iters = 1184, 100, int(sys.argv[1]) if len(sys.argv) > 1 else 41
prob = D.affine_quadratic(8, 4, T)
nz, nl = D.sizes(prob)
b = D.Batch(prob, B)
b.upload(L.F_THETA, D.generate_affine_quadratic(8, 4, 0, B))
b.upload(L.F_Z, np.zeros((B, nz)))
b.linearize(); b.assemble_schur(); b.assemble_gamma()
for rep in range(3):
    b.upload(L.F_LAMBDA, np.zeros((B, nl)))
    b.pcg_solve(D.PcgConfig(epsilon=1e-300, max_iters=iters, mode="fast"))
b.sync()
print("ok")
