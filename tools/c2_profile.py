import sys, os, json
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tools')
import numpy as np, torch
import paper_2510_06179_b200 as D
from paper_2510_06179_b200 import _lib as L
T, B = 50, 4096
prob = D.cartpole(T); nz, nl = D.sizes(prob)
x0 = D.generate_cartpole_x0(0, B)
EXPERT = np.array([1.0, 2.0, 1.5, 1.0])
th = np.concatenate([np.tile(EXPERT, (B, 1)), np.full((B, 1), 0.05), x0], axis=1)
z0 = np.zeros((B, nz))
for t in range(T + 1):
    o = D.flat_offset(4, 1, t, True); z0[:, o:o + 4] = x0
b = D.Batch(prob, B)
b.upload(L.F_THETA, th); b.upload(L.F_Z, z0); b.upload(L.F_LAMBDA, np.zeros((B, nl)))
b.sqp_solve(D.SqpConfig(max_sqp_iters=100, convergence_tol=1e-9))
demos = torch.tensor(b.download(L.F_Z), device="cuda")
b.upload(L.F_LAMBDA, np.zeros((B, nl))); b.upload(L.F_LAMBDA_TILDE, np.zeros((B, nl)))
w = torch.tensor(D.generate_uniform(0, 4), device="cuda"); out = torch.zeros(5, dtype=torch.float64, device="cuda")
cfg = D.SqpConfig(max_sqp_iters=5)
for _ in range(3):
    b.il_epoch(cfg, w.data_ptr(), 0, 4, demos.data_ptr(), float(B), out.data_ptr(), out.data_ptr() + 8); w.sub_(1e-2 * out[1:])
b.profile_begin()
for _ in range(10):
    b.il_epoch(cfg, w.data_ptr(), 0, 4, demos.data_ptr(), float(B), out.data_ptr(), out.data_ptr() + 8); w.sub_(1e-2 * out[1:])
p = b.profile_end()
print(json.dumps({k: round(v["ms"] / 10, 3) for k, v in p["kernels"].items()}), p["pcg_iterations"] / max(1, p["pcg_solves"]), p["gap_ms"] / 10, p["span_ms"] / 10)
