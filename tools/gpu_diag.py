"""Quick GPU diagnostic: runs each hot-path stage against the oracle port and
prints diffs (does not stop at the first mismatch)."""
import os, sys, time, traceback
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import pyoracle as po
import paper_2510_06179_b200 as D
from paper_2510_06179_b200 import _lib as L

def rel(a, b): return np.linalg.norm(a - b) / max(1.0, np.linalg.norm(b))

def stage(name, fn):
    try:
        t = time.time(); fn(); print(f"[ok] {name} ({time.time()-t:.2f}s)", flush=True)
    except Exception:
        print(f"[FAIL] {name}"); traceback.print_exc(); sys.stdout.flush()

def assembly(nx, nu, T):
    th = po.gen_aq(nx, nu, T, 3, 2) if po.available("ref") else None
    b = D.Batch(D.affine_quadratic(nx, nu, T), 2)
    z = np.random.default_rng(0).standard_normal((2, b.nz))
    b.upload(L.F_THETA, th); b.upload(L.F_Z, z); b.linearize(); b.assemble_schur(); b.assemble_gamma()
    print("  status", [ (s.code, s.where, s.index) for s in b.statuses()])
    blocks = b.download_schur(); g = b.download(L.F_GAMMA)
    o = po.Oracle("port", po.aq_problem(nx, nu, T)); o.linearize(th[0], z[0]); o.assemble(); w = o.schur()
    for k in range(4): print("  block", k, "maxdiff", np.abs(blocks[k][0] - w[k]).max())
    print("  gamma maxdiff", np.abs(g[0] - o.gamma(o.flat_b(), o.flat_d())).max())

def pcg(nx, nu, T, mode):
    th = po.gen_aq(nx, nu, T, 5, 2)
    o = po.Oracle("port", po.aq_problem(nx, nu, T)); o.linearize(th[0], np.zeros(o.nz)); o.assemble()
    gam = o.gamma(o.flat_b(), o.flat_d()); lam, it, eta, conv = o.pcg(gam, np.zeros(o.nl))
    b = D.Batch(D.affine_quadratic(nx, nu, T), 1)
    b.upload_schur(*[x[None] for x in o.schur()]); b.upload(L.F_GAMMA, gam[None]); b.upload(L.F_LAMBDA, np.zeros((1, o.nl)))
    b.pcg_solve(D.PcgConfig(mode=mode))
    print("  iters gpu", b.download(L.F_PCG_ITERS)[0,0], "oracle", it, "status", (b.statuses()[0].code, b.statuses()[0].where),
          "rel", rel(b.download(L.F_LAMBDA)[0], lam), "bitwise", np.array_equal(b.download(L.F_LAMBDA)[0], lam),
          "eta", b.download(L.F_FINAL_ETA)[0,0], eta)

def sqp(nx, nu, T, mode, B=3):
    th = po.gen_aq(nx, nu, T, 9, B); prob = D.affine_quadratic(nx, nu, T); nz, nl = D.sizes(prob)
    cfg = D.SqpConfig(max_sqp_iters=5, pcg=D.PcgConfig(mode=mode))
    res, errs = D.sqp_solve_batch(prob, th, np.zeros((B, nz)), np.zeros((B, nl)), cfg)
    lg = np.random.default_rng(1).standard_normal((B, nz))
    gr, lt, its, errs2 = D.backward_vjp_batch(res[0].batch, lg, np.zeros((B, nl)), cfg.pcg)
    for j in range(B):
        o = po.Oracle("port", po.aq_problem(nx, nu, T)); s = o.sqp_solve(th[j], np.zeros(nz), np.zeros(nl), po.sqp_config(max_sqp_iters=5))
        g, l2, it = o.backward(th[j], lg[j], np.zeros(nl))
        print(f"  [{j}] err {errs[j]} {errs2[j]} sqp {res[j].sqp_iters}/{s.sqp_iters} pcg {res[j].pcg_iters}/{s.pcg_iters} bwd {its[j]}/{it}",
              "z", rel(res[j].z, s.z), "lam", rel(res[j].lam, s.lam), "g", rel(gr[j], g), "kkt", res[j].kkt_inf_norm, s.kkt)

print(D.describe(D.affine_quadratic(8, 4, 100)))
stage("assembly 4,2,20", lambda: assembly(4, 2, 20))
stage("assembly 8,4,100", lambda: assembly(8, 4, 100))
stage("assembly 5,2,9", lambda: assembly(5, 2, 9))
for m in ("parity", "fast"):
    stage(f"pcg 8,4,100 {m}", lambda: pcg(8, 4, 100, m))
    stage(f"pcg 4,2,20 {m}", lambda: pcg(4, 2, 20, m))
    stage(f"pcg 6,3,12 {m}", lambda: pcg(6, 3, 12, m))
    stage(f"pcg 16,8,30 {m}", lambda: pcg(16, 8, 30, m))
    stage(f"sqp 8,4,100 {m}", lambda: sqp(8, 4, 100, m))
    stage(f"sqp 4,2,20 {m}", lambda: sqp(4, 2, 20, m))
print("launches", D.kernel_launches(), "pcg solves", D.pcg_invocations())
