#!/usr/bin/env python3
"""Generates tests/golden/*.npz from the REFERENCE itself (oracle/_ref, the
unmodified reference headers compiled against eigen_lite).

TEST INFRASTRUCTURE. Run here (where /root/reference exists):
    make -C oracle ref && python oracle/gen_golden.py
The fixtures travel with the repo so GPU-box tests never need /root/reference.

Inputs come from the reference's own generators (bench/generators.hpp), outputs
from sqp_solve / backward_vjp / train_il (sqp.hpp, backward.hpp, train.hpp).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import pyoracle as po  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")


def aq_case(nx, nu, T, seed, B, max_sqp_iters=20):
    th = po.gen_aq(nx, nu, T, seed, B)
    prob = po.aq_problem(nx, nu, T)
    nz, nl = po.sizes(prob)
    rng = np.random.default_rng(seed)
    z0 = rng.standard_normal((B, nz))
    lg = rng.standard_normal((B, nz))
    cfg = po.sqp_config(max_sqp_iters=max_sqp_iters)
    out = {k: [] for k in ("z", "lam", "sqp_iters", "pcg_iters", "kkt", "grad", "lt", "bwd_iters", "S_diag", "S_sub",
                           "P_diag", "P_super")}
    for j in range(B):
        o = po.Oracle("ref", prob)
        s = o.sqp_solve(th[j], z0[j], np.zeros(nl), cfg)
        g, lt, it = o.backward(th[j], lg[j], np.zeros(nl))
        sd, ss, pd, ps = o.schur()
        out["z"].append(s.z)
        out["lam"].append(s.lam)
        out["sqp_iters"].append(s.sqp_iters)
        out["pcg_iters"].append(s.pcg_iters + [-1] * (max_sqp_iters - len(s.pcg_iters)))
        out["kkt"].append(s.kkt)
        out["grad"].append(g)
        out["lt"].append(lt)
        out["bwd_iters"].append(it)
        out["S_diag"].append(sd)
        out["S_sub"].append(ss)
        out["P_diag"].append(pd)
        out["P_super"].append(ps)
    np.savez_compressed(os.path.join(OUT, f"aq_{nx}_{nu}_{T}_seed{seed}.npz"), theta=th, z0=z0, loss_grad=lg,
                        max_sqp_iters=max_sqp_iters, **{k: np.array(v) for k, v in out.items()})


def cartpole_case(T, seed, n_demos):
    x0, demos = po.gen_cartpole(seed, T, n_demos)
    prob = po.cartpole_problem(T)
    nz, nl = po.sizes(prob)
    w = np.array([0.3, 0.8, 0.5, 0.9])
    th = np.array([np.concatenate([w, [0.05], x]) for x in x0])
    cfg = po.sqp_config(max_sqp_iters=5)
    z, lam, its, pcg, grads, lts, bwd = [], [], [], [], [], [], []
    for j in range(n_demos):
        o = po.Oracle("ref", prob)
        s = o.sqp_solve(th[j], demos[j], np.zeros(nl), cfg)
        lg = np.zeros(nz)
        for t in range(T):
            k = t * 5 + 4
            lg[k] = 2.0 / n_demos * (s.z[k] - demos[j, k])
        g, lt, it = o.backward(th[j], lg, np.zeros(nl))
        z.append(s.z), lam.append(s.lam), its.append(s.sqp_iters), pcg.append(s.pcg_iters + [-1] * (5 - len(s.pcg_iters)))
        grads.append(g), lts.append(lt), bwd.append(it)
    np.savez_compressed(os.path.join(OUT, f"cartpole_T{T}_seed{seed}.npz"), x0=x0, demos=demos, theta=th,
                        z=np.array(z), lam=np.array(lam), sqp_iters=np.array(its), pcg_iters=np.array(pcg),
                        grad=np.array(grads), lt=np.array(lts), bwd_iters=np.array(bwd))


def train_il_case():
    """bench::train_il itself, two epochs on 8 demonstrations (train.hpp:53-145)."""
    import ctypes as C
    lib = po.load("ref")
    objectives = np.zeros(2)
    sqp_it, pcg_it = (C.c_long * 2)(), (C.c_long * 2)()
    w0 = np.array([0.2, 0.5, 0.9, 0.4])
    final = np.zeros(4)
    st = po.Status()
    rc = lib.ref_train_il_cartpole(3, 40, 8, w0.ctypes.data_as(C.POINTER(C.c_double)), 2, 1e-2,
                                   objectives.ctypes.data_as(C.POINTER(C.c_double)), sqp_it, pcg_it,
                                   final.ctypes.data_as(C.POINTER(C.c_double)), C.byref(st))
    assert rc == 0, st.message
    x0, demos = po.gen_cartpole(3, 40, 8)
    np.savez_compressed(os.path.join(OUT, "train_il_cartpole_seed3.npz"), w0=w0, objectives=objectives,
                        sqp_iters=np.array(list(sqp_it)), pcg_iters=np.array(list(pcg_it)), final_weights=final,
                        x0=x0, demos=demos, lr=1e-2)


def generators_case():
    """random_convex_instance / random_linear_instance draws (generators.hpp:52-111)."""
    np.savez_compressed(os.path.join(OUT, "generators.npz"), convex_8_4_100_seed0=po.gen_aq(8, 4, 100, 0, 16),
                        linear_8_4_40_seed0=po.gen_aq(8, 4, 40, 0, 16, convex=False))


def main():
    assert po.available("ref"), "build the reference first: make -C oracle ref"
    os.makedirs(OUT, exist_ok=True)
    aq_case(1, 1, 1, 0, 1)
    aq_case(4, 2, 20, 1, 4)
    aq_case(8, 4, 30, 2, 4)
    aq_case(8, 4, 100, 3, 2, max_sqp_iters=5)
    aq_case(16, 8, 30, 4, 2)
    cartpole_case(40, 0, 8)
    cartpole_case(50, 0, 4)
    train_il_case()
    generators_case()
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
