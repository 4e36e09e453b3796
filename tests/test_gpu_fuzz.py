"""Randomised shape sweep of the whole forward + backward path against the
oracle (plain-C port, pinned bitwise to the reference in tests/test_oracle.py).

Covers every kernel variant the dispatcher can pick — n_x = 8 single-CTA and
cluster forms (h8f), n_x = 16 (h16f), n_x = 4, the runtime-shape kernels for
other n_x, resident and streaming records — with PARITY bit-identical and
FAST at equal iteration counts within 1e-9.
"""
import numpy as np
import pytest

import pyoracle as po

pytestmark = pytest.mark.gpu

RTOL_FAST = 1e-9

# (n_x, n_u, T): every PCG / K1 variant, including cluster sizes 2, 3, 4, 5, 6, 7, 8 for n_x = 8
SHAPES = [(1, 1, 3), (2, 1, 9), (3, 3, 17), (4, 1, 50), (4, 2, 20), (5, 2, 33), (6, 2, 64), (7, 3, 25),
          (8, 2, 100), (8, 4, 1), (8, 4, 2), (8, 4, 113), (8, 4, 114), (8, 4, 200), (8, 4, 240), (8, 4, 256), (8, 4, 320), (8, 4, 400), (8, 4, 512), (8, 4, 600), (8, 4, 700), (8, 4, 800),
          (9, 2, 40), (12, 4, 20), (16, 8, 6), (16, 8, 60)]


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(1.0, np.linalg.norm(b))


@pytest.mark.parametrize("nx,nu,T", SHAPES)
def test_fuzz_shapes(nx, nu, T):
    import paper_2510_06179_b200 as D
    seed = 1000 + 7 * nx + 3 * nu + T
    B = 3
    th = D.generate_affine_quadratic(nx, nu, seed, B)
    prob = D.affine_quadratic(nx, nu, T)
    nz, nl = D.sizes(prob)
    rng = np.random.default_rng(seed)
    z0 = rng.standard_normal((B, nz))
    lg = rng.standard_normal((B, nz))
    want = []
    for j in range(B):
        o = po.Oracle("port", po.aq_problem(nx, nu, T))
        s = o.sqp_solve(th[j], z0[j], np.zeros(nl), po.sqp_config(max_sqp_iters=4))
        g, lt, it = o.backward(th[j], lg[j], np.zeros(nl))
        want.append((s, g, lt, it))
    # PARITY runs the one-thread-per-block-row kernel, which stops at T = 511;
    # FAST n_x = 8 goes further on thread-block clusters
    modes = ("fast",) if T > 511 else ("parity", "fast")
    for mode in modes:
        cfg = D.SqpConfig(max_sqp_iters=4, pcg=D.PcgConfig(mode=mode))
        res, errs = D.sqp_solve_batch(prob, th, z0, np.zeros((B, nl)), cfg)
        assert all(e is None for e in errs), (mode, errs)
        grads, lts, its, errs = D.backward_vjp_batch(res[0].batch, lg, np.zeros((B, nl)), cfg.pcg)
        assert all(e is None for e in errs), (mode, errs)
        for j, (s, g, lt, it) in enumerate(want):
            assert res[j].sqp_iters == s.sqp_iters and res[j].pcg_iters == s.pcg_iters and its[j] == it, \
                (mode, j, res[j].pcg_iters, s.pcg_iters, its[j], it, D.describe(prob))
            if mode == "parity":
                assert np.array_equal(res[j].z, s.z) and np.array_equal(grads[j], g) and np.array_equal(lts[j], lt)
            else:
                for got, w in ((res[j].z, s.z), (res[j].lam, s.lam), (grads[j], g), (lts[j], lt)):
                    assert rel(got, w) <= RTOL_FAST, (mode, j, rel(got, w), D.describe(prob))
