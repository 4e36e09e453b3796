"""The drifting family's model definition (include/docp_drift_model.h) on the
host, through the reference-solver harness (oracle/_ref): Jacobians against
central differences, the nominal reference state is an equilibrium, and the
reference solver converges on the benchmark instances. No GPU needed.

The model has no reference implementation ("parity
unpinned"); these checks pin its internal consistency, the GPU tests
(test_gpu_drift.py) pin the GPU solver on it against the reference solver."""
import ctypes as C

import numpy as np
import pytest

import pyoracle as po

pytestmark = pytest.mark.skipif(not po.available("ref"), reason="oracle/_ref not built")


def step(th, xb, u, dt=0.1, jac=True):
    lib = po.load("ref")
    p = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
    xn, jx, ju = np.zeros(8), np.zeros(64), np.zeros(16)
    th, xb, u = (np.ascontiguousarray(a, dtype=np.float64) for a in (th, xb, u))
    lib.ref_drift_step(p(th), dt, p(xb), p(u), p(xn), p(jx) if jac else None, p(ju) if jac else None)
    return xn, jx.reshape(8, 8, order="F"), ju.reshape(8, 2, order="F")


@pytest.fixture(scope="module")
def D():
    import paper_2510_06179_b200 as D
    return D


def test_jacobians_match_central_differences(D):
    th = D.drift_thetas(3, seed=5)
    rng = np.random.default_rng(0)
    for j in range(3):
        xb = th[j, 10:18] + 0.05 * rng.standard_normal(8)
        u = 0.1 * rng.standard_normal(2)
        xn, jx, ju = step(th[j], xb, u)
        xn2, _, _ = step(th[j], xb, u, jac=False)
        assert np.array_equal(xn, xn2)  # the dual-number and plain paths agree bit for bit
        for k in range(8):
            h = 1e-6 * max(1.0, abs(xb[k] + th[j, 18 + k]))
            e = np.zeros(8)
            e[k] = h
            fd = (step(th[j], xb + e, u, jac=False)[0] - step(th[j], xb - e, u, jac=False)[0]) / (2 * h)
            assert np.allclose(jx[:, k], fd, rtol=1e-6, atol=1e-7), k
        for k in range(2):
            e = np.zeros(2)
            e[k] = 1e-6
            fd = (step(th[j], xb, u + e, jac=False)[0] - step(th[j], xb, u - e, jac=False)[0]) / 2e-6
            assert np.allclose(ju[:, k], fd, rtol=1e-6, atol=1e-7), k


def test_reference_state_is_a_steady_state(D):
    th = D.drift_thetas(1, seed=0, spread=0.0)[0]
    xn, _, _ = step(th, np.zeros(8), np.zeros(2))
    # all states but the path distance s (which advances by V cos(beta) dt) stay put
    assert np.abs(np.delete(xn, 5)).max() < 1e-10
    assert abs(xn[5] - 0.1 * 8.0) < 1e-10  # ds/dt = V cos(dphi + beta) / (1 - kappa e) = V


def test_reference_solver_converges_on_benchmark_instances(D):
    T, B = 30, 4
    pp = po.drift_problem(T, 0.1)
    nz, nl = po.sizes(pp)
    th = D.drift_thetas(B, seed=0)
    for j in range(B):
        s = po.Oracle("ref", pp).sqp_solve(th[j], np.zeros(nz), np.zeros(nl), po.sqp_config(max_sqp_iters=20))
        assert s.converged and s.kkt < 1e-5, (j, s.sqp_iters, s.kkt)
