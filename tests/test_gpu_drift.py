"""The drifting family (DOCP_DRIFT) on the GPU against the
REFERENCE solver (sqp_solve, backward_vjp, the train_il epoch body compiled
from /root/reference in oracle/_ref) running the same model definition
(include/docp_drift_model.h). PARITY: bit for bit, equal SQP and PCG counts.
FAST: equal SQP counts, <= 1e-9 relative, PCG counts equal but for a warm
start on the exit threshold. The model itself has no reference (unpinned)."""
import numpy as np
import pytest

import pyoracle as po

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not po.available("ref"), reason="oracle/_ref not built")]

RTOL_FAST = 1e-9


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(1.0, np.linalg.norm(b))


@pytest.fixture(scope="module")
def D():
    import paper_2510_06179_b200 as D
    return D


@pytest.mark.parametrize("mode", ["parity", "fast"])
def test_drift_solve_and_backward_match_reference(D, mode):
    T, B = 30, 6
    prob, pp = D.drift(T, 0.1), po.drift_problem(T, 0.1)
    nz, nl = D.sizes(prob)
    th = D.drift_thetas(B, seed=1)
    rng = np.random.default_rng(2)
    lg = rng.standard_normal((B, nz))
    # FAST is compared over the first 4 SQP iterations (full steps): later, at
    # the merit's noise floor (KKT ~ 1e-7), the line search's "first alpha with
    # a strictly negative merit change" decides on differences of 1e-13 and
    # FAST's rounding can pick another candidate; PARITY runs to convergence.
    its_max = 10 if mode == "parity" else 4
    cfg = D.SqpConfig(max_sqp_iters=its_max, pcg=D.PcgConfig(mode=mode))
    res, errs = D.sqp_solve_batch(prob, th, np.zeros((B, nz)), np.zeros((B, nl)), cfg)
    assert all(e is None for e in errs), errs
    g, lt, its, errs = D.backward_vjp_batch(res[0].batch, lg, np.zeros((B, nl)), cfg.pcg)
    assert all(e is None for e in errs), errs
    for j in range(B):
        o = po.Oracle("ref", pp)
        s = o.sqp_solve(th[j], np.zeros(nz), np.zeros(nl), po.sqp_config(max_sqp_iters=its_max))
        gj, ltj, itj = o.backward(th[j], lg[j], np.zeros(nl))
        assert res[j].sqp_iters == s.sqp_iters, j
        if mode == "parity":
            assert list(res[j].pcg_iters) == list(s.pcg_iters) and its[j] == itj, j
            assert np.array_equal(res[j].z, s.z) and np.array_equal(res[j].lam, s.lam), j
            assert np.array_equal(g[j], gj) and np.array_equal(lt[j], ltj), j
            assert res[j].step_sizes == s.step_sizes and res[j].kkt_inf_norm == s.kkt, j
        else:
            d = [abs(a - b) for a, b in zip(res[j].pcg_iters, s.pcg_iters)] + [abs(its[j] - itj)]
            assert max(d) <= 1, (j, res[j].pcg_iters, s.pcg_iters)
            for a, b in ((res[j].z, s.z), (res[j].lam, s.lam), (g[j], gj), (lt[j], ltj)):
                assert rel(a, b) <= RTOL_FAST, j


def test_drift_il_epoch_matches_reference(D):
    """train_il epoch body (train.hpp:82-131) on the drifting family: learnable
    state-cost weights, demonstrations from the expert weights, PARITY, two
    epochs with warm caches, bit for bit."""
    import torch
    T, B = 30, 8
    prob, pp = D.drift(T, 0.1), po.drift_problem(T, 0.1)
    nz, nl = D.sizes(prob)
    th = D.drift_thetas(B, seed=3)
    demos = np.array([po.Oracle("ref", pp).sqp_solve(th[j], np.zeros(nz), np.zeros(nl), po.sqp_config()).z
                      for j in range(B)])
    w = th[0, :8] * np.random.default_rng(4).uniform(0.5, 1.5, 8)
    cfg = D.SqpConfig(max_sqp_iters=5, pcg=D.PcgConfig(mode="parity"))
    b = D.Batch(prob, B)
    b.upload(D._lib.F_THETA, th)
    dev = torch.device("cuda")
    demos_t = torch.tensor(demos, device=dev)
    out = torch.zeros(9, dtype=torch.float64, device=dev)
    lam_c, lt_c = np.zeros((B, nl)), np.zeros((B, nl))
    for epoch in range(2):
        wt = torch.tensor(w, device=dev)
        b.il_epoch(cfg, wt.data_ptr(), 0, 8, demos_t.data_ptr(), float(B), out.data_ptr(), out.data_ptr() + 8)
        b.il_check(epoch)
        th_e = th.copy()
        th_e[:, :8] = w
        loss, grad, losses, grads, sqp_it, pcg_it = po.il_epoch("ref", pp, th_e, demos, lam_c, lt_c,
                                                                 po.sqp_config(max_sqp_iters=5), 0, 8)
        o = out.cpu().numpy()
        assert o[0] == loss and np.array_equal(o[1:], grad)
        assert np.array_equal(b.download(D._lib.F_LAMBDA), lam_c)
        assert np.array_equal(b.download(D._lib.F_LAMBDA_TILDE), lt_c)
        w = w - 1e-3 * grad
