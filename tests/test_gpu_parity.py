"""GPU parity tests: the CUDA path (through the C ABI) against the oracle.

The checker is the plain-C restatement (oracle/port), itself pinned
bit-for-bit to the reference headers (tests/test_oracle_port.py). Bars:
  * PARITY PCG mode: bit-identical z, lambda, lambda~, dtheta and equal
    iteration counts (cart-pole: <= 1e-12 relative, device sin/cos differ from
    glibc's by <= 2 ulp);
  * FAST mode (FMA + tree reductions): equal PCG / SQP iteration counts and
    <= 1e-9 relative error (north_star's fp64 bar).
"""
import numpy as np
import pytest

import pyoracle as po

pytestmark = pytest.mark.gpu

RTOL_FAST = 1e-9


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(1.0, np.linalg.norm(b))


@pytest.fixture(scope="module")
def D():
    import paper_2510_06179_b200 as D
    return D


def aq_thetas(nx, nu, T, seed, count):
    """random_convex_instance draws (generators.hpp:102-111) via the reference
    when available, else the golden fixture set."""
    if po.available("ref"):
        return po.gen_aq(nx, nu, T, seed, count)
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        A = np.eye(nx) + 0.1 * rng.standard_normal((nx, nx))
        rho = max(abs(np.linalg.eigvals(A)))
        if rho > 0.99:
            A *= 0.99 / rho
        out.append(np.concatenate([rng.uniform(0.5, 2, nx), rng.uniform(0.5, 2, nu), A.T.ravel(),
                                   rng.standard_normal((nu, nx)).ravel(), 1e-2 * rng.standard_normal(nx),
                                   rng.standard_normal(nx)]))
    return np.array(out)


def port_problem(p):
    if p.family == 2:
        return po.cartpole_problem(p.horizon, p.cart_mass, p.pole_mass, p.length, p.gravity, p.dt)
    return po.aq_problem(p.n_x, p.n_u, p.horizon, p.cost_scale)


# ----------------------------------------------------------------- PCG KATs (test_pcg.cpp)


def test_pcg_scalar_kat(D):
    """test_pcg.cpp:46-61: gamma_stored = (-1, 0), lambda = (-1.5, -0.5), <= 2 iterations."""
    prob = D.affine_quadratic(1, 1, 1, cost_scale=0.5)
    theta = np.array([1.0, 1.0, 1.0, 1.0, 0.0, 1.0])
    b = D.Batch(prob, 1)
    b.upload(D._lib.F_THETA, theta)
    b.upload(D._lib.F_Z, np.zeros(3))
    b.linearize()
    b.assemble_schur()
    b.assemble_gamma()
    g = b.download(D._lib.F_GAMMA)[0]
    assert g[0] == pytest.approx(-1.0) and abs(g[1]) <= 1e-15
    for mode in ("fast", "parity"):
        b.upload(D._lib.F_LAMBDA, np.zeros(2))
        b.pcg_solve(D.PcgConfig(mode=mode))
        lam = b.download(D._lib.F_LAMBDA)[0]
        assert b.download(D._lib.F_PCG_ITERS)[0, 0] <= 2
        assert b.download(D._lib.F_PCG_CONVERGED)[0, 0] == 1
        assert lam == pytest.approx([-1.5, -0.5])
    sd, ss, pd, ps = b.download_schur()
    assert sd[0, :, 0, 0] == pytest.approx([1.0, 3.0]) and ss[0, 0, 0, 0] == pytest.approx(-1.0)
    assert pd[0, :, 0, 0] == pytest.approx([1.0, 1.0 / 3.0]) and ps[0, 0, 0, 0] == pytest.approx(1.0 / 3.0)


@pytest.mark.parametrize("nx,T", [(3, 5), (4, 6), (8, 4)])
def test_pcg_identity_system_one_iteration(D, nx, T):
    """test_pcg.cpp:32-44: a decoupled instance gives -S = Phi^-1 = I."""
    prob = D.affine_quadratic(nx, nx, T, cost_scale=0.5)
    theta = np.concatenate([np.ones(2 * nx), np.zeros(2 * nx * nx + 2 * nx)])
    b = D.Batch(prob, 2)
    b.upload(D._lib.F_THETA, np.tile(theta, (2, 1)))
    b.upload(D._lib.F_Z, np.zeros((2, b.nz)))
    b.linearize()
    b.assemble_schur()
    rng = np.random.default_rng(1)
    gamma = rng.standard_normal((2, b.nl))
    b.upload(D._lib.F_GAMMA, gamma)
    for mode in ("fast", "parity"):
        b.upload(D._lib.F_LAMBDA, np.zeros((2, b.nl)))
        b.pcg_solve(D.PcgConfig(mode=mode))
        assert (b.download(D._lib.F_PCG_ITERS)[:, 0] == 1).all()
        assert np.abs(b.download(D._lib.F_LAMBDA) - gamma).max() < 1e-12


def test_pcg_breakdown_and_cap(D):
    """test_pcg.cpp:162-190: indefinite system -> BreakdownError(iteration 0);
    max_iters = 2 -> 2 iterations, unconverged."""
    prob = D.affine_quadratic(2, 2, 3, cost_scale=0.5)
    b = D.Batch(prob, 1)
    nb = 4
    eye = np.tile(np.eye(2), (1, nb, 1, 1))
    zero = np.zeros((1, nb - 1, 2, 2))
    b.upload_schur(-eye, zero, eye, zero)
    b.upload(D._lib.F_GAMMA, np.ones((1, b.nl)))
    b.upload(D._lib.F_LAMBDA, np.zeros((1, b.nl)))
    b.pcg_solve(D.PcgConfig())
    err = b.errors()[0]
    assert isinstance(err, D.BreakdownError) and err.iteration == 0

    th = aq_thetas(8, 4, 30, 7, 1)
    p2 = D.affine_quadratic(8, 4, 30)
    b2 = D.Batch(p2, 1)
    b2.upload(D._lib.F_THETA, th)
    b2.upload(D._lib.F_Z, np.zeros((1, b2.nz)))
    b2.linearize()
    b2.assemble_schur()
    b2.upload(D._lib.F_GAMMA, np.random.default_rng(7).standard_normal((1, b2.nl)))
    b2.upload(D._lib.F_LAMBDA, np.zeros((1, b2.nl)))
    b2.pcg_solve(D.PcgConfig(epsilon=1e-14, max_iters=2))
    assert b2.download(D._lib.F_PCG_ITERS)[0, 0] == 2
    assert b2.download(D._lib.F_PCG_CONVERGED)[0, 0] == 0


@pytest.mark.parametrize("nx,nu,T,seed", [(4, 2, 10, 1), (8, 4, 30, 2), (8, 4, 100, 3), (6, 3, 12, 4),
                                          (16, 8, 30, 5), (9, 2, 40, 6), (8, 4, 4, 7),
                                          # long horizons: FAST runs on a 2-, 3-, 4- and 6-CTA cluster
                                          (8, 4, 128, 8), (8, 4, 256, 9), (8, 4, 500, 10), (8, 4, 700, 11)])
def test_pcg_on_oracle_blocks(D, nx, nu, T, seed):
    """K2 alone: blocks and gamma assembled by the oracle; PARITY is
    bit-identical to the oracle's pcg_solve, FAST within 1e-9 with equal
    iteration counts."""
    th = aq_thetas(nx, nu, T, seed, 3)
    pp = po.aq_problem(nx, nu, T)
    o = po.Oracle("port", pp)
    blocks, gammas, want = [], [], []
    for j in range(3):
        o.linearize(th[j], np.zeros(o.nz))
        o.assemble()
        g = o.gamma(o.flat_b(), o.flat_d())
        blocks.append(o.schur())
        gammas.append(g)
        want.append(o.pcg(g, np.zeros(o.nl)))
    b = D.Batch(D.affine_quadratic(nx, nu, T), 3)
    b.upload_schur(*[np.stack([bl[k] for bl in blocks]) for k in range(4)])
    b.upload(D._lib.F_GAMMA, np.stack(gammas))
    # PARITY on uploaded blocks runs one thread per block row, up to T = 511
    for mode in ("parity", "fast") if T <= 511 else ("fast",):
        b.upload(D._lib.F_LAMBDA, np.zeros((3, b.nl)))
        b.pcg_solve(D.PcgConfig(mode=mode))
        lam = b.download(D._lib.F_LAMBDA)
        its = b.download(D._lib.F_PCG_ITERS)[:, 0]
        for j in range(3):
            assert its[j] == want[j][1], (mode, j, its[j], want[j][1])
            if mode == "parity":
                assert np.array_equal(lam[j], want[j][0])
            else:
                assert rel(lam[j], want[j][0]) <= RTOL_FAST


# ----------------------------------------------------------------- K1 assembly


@pytest.mark.parametrize("nx,nu,T,seed", [(1, 1, 1, 0), (4, 2, 20, 1), (8, 4, 100, 2), (5, 2, 9, 3),
                                          (16, 8, 30, 4)])
def test_assembly_bitwise(D, nx, nu, T, seed):
    """linearize + assemble_schur + assemble_gamma at a random z are
    bit-identical to the oracle (diagonal Hessians specialised exactly)."""
    th = aq_thetas(nx, nu, T, seed, 2)
    rng = np.random.default_rng(seed)
    prob = D.affine_quadratic(nx, nu, T)
    b = D.Batch(prob, 2)
    z = rng.standard_normal((2, b.nz))
    b.upload(D._lib.F_THETA, th)
    b.upload(D._lib.F_Z, z)
    b.linearize()
    b.assemble_schur()
    b.assemble_gamma()
    blocks = b.download_schur()
    qp = b.download_qp()
    gam = b.download(D._lib.F_GAMMA)
    for j in range(2):
        o = po.Oracle("port", po.aq_problem(nx, nu, T))
        o.linearize(th[j], z[j])
        o.assemble()
        want = o.schur()
        for k in range(4):
            assert np.array_equal(blocks[k][j], want[k]), k
        oq = o.qp()
        for k in ("Q", "q", "R", "r", "A", "B", "C", "x_s"):
            assert np.array_equal(qp[k][j], oq[k]), k
        assert np.array_equal(gam[j], o.gamma(o.flat_b(), o.flat_d()))


@pytest.mark.parametrize("nx,nu,T", [(8, 4, 20), (4, 2, 12), (4, 1, 9), (5, 2, 9)])
def test_linearize_errors_and_projection(D, nx, nu, T):
    """K1 phase A (per-entry for compile-time affine-quadratic shapes, per-stage
    otherwise): the first failing stage in the reference's order, the
    project_pd clamps and the QpData, against the oracle."""
    B = 8
    th = aq_thetas(nx, nu, T, 5, B)
    rng = np.random.default_rng(9)
    prob = D.affine_quadratic(nx, nu, T)
    b = D.Batch(prob, B)
    z = rng.standard_normal((B, b.nz))
    sz = nx + nu
    th[1, 2 % nx] = 1e-9                     # Q below eps_pd: projected (problem.hpp:157-181)
    th[2, nx] = -1.0                         # R indefinite: projected
    z[3, 7 % T * sz + 1 % nx] = 1e200        # state cost overflows at stage 7 % T
    z[4, 3 % T * sz + nx] = np.inf           # control (and dynamics) at stage 3 % T
    th[5, nx + nu + 1] = np.nan              # A: dynamics non-finite from stage 0
    z[6, T * sz] = np.nan                    # terminal state
    th[7, -1] = np.nan                       # x_s
    b.upload(D._lib.F_THETA, th)
    b.upload(D._lib.F_Z, z)
    b.linearize()
    errs = b.errors()
    qp = b.download_qp()
    for j in range(B):
        o = po.Oracle("port", po.aq_problem(nx, nu, T))
        try:
            o.linearize(th[j], z[j])
        except po.OracleError as e:
            assert errs[j] is not None and str(errs[j]) == e.message, (j, errs[j], e.message)
            continue
        assert errs[j] is None, (j, errs[j])
        oq = o.qp()
        for k in ("Q", "q", "R", "r", "A", "B", "C", "x_s"):
            assert np.array_equal(qp[k][j], oq[k]), (j, k)
    assert [e is None for e in errs] == [True, True, True, False, False, False, False, False]


def test_assembly_cartpole(D):
    x0, demos = _cartpole_demos(4)
    prob = D.cartpole(40)
    b = D.Batch(prob, 4)
    th = np.array([np.concatenate([[1, 2, 1.5, 1], [0.05], x]) for x in x0])
    z = demos * 0.97
    b.upload(D._lib.F_THETA, th)
    b.upload(D._lib.F_Z, z)
    b.linearize()
    b.assemble_schur()
    blocks = b.download_schur()
    for j in range(4):
        o = po.Oracle("port", po.cartpole_problem(40))
        o.linearize(th[j], z[j])
        o.assemble()
        want = o.schur()
        for k in range(4):
            assert rel(blocks[k][j], want[k]) <= 1e-12


# ----------------------------------------------------------------- full SQP + backward


def _cartpole_demos(n, T=40, seed=0):
    if po.available("ref"):
        return po.gen_cartpole(seed, T, n)
    import json, os
    path = os.path.join(os.path.dirname(__file__), "golden", f"cartpole_T{T}_seed{seed}.npz")
    g = np.load(path)
    return g["x0"][:n], g["demos"][:n]


def _oracle_solve_and_grad(pprob, th, z0, lam0, cfg_port, lg, lt0):
    o = po.Oracle("port", pprob)
    s = o.sqp_solve(th, z0, lam0, cfg_port)
    g, lt, it = o.backward(th, lg, lt0)
    return s, g, lt, it


@pytest.mark.parametrize("mode", ["parity", "fast"])
@pytest.mark.parametrize("nx,nu,T,seed,max_it", [(4, 2, 20, 11, 20), (8, 4, 30, 12, 20), (8, 4, 100, 13, 5),
                                                 (8, 4, 127, 16, 5), (3, 2, 4, 14, 20), (16, 8, 30, 15, 20),
                                                 (9, 2, 100, 17, 5)])
def test_sqp_backward_affine_quadratic(D, mode, nx, nu, T, seed, max_it):
    B = 4
    th = aq_thetas(nx, nu, T, seed, B)
    prob = D.affine_quadratic(nx, nu, T)
    rng = np.random.default_rng(seed)
    nz, nl = D.sizes(prob)
    z0 = rng.standard_normal((B, nz))
    lg = rng.standard_normal((B, nz))
    cfg = D.SqpConfig(max_sqp_iters=max_it, pcg=D.PcgConfig(mode=mode))
    res, errs = D.sqp_solve_batch(prob, th, z0, np.zeros((B, nl)), cfg)
    assert all(e is None for e in errs)
    b = res[0].batch
    grads, lts, its, errs = D.backward_vjp_batch(b, lg, np.zeros((B, nl)), cfg.pcg)
    assert all(e is None for e in errs)
    for j in range(B):
        s, g, lt, it = _oracle_solve_and_grad(po.aq_problem(nx, nu, T), th[j], z0[j], np.zeros(nl),
                                              po.sqp_config(max_sqp_iters=max_it), lg[j], np.zeros(nl))
        assert res[j].sqp_iters == s.sqp_iters and res[j].pcg_iters == s.pcg_iters and its[j] == it
        assert res[j].converged == s.converged
        if mode == "parity":
            assert np.array_equal(res[j].z, s.z) and np.array_equal(res[j].lam, s.lam)
            assert np.array_equal(grads[j], g) and np.array_equal(lts[j], lt)
            assert res[j].kkt_inf_norm == s.kkt and res[j].step_sizes == s.step_sizes
        else:
            for got, want in ((res[j].z, s.z), (res[j].lam, s.lam), (grads[j], g), (lts[j], lt)):
                assert rel(got, want) <= RTOL_FAST


@pytest.mark.parametrize("mode", ["parity", "fast"])
def test_sqp_backward_cartpole(D, mode):
    B, T = 6, 40
    x0, demos = _cartpole_demos(B, T)
    prob = D.cartpole(T)
    nz, nl = D.sizes(prob)
    w = np.array([0.3, 0.8, 0.5, 0.9])
    th = np.array([np.concatenate([w, [0.05], x]) for x in x0])
    cfg = D.SqpConfig(max_sqp_iters=5, pcg=D.PcgConfig(mode=mode))
    res, errs = D.sqp_solve_batch(prob, th, demos, np.zeros((B, nl)), cfg)
    assert all(e is None for e in errs)
    lg = np.zeros((B, nz))
    for j in range(B):
        for t in range(T):
            k = D.flat_offset(4, 1, t, False)
            lg[j, k] = 2.0 / B * (res[j].z[k] - demos[j, k])
    grads, lts, its, errs = D.backward_vjp_batch(res[0].batch, lg, np.zeros((B, nl)), cfg.pcg)
    for j in range(B):
        s, g, lt, it = _oracle_solve_and_grad(po.cartpole_problem(T), th[j], demos[j], np.zeros(nl),
                                              po.sqp_config(max_sqp_iters=5), lg[j], np.zeros(nl))
        assert res[j].sqp_iters == s.sqp_iters and res[j].pcg_iters == s.pcg_iters and its[j] == it
        errs_j = [rel(got, want) for got, want in ((res[j].z, s.z), (res[j].lam, s.lam), (grads[j], g), (lts[j], lt))]
        print(f"cartpole[{mode}] {j}: steps gpu {res[j].step_sizes} oracle {s.step_sizes} kkt {s.kkt:.2e} "
              f"rel z/lam/grad/lt {['%.1e' % e for e in errs_j]}")
        assert max(errs_j) <= RTOL_FAST


@pytest.mark.parametrize("mode", ["parity", "fast"])
def test_il_epoch_matches_oracle(D, mode):
    """One train_il epoch body (C3 shape, scaled down): per-instance solve from
    the demonstration, MSE loss, warm-started backward, fixed-order sums
    (PARITY: bit for bit; FAST, whose sums are a tree: <= 1e-9)."""
    import torch
    nx, nu, T, B = 8, 4, 30, 16
    th = aq_thetas(nx, nu, T, 21, B)
    prob = D.affine_quadratic(nx, nu, T)
    nz, nl = D.sizes(prob)
    expert = np.array([1, 2, 1.5, 1, 1, 2, 1.5, 1.0])
    th[:, :nx] = expert
    pp = po.aq_problem(nx, nu, T)
    demos = np.array([po.Oracle("port", pp).sqp_solve(th[j], np.zeros(nz), np.zeros(nl), po.sqp_config()).z
                      for j in range(B)])
    w = np.random.default_rng(0).uniform(0, 1, nx)
    cfg = D.SqpConfig(max_sqp_iters=5, pcg=D.PcgConfig(mode=mode))
    b = D.Batch(prob, B)
    b.upload(D._lib.F_THETA, th)
    dev = torch.device("cuda")
    wt = torch.tensor(w, device=dev)
    demos_t = torch.tensor(demos, device=dev)
    loss_t = torch.zeros(1, dtype=torch.float64, device=dev)
    grad_t = torch.zeros(nx, dtype=torch.float64, device=dev)
    lam_c, lt_c = np.zeros((B, nl)), np.zeros((B, nl))
    for epoch in range(2):
        b.il_epoch(cfg, wt.data_ptr(), 0, nx, demos_t.data_ptr(), float(B), loss_t.data_ptr(), grad_t.data_ptr())
        b.sync()
        th_e = th.copy()
        th_e[:, :nx] = w
        loss, grad, *_ = po.il_epoch("port", pp, th_e, demos, lam_c, lt_c, po.sqp_config(max_sqp_iters=5), 0, nx)
        if mode == "parity":
            assert loss_t.item() == loss
            assert np.array_equal(grad_t.cpu().numpy(), grad)
            assert np.array_equal(b.download(D._lib.F_LAMBDA), lam_c)
            assert np.array_equal(b.download(D._lib.F_LAMBDA_TILDE), lt_c)
        else:
            assert abs(loss_t.item() - loss) <= RTOL_FAST * max(1.0, abs(loss))
            assert rel(grad_t.cpu().numpy(), grad) <= RTOL_FAST
            assert rel(b.download(D._lib.F_LAMBDA), lam_c) <= RTOL_FAST
            assert rel(b.download(D._lib.F_LAMBDA_TILDE), lt_c) <= RTOL_FAST
        w = w - 1e-2 * grad
        wt = torch.tensor(w, device=dev)


@pytest.mark.parametrize("mode", ["parity", "fast"])
def test_il_epoch_c3_shape_matches_reference(D, mode):
    """The benched function at the benched shape: docp_il_epoch at C3
    (random_convex_instance(8,4,100), shared expert w*, max 5 SQP iterations,
    eps 1e-12) over the first 256 problems of bench.py's batch, two epochs with
    warm caches, against the reference build's train_il epoch body
    (oracle/_ref, train.hpp:82-131) on the same inputs. PARITY: every field
    bit for bit and equal per-instance SQP and PCG counts. FAST: equal SQP
    counts, PCG counts equal except at a warm start on the exit threshold
    (one iteration apart), <= 1e-9 relative."""
    import torch
    if not po.available("ref"):
        pytest.skip("oracle/_ref not built")
    nx, nu, T, B = 8, 4, 100, 256
    th = D.generate_affine_quadratic(nx, nu, 0, B)
    assert np.array_equal(th, po.gen_aq(nx, nu, T, 0, B))
    prob = D.affine_quadratic(nx, nu, T)
    nz, nl = D.sizes(prob)
    pp = po.aq_problem(nx, nu, T)
    expert = th.copy()
    expert[:, :nx] = np.array([1, 2, 1.5, 1, 1, 2, 1.5, 1.0])
    demos = np.array([po.Oracle("ref", pp).sqp_solve(expert[j], np.zeros(nz), np.zeros(nl), po.sqp_config()).z
                      for j in range(B)])
    w = po.gen_uniform(0, nx)
    cfg = D.SqpConfig(max_sqp_iters=5, pcg=D.PcgConfig(epsilon=1e-12, mode=mode))
    b = D.Batch(prob, B)
    b.upload(D._lib.F_THETA, th)
    b.upload(D._lib.F_LAMBDA, np.zeros((B, nl)))
    b.upload(D._lib.F_LAMBDA_TILDE, np.zeros((B, nl)))
    dev = torch.device("cuda")
    demos_t = torch.tensor(demos, device=dev)
    out_t = torch.zeros(1 + nx, dtype=torch.float64, device=dev)
    lam_c, lt_c = np.zeros((B, nl)), np.zeros((B, nl))
    count_diffs = 0
    for epoch in range(2):
        wt = torch.tensor(w, device=dev)
        b.il_epoch(cfg, wt.data_ptr(), 0, nx, demos_t.data_ptr(), float(B), out_t.data_ptr(),
                   out_t.data_ptr() + 8)
        b.il_check(epoch)
        th_e = th.copy()
        th_e[:, :nx] = w
        loss, grad, losses, grads, sqp_it, pcg_it = po.il_epoch("ref", pp, th_e, demos, lam_c, lt_c,
                                                                 po.sqp_config(max_sqp_iters=5), 0, nx)
        g_sqp = b.download(D._lib.F_SQP_ITERS).ravel()
        hist = b.download(D._lib.F_PCG_HISTORY)
        g_pcg = np.array([hist[j, :g_sqp[j]].sum() for j in range(B)]) + b.download(D._lib.F_PCG_ITERS).ravel()
        out = out_t.cpu().numpy()
        assert np.array_equal(g_sqp, sqp_it), "SQP iteration counts"
        if mode == "parity":
            assert np.array_equal(g_pcg, pcg_it), "PCG iteration counts"
            assert out[0] == loss and np.array_equal(out[1:], grad)
            assert np.array_equal(b.download(D._lib.F_LOSS).ravel(), losses)
            assert np.array_equal(b.download(D._lib.F_LAMBDA), lam_c)
            assert np.array_equal(b.download(D._lib.F_LAMBDA_TILDE), lt_c)
        else:
            d = np.abs(g_pcg - pcg_it)
            count_diffs += int(np.sum(d != 0))
            assert d.max() <= 1
            assert abs(out[0] - loss) <= RTOL_FAST * max(1.0, abs(loss))
            assert rel(out[1:], grad) <= RTOL_FAST
            assert rel(b.download(D._lib.F_LAMBDA), lam_c) <= RTOL_FAST
            assert rel(b.download(D._lib.F_LAMBDA_TILDE), lt_c) <= RTOL_FAST
        w = w - 1e-2 * grad
    print(f"{mode}: instances whose PCG total differs from the reference by one: {count_diffs} of {2 * B}")
    assert count_diffs <= 2


def test_il_epoch_failed_demonstration_is_reported(D):
    """A demonstration whose solve throws fails the epoch as train_il does
    (train.hpp:111-119): it contributes nothing to the sums, is counted on the
    device, and il_check raises "epoch E, demonstration J: <reference message>"."""
    import torch
    nx, nu, T, B = 4, 2, 10, 4
    prob = D.affine_quadratic(nx, nu, T)
    nz, nl = D.sizes(prob)
    th = D.generate_affine_quadratic(nx, nu, 0, B)
    th[2, nx + nu] = np.nan  # A(0, 0) of instance 2: non-finite dynamics at stage 0
    cfg = D.SqpConfig(max_sqp_iters=3, pcg=D.PcgConfig(mode="parity"))
    b = D.Batch(prob, B)
    b.upload(D._lib.F_THETA, th)
    dev = torch.device("cuda")
    demos = torch.zeros((B, nz), dtype=torch.float64, device=dev)
    w = torch.full((nx,), 0.5, dtype=torch.float64, device=dev)
    out = torch.zeros(1 + nx, dtype=torch.float64, device=dev)
    b.il_epoch(cfg, w.data_ptr(), 0, nx, demos.data_ptr(), float(B), out.data_ptr(), out.data_ptr() + 8)
    with pytest.raises(D.EvaluationError, match=r"^epoch 3, demonstration 2: .*non-finite"):
        b.il_check(3)
    assert np.isfinite(out.cpu().numpy()).all()
    losses = b.download(D._lib.F_LOSS).ravel()
    assert out[0].item() == ((0.0 + losses[0]) + losses[1]) + losses[3]
    assert b.il_failures() == (0, -1)  # reset by the check


@pytest.mark.parametrize("nx,nu,T", [(4, 2, 10), (8, 4, 30)])
def test_error_statuses(D, nx, nu, T):
    """Per-problem failures become the reference's errors; the rest of the
    batch is unaffected (batch.hpp:92-101). The PCG kernels skip the failed
    problems of their work list (n_x = 8: pcg_kernel_h8s's skip path)."""
    B = 7
    th = aq_thetas(nx, nu, T, 31, B)
    for j in (1, 3, 4):
        th[j, -nx] = np.nan  # non-finite x_s (test_batch.cpp:88-105)
    prob = D.affine_quadratic(nx, nu, T)
    nz, nl = D.sizes(prob)
    res, errs = D.sqp_solve_batch(prob, th, np.zeros((B, nz)), np.zeros((B, nl)),
                                  D.SqpConfig(pcg=D.PcgConfig(mode="fast")))
    for j in range(B):
        if j in (1, 3, 4):
            assert isinstance(errs[j], D.EvaluationError) and "initial_state" in str(errs[j])
            continue
        assert errs[j] is None
        o = po.Oracle("port", po.aq_problem(nx, nu, T))
        s = o.sqp_solve(th[j], np.zeros(nz), np.zeros(nl), po.sqp_config())
        assert res[j].pcg_iters == s.pcg_iters and rel(res[j].z, s.z) <= RTOL_FAST
    with pytest.raises(D.DimensionError):
        D.sqp_solve(prob, th[0], np.full(nz, np.inf), np.zeros(nl))
    with pytest.raises(D.DimensionError):
        D.sqp_solve(prob, th[0], np.zeros(nz), np.zeros(nl), D.SqpConfig(step_candidates=(1.0, 1.0)))


# ----------------------------------------------------------------- rollouts


@pytest.mark.skipif(not po.available("ref"), reason="needs the reference build (oracle/_ref)")
@pytest.mark.parametrize("mode", ["parity", "fast"])
@pytest.mark.parametrize("one_step", [True, False])
def test_rollout_affine_matches_reference(D, mode, one_step):
    """rollout + rollout_backward (batch.hpp:172-258) with the affine
    environment (train.hpp:195-213) against the reference's own functions:
    total rewards and d(reward)/dtheta bit-identical in PARITY, 1e-9 in FAST;
    a NaN-weighted instance is truncated with the reference's message."""
    import torch
    nx, nu, T, B, H = 4, 2, 20, 6, 5
    th = po.gen_aq(nx, nu, T, 5, B, convex=False)   # random_linear_instance (make_linear_rl_task)
    th[4, 0] = np.nan                                 # solve fails at step 0
    x0 = th[:, -nx:].copy()                           # x_inits = inst.x_s
    if one_step:  # the benchmark's real-time mode (train.hpp:226-230)
        ocfg = po.sqp_config(max_sqp_iters=1, alphas=(1.0,))
        gcfg = D.SqpConfig(max_sqp_iters=1, step_candidates=[1.0], pcg=D.PcgConfig(mode=mode))
    else:
        ocfg = po.sqp_config()
        gcfg = D.SqpConfig(pcg=D.PcgConfig(mode=mode))
    want_r, want_g, ok, msgs = po.rollout_affine(nx, nu, T, th, x0, H, ocfg)
    assert not ok[4] and ok.sum() == B - 1
    b = D.Batch(D.affine_quadratic(nx, nu, T), B)
    b.upload(D._lib.F_THETA, th)
    xi = torch.tensor(x0, device="cuda")
    # one_step: on a side stream, so the rollout and its backward run as captured CUDA graphs
    # (second call replays them); otherwise eagerly on the default stream
    side = torch.cuda.Stream() if one_step else None
    if side is not None:
        b.set_stream(side.cuda_stream)
    for rep in range(2 if one_step else 1):
        b.rollout(gcfg, xi.data_ptr() if one_step else x0, H)  # device and host x_init paths
        b.rollout_backward(gcfg.pcg)
    b.sync()
    got_r = b.download(D._lib.F_REWARD)[:, 0]
    got_g = b.download(D._lib.F_GRAD_THETA)
    errs = b.rollout_errors()
    for j in range(B):
        if not ok[j]:
            assert isinstance(errs[j], D.RolloutTruncation) and str(errs[j]) == msgs[j], (str(errs[j]), msgs[j])
            continue
        assert errs[j] is None
        if mode == "parity":
            assert got_r[j] == want_r[j], (j, got_r[j], want_r[j])
            assert np.array_equal(got_g[j], want_g[j]), (j, np.abs(got_g[j] - want_g[j]).max())
        else:
            assert abs(got_r[j] - want_r[j]) <= RTOL_FAST * max(1.0, abs(want_r[j]))
            assert rel(got_g[j], want_g[j]) <= RTOL_FAST


# ----------------------------------------------------------------- attitude family


def _attitude_set(B, seed):
    rng = np.random.default_rng(seed)
    inertia = rng.uniform(0.5, 2.0, (B, 3))
    w0 = rng.uniform(-1.0, 1.0, (B, 3))
    th9 = np.concatenate([np.ones((B, 3)), np.ones((B, 3)), w0], axis=1)  # make_attitude_theta, Q = R = I
    return th9, inertia


@pytest.mark.skipif(not po.available("ref"), reason="needs the reference build (oracle/_ref)")
@pytest.mark.parametrize("mode", ["parity", "fast"])
def test_sqp_backward_attitude(D, mode):
    """Attitude-rate family (attitude.hpp) against the reference: SQP from
    z = 0 (4 iterations, make_attitude_rl_task) and the backward pass."""
    B, T = 5, 25
    th9, inertia = _attitude_set(B, 3)
    prob = D.attitude(T, 0.1)
    nz, nl = D.sizes(prob)
    th = np.concatenate([th9, inertia], axis=1)
    cfg = D.SqpConfig(max_sqp_iters=4, pcg=D.PcgConfig(mode=mode))
    res, errs = D.sqp_solve_batch(prob, th, np.zeros((B, nz)), np.zeros((B, nl)), cfg)
    assert all(e is None for e in errs)
    lg = np.random.default_rng(4).standard_normal((B, nz))
    grads, lts, its, errs = D.backward_vjp_batch(res[0].batch, lg, np.zeros((B, nl)), cfg.pcg)
    assert all(e is None for e in errs)
    for j in range(B):
        o = po.Oracle("ref", po.attitude_problem(T, inertia[j], 0.1))
        s = o.sqp_solve(th9[j], np.zeros(nz), np.zeros(nl), po.sqp_config(max_sqp_iters=4))
        g, lt, it = o.backward(th9[j], lg[j], np.zeros(nl))
        assert res[j].sqp_iters == s.sqp_iters and res[j].pcg_iters == s.pcg_iters and its[j] == it
        assert np.all(grads[j][9:] == 0.0)
        if mode == "parity":
            assert np.array_equal(res[j].z, s.z) and np.array_equal(res[j].lam, s.lam)
            assert np.array_equal(grads[j][:9], g) and np.array_equal(lts[j], lt)
            assert res[j].kkt_inf_norm == s.kkt and res[j].step_sizes == s.step_sizes
        else:
            for got, want in ((res[j].z, s.z), (res[j].lam, s.lam), (grads[j][:9], g), (lts[j], lt)):
                assert rel(got, want) <= RTOL_FAST


@pytest.mark.skipif(not po.available("ref"), reason="needs the reference build (oracle/_ref)")
@pytest.mark.parametrize("mode", ["parity", "fast"])
def test_rollout_attitude_matches_reference(D, mode):
    """rollout + rollout_backward with the attitude RL environment
    (make_attitude_rl_task, train.hpp:239-263) against the reference."""
    B, T, H = 5, 25, 4
    th9, inertia = _attitude_set(B, 8)
    x0 = th9[:, 6:9].copy()
    want_r, want_g, ok, msgs = po.rollout_attitude(T, 0.1, th9, inertia, x0, H, po.sqp_config(max_sqp_iters=4))
    assert ok.all(), msgs
    b = D.Batch(D.attitude(T, 0.1), B)
    b.upload(D._lib.F_THETA, np.concatenate([th9, inertia], axis=1))
    cfg = D.SqpConfig(max_sqp_iters=4, pcg=D.PcgConfig(mode=mode))
    b.rollout(cfg, x0, H)
    b.rollout_backward(cfg.pcg)
    assert all(e is None for e in b.rollout_errors())
    got_r = b.download(D._lib.F_REWARD)[:, 0]
    got_g = b.download(D._lib.F_GRAD_THETA)[:, :9]
    for j in range(B):
        if mode == "parity":
            assert got_r[j] == want_r[j] and np.array_equal(got_g[j], want_g[j]), (j, got_r[j], want_r[j])
        else:
            assert abs(got_r[j] - want_r[j]) <= RTOL_FAST * abs(want_r[j])
            assert rel(got_g[j], want_g[j]) <= RTOL_FAST


# ----------------------------------------------------------------- pcg_study


@pytest.mark.skipif(not po.available("ref"), reason="needs the reference build (oracle/_ref)")
def test_pcg_study_matches_reference(D):
    """The GPU warm-vs-cold study reproduces the reference's pcg_study
    iteration counts (study.hpp:56-145) for every tol, step and pass."""
    from paper_2510_06179_b200.study import pcg_study
    tols, steps = [1e-4, 1e-8, 1e-12], 6
    want_c, want_w = po.pcg_study(tols, steps, seed=0)
    cold, warm, _, _ = pcg_study(tols, steps, seed=0, sequences=1, mode="parity")
    assert np.array_equal(cold[..., 0], want_c) and np.array_equal(warm[..., 0], want_w)


@pytest.mark.parametrize("nx,nu,T", [(8, 4, 256), (16, 8, 30), (8, 4, 100)])
def test_pcg_breakdown_all_kernels(D, nx, nu, T):
    """An indefinite diagonal block deep in the system: every FAST kernel
    (single CTA, and the cluster forms whose CTAs must take the same
    decision) reports the reference's BreakdownError at the oracle's
    iteration, and the batch's other problems solve normally."""
    th = aq_thetas(nx, nu, T, 31, 2)
    pp = po.aq_problem(nx, nu, T)
    o = po.Oracle("port", pp)
    blocks, gammas = [], []
    for j in range(2):
        o.linearize(th[j], np.zeros(o.nz))
        o.assemble()
        blocks.append([np.array(a) for a in o.schur()])
        gammas.append(o.gamma(o.flat_b(), o.flat_d()))
    blocks[0][0][T // 2] = -blocks[0][0][T // 2]  # -S diag block of a mid-horizon stage
    with pytest.raises(po.OracleError) as ei:
        po.pcg_blocks("port", blocks[0][0], blocks[0][1], blocks[0][2], blocks[0][3], gammas[0], np.zeros(o.nl))
    want_it = ei.value.iteration
    want_ok = po.pcg_blocks("port", *blocks[1], gammas[1], np.zeros(o.nl))
    b = D.Batch(D.affine_quadratic(nx, nu, T), 2)
    b.upload_schur(*[np.stack([bl[k] for bl in blocks]) for k in range(4)])
    b.upload(D._lib.F_GAMMA, np.stack(gammas))
    for mode in ("parity", "fast"):
        b.upload(D._lib.F_LAMBDA, np.zeros((2, b.nl)))
        b.pcg_solve(D.PcgConfig(mode=mode))
        errs = b.errors()
        assert isinstance(errs[0], D.BreakdownError) and errs[0].iteration == want_it, (mode, errs[0])
        assert errs[1] is None
        assert b.download(D._lib.F_PCG_ITERS)[1, 0] == want_ok[1]


@pytest.mark.parametrize("nx,nu,T", [(8, 4, 1), (8, 4, 2), (8, 4, 30), (8, 4, 100), (8, 4, 113), (8, 4, 120),
                                     (8, 4, 127), (8, 4, 128), (8, 4, 134), (8, 4, 135), (8, 4, 143), (8, 4, 160),
                                     (8, 4, 191)])
def test_fast_nx8_kernels_agree(D, nx, nu, T, monkeypatch):
    """The n_x = 8 single-CTA FAST kernels: pcg_kernel_h8r (-S in registers)
    and pcg_kernel_h8f fold every sum in the same order and agree bit for bit;
    pcg_kernel_h8s (the default for device-assembled systems: both symmetric
    diagonal blocks packed in registers; T > 113: the 288-thread form without
    the prefetch, against the h8f cluster) folds the diagonal products in
    another order: same iteration counts, iterates within 1e-12."""
    if T > 113:
        assert "no-prefetch" in D.describe(D.affine_quadratic(nx, nu, T))
    th = aq_thetas(nx, nu, T, 77, 5)
    b = D.Batch(D.affine_quadratic(nx, nu, T), 5)
    b.upload(D._lib.F_THETA, th)
    b.upload(D._lib.F_Z, np.zeros((5, b.nz)))
    b.linearize()
    b.assemble_schur()
    b.assemble_gamma()
    got = {}
    for variant in ("", "h8r", "h8f"):
        monkeypatch.setenv("DOCP_PCG_VARIANT", variant)
        b.upload(D._lib.F_LAMBDA, np.zeros((5, b.nl)))
        b.pcg_solve(D.PcgConfig(mode="fast"))
        got[variant] = (b.download(D._lib.F_LAMBDA), b.download(D._lib.F_PCG_ITERS)[:, 0])
    assert np.array_equal(got["h8f"][1], got["h8r"][1]) and np.array_equal(got["h8f"][0], got["h8r"][0])
    assert np.array_equal(got[""][1], got["h8r"][1])
    for j in range(5):
        assert rel(got[""][0][j], got["h8r"][0][j]) <= 1e-12


@pytest.mark.parametrize("mode", ["parity", "fast"])
def test_aq_blocks_kept_across_sqp_iterations(D, mode, monkeypatch):
    """The affine-quadratic family's -S / Phi^-1 depend on theta only, so
    docp_sqp_solve assembles them once per solve and later iterations (and
    the final refresh, sqp.hpp:254-259) only re-linearise. The kept blocks
    must equal a fresh assembly at the returned trajectory bit for bit, and
    the whole solve + backward must equal a run that re-assembles every
    iteration (DOCP_REASSEMBLE)."""
    nx, nu, T, B = 8, 4, 30, 8
    th = aq_thetas(nx, nu, T, 31, B)
    prob = D.affine_quadratic(nx, nu, T)
    nz, nl = D.sizes(prob)
    z0 = np.random.default_rng(3).standard_normal((B, nz))
    cfg = D.SqpConfig(max_sqp_iters=5, pcg=D.PcgConfig(mode=mode))
    lg = np.random.default_rng(4).standard_normal((B, nz))

    def run():
        b = D.Batch(prob, B)
        b.upload(D._lib.F_THETA, th)
        b.upload(D._lib.F_Z, z0)
        b.upload(D._lib.F_LAMBDA, np.zeros((B, nl)))
        b.sqp_solve(cfg)
        assert all(e is None for e in b.errors())
        assert (b.download(D._lib.F_SQP_ITERS) >= 2).all()  # blocks were reused at least once
        kept = b.download_schur()
        b.upload(D._lib.F_LOSS_GRAD_Z, lg)
        b.upload(D._lib.F_LAMBDA_TILDE, np.zeros((B, nl)))
        b.backward_vjp(cfg.pcg)
        out = [b.download(f) for f in (D._lib.F_Z, D._lib.F_LAMBDA, D._lib.F_GRAD_THETA, D._lib.F_LAMBDA_TILDE,
                                       D._lib.F_KKT, D._lib.F_PCG_HISTORY, D._lib.F_STEP_SIZES)]
        if mode == "parity":  # docp_assemble_schur is the reference's arithmetic
            b.linearize()          # fresh assembly at the returned trajectory
            b.assemble_schur()
            fresh = b.download_schur()
            for k, f in zip(kept, fresh):
                assert np.array_equal(k, f)
        return out + list(kept)

    kept_run = run()
    monkeypatch.setenv("DOCP_REASSEMBLE", "1")
    full_run = run()
    for a, c in zip(kept_run, full_run):
        assert np.array_equal(a, c)


def test_solve_and_backward_graphs_replay_bitwise(D):
    """With a batch stream, sqp_solve (<= 4 SQP iterations) and backward_vjp run
    as cached CUDA graphs (the C1 small-batch path): the first call captures,
    later calls replay. Replays on new inputs equal the direct launches bit
    for bit."""
    import torch
    nx, nu, T, B = 4, 2, 20, 3
    prob = D.affine_quadratic(nx, nu, T)
    nz, nl = D.sizes(prob)
    cfg = D.one_shot_config(mode="parity")
    outs = {}
    for graphs in (True, False):
        b = D.Batch(prob, B)
        if graphs:
            stream = torch.cuda.Stream()
            b.set_stream(stream.cuda_stream)
        res = []
        for seed in (0, 1, 2):  # capture, then two replays on different data
            th = D.generate_affine_quadratic(nx, nu, seed, B)
            b.upload(D._lib.F_THETA, th)
            b.upload(D._lib.F_Z, np.zeros((B, nz)))
            b.upload(D._lib.F_LAMBDA, np.zeros((B, nl)))
            l0 = D.kernel_launches()
            b.sqp_solve(cfg)
            z = b.download(D._lib.F_Z)
            b.upload(D._lib.F_LOSS_GRAD_Z, 2.0 * z)
            b.upload(D._lib.F_LAMBDA_TILDE, np.zeros((B, nl)))
            b.backward_vjp(cfg.pcg)
            b.sync()
            res.append((z.copy(), b.download(D._lib.F_GRAD_THETA).copy(), D.kernel_launches() - l0))
        outs[graphs] = res
    for (zg, gg, ng), (zd, gd, nd) in zip(outs[True], outs[False]):
        assert np.array_equal(zg, zd) and np.array_equal(gg, gd)
        assert ng == nd  # launches inside a replayed graph are still counted
