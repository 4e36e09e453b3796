"""CPU tests of the parity CHECKER (oracle/port, the plain-C restatement).

Pins the restatement three ways:
  1. against golden vectors produced by the reference itself (tests/golden,
     oracle/gen_golden.py) — bit-for-bit;
  2. against the reference's own known-answer tests (the §4 rows of SURVEY.md,
     restated here with their file:line);
  3. against the live reference build (oracle/_ref) on fresh random instances,
     and by running the reference's own unit-test binary, when present.
"""
import os
import subprocess

import numpy as np
import pytest

import pyoracle as po

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not po.available("port"):
        subprocess.run(["make", "-s", "-C", os.path.join(os.path.dirname(po.HERE), "oracle"), "port"], check=True)


# ------------------------------------------------------------------ golden vectors (reference outputs)


@pytest.mark.parametrize("name", ["aq_1_1_1_seed0.npz", "aq_4_2_20_seed1.npz", "aq_8_4_30_seed2.npz",
                                  "aq_8_4_100_seed3.npz", "aq_16_8_30_seed4.npz"])
def test_port_matches_reference_golden_aq(name):
    g = golden(name)
    th = g["theta"]
    B = th.shape[0]
    nx, nu, T = [int(s) for s in name.split("_")[1:4]]
    prob = po.aq_problem(nx, nu, T)
    nz, nl = po.sizes(prob)
    cfg = po.sqp_config(max_sqp_iters=int(g["max_sqp_iters"]))
    for j in range(B):
        o = po.Oracle("port", prob)
        s = o.sqp_solve(th[j], g["z0"][j], np.zeros(nl), cfg)
        assert np.array_equal(s.z, g["z"][j]) and np.array_equal(s.lam, g["lam"][j])
        assert s.sqp_iters == g["sqp_iters"][j]
        assert s.pcg_iters == [int(x) for x in g["pcg_iters"][j] if x >= 0]
        assert s.kkt == g["kkt"][j]
        sd, ss, pd, ps = o.schur()
        for got, key in ((sd, "S_diag"), (ss, "S_sub"), (pd, "P_diag"), (ps, "P_super")):
            assert np.array_equal(got, g[key][j]), key
        grad, lt, it = o.backward(th[j], g["loss_grad"][j], np.zeros(nl))
        assert np.array_equal(grad, g["grad"][j]) and np.array_equal(lt, g["lt"][j]) and it == g["bwd_iters"][j]


@pytest.mark.parametrize("T", [40, 50])
def test_port_matches_reference_golden_cartpole(T):
    g = golden(f"cartpole_T{T}_seed0.npz")
    prob = po.cartpole_problem(T)
    nz, nl = po.sizes(prob)
    n = g["theta"].shape[0]
    for j in range(n):
        o = po.Oracle("port", prob)
        s = o.sqp_solve(g["theta"][j], g["demos"][j], np.zeros(nl), po.sqp_config(max_sqp_iters=5))
        assert np.array_equal(s.z, g["z"][j]) and np.array_equal(s.lam, g["lam"][j])
        assert s.pcg_iters == [int(x) for x in g["pcg_iters"][j] if x >= 0]
        lg = np.zeros(nz)
        for t in range(T):
            k = t * 5 + 4
            lg[k] = 2.0 / n * (s.z[k] - g["demos"][j, k])
        grad, lt, it = o.backward(g["theta"][j], lg, np.zeros(nl))
        assert np.array_equal(grad, g["grad"][j]) and np.array_equal(lt, g["lt"][j]) and it == g["bwd_iters"][j]


def test_port_epoch_reproduces_reference_train_il():
    """Two epochs of the reference's bench::train_il (train.hpp:53-145) from
    the golden record; the port's epoch body + host GD step reproduce the
    objectives, the iteration counters and the final weights bit for bit."""
    g = golden("train_il_cartpole_seed3.npz")
    T, B = 40, g["x0"].shape[0]
    prob = po.cartpole_problem(T)
    nz, nl = po.sizes(prob)
    w = g["w0"].copy()
    lam_c, lt_c = np.zeros((B, nl)), np.zeros((B, nl))
    for epoch in range(2):
        th = np.array([np.concatenate([w, [0.05], x]) for x in g["x0"]])
        loss, grad, _, _, sqp_it, pcg_it = po.il_epoch("port", prob, th, g["demos"], lam_c, lt_c,
                                                       po.sqp_config(max_sqp_iters=5), 0, 4)
        assert loss == g["objectives"][epoch]
        assert sqp_it.sum() == g["sqp_iters"][epoch] and pcg_it.sum() == g["pcg_iters"][epoch]
        w = w - float(g["lr"]) * grad
    assert np.array_equal(w, g["final_weights"])


# ------------------------------------------------------------------ known-answer tests of the reference suite


def scalar():
    """scalar_one_step_problem (affine_quadratic.hpp:124-135): x^2/2 + u^2/2,
    x+ = x + u, x_s = 1."""
    prob = po.aq_problem(1, 1, 1, cost_scale=0.5)
    theta = np.array([1.0, 1.0, 1.0, 1.0, 0.0, 1.0])
    return prob, theta


def test_kat_scalar_linearize_and_schur():
    prob, th = scalar()
    o = po.Oracle("port", prob)
    o.linearize(th, np.zeros(3))
    qp = o.qp()  # test_problem.cpp:55-73
    assert qp["Q"][:, 0, 0].tolist() == [1.0, 1.0] and qp["R"][0, 0, 0] == 1.0
    assert qp["q"].ravel().tolist() == [0.0, 0.0] and qp["r"][0, 0] == 0.0
    assert qp["Ap"][0, 0, 0] == 1.0 and qp["A"][0, 0, 0] == -1.0 and qp["B"][0, 0, 0] == -1.0
    assert qp["C"][0, 0] == 0.0 and qp["x_s"][0] == 1.0 and not qp["pd_projected"]
    o.assemble()
    sd, ss, pd, ps = o.schur()  # test_schur.cpp:21-35
    assert sd[:, 0, 0].tolist() == pytest.approx([1.0, 3.0]) and ss[0, 0, 0] == pytest.approx(-1.0)
    assert pd[:, 0, 0].tolist() == pytest.approx([1.0, 1.0 / 3.0]) and ps[0, 0, 0] == pytest.approx(1.0 / 3.0)
    gam = o.gamma(o.flat_b(), o.flat_d())  # test_pcg.cpp:46-61
    assert gam[0] == pytest.approx(-1.0) and abs(gam[1]) <= 1e-15
    lam, it, _, conv = o.pcg(gam, np.zeros(2))
    assert it <= 2 and conv and lam.tolist() == pytest.approx([-1.5, -0.5])


def test_kat_scalar_sqp_and_backward():
    prob, th = scalar()
    o = po.Oracle("port", prob)
    s = o.sqp_solve(th, np.zeros(3), np.zeros(2), po.sqp_config(max_sqp_iters=1, alphas=(1.0,)))
    assert s.z.tolist() == pytest.approx([1.0, -0.5, 0.5])  # test_sqp.cpp:44-58 (x0, u0, x1)
    assert s.z[1] == pytest.approx(-0.5)  # policy_first_control, test_sqp.cpp:279-285
    assert o.merit(th, np.zeros(3), 2.0) == pytest.approx(2.0)  # test_sqp.cpp:92-96
    lg = np.array([0.0, 0.0, 1.0])  # loss = x_1 (test_backward.cpp:34-53)
    grad, lt, _ = o.backward(th, lg, np.zeros(2))
    assert lt.tolist() == pytest.approx([0.5, 0.5])
    assert grad[1] == pytest.approx(0.25) and grad[5] == pytest.approx(0.5)


def test_kat_zero_cotangent_zero_iterations():
    """test_backward.cpp:20-32"""
    prob, th = scalar()
    o = po.Oracle("port", prob)
    o.sqp_solve(th, np.zeros(3), np.zeros(2), po.sqp_config())
    grad, lt, it = o.backward(th, np.zeros(3), np.zeros(2))
    assert it == 0 and not grad.any()


def decoupled(nx, T):
    return po.aq_problem(nx, nx, T, cost_scale=0.5), np.concatenate([np.ones(2 * nx), np.zeros(2 * nx * nx + 2 * nx)])


def test_kat_pcg_identity_one_iteration():
    """test_pcg.cpp:32-44"""
    prob, th = decoupled(3, 5)
    o = po.Oracle("port", prob)
    o.linearize(th, np.zeros(o.nz))
    o.assemble()
    gam = np.random.default_rng(1).standard_normal(o.nl)
    lam, it, _, conv = o.pcg(gam, np.zeros(o.nl))
    assert it == 1 and conv and np.abs(lam - gam).max() < 1e-12


def test_kat_pcg_warm_start_breakdown_cap_rerun():
    g = golden("generators.npz")
    th = g["convex_8_4_100_seed0"][0]
    prob = po.aq_problem(8, 4, 100)
    o = po.Oracle("port", prob)
    o.linearize(th, np.zeros(o.nz))
    o.assemble()
    gam = o.gamma(o.flat_b(), o.flat_d())
    cold = o.pcg(gam, np.zeros(o.nl))
    warm = o.pcg(gam, cold[0])  # test_pcg.cpp:63-78
    assert warm[1] == 0 and warm[3] and np.array_equal(warm[0], cold[0])
    again = o.pcg(gam, np.zeros(o.nl))  # test_pcg.cpp:192-206
    assert again[1] == cold[1] and np.array_equal(again[0], cold[0]) and again[2] == cold[2]
    capped = o.pcg(gam, np.zeros(o.nl), epsilon=1e-14, max_iters=2)  # test_pcg.cpp:175-190
    assert capped[1] == 2 and not capped[3]
    # test_pcg.cpp:162-173: negated -S -> BreakdownError at iteration 0
    sd, ss, pd, ps = o.schur()
    with pytest.raises(po.OracleError) as e:
        po.pcg_blocks("port", -sd, ss, pd, ps, gam, np.zeros(o.nl), s_super=np.swapaxes(ss, 1, 2))
    assert e.value.code == "BREAKDOWN" and e.value.iteration == 0


def test_kat_dense_kkt_agreement():
    """pcg/recover agree with a dense KKT solve (test_pcg.cpp:80-95)."""
    th = golden("generators.npz")["linear_8_4_40_seed0"][0]
    prob = po.aq_problem(8, 4, 40)
    o = po.Oracle("port", prob)
    o.linearize(th, np.zeros(o.nz))
    o.assemble()
    b, d = o.flat_b(), o.flat_d()
    lam, it, _, conv = o.pcg(o.gamma(b, d), np.zeros(o.nl), epsilon=1e-12)
    z = o.recover(lam, b)
    qp = o.qp()
    nx, nu, T = 8, 4, 40
    nz, nl = o.nz, o.nl
    G, H = np.zeros((nz, nz)), np.zeros((nl, nz))
    for t in range(T + 1):
        G[t * 12:t * 12 + 8, t * 12:t * 12 + 8] = qp["Q"][t]
    for t in range(T):
        G[t * 12 + 8:t * 12 + 12, t * 12 + 8:t * 12 + 12] = qp["R"][t]
    H[:8, :8] = np.eye(8)
    for t in range(T):
        H[(t + 1) * 8:(t + 2) * 8, t * 12:t * 12 + 8] = qp["A"][t]
        H[(t + 1) * 8:(t + 2) * 8, t * 12 + 8:t * 12 + 12] = qp["B"][t]
        H[(t + 1) * 8:(t + 2) * 8, (t + 1) * 12:(t + 1) * 12 + 8] = qp["Ap"][t]
    K = np.block([[G, H.T], [H, np.zeros((nl, nl))]])
    sol = np.linalg.solve(K, np.concatenate([-b, d]))
    assert np.linalg.norm(z - sol[:nz]) / max(1, np.linalg.norm(sol[:nz])) < 1e-8
    assert np.linalg.norm(lam - sol[nz:]) / max(1, np.linalg.norm(sol[nz:])) < 1e-8


def test_port_error_messages():
    prob, th = scalar()
    o = po.Oracle("port", prob)
    bad = th.copy()
    bad[5] = np.nan
    with pytest.raises(po.OracleError) as e:  # problem.hpp:187-193
        o.sqp_solve(bad, np.zeros(3), np.zeros(2), po.sqp_config())
    assert e.value.code == "EVALUATION" and "initial_state returned non-finite values at stage 0" in e.value.message
    with pytest.raises(po.OracleError) as e:
        o.sqp_solve(th, np.array([np.inf, 0, 0]), np.zeros(2), po.sqp_config())
    assert e.value.code == "DIMENSION"


# ------------------------------------------------------------------ live reference (where built)

needs_ref = pytest.mark.skipif(not po.available("ref"), reason="oracle/_ref not built (needs /root/reference)")


@needs_ref
@pytest.mark.parametrize("nx,nu,T,seed", [(3, 2, 6, 1), (5, 2, 9, 2), (6, 3, 12, 3), (8, 4, 40, 4), (9, 2, 20, 5)])
def test_port_bitwise_vs_live_reference(nx, nu, T, seed):
    th = po.gen_aq(nx, nu, T, seed, 2)
    prob = po.aq_problem(nx, nu, T, cost_scale=0.5 if seed % 2 else 1.0)
    rng = np.random.default_rng(seed)
    for j in range(2):
        z0 = rng.standard_normal(po.sizes(prob)[0])
        lg = rng.standard_normal(po.sizes(prob)[0])
        outs = []
        for kind in ("port", "ref"):
            o = po.Oracle(kind, prob)
            s = o.sqp_solve(th[j], z0, np.zeros(o.nl), po.sqp_config())
            outs.append((s, *o.backward(th[j], lg, np.zeros(o.nl))))
        (a, ga, la, ia), (b, gb, lb, ib) = outs
        assert np.array_equal(a.z, b.z) and np.array_equal(a.lam, b.lam) and a.pcg_iters == b.pcg_iters
        assert np.array_equal(ga, gb) and np.array_equal(la, lb) and ia == ib and a.kkt == b.kkt


@needs_ref
def test_port_line_search_and_merit_vs_live_reference():
    th = po.gen_aq(4, 2, 10, 9, 1)[0]
    prob = po.aq_problem(4, 2, 10)
    rng = np.random.default_rng(9)
    z_old, z_qp = rng.standard_normal((2, po.sizes(prob)[0]))
    lam = rng.standard_normal(po.sizes(prob)[1])
    res = []
    for kind in ("port", "ref"):
        o = po.Oracle(kind, prob)
        o.linearize(th, z_old)
        z_new, alpha, acc, mu = o.line_search(th, z_old, z_qp, po.sqp_config(), 1.0)
        res.append((z_new, alpha, acc, mu, o.merit(th, z_qp, 3.0), o.kkt_inf_norm(th, z_old, lam)))
    a, b = res
    assert np.array_equal(a[0], b[0]) and a[1:] == b[1:]


REF_TESTS = os.path.join(po.HERE, "_ref", "docp_ref_tests")
# Reference tests that also fail against the reference's algorithm itself
# (cart-pole Gauss-Newton limits): non-monotone KKT on
# the swing-up and a 3.4e-6 (> 1e-6) stationarity residual at the expert.
KNOWN_REFERENCE_FAILURES = {"sqp_solve: cart-pole swing-up converges within five iterations",
                            "train_il: the expert weights are a stationary point"}


@pytest.mark.skipif(not os.path.exists(REF_TESTS), reason="reference unit tests not built")
def test_reference_unit_suite_runs_on_eigen_lite():
    """The reference's own Catch2 suite (proj/tests, 93 cases outside the CLI
    file), compiled unmodified against eigen_lite + catch2_lite."""
    r = subprocess.run([REF_TESTS], capture_output=True, text=True, timeout=900)
    failed = {line[5:] for line in r.stdout.splitlines() if line.startswith("FAIL ")}
    passed = [line for line in r.stdout.splitlines() if line.startswith("PASS ")]
    assert failed <= KNOWN_REFERENCE_FAILURES, failed - KNOWN_REFERENCE_FAILURES
    assert len(passed) >= 91
