"""The `docp_gpu` CLI (paper_2510_06179_b200/cli): the reference CLI's `solve`
and `grad-check` (proj/tools/docp_main.cpp:67-175) on aq-ocp/1 problem files
(problems/affine_quadratic_io.hpp:9-77), run on the GPU path.

CPU tests cover argument handling and every problem-file rejection (they
exit before any device call). GPU tests check the written solution against
the oracle bit for bit (PARITY is the CLI default) and that grad-check passes.
"""
import json
import os
import subprocess

import numpy as np
import pytest

import pyoracle as po

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2510_06179_b200", "lib", "docp_gpu")

pytestmark = pytest.mark.skipif(not os.path.exists(CLI), reason="docp_gpu not built (python build.py)")


def run(*args, cwd=None):
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=600, cwd=cwd)


def double_integrator(T=20, dt=0.1):
    """C1: the planar double integrator of the reference tests."""
    A = np.block([[np.eye(2), dt * np.eye(2)], [np.zeros((2, 2)), np.eye(2)]])
    B = np.vstack([0.5 * dt * dt * np.eye(2), dt * np.eye(2)])
    return {"format": "aq-ocp/1", "n_x": 4, "n_u": 2, "T": T, "Q": [1.0, 1.0, 0.1, 0.1], "R": [0.1, 0.1],
            "A": A.tolist(), "B": B.tolist(), "b_affine": [0.0] * 4, "x_s": [1.0, -1.0, 0.0, 0.0]}


def random_problem(nx, nu, T, seed):
    rng = np.random.default_rng(seed)
    A = np.eye(nx) + 0.1 * rng.standard_normal((nx, nx))
    A *= min(1.0, 0.99 / max(abs(np.linalg.eigvals(A))))
    return {"format": "aq-ocp/1", "n_x": nx, "n_u": nu, "T": T, "Q": rng.uniform(0.5, 2, nx).tolist(),
            "R": rng.uniform(0.5, 2, nu).tolist(), "A": A.tolist(), "B": rng.standard_normal((nx, nu)).tolist(),
            "b_affine": (1e-2 * rng.standard_normal(nx)).tolist(), "x_s": rng.standard_normal(nx).tolist()}


def theta_of(p):
    """AffineQuadratic::make_theta (affine_quadratic.hpp:27-37), column-major A and B."""
    A, B = np.asarray(p["A"]), np.asarray(p["B"])
    return np.concatenate([p["Q"], p["R"], A.flatten(order="F"), B.flatten(order="F"), p["b_affine"], p["x_s"]])


def write(tmp_path, obj, name="problem.json"):
    path = tmp_path / name
    path.write_text(obj if isinstance(obj, str) else json.dumps(obj))
    return str(path)


# ------------------------------------------------------------------ CPU: input handling


def test_help_and_usage():
    r = run("--help")
    assert r.returncode == 0 and "solve <problem.json>" in r.stdout
    assert run().returncode == 1                      # a sub-command is required (CLI11)
    assert run("solve").returncode == 1               # ... and its problem argument
    assert run("frobnicate", "x.json").returncode == 1


@pytest.mark.parametrize("mutate, message", [
    (lambda p: p.pop("format"), "problem file: missing or unsupported format key"),
    (lambda p: p.update(format="aq-ocp/2"), "problem file: missing or unsupported format key"),
    (lambda p: p.update(T=0), "problem file: dimensions must be positive"),
    (lambda p: p.update(Q=[1.0, 1.0]), "problem file: bad length for Q"),
    (lambda p: p.update(R=[1.0]), "problem file: bad length for R"),
    (lambda p: p.update(A=p["A"][:3]), "problem file: bad row count for A"),
    (lambda p: p["B"][2].append(0.0), "problem file: bad column count for B"),
    (lambda p: p.update(x_s=[0.0] * 5), "problem file: bad length for x_s"),
    (lambda p: p.pop("b_affine"), "problem file is not valid JSON: [json.exception.out_of_range.403] key 'b_affine' not found"),
])
def test_invalid_problem_files(tmp_path, mutate, message):
    """affine_quadratic_from_json's checks and load_problem's wrapping (exit 3)."""
    p = double_integrator()
    mutate(p)
    for cmd in ("solve", "grad-check"):
        r = run(cmd, write(tmp_path, p), "--out", str(tmp_path / "out"))
        assert r.returncode == 3, r.stderr
        assert r.stderr.strip() == "invalid input: " + message


def test_unreadable_and_malformed_files(tmp_path):
    r = run("solve", str(tmp_path / "missing.json"))
    assert r.returncode == 3 and "cannot open problem file: " in r.stderr
    r = run("solve", write(tmp_path, '{"format": "aq-ocp/1", "n_x": [1,'))
    assert r.returncode == 3 and r.stderr.startswith("invalid input: problem file is not valid JSON: ")


# ------------------------------------------------------------------ GPU: results


def oracle_solve(p):
    prob = po.aq_problem(p["n_x"], p["n_u"], p["T"])
    o = po.Oracle("port", prob)
    return o.sqp_solve(theta_of(p), np.zeros(o.nz), np.zeros(o.nl), po.sqp_config()), o


def flat_z(sol, nx, nu, T):
    x, u = np.asarray(sol["trajectory"]["x"]), np.asarray(sol["trajectory"]["u"])
    assert x.shape == (T + 1, nx) and u.shape == (T, nu)
    z = []
    for t in range(T + 1):
        z.extend(x[t])
        if t < T:
            z.extend(u[t])
    return np.asarray(z)


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["c1", "random8"])
def test_solve_matches_oracle_bitwise(tmp_path, case):
    p = double_integrator() if case == "c1" else random_problem(8, 4, 40, 3)
    path = write(tmp_path, p)
    out = tmp_path / "out"
    r = run("--seed", "7", "--workers", "3", "--out", str(out), "solve", path)
    assert r.returncode == 0, r.stderr
    sol = json.loads((out / "solution.json").read_text())
    s, _ = oracle_solve(p)
    assert sol["format"] == "docp-bench/1" and sol["command"] == "solve" and sol["seed"] == 7 and sol["workers"] == 3
    assert sol["problem"] == path
    # the JSON numbers are shortest round-trip, so == compares the device bits
    assert np.array_equal(flat_z(sol, p["n_x"], p["n_u"], p["T"]), s.z)
    assert np.array_equal(np.asarray(sol["lambda"]), s.lam)
    assert sol["sqp_iters"] == s.sqp_iters and sol["pcg_iters"] == s.pcg_iters
    assert sol["converged"] == s.converged and sol["kkt_inf_norm"] == s.kkt
    assert r.stdout.strip() == (f"solved {path}: sqp_iters={s.sqp_iters} kkt_inf_norm={s.kkt:g} "
                                f"converged={'yes' if s.converged else 'no'}")
    assert list(sol) == sorted(sol)  # nlohmann::json object key order


@pytest.mark.gpu
def test_solve_fast_mode(tmp_path):
    p = random_problem(8, 4, 100, 5)
    out = tmp_path / "out"
    r = run("--mode", "fast", "--out", str(out), "solve", write(tmp_path, p))
    assert r.returncode == 0, r.stderr
    sol = json.loads((out / "solution.json").read_text())
    s, _ = oracle_solve(p)
    z = flat_z(sol, 8, 4, 100)
    assert np.linalg.norm(z - s.z) <= 1e-9 * max(1.0, np.linalg.norm(s.z))
    assert sol["sqp_iters"] == s.sqp_iters and sol["pcg_iters"] == s.pcg_iters


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["c1", "random6"])
def test_grad_check_passes(tmp_path, case):
    p = double_integrator() if case == "c1" else random_problem(6, 3, 30, 11)
    out = tmp_path / "out"
    r = run("--out", str(out), "grad-check", write(tmp_path, p), "--tol", "1e-5")
    assert r.returncode == 0, r.stdout + r.stderr
    g = json.loads((out / "gradcheck.json").read_text())
    assert g["command"] == "grad-check" and g["pass"] is True and g["tolerance"] == 1e-5
    assert set(g["max_rel_error"]) == {"control_cost", "dynamics", "initial_state", "state_cost"}
    assert g["overall_max_rel_error"] == max(g["max_rel_error"].values()) <= 1e-5
    assert r.stdout.splitlines()[-1].endswith("(pass)")
    # an impossible tolerance fails with the solver-failure exit code
    r = run("--out", str(out), "grad-check", write(tmp_path, p), "--tol", "0")
    assert r.returncode == 2 and r.stdout.splitlines()[-1].endswith("(FAIL)")


@pytest.mark.gpu
def test_solver_failure_exit_code(tmp_path):
    """A non-finite evaluation is a docp::EvaluationError -> exit 2 with the
    reference's message (here the merit's, sqp.hpp:98-133)."""
    p = double_integrator()
    p["b_affine"] = [1e308, 1e308, 0.0, 0.0]
    p["A"] = (1e10 * np.asarray(p["A"])).tolist()
    r = run("--out", str(tmp_path / "out"), "solve", write(tmp_path, p))
    assert r.returncode == 2, r.stdout + r.stderr
    with pytest.raises(po.OracleError) as e:
        oracle_solve(p)
    assert r.stderr.strip() == "solver failure: " + e.value.message
