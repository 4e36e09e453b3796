"""Small solve + backward cases that route through every K2 variant (and K1,
K3, K4), for compute-sanitizer runs (racecheck / synccheck / memcheck; one
tool per gpurun call). Each FAST case is checked against the PARITY solve of
the same batch (PARITY is bit-identical to the reference; test_gpu_parity.py):
equal SQP counts, PCG counts within one, <= 1e-9 relative.

  python tools/sanitize_cases.py [case ...]      (default: all)
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2510_06179_b200 as D  # noqa: E402

# name: (n_x, n_u, T, B, env overrides, modes)
CASES = {
    "h8s": (8, 4, 30, 3, {}, ("fast",)),
    "h8s_np": (8, 4, 30, 3, {"DOCP_PCG_VARIANT": "h8s_np"}, ("fast",)),
    "h8s_wide": (8, 4, 140, 2, {}, ("fast",)),
    "h8r": (8, 4, 30, 3, {"DOCP_PCG_VARIANT": "h8r"}, ("fast",)),
    "h8f_cl1": (8, 4, 30, 3, {"DOCP_PCG_VARIANT": "h8f"}, ("fast",)),
    "h8f_cl2": (8, 4, 60, 2, {"DOCP_PCG_VARIANT": "h8f", "DOCP_H8F_CLUSTER": "2"}, ("fast",)),
    "h8f_cl3": (8, 4, 60, 2, {"DOCP_PCG_VARIANT": "h8f", "DOCP_H8F_CLUSTER": "3"}, ("fast",)),
    "h8s_cl2": (8, 4, 200, 2, {}, ("fast",)),
    "h8s_cl3": (8, 4, 320, 1, {}, ("fast",)),
    "h8f_cl4": (8, 4, 60, 2, {"DOCP_PCG_VARIANT": "h8f", "DOCP_H8F_CLUSTER": "4"}, ("fast",)),
    "h8f_cl6": (8, 4, 60, 2, {"DOCP_PCG_VARIANT": "h8f", "DOCP_H8F_CLUSTER": "6"}, ("fast",)),
    "h8f_cl4_nodbuf": (8, 4, 400, 1, {}, ("fast",)),  # R = 101: the barrier form (no second buffer pair)
    "h8_fast": (8, 4, 30, 3, {"DOCP_PCG_VARIANT": "h8"}, ("fast",)),
    "h8p": (8, 4, 30, 3, {}, ("parity",)),
    "h4f": (4, 2, 20, 3, {}, ("fast", "parity")),
    "h16f": (16, 8, 10, 2, {}, ("fast", "parity")),
    "generic": (6, 3, 20, 3, {}, ("fast", "parity")),
    "fp32": (8, 4, 30, 3, {}, ("fp32",)),
}


def run(nx, nu, T, B, mode):
    prob = D.affine_quadratic(nx, nu, T)
    nz, nl = D.sizes(prob)
    th = D.generate_affine_quadratic(nx, nu, 0, B)
    rng = np.random.default_rng(0)
    z0 = 0.1 * rng.standard_normal((B, nz))
    lg = rng.standard_normal((B, nz))
    cfg = D.SqpConfig(max_sqp_iters=5, pcg=D.PcgConfig(mode=mode))
    res, errs = D.sqp_solve_batch(prob, th, z0, np.zeros((B, nl)), cfg)
    assert all(e is None for e in errs), errs
    g, lt, its, errs = D.backward_vjp_batch(res[0].batch, lg, np.zeros((B, nl)), cfg.pcg)
    assert all(e is None for e in errs), errs
    return (np.stack([r.z for r in res]), [r.pcg_iters for r in res], [r.sqp_iters for r in res], g.copy(),
            list(its))


def main(names):
    for name in names:
        nx, nu, T, B, env, modes = CASES[name]
        ref = None
        saved = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        try:
            outs = {m: run(nx, nu, T, B, m) for m in modes}
        finally:
            for k, v in saved.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        ref = run(nx, nu, T, B, "parity") if "parity" not in outs else outs["parity"]
        for m, (z, h, s, g, it) in outs.items():
            tol = 1e-4 if m == "fp32" else 1e-9
            rz = np.abs(z - ref[0]).max() / max(1.0, np.abs(ref[0]).max())
            rg = np.abs(g - ref[3]).max() / max(1.0, np.abs(ref[3]).max())
            ok = rz <= tol and rg <= tol and (m == "fp32" or (s == ref[2] and all(
                abs(a - b) <= 1 for ha, hb in zip(h, ref[1]) for a, b in zip(ha, hb))))
            print(f"{name:9s} {m:6s} n_x={nx} T={T} B={B}: rel z {rz:.1e} grad {rg:.1e} "
                  f"sqp {s} pcg {h} bwd {it} {'ok' if ok else 'MISMATCH'}", flush=True)
            if not ok:
                raise SystemExit(1)
    print("sanitize cases ok")


if __name__ == "__main__":
    main(sys.argv[1:] or [k for k in CASES if k != "fp32"])
