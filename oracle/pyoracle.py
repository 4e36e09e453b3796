"""ctypes bindings for the parity CHECKERS (test infrastructure only).

Two interchangeable back ends with one signature set (oracle/port/docp_port.h):
  * ``Oracle("port")`` — the plain-C restatement, oracle/_build/libdocp_port.so
  * ``Oracle("ref")``  — the UNMODIFIED reference headers compiled against
    eigen_lite, oracle/_ref/libdocp_ref.so (built where /root/reference exists;
    the prebuilt .so travels to the GPU box).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import
this module, and only as the checker — never as the product path.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "port": os.path.join(HERE, "_build", "libdocp_port.so"),
    "ref": os.path.join(HERE, "_ref", "libdocp_ref.so"),
}

AFFINE_QUADRATIC, CARTPOLE, ATTITUDE, DRIFT = 1, 2, 3, 4
CODES = {0: "OK", 1: "DIMENSION", 2: "EVALUATION", 3: "NUMERICAL", 4: "BREAKDOWN", 5: "DIVERGENCE", 99: "ERROR"}


class Problem(C.Structure):
    _fields_ = [
        ("family", C.c_int), ("nx", C.c_int), ("nu", C.c_int), ("horizon", C.c_int),
        ("cost_scale", C.c_double), ("cart_mass", C.c_double), ("pole_mass", C.c_double),
        ("length", C.c_double), ("gravity", C.c_double), ("dt", C.c_double),
        ("inertia", C.c_double * 3),
    ]


class Status(C.Structure):
    _fields_ = [("code", C.c_int), ("iteration", C.c_int), ("message", C.c_char * 192)]


class SqpConfig(C.Structure):
    _fields_ = [
        ("max_sqp_iters", C.c_int), ("n_alphas", C.c_int), ("alphas", C.c_double * 8),
        ("eta_armijo", C.c_double), ("rho_penalty", C.c_double), ("pcg_epsilon", C.c_double),
        ("pcg_max_iters", C.c_int), ("convergence_tol", C.c_double),
        ("mu_floor_denominator", C.c_double), ("eps_pd", C.c_double),
    ]


def sqp_config(max_sqp_iters=20, alphas=(1.0, 0.7, 0.3, 0.1, 0.01), eta_armijo=0.4, rho_penalty=0.5,
               pcg_epsilon=1e-12, pcg_max_iters=0, convergence_tol=1e-8, mu_floor_denominator=1e-12,
               eps_pd=1e-6) -> SqpConfig:
    """SqpConfig defaults of sqp.hpp:7-22 (PcgConfig pcg.hpp:7-23)."""
    c = SqpConfig()
    c.max_sqp_iters = max_sqp_iters
    c.n_alphas = len(alphas)
    for i, a in enumerate(alphas):
        c.alphas[i] = a
    c.eta_armijo, c.rho_penalty = eta_armijo, rho_penalty
    c.pcg_epsilon, c.pcg_max_iters = pcg_epsilon, pcg_max_iters
    c.convergence_tol, c.mu_floor_denominator, c.eps_pd = convergence_tol, mu_floor_denominator, eps_pd
    return c


def aq_problem(nx, nu, T, cost_scale=1.0) -> Problem:
    return Problem(AFFINE_QUADRATIC, nx, nu, T, cost_scale, 0, 0, 0, 0, 0)


def cartpole_problem(T=40, cart_mass=1.0, pole_mass=0.1, length=0.5, gravity=9.81, dt=0.05) -> Problem:
    """CartpoleParams defaults (cartpole.hpp:17-26)."""
    return Problem(CARTPOLE, 4, 1, T, 0.5, cart_mass, pole_mass, length, gravity, dt)


def attitude_problem(T=25, inertia=(1.0, 1.0, 1.0), dt=0.1) -> Problem:
    """AttitudeParams (attitude.hpp:10-14); ref build only."""
    p = Problem(ATTITUDE, 3, 3, T, 0.5, 0.0, 0.0, 0.0, 0.0, dt)
    for k in range(3):
        p.inertia[k] = inertia[k]
    return p


def drift_problem(T=100, dt=0.1) -> Problem:
    """The drifting family (include/docp_drift_model.h; ref build only: the
    reference solver on the shared model definition)."""
    return Problem(DRIFT, 8, 2, T, 0.5, 0.0, 0.0, 0.0, 0.0, dt)


def theta_size(p: Problem) -> int:
    if p.family == DRIFT:
        return 36
    if p.family in (CARTPOLE, ATTITUDE):
        return 2 * p.nx + p.nu
    return p.nx + p.nu + p.nx * p.nx + p.nx * p.nu + 2 * p.nx


def sizes(p: Problem):
    nl = p.nx * (p.horizon + 1)
    nz = nl + p.nu * p.horizon
    return nz, nl


class OracleError(RuntimeError):
    def __init__(self, st: Status):
        self.code = CODES.get(st.code, str(st.code))
        self.iteration = st.iteration
        self.message = st.message.decode()
        super().__init__(f"{self.code}: {self.message}")


def _p(a):
    return a.ctypes.data_as(C.POINTER(C.c_double)) if a is not None else None


def _arr(a, n=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if n is not None and a.size != n:
        raise ValueError(f"expected {n} values, got {a.size}")
    return a


_loaded = {}


def available(kind: str) -> bool:
    return os.path.exists(LIBS[kind])


def load(kind: str):
    if kind not in _loaded:
        lib = C.CDLL(LIBS[kind])
        pre = kind + "_"
        dp = C.POINTER(C.c_double)
        ip = C.POINTER(C.c_int)
        sp = C.POINTER(Status)
        vp = C.c_void_p
        sig = {
            "create": (vp, [C.POINTER(Problem)]),
            "destroy": (None, [vp]),
            "linearize": (C.c_int, [vp, dp, dp, C.c_double, sp]),
            "assemble": (C.c_int, [vp, sp]),
            "flat_b": (None, [vp, dp]),
            "flat_d": (None, [vp, dp]),
            "gamma": (C.c_int, [vp, dp, dp, dp, sp]),
            "pcg": (C.c_int, [vp, dp, dp, C.c_double, C.c_int, dp, ip, dp, ip, dp, C.c_int, sp]),
            "recover": (C.c_int, [vp, dp, dp, dp, sp]),
            "merit": (C.c_int, [vp, dp, dp, C.c_double, dp, sp]),
            "line_search": (C.c_int, [vp, dp, dp, dp, C.POINTER(SqpConfig), C.c_double, dp, dp, ip, dp, sp]),
            "kkt_inf_norm": (C.c_int, [vp, dp, dp, dp, dp, sp]),
            "sqp_solve": (C.c_int, [vp, dp, dp, dp, C.POINTER(SqpConfig), dp, dp, ip, ip, dp, ip, dp, sp]),
            "backward": (C.c_int, [vp, dp, dp, dp, C.c_double, C.c_int, dp, dp, ip, sp]),
            "get_qp": (None, [vp, dp, dp, dp, dp, dp, dp, dp, dp, dp, ip]),
            "get_schur": (None, [vp, dp, dp, dp, dp]),
            "pcg_blocks": (C.c_int, [C.c_int, C.c_int, dp, dp, dp, dp, dp, dp, dp, dp, C.c_double, C.c_int, dp, ip,
                                     dp, ip, sp]),
            "il_epoch": (C.c_int, [C.POINTER(Problem), C.c_int, dp, dp, dp, dp, C.POINTER(SqpConfig), C.c_int,
                                   C.c_int, dp, dp, dp, dp, ip, C.POINTER(C.c_long), sp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(lib, pre + name)
            f.restype, f.argtypes = res, args
        if kind == "ref":
            lib.ref_gen_aq.restype = None
            lib.ref_gen_aq.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int, dp]
            lib.ref_gen_cartpole.restype = C.c_int
            lib.ref_gen_cartpole.argtypes = [C.c_uint64, C.c_int, C.c_int, dp, dp, sp]
            lib.ref_train_il_cartpole.restype = C.c_int
            lib.ref_train_il_cartpole.argtypes = [C.c_uint64, C.c_int, C.c_int, dp, C.c_int, C.c_double, dp,
                                                  C.POINTER(C.c_long), C.POINTER(C.c_long), dp, sp]
            lib.ref_drift_step.restype = None
            lib.ref_drift_step.argtypes = [dp, C.c_double, dp, dp, dp, dp, dp]
            lib.ref_gen_uniform.restype = None
            lib.ref_gen_uniform.argtypes = [C.c_uint64, C.c_int, C.c_double, C.c_double, dp]
            lib.ref_spectral_radius.restype = C.c_double
            lib.ref_spectral_radius.argtypes = [dp, C.c_int]
            lib.ref_pcg_invocations.restype = C.c_ulonglong
            lib.ref_pcg_study.restype = C.c_int
            lib.ref_pcg_study.argtypes = [dp, C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_int, ip, ip]
            lib.ref_rollout_attitude.restype = C.c_int
            lib.ref_rollout_attitude.argtypes = [C.c_int, C.c_double, C.c_int, dp, dp, dp, C.c_int,
                                                 C.POINTER(SqpConfig), dp, dp, ip, C.c_char_p]
            lib.ref_rollout_affine.restype = C.c_int
            lib.ref_rollout_affine.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, dp, dp, C.c_int,
                                               C.POINTER(SqpConfig), dp, dp, ip, C.c_char_p]
        _loaded[kind] = lib
    return _loaded[kind]


@dataclass
class SolveOut:
    z: np.ndarray
    lam: np.ndarray
    sqp_iters: int
    converged: bool
    kkt: float
    pcg_iters: list = field(default_factory=list)
    step_sizes: list = field(default_factory=list)


class Oracle:
    """One problem's solver state in the chosen checker (port or ref)."""

    def __init__(self, kind: str, prob: Problem):
        self.kind, self.prob = kind, prob
        self.lib = load(kind)
        self.nz, self.nl = sizes(prob)
        self.nth = theta_size(prob)
        self.h = getattr(self.lib, kind + "_create")(C.byref(prob))
        if not self.h:
            raise ValueError("oracle: unsupported problem")

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            getattr(self.lib, self.kind + "_destroy")(h)
            self.h = None

    def _f(self, name):
        return getattr(self.lib, self.kind + "_" + name)

    @staticmethod
    def _check(rc, st):
        if rc != 0:
            raise OracleError(st)

    def linearize(self, theta, z, eps_pd=1e-6):
        st = Status()
        self._check(self._f("linearize")(self.h, _p(_arr(theta, self.nth)), _p(_arr(z, self.nz)), eps_pd,
                                         C.byref(st)), st)

    def assemble(self):
        st = Status()
        self._check(self._f("assemble")(self.h, C.byref(st)), st)

    def flat_b(self):
        b = np.zeros(self.nz)
        self._f("flat_b")(self.h, _p(b))
        return b

    def flat_d(self):
        d = np.zeros(self.nl)
        self._f("flat_d")(self.h, _p(d))
        return d

    def gamma(self, b, d):
        out = np.zeros(self.nl)
        st = Status()
        self._check(self._f("gamma")(self.h, _p(_arr(b, self.nz)), _p(_arr(d, self.nl)), _p(out), C.byref(st)), st)
        return out

    def pcg(self, gamma, lambda0, epsilon=1e-12, max_iters=0):
        lam = np.zeros(self.nl)
        it, conv, feta, st = C.c_int(), C.c_int(), C.c_double(), Status()
        self._check(self._f("pcg")(self.h, _p(_arr(gamma, self.nl)), _p(_arr(lambda0, self.nl)), epsilon, max_iters,
                                   _p(lam), C.byref(it), C.byref(feta), C.byref(conv), None, 0, C.byref(st)), st)
        return lam, it.value, feta.value, bool(conv.value)

    def recover(self, lam, b):
        z = np.zeros(self.nz)
        st = Status()
        self._check(self._f("recover")(self.h, _p(_arr(lam, self.nl)), _p(_arr(b, self.nz)), _p(z), C.byref(st)), st)
        return z

    def merit(self, theta, z, mu):
        out, st = C.c_double(), Status()
        self._check(self._f("merit")(self.h, _p(_arr(theta, self.nth)), _p(_arr(z, self.nz)), mu, C.byref(out),
                                     C.byref(st)), st)
        return out.value

    def line_search(self, theta, z_old, z_qp, cfg, mu_prev=1.0):
        zn = np.zeros(self.nz)
        a, acc, mu, st = C.c_double(), C.c_int(), C.c_double(), Status()
        self._check(self._f("line_search")(self.h, _p(_arr(theta, self.nth)), _p(_arr(z_old, self.nz)),
                                           _p(_arr(z_qp, self.nz)), C.byref(cfg), mu_prev, _p(zn), C.byref(a),
                                           C.byref(acc), C.byref(mu), C.byref(st)), st)
        return zn, a.value, bool(acc.value), mu.value

    def kkt_inf_norm(self, theta, z, lam):
        out, st = C.c_double(), Status()
        self._check(self._f("kkt_inf_norm")(self.h, _p(_arr(theta, self.nth)), _p(_arr(z, self.nz)),
                                            _p(_arr(lam, self.nl)), C.byref(out), C.byref(st)), st)
        return out.value

    def sqp_solve(self, theta, z0, lambda0, cfg) -> SolveOut:
        z, lam = np.zeros(self.nz), np.zeros(self.nl)
        it, conv, kkt = C.c_int(), C.c_int(), C.c_double()
        pcg = (C.c_int * max(cfg.max_sqp_iters, 1))()
        steps = (C.c_double * max(cfg.max_sqp_iters, 1))()
        st = Status()
        self._check(self._f("sqp_solve")(self.h, _p(_arr(theta, self.nth)), _p(_arr(z0, self.nz)),
                                         _p(_arr(lambda0, self.nl)), C.byref(cfg), _p(z), _p(lam), C.byref(it),
                                         C.byref(conv), C.byref(kkt), pcg, steps, C.byref(st)), st)
        n = it.value
        return SolveOut(z, lam, n, bool(conv.value), kkt.value, list(pcg[:n]), list(steps[:n]))

    def backward(self, theta, loss_grad_z, lambda_tilde0, epsilon=1e-12, max_iters=0):
        g, lt = np.zeros(self.nth), np.zeros(self.nl)
        it, st = C.c_int(), Status()
        self._check(self._f("backward")(self.h, _p(_arr(theta, self.nth)), _p(_arr(loss_grad_z, self.nz)),
                                        _p(_arr(lambda_tilde0, self.nl)), epsilon, max_iters, _p(g), _p(lt),
                                        C.byref(it), C.byref(st)), st)
        return g, lt, it.value

    def qp(self):
        nx, nu, T = self.prob.nx, self.prob.nu, self.prob.horizon
        out = dict(Q=np.zeros((T + 1, nx, nx)), q=np.zeros((T + 1, nx)), R=np.zeros((T, nu, nu)),
                   r=np.zeros((T, nu)), Ap=np.zeros((T, nx, nx)), A=np.zeros((T, nx, nx)), B=np.zeros((T, nu, nx)),
                   C=np.zeros((T, nx)), x_s=np.zeros(nx))
        pd = C.c_int()
        self._f("get_qp")(self.h, *[_p(out[k]) for k in ("Q", "q", "R", "r", "Ap", "A", "B", "C", "x_s")],
                          C.byref(pd))
        # blocks are column-major: reinterpret (n_cols, n_rows) storage as matrices
        for k in ("Q", "R", "Ap", "A"):
            out[k] = np.ascontiguousarray(np.swapaxes(out[k], 1, 2))
        out["B"] = np.ascontiguousarray(np.swapaxes(out["B"], 1, 2))  # (T, nx, nu)
        out["pd_projected"] = bool(pd.value)
        return out

    def schur(self):
        """(S_diag, S_sub, P_diag, P_super) as (n, nx, nx) row-major matrices."""
        nx, T = self.prob.nx, self.prob.horizon
        sd, ss = np.zeros((T + 1, nx, nx)), np.zeros((T, nx, nx))
        pd, ps = np.zeros((T + 1, nx, nx)), np.zeros((T, nx, nx))
        self._f("get_schur")(self.h, _p(sd), _p(ss), _p(pd), _p(ps))
        return tuple(np.ascontiguousarray(np.swapaxes(a, 1, 2)) for a in (sd, ss, pd, ps))


def pcg_blocks(kind, s_diag, s_sub, p_diag, p_super, gamma, lambda0, epsilon=1e-12, max_iters=0,
               s_super=None, p_sub=None):
    """pcg_solve on explicit blocks given as (n, nx, nx) row-major matrices."""
    lib = load(kind)
    nb, nx, _ = s_diag.shape
    cm = lambda a: np.ascontiguousarray(np.swapaxes(a, 1, 2))  # to column-major blocks
    s_super = np.swapaxes(s_sub, 1, 2) if s_super is None else s_super
    p_sub = np.swapaxes(p_super, 1, 2) if p_sub is None else p_sub
    blocks = [cm(a) for a in (s_diag, s_sub, s_super, p_diag, p_sub, p_super)]
    lam = np.zeros(nb * nx)
    it, conv, feta, st = C.c_int(), C.c_int(), C.c_double(), Status()
    rc = getattr(lib, kind + "_pcg_blocks")(nx, nb, *[_p(b) for b in blocks], _p(_arr(gamma)), _p(_arr(lambda0)),
                                            epsilon, max_iters, _p(lam), C.byref(it), C.byref(feta), C.byref(conv),
                                            C.byref(st))
    if rc:
        raise OracleError(st)
    return lam, it.value, feta.value, bool(conv.value)


def il_epoch(kind, prob, thetas, demos, lam_cache, lt_cache, cfg, learn_start, learn_size):
    """train_il epoch body; caches are updated in place."""
    lib = load(kind)
    B = thetas.shape[0]
    loss = C.c_double()
    grad = np.zeros(learn_size)
    losses, grads = np.zeros(B), np.zeros((B, learn_size))
    sqp_it, pcg_it = np.zeros(B, np.int32), np.zeros(B, np.int64)
    st = Status()
    rc = getattr(lib, kind + "_il_epoch")(C.byref(prob), B, _p(_arr(thetas)), _p(_arr(demos)), _p(lam_cache),
                                          _p(lt_cache), C.byref(cfg), learn_start, learn_size, C.byref(loss),
                                          _p(grad), _p(losses), _p(grads),
                                          sqp_it.ctypes.data_as(C.POINTER(C.c_int)),
                                          pcg_it.ctypes.data_as(C.POINTER(C.c_long)), C.byref(st))
    if rc:
        raise OracleError(st)
    return loss.value, grad, losses, grads, sqp_it, pcg_it


def gen_uniform(seed, n, lo=0.0, hi=1.0):
    """Reference recipe of train_il's learnable-weight draw (train.hpp:61-64; ref only)."""
    out = np.zeros(n)
    load("ref").ref_gen_uniform(seed, n, lo, hi, _p(out))
    return out


def gen_aq(nx, nu, T, seed, count, convex=True):
    """Reference generators (ref only): thetas of sequential random instances."""
    lib = load("ref")
    th = np.zeros((count, nx + nu + nx * nx + nx * nu + 2 * nx))
    lib.ref_gen_aq(nx, nu, T, seed, count, 1 if convex else 0, _p(th))
    return th


def rollout_affine(nx, nu, T, thetas, x_inits, episode_length, cfg):
    """The reference's rollout + rollout_backward per instance (ref only):
    (rewards, grads, ok, messages)."""
    lib = load("ref")
    B = thetas.shape[0]
    rewards, grads = np.zeros(B), np.zeros_like(np.asarray(thetas, np.float64))
    ok = np.zeros(B, np.int32)
    msgs = C.create_string_buffer(256 * B)
    lib.ref_rollout_affine(nx, nu, T, B, _p(_arr(thetas)), _p(_arr(x_inits)), episode_length, C.byref(cfg),
                           _p(rewards), _p(grads), ok.ctypes.data_as(C.POINTER(C.c_int)), msgs)
    raw = msgs.raw
    messages = [raw[256 * j:256 * (j + 1)].split(b"\0")[0].decode() for j in range(B)]
    return rewards, grads, ok.astype(bool), messages


def rollout_attitude(T, dt, thetas, inertias, x_inits, episode_length, cfg):
    """The reference's rollout + rollout_backward with the attitude RL environment
    (train.hpp:239-263), per instance (ref only): (rewards, grads[9], ok, messages)."""
    lib = load("ref")
    B = thetas.shape[0]
    rewards, grads = np.zeros(B), np.zeros((B, 9))
    ok = np.zeros(B, np.int32)
    msgs = C.create_string_buffer(256 * B)
    lib.ref_rollout_attitude(T, dt, B, _p(_arr(thetas)), _p(_arr(inertias)), _p(_arr(x_inits)), episode_length,
                             C.byref(cfg), _p(rewards), _p(grads), ok.ctypes.data_as(C.POINTER(C.c_int)), msgs)
    raw = msgs.raw
    return rewards, grads, ok.astype(bool), [raw[256 * j:256 * (j + 1)].split(b"\0")[0].decode() for j in range(B)]


def pcg_study(tols, steps, seed=0, nx=8, nu=4, T=30):
    """The reference's pcg_study iteration counts: arrays [tol][step][pass] of
    (cold, warm) with pass 0 = forward, 1 = backward (ref only)."""
    lib = load("ref")
    n = len(tols) * steps * 2
    cold, warm = np.zeros(n, np.int32), np.zeros(n, np.int32)
    ip_ = C.POINTER(C.c_int)
    lib.ref_pcg_study(_p(_arr(np.asarray(tols, np.float64))), len(tols), steps, seed, nx, nu, T,
                      cold.ctypes.data_as(ip_), warm.ctypes.data_as(ip_))
    return cold.reshape(len(tols), steps, 2), warm.reshape(len(tols), steps, 2)


def gen_cartpole(seed, horizon, n_demos):
    lib = load("ref")
    x0 = np.zeros((n_demos, 4))
    nz = 4 * (horizon + 1) + horizon
    demos = np.zeros((n_demos, nz))
    st = Status()
    if lib.ref_gen_cartpole(seed, horizon, n_demos, _p(x0), _p(demos), C.byref(st)):
        raise OracleError(st)
    return x0, demos
