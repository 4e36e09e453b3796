"""Python mirror of the reference solver API (namespace docp, proj/include/docp)
over the C ABI of libdocp_cuda.so.

Names, argument meaning and error behaviour follow the reference:

    sqp_solve(problem, theta, z0, lambda0, cfg)        sqp.hpp:213-261
    backward_vjp(result, loss_grad_z, lambda_tilde0, cfg)  backward.hpp:27-50
    batch_solve(problem, thetas, cache, cfg)           batch.hpp:83-108
    pcg_solve / assemble_* / linearize / ...           via Batch (one call per batch)
    Error, DimensionError, EvaluationError, NumericalError, BreakdownError,
    DivergenceError                                    common.hpp:18-54
    SqpConfig, PcgConfig                               sqp.hpp:7-34, pcg.hpp:7-23
    WarmStartCache                                     batch.hpp:10-65

A "problem" is a family descriptor (the reference's OcpDefinition callbacks
cannot cross to the GPU); theta is the family's packed parameter vector, z the
flat interleaved trajectory (x_0, u_0, ..., x_T), lambda n_x (T+1).
Every compute call runs on the GPU; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _lib as L

# --------------------------------------------------------------------------- errors


class Error(RuntimeError):
    """docp::Error (common.hpp:18-22)."""


class DimensionError(Error):
    """Input sizes do not match the problem definition."""


class EvaluationError(Error):
    """A callback (family function) produced a non-finite value."""


class NumericalError(Error):
    """A factorization failed."""


class BreakdownError(Error):
    """Conjugate-gradient breakdown; carries the iteration (common.hpp:43-48)."""

    def __init__(self, msg: str, iteration: int):
        super().__init__(msg)
        self.iteration = iteration


class DivergenceError(Error):
    """Iterates became non-finite."""


class RolloutTruncation(Error):
    """A rollout abandoned because a solve failed mid-episode (batch.hpp:146-153)."""

    def __init__(self, msg, step):
        super().__init__(msg)
        self.step = step


class CudaError(Error):
    """The CUDA runtime or the ABI rejected a call."""


_BY_CODE = {L.DIMENSION: DimensionError, L.EVALUATION: EvaluationError, L.NUMERICAL: NumericalError,
            L.DIVERGENCE: DivergenceError}


def _raise_call(rc: int):
    if rc == L.OK:
        return
    msg = L.lib().docp_last_error().decode()
    cls = _BY_CODE.get(rc, CudaError)
    raise cls(msg)


def status_error(st: L.Status) -> Optional[Error]:
    """The docp::Error a per-problem status word stands for (None when OK)."""
    if st.code == L.OK:
        return None
    buf = C.create_string_buffer(256)
    L.lib().docp_format_status(C.byref(st), buf, 256)
    msg = buf.value.decode()
    if st.step > 0:
        return RolloutTruncation(msg, st.step - 1)
    if st.where == L.AT_ROLLOUT_ENV:
        return RolloutTruncation(msg, st.index)
    if st.code == L.BREAKDOWN:
        return BreakdownError(msg, st.index)
    return _BY_CODE.get(st.code, Error)(msg)


# --------------------------------------------------------------------------- configs


@dataclass
class PcgConfig:
    """PcgConfig (pcg.hpp:7-23). mode: "fast" (FMA, tree reductions) or
    "parity" (the reference's operation order, bit-identical results)."""

    epsilon: float = 1e-12
    max_iters: int = 0
    mode: str = "fast"

    def c(self) -> L.PcgConfigC:
        modes = {"fast": L.PCG_FAST, "parity": L.PCG_PARITY, "fp32": L.PCG_FP32}
        if self.mode not in modes:
            raise ValueError(f"PcgConfig.mode must be one of {sorted(modes)}, not {self.mode!r}")
        return L.PcgConfigC(self.epsilon, self.max_iters, modes[self.mode])


@dataclass
class SqpConfig:
    """SqpConfig (sqp.hpp:7-34)."""

    max_sqp_iters: int = 20
    step_candidates: Sequence[float] = (1.0, 0.7, 0.3, 0.1, 0.01)
    eta_armijo: float = 0.4
    rho_penalty: float = 0.5
    pcg: PcgConfig = field(default_factory=PcgConfig)
    convergence_tol: float = 1e-8
    mu_floor_denominator: float = 1e-12
    eps_pd: float = 1e-6

    def c(self) -> L.SqpConfigC:
        s = L.SqpConfigC()
        s.max_sqp_iters = self.max_sqp_iters
        s.n_step_candidates = len(self.step_candidates)
        if len(self.step_candidates) > L.MAX_STEP_CANDIDATES:
            raise DimensionError(f"at most {L.MAX_STEP_CANDIDATES} step candidates")
        for i, a in enumerate(self.step_candidates):
            s.step_candidates[i] = a
        s.eta_armijo, s.rho_penalty = self.eta_armijo, self.rho_penalty
        s.pcg = self.pcg.c()
        s.convergence_tol, s.mu_floor_denominator, s.eps_pd = (self.convergence_tol, self.mu_floor_denominator,
                                                               self.eps_pd)
        return s


def one_shot_config(epsilon: float = 1e-12, mode: str = "fast") -> SqpConfig:
    """test_support.hpp:13-19 / the CLI grad-check config (docp_main.cpp:104-106)."""
    return SqpConfig(max_sqp_iters=1, step_candidates=(1.0,), pcg=PcgConfig(epsilon, 0, mode))


# --------------------------------------------------------------------------- problems


def affine_quadratic(n_x: int, n_u: int, horizon: int, cost_scale: float = 1.0) -> L.Problem:
    """AffineQuadratic family (affine_quadratic.hpp:14-120); theta =
    [w_x | w_u | vec(A) | vec(B) | b | x_s] (column-major A, B)."""
    return L.Problem(L.AFFINE_QUADRATIC, n_x, n_u, horizon, cost_scale, 0.0, 0.0, 0.0, 0.0, 0.0)


def cartpole(horizon: int = 40, cart_mass: float = 1.0, pole_mass: float = 0.1, length: float = 0.5,
             gravity: float = 9.81, dt: float = 0.05) -> L.Problem:
    """Cart-pole family (cartpole.hpp:17-107); theta = [w_x(4) | w_u(1) | x_0(4)]."""
    return L.Problem(L.CARTPOLE, 4, 1, horizon, 0.5, cart_mass, pole_mass, length, gravity, dt)


def attitude(horizon: int = 25, dt: float = 0.1) -> L.Problem:
    """Attitude-rate family (attitude.hpp:10-72). Device theta =
    [w_x(3) | w_u(3) | omega_0(3) | inertia(3)]: make_attitude_theta's 9
    entries, then the instance's AttitudeParams::inertia (d theta of it is 0)."""
    return L.Problem(L.ATTITUDE, 3, 3, horizon, 0.5, 0.0, 0.0, 0.0, 0.0, dt)


# The drifting family (include/docp_drift_model.h). No
# reference implementation or generator exists. Nominal vehicle: the paper's
# Table (a, b, m, r_w, C_f, C_r, mu_f, mu_r) plus our I_z and path curvature
# kappa (a 10 m circle); the reference state is the model's steady cornering
# equilibrium at 8 m/s on that circle, heading offset -beta so the velocity is
# tangent to the path (f(X_ref, 0) = 0 to 1e-15 except ds/dt = V, computed with
# scipy.optimize.fsolve on the model); the weights follow the paper's emphasis
# on sideslip, heading and lateral error, rescaled so the QPs stay well posed.
DRIFT_PARAMS = np.array([1.239, 1.209, 1476.0, 2200.0, 0.323, 54000.0, 220000.0, 0.99, 0.90, 0.1])
DRIFT_REF_STATE = np.array([0.80000000000000004, 8.0, 0.089764022782235914, -0.089764022782235914, 0.0, 0.0,
                            0.33936077951463062, 0.79350102041864212])
DRIFT_W_X = np.array([1.0, 0.1, 50.0, 20.0, 30.0, 1e-3, 1.0, 1.0])
DRIFT_W_U = np.array([10.0, 1.0])
_DRIFT_X0_SPREAD = np.array([0.05, 0.3, 0.03, 0.05, 0.2, 0.0, 0.02, 0.06])


def drift(horizon: int = 100, dt: float = 0.1) -> L.Problem:
    """Drifting family: n_x = 8 (6 vehicle / path states + steering and drive
    force), n_u = 2 (their rates), Heun sub-steps over dt. theta = [w_x 8 |
    w_u 2 | xbar_0 8 | X_ref 8 | a, b, m, I_z, r_w, C_f, C_r, mu_f, mu_r, kappa]."""
    return L.Problem(L.DRIFT, 8, 2, horizon, 0.5, 0.0, 0.0, 0.0, 0.0, dt)


def drift_thetas(count: int, seed: int = 0, spread: float = 0.1, w_x=None, w_u=None) -> np.ndarray:
    """Domain-randomised drifting instances [count][36]: every vehicle parameter
    drawn from U(1 - spread, 1 + spread) times nominal, the initial deviation
    from U(-1, 1) times a per-state scale (numpy PCG64, seeded)."""
    rng = np.random.default_rng(seed)
    th = np.zeros((count, 36))
    th[:, 0:8] = DRIFT_W_X if w_x is None else w_x
    th[:, 8:10] = DRIFT_W_U if w_u is None else w_u
    th[:, 10:18] = rng.uniform(-1.0, 1.0, (count, 8)) * _DRIFT_X0_SPREAD
    th[:, 18:26] = DRIFT_REF_STATE
    th[:, 26:36] = DRIFT_PARAMS * rng.uniform(1.0 - spread, 1.0 + spread, (count, 10))
    return th


def theta_size(problem: L.Problem) -> int:
    return L.lib().docp_theta_size(C.byref(problem))


def sizes(problem: L.Problem):
    """(n_z, n_lambda) — OcpDefinition::primal_size / dual_size (problem.hpp:56-62)."""
    nl = problem.n_x * (problem.horizon + 1)
    return nl + problem.n_u * problem.horizon, nl


def flat_offset(n_x: int, n_u: int, t: int, state: bool) -> int:
    """trajectory.hpp:72-74"""
    return t * (n_x + n_u) + (0 if state else n_x)


def describe(problem: L.Problem) -> str:
    buf = C.create_string_buffer(256)
    L.lib().docp_describe(C.byref(problem), buf, 256)
    return buf.value.decode()


def pcg_invocations() -> int:
    """stats::pcg_invocations (common.hpp:112-115): solves performed."""
    return int(L.lib().docp_pcg_invocations())


def kernel_launches() -> int:
    return int(L.lib().docp_kernel_launches())


# --------------------------------------------------------------------------- synthetic inputs


def generate_affine_quadratic(n_x: int, n_u: int, seed: int, count: int, convex: bool = True) -> np.ndarray:
    """Sequential random_convex_instance / random_linear_instance draws
    (generators.hpp:52-111) as thetas [count][n_theta]."""
    out = np.zeros((count, n_x + n_u + n_x * n_x + n_x * n_u + 2 * n_x))
    _raise_call(L.lib().docp_generate_affine_quadratic(n_x, n_u, seed, count, 1 if convex else 0,
                                                       out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


def generate_drift_sequence(n_x: int, n_u: int, seed: int, steps: int, magnitude: float = 0.01) -> np.ndarray:
    """pcg_study's slowly drifting instance sequence (study.hpp:37-48, 74-124), [steps][n_theta]."""
    out = np.zeros((steps, n_x + n_u + n_x * n_x + n_x * n_u + 2 * n_x))
    _raise_call(L.lib().docp_generate_drift_sequence(n_x, n_u, seed, steps, magnitude,
                                                     out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


def generate_uniform(seed: int, n: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
    out = np.zeros(n)
    _raise_call(L.lib().docp_generate_uniform(seed, n, lo, hi, out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


def generate_cartpole_x0(seed: int, n: int) -> np.ndarray:
    """gen_cartpole initial states (generators.hpp:142-152)."""
    out = np.zeros((n, 4))
    _raise_call(L.lib().docp_generate_cartpole_x0(seed, n, out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


# --------------------------------------------------------------------------- batch

_FLOAT_FIELDS = {L.F_THETA, L.F_Z, L.F_LAMBDA, L.F_LAMBDA_TILDE, L.F_LOSS_GRAD_Z, L.F_GRAD_THETA, L.F_GAMMA,
                 L.F_Z_QP, L.F_KKT, L.F_FINAL_ETA, L.F_STEP_SIZES, L.F_MU, L.F_ALPHA, L.F_LOSS, L.F_REWARD}


class Batch:
    """A device-resident batch of same-shaped problems (docp_batch)."""

    def __init__(self, problem: L.Problem, batch_size: int, device: int = 0):
        self.problem = problem
        self.B = int(batch_size)
        self.nz, self.nl = sizes(problem)
        self.nth = theta_size(problem)
        h = C.c_void_p()
        _raise_call(L.lib().docp_batch_create(C.byref(problem), self.B, device, C.byref(h)))
        self.h = h

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            try:
                L.lib().docp_batch_destroy(h)
            except TypeError:  # interpreter shutdown: module globals already cleared
                pass
            self.h = None

    # ---- data
    def field_ptr(self, f: int):
        p, n = C.c_void_p(), C.c_size_t()
        _raise_call(L.lib().docp_batch_field_ptr(self.h, f, C.byref(p), C.byref(n)))
        return p.value, n.value

    def set_stream(self, stream_handle: int):
        _raise_call(L.lib().docp_batch_set_stream(self.h, C.c_void_p(stream_handle)))

    def sync(self):
        _raise_call(L.lib().docp_batch_sync(self.h))

    def upload(self, f: int, a):
        """Host array (synchronous copy) or a CUDA tensor (device-to-device
        copy ordered on the batch's stream)."""
        if getattr(a, "is_cuda", False):
            _, n = self.field_ptr(f)
            if not a.is_contiguous() or a.numel() * a.element_size() != n:
                raise DimensionError(f"field {f}: expected {n} contiguous bytes")
            _raise_call(L.lib().docp_batch_upload(self.h, f, C.c_void_p(a.data_ptr()), 1))
            return
        dtype = np.float64 if f in _FLOAT_FIELDS else np.int32
        arr = np.ascontiguousarray(a, dtype=dtype)
        _, n = self.field_ptr(f)
        if arr.nbytes != n:
            raise DimensionError(f"field {f}: expected {n} bytes, got {arr.nbytes}")
        _raise_call(L.lib().docp_batch_upload(self.h, f, arr.ctypes.data, 0))

    def download(self, f: int) -> np.ndarray:
        _, n = self.field_ptr(f)
        if f in (L.F_STATUS, L.F_ROLLOUT_STATUS):
            arr = np.zeros((self.B, 4), np.int32)
        else:
            dtype = np.float64 if f in _FLOAT_FIELDS else np.int32
            arr = np.zeros(n // np.dtype(dtype).itemsize, dtype)
            arr = arr.reshape(self.B, -1)
        _raise_call(L.lib().docp_batch_download(self.h, f, arr.ctypes.data, 0))
        return arr

    def statuses(self) -> List[L.Status]:
        raw = self.download(L.F_STATUS)
        return [L.Status(*map(int, row)) for row in raw]

    def errors(self) -> List[Optional[Error]]:
        return [status_error(s) for s in self.statuses()]

    def upload_schur(self, s_diag, s_sub, p_diag, p_super):
        """Blocks as (B, n, n_x, n_x) row-major matrices (reference semantics)."""
        cm = lambda a: np.ascontiguousarray(np.swapaxes(np.asarray(a, np.float64), -1, -2))
        arrs = [cm(a) for a in (s_diag, s_sub, p_diag, p_super)]
        ptr = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
        _raise_call(L.lib().docp_batch_upload_schur(self.h, *[ptr(a) for a in arrs]))

    def download_schur(self):
        nx, T = self.problem.n_x, self.problem.horizon
        sd, ss = np.zeros((self.B, T + 1, nx, nx)), np.zeros((self.B, T, nx, nx))
        pd, ps = np.zeros((self.B, T + 1, nx, nx)), np.zeros((self.B, T, nx, nx))
        ptr = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
        _raise_call(L.lib().docp_batch_download_schur(self.h, ptr(sd), ptr(ss), ptr(pd), ptr(ps)))
        sw = lambda a: np.ascontiguousarray(np.swapaxes(a, -1, -2))
        return sw(sd), sw(ss), sw(pd), sw(ps)

    def download_qp(self):
        nx, nu, T, B = self.problem.n_x, self.problem.n_u, self.problem.horizon, self.B
        out = dict(Q=np.zeros((B, T + 1, nx, nx)), q=np.zeros((B, T + 1, nx)), R=np.zeros((B, T, nu, nu)),
                   r=np.zeros((B, T, nu)), A=np.zeros((B, T, nx, nx)), B=np.zeros((B, T, nu, nx)),
                   C=np.zeros((B, T, nx)), x_s=np.zeros((B, nx)))
        ptr = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
        _raise_call(L.lib().docp_batch_download_qp(self.h, *[ptr(out[k]) for k in
                                                             ("Q", "q", "R", "r", "A", "B", "C", "x_s")]))
        for k in ("Q", "R", "A", "B"):
            out[k] = np.ascontiguousarray(np.swapaxes(out[k], -1, -2))
        return out

    # ---- profiling (CUDA events around every launch on the batch stream)
    def profile_begin(self):
        _raise_call(L.lib().docp_profile_begin(self.h))

    def profile_end(self) -> dict:
        p = L.Profile()
        _raise_call(L.lib().docp_profile_end(self.h, C.byref(p)))
        kinds = {n: {"launches": int(p.launches[i]), "ms": float(p.ms[i])} for i, n in enumerate(L.PROF_NAMES)}
        return {"kernels": kinds, "pcg_iterations": int(p.pcg_iterations), "pcg_solves": int(p.pcg_solves),
                "pcg_bytes_per_iteration": float(p.pcg_bytes_per_iteration),
                "pcg_algorithmic_bytes": float(p.pcg_algorithmic_bytes),
                "span_ms": float(p.span_ms), "gap_ms": float(p.gap_ms), "max_gap_ms": float(p.max_gap_ms),
                "max_gap_between": [L.PROF_NAMES[k] if 0 <= k < len(L.PROF_NAMES) else None
                                    for k in (p.max_gap_after, p.max_gap_before)]}

    # ---- primitives (one call each for the whole batch)
    def linearize(self, eps_pd: float = 1e-6):
        _raise_call(L.lib().docp_linearize(self.h, eps_pd))

    def assemble_schur(self):
        _raise_call(L.lib().docp_assemble_schur(self.h))

    def assemble_gamma(self, rhs: int = L.RHS_FORWARD):
        _raise_call(L.lib().docp_assemble_gamma(self.h, rhs))

    def pcg_solve(self, cfg: PcgConfig, solution_field: int = L.F_LAMBDA):
        c = cfg.c()
        _raise_call(L.lib().docp_pcg_solve(self.h, C.byref(c), solution_field))

    def recover_primal(self, lambda_field: int = L.F_LAMBDA, rhs: int = L.RHS_FORWARD):
        _raise_call(L.lib().docp_recover_primal(self.h, lambda_field, rhs))

    def line_search(self, cfg: SqpConfig):
        c = cfg.c()
        _raise_call(L.lib().docp_line_search(self.h, C.byref(c)))

    def kkt_residual(self):
        _raise_call(L.lib().docp_kkt_residual(self.h))

    def sqp_solve(self, cfg: SqpConfig):
        c = cfg.c()
        _raise_call(L.lib().docp_sqp_solve(self.h, C.byref(c)))

    def backward_vjp(self, cfg: PcgConfig):
        c = cfg.c()
        _raise_call(L.lib().docp_backward_vjp(self.h, C.byref(c)))

    def il_epoch(self, cfg: SqpConfig, weights_ptr: int, learn_start: int, learn_size: int, demos_ptr: int,
                 loss_denominator: float, loss_sum_ptr: int, grad_sum_ptr: int):
        """Device pointers in, device pointers out (train.hpp:82-131)."""
        c = cfg.c()
        _raise_call(L.lib().docp_il_epoch(self.h, C.byref(c), weights_ptr, learn_start, learn_size, demos_ptr,
                                          loss_denominator, loss_sum_ptr, grad_sum_ptr))

    def il_failures(self) -> Tuple[int, int]:
        """(failed demonstrations since the last call, first failed index or -1);
        waits for the batch's stream and resets the count."""
        n, first = C.c_int32(0), C.c_int32(0)
        _raise_call(L.lib().docp_il_failures(self.h, C.byref(n), C.byref(first)))
        return int(n.value), int(first.value)

    def il_check(self, epoch: int = 0):
        """Raises like train_il (train.hpp:111-119) when a demonstration of the
        epochs since the last check failed: "epoch E, demonstration J: <error>"."""
        n, first = self.il_failures()
        if n:
            st = self.download(L.F_STATUS)[first]
            err = status_error(L.Status(*[int(x) for x in st]))
            msg = f"epoch {epoch}, demonstration {first}: {err}"
            if isinstance(err, BreakdownError):
                raise BreakdownError(msg, err.iteration)
            raise type(err)(msg)


    def rollout(self, cfg: SqpConfig, x_init, episode_length: int):
        """Closed-loop MPC rollouts (batch.hpp:172-212) from x_init [B][n_x]
        (a device pointer as int, or a host array); totals in REWARD,
        truncations in ROLLOUT_STATUS."""
        c = cfg.c()
        if isinstance(x_init, int):
            _raise_call(L.lib().docp_rollout(self.h, C.byref(c), x_init, 1, episode_length))
        else:
            arr = np.ascontiguousarray(x_init, dtype=np.float64)
            if arr.size != self.B * self.problem.n_x:
                raise DimensionError("rollout: initial state length mismatch")
            _raise_call(L.lib().docp_rollout(self.h, C.byref(c), arr.ctypes.data, 0, episode_length))

    def rollout_backward(self, cfg: PcgConfig):
        """rollout_backward (batch.hpp:221-258) of the last rollout into GRAD_THETA."""
        c = cfg.c()
        _raise_call(L.lib().docp_rollout_backward(self.h, C.byref(c)))

    def rollout_errors(self) -> List[Optional[Error]]:
        st = self.download(L.F_ROLLOUT_STATUS)
        return [status_error(L.Status(*[int(x) for x in st[j]])) for j in range(self.B)]


# --------------------------------------------------------------------------- results


@dataclass
class SolveResult:
    """SolveResult (sqp.hpp:40-52). qp/schur stay device-resident in `batch`
    (slot `index`) for backward_vjp."""

    z: np.ndarray
    lam: np.ndarray
    sqp_iters: int
    kkt_inf_norm: float
    converged: bool
    pcg_iters: List[int]
    step_sizes: List[float]
    batch: Batch = field(repr=False, default=None)
    index: int = 0


@dataclass
class BackwardResult:
    """BackwardResult (backward.hpp:7-12)."""

    grad_theta: np.ndarray
    lambda_tilde: np.ndarray
    pcg_iters: int


@dataclass
class BatchItem:
    """BatchItem (batch.hpp:72-77)."""

    ok: bool
    result: Optional[SolveResult]
    error: str = ""


def _results(b: Batch, cfg: SqpConfig):
    z, lam = b.download(L.F_Z), b.download(L.F_LAMBDA)
    it, conv, kkt = b.download(L.F_SQP_ITERS)[:, 0], b.download(L.F_CONVERGED)[:, 0], b.download(L.F_KKT)[:, 0]
    hist, steps = b.download(L.F_PCG_HISTORY), b.download(L.F_STEP_SIZES)
    out = []
    for j in range(b.B):
        n = int(it[j])
        out.append(SolveResult(z[j].copy(), lam[j].copy(), n, float(kkt[j]), bool(conv[j]),
                               [int(x) for x in hist[j, :n]], [float(x) for x in steps[j, :n]], b, j))
    return out


def sqp_solve_batch(problem: L.Problem, thetas, z0, lambda0, cfg: SqpConfig = None, device: int = 0):
    """Batched sqp_solve: returns (results, errors) with one entry per problem."""
    cfg = cfg or SqpConfig()
    thetas = np.atleast_2d(np.asarray(thetas, np.float64))
    b = Batch(problem, thetas.shape[0], device)
    b.upload(L.F_THETA, thetas)
    b.upload(L.F_Z, np.broadcast_to(np.asarray(z0, np.float64), (b.B, b.nz)))
    b.upload(L.F_LAMBDA, np.broadcast_to(np.asarray(lambda0, np.float64), (b.B, b.nl)))
    b.sqp_solve(cfg)
    return _results(b, cfg), b.errors()


def sqp_solve(problem: L.Problem, theta, z0, lambda0, cfg: SqpConfig = None, device: int = 0) -> SolveResult:
    """sqp_solve (sqp.hpp:213-261) for one problem; raises the docp error."""
    theta = np.asarray(theta, np.float64)
    nz, nl = sizes(problem)
    if theta.size != theta_size(problem) or np.asarray(z0).size != nz:
        raise DimensionError("trajectory dimensions do not match the problem")
    if np.asarray(lambda0).size != nl:
        raise DimensionError("sqp: dual guess length mismatch")
    res, errs = sqp_solve_batch(problem, theta[None], np.asarray(z0)[None], np.asarray(lambda0)[None], cfg, device)
    if errs[0] is not None:
        raise errs[0]
    return res[0]


def backward_vjp(result: SolveResult, loss_grad_z, lambda_tilde0, cfg: PcgConfig = None) -> BackwardResult:
    """backward_vjp (backward.hpp:27-50) on the resident forward result. For
    a result from a batch, runs the backward pass of the whole batch slot set
    with zero cotangents elsewhere untouched (use backward_vjp_batch)."""
    b = result.batch
    grads, lts, its, errs = backward_vjp_batch(
        b, _only(b, result.index, loss_grad_z, b.nz), _only(b, result.index, lambda_tilde0, b.nl), cfg)
    if errs[result.index] is not None:
        raise errs[result.index]
    return BackwardResult(grads[result.index], lts[result.index], int(its[result.index]))


def _only(b: Batch, j: int, vec, n: int):
    vec = np.asarray(vec, np.float64)
    if vec.size != n:
        raise DimensionError("backward_vjp: cotangent length mismatch" if n == b.nz else
                             "backward_vjp: warm start length mismatch")
    out = np.zeros((b.B, n))
    out[j] = vec
    return out


def backward_vjp_batch(b: Batch, loss_grad_z, lambda_tilde0, cfg: PcgConfig = None):
    cfg = cfg or PcgConfig()
    b.upload(L.F_LOSS_GRAD_Z, loss_grad_z)
    b.upload(L.F_LAMBDA_TILDE, lambda_tilde0)
    b.backward_vjp(cfg)
    return (b.download(L.F_GRAD_THETA), b.download(L.F_LAMBDA_TILDE), b.download(L.F_PCG_ITERS)[:, 0], b.errors())


class WarmStartCache:
    """WarmStartCache (batch.hpp:10-65): per-instance (z, lambda, lambda~);
    cleared slots read as zeros."""

    def __init__(self, problem: L.Problem, n: int = 0):
        self.nz, self.nl = sizes(problem)
        self.resize(n)
        self.generation = 0

    def resize(self, n: int):
        self.z = np.zeros((n, self.nz))
        self.lam = np.zeros((n, self.nl))
        self.lam_tilde = np.zeros((n, self.nl))
        self.valid = np.zeros(n, bool)

    def __len__(self):
        return len(self.valid)

    def store(self, i, z, lam):
        self.z[i], self.lam[i], self.valid[i] = z, lam, True

    def store_backward(self, i, lam_tilde):
        self.lam_tilde[i] = lam_tilde


def batch_solve(problem: L.Problem, thetas, cache: WarmStartCache, cfg: SqpConfig = None,
                device: int = 0) -> List[BatchItem]:
    """batch_solve (batch.hpp:83-108): warm-started from the cache, per-item
    failures reported without aborting the batch, cache stored afterwards."""
    thetas = np.atleast_2d(np.asarray(thetas, np.float64))
    if len(cache) != thetas.shape[0]:
        cache.resize(thetas.shape[0])
    res, errs = sqp_solve_batch(problem, thetas, cache.z, cache.lam, cfg, device)
    items = [BatchItem(e is None, r if e is None else None, "" if e is None else str(e)) for r, e in zip(res, errs)]
    for i, it in enumerate(items):
        if it.ok:
            cache.store(i, it.result.z, it.result.lam)
    cache.generation += 1
    return items
