// k_step.cuh — K3 (SQP merit + line search + convergence test), the KKT
// diagnostic, K4's theta-VJP contraction and the imitation-learning epoch
// helpers.
//
//   line_search + sqp loop body   sqp.hpp:151-206, 236-251
//   merit_parts                   sqp.hpp:98-123
//   kkt_residual                  problem.hpp:263-300
//   theta_vjp                     affine_quadratic.hpp:82-117, quadratic_cost.hpp:24-45
//   train_il epoch body           train.hpp:87-131
//
// Per-stage terms are evaluated in parallel (one thread per (candidate,
// stage) task); every sum the reference accumulates is then folded by one
// thread in the reference's order, so the line-search decision sees exactly
// the reference's numbers.
#pragma once

#include "families.cuh"

namespace docp_dev {

constexpr int kStepThreads = 128;

struct StepCfg {
  int n_alpha;
  double alphas[DOCP_MAX_STEP_CANDIDATES];
  double eta_armijo, rho_penalty, mu_floor, conv_tol;
  int iter;       // SQP iteration index (history slot)
  int max_iters;  // cfg.max_sqp_iters
  int is_loop;    // 1: sqp loop body (update counters/convergence); 0: bare line_search
};

/// Stage terms of merit_parts at one trajectory version (old or a trial).
/// Slots: state value t -> t, control value t -> T+1+t, dynamics |res|_1
/// t -> 2T+1+t, initial-condition |x_0 - x_s|_1 -> 3T+1. zo, zq, th are the
/// problem's shared-memory copies; a non-finite cost value lowers *first_bad
/// to its slot (merit_parts throws at the first one in slot order).
template <int NX, int NU, bool DR = (NX == 0)>
__device__ inline void merit_task(const Dims& d, const Family& fam, const double* th, const double* zo,
                                  const double* zq, int P, double alpha, bool trial, int task, double* slots,
                                  int* first_bad) {
  const int nx = NX ? NX : d.nx, nu = NU ? NU : d.nu, T = d.T;
  auto xo = [&](int t) { return t * P; };       // x_t in the padded SMEM copy
  auto uo = [&](int t) { return t * P + nx; };  // u_t
  constexpr int AX = NX ? NX : kMaxNx, AU = NU ? NU : kMaxNx;
  double a[AX], b[AU], c[AX], res[AX];
  auto get = [&](int off, int n, double* out) {
#pragma unroll
    for (int i = 0; i < (NX ? (NX > NU ? NX : NU) : kMaxNx); ++i)
      if (i < n) out[i] = trial ? zo[off + i] + alpha * (zq[off + i] - zo[off + i]) : zo[off + i];
  };
  if (task <= T) {
    get(xo(task), nx, a);
    const double val = diag_cost_value<NX>(fam.scale, fam.w_x(d, th), a, nx);
    slots[task] = val;
    if (!isfinite(val)) atomicMin(first_bad, task);
  } else if (task < 2 * T + 1) {
    const int t = task - (T + 1);
    get(xo(t), nx, a);
    get(uo(t), nu, b);
    get(xo(t + 1), nx, c);
    const double val = diag_cost_value<NU>(fam.scale, fam.w_u(d, th), b, nu);
    slots[T + 1 + t] = val;
    if (!isfinite(val)) atomicMin(first_bad, T + 1 + t);
    fam.dynamics<NX, NU, DR>(d, th, c, a, b, res, nullptr, nullptr);
    double s = fabs(res[0]);
#pragma unroll
    for (int i = 1; i < nx; ++i) s = s + fabs(res[i]);
    slots[2 * T + 1 + t] = s;
  } else {
    get(xo(0), nx, a);
    const double* x_s = fam.x_s(d, th);
    double s = fabs(a[0] - x_s[0]);
#pragma unroll
    for (int i = 1; i < nx; ++i) s = s + fabs(a[i] - x_s[i]);
    slots[3 * T + 1] = s;
  }
}

/// Folds one version's slots in merit_parts order (sqp.hpp:102-121). Only
/// called when every cost slot is finite.
__device__ inline void merit_fold(const Dims& d, const double* slots, double* cost, double* viol) {
  const int T = d.T;
  double c = 0.0, v = 0.0;
#pragma unroll 4
  for (int t = 0; t <= T; ++t) c = c + slots[t];
#pragma unroll 4
  for (int t = 0; t < T; ++t) {
    c = c + slots[T + 1 + t];
    v = v + slots[2 * T + 1 + t];
  }
  v = v + slots[3 * T + 1];
  *cost = c;
  *viol = v;
}

/// Dynamic shared memory of step_kernel (doubles): z_old, z_qp, theta, the
/// merit slots of every version and the d_cost / curvature stage terms.
/// z is staged with stage stride P = n_x + n_u + 1 (odd: the per-stage walks
/// of consecutive threads land on distinct banks).
/// Long horizons whose staged copies do not fit read z and theta from global
/// memory instead (STAGE = false), keeping only the merit slots in SMEM.
__host__ __device__ inline int step_stride(const Dims& d) { return d.nx + d.nu + 1; }
__host__ __device__ inline long step_smem_doubles(const Dims& d, int n_alpha, bool stage = true) {
  const long zs = stage ? static_cast<long>(d.T + 1) * step_stride(d) : 0;
  return 2L * zs + (stage ? d.nth : 0) + static_cast<long>(n_alpha + 1) * (3 * d.T + 2) + 2L * (2 * d.T + 1);
}

/// K3: line search from Z toward Z_QP and the SQP-loop bookkeeping
/// (sqp.hpp:151-206, 236-251). One CTA per problem: the problem's z_old,
/// z_qp and theta are staged in shared memory, the stage terms of every
/// version are evaluated in parallel, and each sum is folded by one thread
/// in the reference's order. NX, NU > 0 fix the block sizes at compile time.
template <int NX, int NU, bool STAGE = true, bool DR = (NX == 0)>
__global__ void __launch_bounds__(kStepThreads) step_kernel(View v, const int* __restrict__ work,
                                                           const int* __restrict__ n_work, StepCfg cfg) {
  extern __shared__ double sm_step[];
  __shared__ double s_dc, s_cv, s_mu, s_alpha, s_step;
  __shared__ double s_cost[DOCP_MAX_STEP_CANDIDATES + 1], s_viol[DOCP_MAX_STEP_CANDIDATES + 1];
  __shared__ int s_bad[DOCP_MAX_STEP_CANDIDATES + 1];
  __shared__ int s_nonfinite, s_accepted;
  const Dims d = v.d;
  const int nx = NX ? NX : d.nx, nu = NU ? NU : d.nu, T = d.T;
  const Family fam = Family::from(v.prob);
  const int tid = threadIdx.x;
  const int nslot = 3 * T + 2;
  const int nver = cfg.n_alpha + 1;
  const int P = STAGE ? step_stride(d) : nx + nu;  // stage stride of the z copies read below
  const int zs = STAGE ? (T + 1) * P : 0;
  double* szo = sm_step;                                   // [T+1][P] padded stages (STAGE)
  double* szq = szo + zs;                                  // [T+1][P]
  double* sth = szq + zs;                                  // [nth]
  double* slots = sth + (STAGE ? d.nth : 0);               // [nver][nslot]
  double* dterm = slots + static_cast<long>(nver) * nslot;  // [2T+1] d_cost terms
  double* cterm = dterm + 2 * T + 1;                       // [2T+1] curvature terms

  for (int w = blockIdx.x; w < *n_work; w += gridDim.x) {
    const int p = work[w];
    if (v.status[p].code != DOCP_OK) continue;
    double* zo = v.z + static_cast<long>(p) * d.nz;
    if constexpr (STAGE) {
      const double* th = v.theta + static_cast<long>(p) * d.nth;
      const double* zq = v.zqp + static_cast<long>(p) * d.nz;
      auto padded = [&](int e) {
        const int t = e / (nx + nu);
        return t * P + (e - t * (nx + nu));
      };
      cta_stage<4>(szo, zo, d.nz, padded);
      cta_stage<4>(szq, zq, d.nz, padded);
      cta_stage(sth, th, d.nth);
    } else {  // the flat layout has the same stage stride: read in place
      szo = zo;
      szq = v.zqp + static_cast<long>(p) * d.nz;
      sth = v.theta + static_cast<long>(p) * d.nth;
    }
    if (tid < nver) s_bad[tid] = 0x7fffffff;
    __syncthreads();
    const double* qd = v.qd + static_cast<long>(p) * d.nb * nx;
    const double* rd = v.rd + static_cast<long>(p) * T * nu;

    // d_cost and curvature stage terms (sqp.hpp:161-172): unprojected
    // gradients at z_old, projected Q / R
    for (int t = tid; t < 2 * T + 1; t += blockDim.x) {
      const bool st = t <= T;
      const int s = st ? t : t - (T + 1);
      const int n = st ? nx : nu;
      const int off = st ? s * P : s * P + nx;
      const double* wt = st ? fam.w_x(d, sth) : fam.w_u(d, sth);
      const double* h = st ? qd + s * nx : rd + s * nu;
      double dc = 0.0, cv = 0.0;
      for (int i = 0; i < n; ++i) {
        const double dx = szq[off + i] - szo[off + i];
        const double g = diag_cost_grad(fam.scale, wt[i], szo[off + i]);
        const double qdx = h[i] * dx;
        dc = i == 0 ? g * dx : dc + g * dx;
        cv = i == 0 ? dx * qdx : cv + dx * qdx;
      }
      dterm[t] = dc;
      cterm[t] = cv;
    }
    for (int task = tid; task < nver * (2 * T + 2); task += blockDim.x) {
      const int ver = task / (2 * T + 2);
      const int tt = task - ver * (2 * T + 2);
      merit_task<NX, NU, DR>(d, fam, sth, szo, szq, P, ver == 0 ? 0.0 : cfg.alphas[ver - 1], ver > 0, tt,
                         slots + static_cast<long>(ver) * nslot, &s_bad[ver]);
    }
    __syncthreads();
    if (tid == 0) {
      double dc = 0.0, cv = 0.0;
#pragma unroll 4
      for (int t = 0; t < 2 * T + 1; ++t) {
        dc = dc + dterm[t];
        cv = cv + cterm[t];
      }
      s_dc = dc;
      s_cv = cv;
    } else if (tid - 1 < nver) {
      const int ver = tid - 1;
      if (s_bad[ver] == 0x7fffffff) {
        double c = 0.0, vv = 0.0;
        merit_fold(d, slots + static_cast<long>(ver) * nslot, &c, &vv);
        s_cost[ver] = c;
        s_viol[ver] = vv;
      }
    }
    __syncthreads();
    if (tid == 0) {
      int err_ver = -1;
      for (int ver = 0; ver < nver; ++ver)
        if (s_bad[ver] != 0x7fffffff) {
          err_ver = ver;
          break;
        }
      if (err_ver >= 0) {
        const int slot = s_bad[err_ver];
        if (slot <= T) set_status(v.status + p, DOCP_EVALUATION, DOCP_AT_MERIT_STATE, slot);
        else set_status(v.status + p, DOCP_EVALUATION, DOCP_AT_MERIT_CONTROL, slot - (T + 1));
        s_alpha = -1.0;
      } else {
        // penalty rule (sqp.hpp:174-183)
        const double viol = s_viol[0];
        double mu = v.mu[p];
        if (viol >= cfg.mu_floor) {
          const double required = (s_dc + 0.5 * s_cv) / ((1.0 - cfg.rho_penalty) * viol);
          if (isfinite(required) && required > mu) mu = required;
        }
        const double phi_old = s_cost[0] + mu * viol;
        const double descent = s_dc - mu * viol;
        double alpha = cfg.alphas[cfg.n_alpha - 1];
        int acc = 0;
        for (int c = 0; c < cfg.n_alpha; ++c) {
          const double merit = s_cost[c + 1] + mu * s_viol[c + 1];
          const double dphi = merit - phi_old - cfg.eta_armijo * cfg.alphas[c] * descent;
          if (dphi < 0.0) {
            alpha = cfg.alphas[c];
            acc = 1;
            break;
          }
        }
        s_mu = mu;
        s_alpha = alpha;
        s_accepted = acc;
      }
      s_nonfinite = 0;
      s_step = 0.0;
    }
    __syncthreads();
    const double alpha = s_alpha;
    if (alpha < 0.0) {  // merit evaluation failed
      __syncthreads();
      continue;
    }
    // z_new = z_old.interpolate(z_qp, alpha) and the step norm (trajectory.hpp:57-68)
    double stepmax = 0.0;
    for (int e = tid; e < d.nz; e += blockDim.x) {
      const int t = e / (nx + nu), k = t * P + (e - t * (nx + nu));
      const double zn = szo[k] + alpha * (szq[k] - szo[k]);
      if (!isfinite(zn)) s_nonfinite = 1;
      stepmax = fmax(stepmax, fabs(zn - szo[k]));
    }
    stepmax = warp_max(stepmax);
    if ((tid & 31) == 0) atomicMax(reinterpret_cast<unsigned long long*>(&s_step), __double_as_longlong(stepmax));
    __syncthreads();
    const bool diverged = s_nonfinite != 0;
    if (!diverged)
      for (int e = tid; e < d.nz; e += blockDim.x) {
        const int t = e / (nx + nu), k = t * P + (e - t * (nx + nu));
        zo[e] = szo[k] + alpha * (szq[k] - szo[k]);
      }
    if (tid == 0) {
      v.mu[p] = s_mu;
      v.alpha[p] = alpha;
      v.accepted[p] = s_accepted;
      if (diverged) {
        set_status(v.status + p, DOCP_DIVERGENCE, DOCP_AT_SQP_ITERATE, cfg.iter + 1);
      } else if (cfg.is_loop) {
        v.step_sizes[static_cast<long>(p) * v.max_hist + cfg.iter] = alpha;
        v.pcg_hist[static_cast<long>(p) * v.max_hist + cfg.iter] = v.pcg_iters[p];
        v.sqp_iters[p] = cfg.iter + 1;
        if (s_step <= cfg.conv_tol) v.converged[p] = 1;
      }
    }
    __syncthreads();
  }
}

/// ||kkt_residual(Z, LAMBDA)||_inf (problem.hpp:263-300), one CTA per
/// problem with z, lambda and theta staged in shared memory, one thread per
/// stage. NX, NU > 0 fix the block sizes at compile time.
constexpr int kKktThreads = 128;
template <int NX, int NU, bool DR = (NX == 0)>
__global__ void __launch_bounds__(kKktThreads, 4) kkt_kernel(View v, const int* __restrict__ work,
                                                        const int* __restrict__ n_work) {
  extern __shared__ double sm_kkt[];
  __shared__ unsigned long long s_max;
  const Dims d = v.d;
  const int nx = NX ? NX : d.nx, nu = NU ? NU : d.nu, T = d.T;
  constexpr int AX = NX ? NX : kMaxNx, AU = NU ? NU : kMaxNx;
  const Family fam = Family::from(v.prob);
  // padded copies (odd strides: consecutive threads' stage walks hit distinct banks)
  const int P = nx + nu + 1, Q = nx + 1;
  double* z = sm_kkt;                 // [T+1][P]: x_t at t P, u_t at t P + n_x
  double* lam = z + (T + 1) * P;      // [T+1][Q]
  double* th = lam + (T + 1) * Q;     // [nth]
  for (int w = blockIdx.x; w < *n_work; w += gridDim.x) {
    const int p = work[w];
    if (v.status[p].code != DOCP_OK) continue;
    if (threadIdx.x == 0) s_max = 0ull;
    cta_stage(z, v.z + static_cast<long>(p) * d.nz, d.nz, [&](int e) {
      const int t = e / (nx + nu);
      return t * P + (e - t * (nx + nu));
    });
    cta_stage(lam, v.lam + static_cast<long>(p) * d.nl, d.nl, [&](int e) { return (e / nx) * Q + e % nx; });
    cta_stage(th, v.theta + static_cast<long>(p) * d.nth, d.nth);
    __syncthreads();
    double m = 0.0;
    for (int t = threadIdx.x; t <= T; t += blockDim.x) {
      double jx[AX * AX], ju[AX * AU], res[AX];
      const double* wx = fam.w_x(d, th);
      // grad_l for x_t: cost grad, + lambda_t (A+_{t-1}' lambda_t, or lambda_0 last), + A_t' lambda_{t+1}
      if (t < T) fam.dynamics<NX, NU, DR>(d, th, z + (t + 1) * P, z + t * P, z + t * P + nx, res, jx, ju);
#pragma unroll
      for (int i = 0; i < AX; ++i) {
        if (i >= nx) break;
        double g = diag_cost_grad(fam.scale, wx[i], z[t * P + i]);
        double a = 0.0;
        if (t < T) {
          a = jx[i * nx] * lam[(t + 1) * Q];
#pragma unroll
          for (int k = 1; k < AX; ++k)
            if (k < nx) a = a + jx[k + i * nx] * lam[(t + 1) * Q + k];
        }
        if (t == 0) {
          if (t < T) g = g + a;
          g = g + lam[i];
        } else {
          g = g + lam[t * Q + i];
          if (t < T) g = g + a;
        }
        m = fmax(m, fabs(g));
      }
      if (t < T) {
        const double* wu = fam.w_u(d, th);
#pragma unroll
        for (int i = 0; i < AU; ++i) {
          if (i >= nu) break;
          double g = diag_cost_grad(fam.scale, wu[i], z[t * P + nx + i]);
          double a = ju[i * nx] * lam[(t + 1) * Q];
#pragma unroll
          for (int k = 1; k < AX; ++k)
            if (k < nx) a = a + ju[k + i * nx] * lam[(t + 1) * Q + k];
          m = fmax(m, fabs(g + a));
        }
#pragma unroll
        for (int i = 0; i < AX; ++i)
          if (i < nx) m = fmax(m, fabs(res[i]));
      } else {
        const double* x_s = fam.x_s(d, th);
        for (int i = 0; i < nx; ++i) m = fmax(m, fabs(z[i] - x_s[i]));
      }
    }
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0) atomicMax(&s_max, __double_as_longlong(m));
    __syncthreads();
    if (threadIdx.x == 0) v.kkt[p] = __longlong_as_double(s_max);
    __syncthreads();
  }
}

/// K4 epilogue: GRAD_THETA = theta_vjp(z, lambda, z~ = Z_QP, lambda~)
/// (affine_quadratic.hpp:82-117, quadratic_cost.hpp:24-45). One CTA per
/// problem: z, z~, lambda and lambda~ are staged in shared memory with
/// coalesced loads (when they fit: `staged`), then one thread per theta
/// entry folds over t in the reference's order. NX, NU > 0 fix the sizes at
/// compile time.
template <int NX = 0, int NU = 0>
__global__ void __launch_bounds__(128) vjp_kernel(View v, const int* __restrict__ work,
                                                  const int* __restrict__ n_work, int staged) {
  extern __shared__ double sm_vjp[];  // z [nz] | z~ [nz] | lambda [nl] | lambda~ [nl]
  const Dims d = v.d;
  const int nx = NX ? NX : d.nx, nu = NU ? NU : d.nu, T = d.T;
  const int nl = (T + 1) * nx, nz = nl + T * nu, sz = nx + nu;
  const Family fam = Family::from(v.prob);
  const double s2 = 2.0 * fam.scale;
  for (int w = blockIdx.x; w < *n_work; w += gridDim.x) {
    const int p = work[w];
    if (v.status[p].code != DOCP_OK) continue;  // block-uniform
    const double* z = v.z + static_cast<long>(p) * nz;
    const double* zt = v.zqp + static_cast<long>(p) * nz;
    const double* lam = v.lam + static_cast<long>(p) * nl;
    const double* lt = v.lt + static_cast<long>(p) * nl;
    if (staged) {
      double* sz_ = sm_vjp;
      double* szt = sz_ + nz;
      double* sl = szt + nz;
      double* slt = sl + nl;
      cta_stage<4>(sz_, z, nz);
      cta_stage<4>(szt, zt, nz);
      cta_stage<4>(sl, lam, nl);
      cta_stage<4>(slt, lt, nl);
      z = sz_, zt = szt, lam = sl, lt = slt;
    }
    __syncthreads();
    for (int k = threadIdx.x; k < d.nth; k += blockDim.x) {
      double acc = 0.0;
      if (k < nx) {  // state-cost weights
        for (int t = 0; t <= T; ++t) acc = acc - s2 * (z[t * sz + k] * zt[t * sz + k]);
      } else if (k < nx + nu) {
        const int i = k - nx;
        for (int t = 0; t < T; ++t) acc = acc - s2 * (z[t * sz + nx + i] * zt[t * sz + nx + i]);
      } else if (fam.kind != DOCP_AFFINE_QUADRATIC) {  // initial state (quadratic_cost.hpp:24-45)
        if (k < 2 * nx + nu) acc = acc + lt[k - nx - nu];  // attitude's inertia tail: 0
      } else {
        const int e = k - nx - nu;
        if (e < nx * nx) {  // dA(i,j) += lam_{t+1,i} z~x_{t,j} + lam~_{t+1,i} x_{t,j}
          const int j = e / nx, i = e - j * nx;
          for (int t = 0; t < T; ++t) {
            acc = acc + lam[(t + 1) * nx + i] * zt[t * sz + j];
            acc = acc + lt[(t + 1) * nx + i] * z[t * sz + j];
          }
        } else if (e < nx * nx + nx * nu) {
          const int f = e - nx * nx;
          const int j = f / nx, i = f - j * nx;
          for (int t = 0; t < T; ++t) {
            acc = acc + lam[(t + 1) * nx + i] * zt[t * sz + nx + j];
            acc = acc + lt[(t + 1) * nx + i] * z[t * sz + nx + j];
          }
        } else if (e < nx * nx + nx * nu + nx) {
          const int i = e - nx * nx - nx * nu;
          for (int t = 0; t < T; ++t) acc = acc + lt[(t + 1) * nx + i];
        } else {
          acc = acc + lt[e - nx * nx - nx * nu - nx];
        }
      }
      v.grad[static_cast<long>(p) * d.nth + k] = acc;
    }
    __syncthreads();
  }
}

/// IL epoch, before the solve: shared learnable segment -> every theta,
/// z0 = demonstration (train.hpp:85-88).
__global__ void il_setup_kernel(View v, const double* __restrict__ weights, int learn_start, int learn_size,
                                const double* __restrict__ demos) {
  const Dims d = v.d;
  const long n = static_cast<long>(v.B) * (learn_size + d.nz);
  for (long g = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; g < n;
       g += static_cast<long>(gridDim.x) * blockDim.x) {
    const int p = static_cast<int>(g / (learn_size + d.nz));
    const int k = static_cast<int>(g % (learn_size + d.nz));
    if (k < learn_size) v.theta[static_cast<long>(p) * d.nth + learn_start + k] = weights[k];
    else v.z[static_cast<long>(p) * d.nz + (k - learn_size)] = demos[static_cast<long>(p) * d.nz + (k - learn_size)];
  }
}

/// IL epoch, after the solve: loss_j = |u - u^|^2 / den and its gradient in
/// the flat layout (train.hpp:89-95). One warp per problem: the gradient row
/// is written coalesced, the squared control errors are staged in shared
/// memory and lane 0 folds them in (t, i) order, as the reference does.
constexpr int kIlLossThreads = 256;
constexpr int kIlLossChunk = 256;  // staged squares per warp per pass
/// FAST = true: every lane accumulates its own squares and the warp sums
/// them as a tree (same value up to rounding; PARITY folds in (t, i) order).
template <bool FAST>
__global__ void __launch_bounds__(kIlLossThreads) il_loss_kernel(View v, const double* __restrict__ demos, double den) {
  __shared__ double sq[kIlLossThreads / 32][kIlLossChunk];
  const Dims d = v.d;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int stage = d.nx + d.nu;
  const int nu_tot = d.T * d.nu;
  const double g2 = 2.0 / den;
  for (int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < v.B; p += warps) {
    const double* z = v.z + static_cast<long>(p) * d.nz;
    const double* dm = demos + static_cast<long>(p) * d.nz;
    double* lg = v.lgz + static_cast<long>(p) * d.nz;
    double acc = 0.0;
    for (int base = 0; base < d.nz; base += kIlLossChunk / d.nu * stage) {
      // this pass covers stages [base/stage, base/stage + kIlLossChunk/nu)
      const int end = min(d.nz, base + kIlLossChunk / d.nu * stage);
      for (int e = base + lane; e < end; e += 32) {
        const int t = e / stage, r = e - t * stage;
        double gv = 0.0;
        if (r >= d.nx && t < d.T) {
          const double du = z[e] - dm[e];
          if constexpr (FAST) acc += du * du;
          else sq[w][(t * d.nu + r - d.nx) - (base / stage) * d.nu] = du * du;
          gv = g2 * du;
        }
        lg[e] = gv;
      }
      if constexpr (FAST) continue;
      __syncwarp();
      if (lane == 0) {
        const int k0 = (base / stage) * d.nu;
        const int k1 = min(nu_tot, k0 + kIlLossChunk);
        for (int k = k0; k < k1; ++k) acc = (k == 0) ? sq[w][0] : acc + sq[w][k - k0];
      }
      __syncwarp();
    }
    if constexpr (FAST) acc = warp_sum(acc);
    if (lane == 0) v.loss[p] = acc / den;
  }
}

/// Fixed-order (instance order) sums of the epoch (train.hpp:126-131). Column
/// 0 is the loss, column 1 + i the i-th learnable gradient entry; CTA c owns
/// columns [c * kIlSumCols, ...). Lane k of warp 0 folds column k in instance
/// order (one dependent chain per column, all columns side by side in one
/// instruction stream) from a shared-memory phase of `rows` instances, while
/// warps 1.. stage the next phase into the other buffer.
constexpr int kIlSumThreads = 256;
constexpr int kIlSumCols = 32;
/// A demonstration whose solve or backward failed contributes nothing (its
/// loss and gradient rows are stale); column 0's pass counts it into
/// fails[0] and the smallest such index into fails[1] (docp_il_failures), so
/// the host can fail the epoch as train.hpp:111-119 does.
__device__ __forceinline__ bool il_row_ok(const View& v, long p, int col, int* fails) {
  if (v.status[p].code == DOCP_OK) return true;
  if (col == 0) {
    atomicAdd(fails, 1);
    atomicMin(fails + 1, static_cast<int>(p));
  }
  return false;
}

__global__ void __launch_bounds__(kIlSumThreads) il_sum_kernel(View v, int learn_start, int learn_size, int rows,
                                                               double* __restrict__ loss_sum,
                                                               double* __restrict__ grad_sum, int* fails) {
  extern __shared__ double stage_buf[];  // [2][ncol][ld]: column-major, odd leading dimension
  const int c0 = blockIdx.x * kIlSumCols;
  const int ncol = min(kIlSumCols, 1 + learn_size - c0);
  const int ld = rows | 1;  // the folding lanes walk their columns on distinct banks
  const int tid = threadIdx.x, k = tid;
  const int nth = v.d.nth;
  // rows [p0, p0 + n) of every column into buffer `which` (warps 1..)
  auto stage = [&](int p0, double* buf) {
    const int n = min(rows, v.B - p0);
    for (int j = tid - 32; j < n; j += kIlSumThreads - 32) {
      const long p = p0 + j;
      const bool ok = il_row_ok(v, p, c0, fails);
      const double* gp = v.grad + p * nth + learn_start - 1;
#pragma unroll 4
      for (int c = 0; c < ncol; ++c)
        buf[c * ld + j] = !ok ? 0.0 : c0 + c == 0 ? v.loss[p] : gp[c0 + c];
    }
  };
  double acc = 0.0;
  if (tid >= 32) stage(0, stage_buf);
  __syncthreads();
  for (int p0 = 0, ph = 0; p0 < v.B; p0 += rows, ph ^= 1) {
    if (tid >= 32) {
      if (p0 + rows < v.B) stage(p0 + rows, stage_buf + (ph ^ 1) * ncol * ld);
    } else if (k < ncol) {
      // instance order (train.hpp:126-131); blocks of 16 loaded one block ahead
      const double* col = stage_buf + ph * ncol * ld + k * ld;
      const int n = min(rows, v.B - p0), n16 = n & ~15;
      double A[16], Bv[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) A[t] = t < n16 ? col[t] : 0.0;
      for (int j = 0; j < n16; j += 32) {
#pragma unroll
        for (int t = 0; t < 16; ++t) Bv[t] = j + 16 + t < n16 ? col[j + 16 + t] : 0.0;
#pragma unroll
        for (int t = 0; t < 16; ++t) acc = acc + A[t];
        if (j + 16 >= n16) break;
#pragma unroll
        for (int t = 0; t < 16; ++t) A[t] = j + 32 + t < n16 ? col[j + 32 + t] : 0.0;
#pragma unroll
        for (int t = 0; t < 16; ++t) acc = acc + Bv[t];
      }
      for (int j = n16; j < n; ++j) acc = acc + col[j];
    }
    __syncthreads();
  }
  if (k < ncol) {
    if (c0 + k == 0) *loss_sum = acc;
    else grad_sum[c0 + k - 1] = acc;
  }
}

/// FAST mode: the same sums as il_sum_kernel, as a fixed-shape tree (one CTA
/// per column: strided per-thread sums, then a warp tree and a pairwise sum
/// of the warp partials). Deterministic; it differs from the instance-order
/// fold only by rounding, so PARITY keeps il_sum_kernel.
constexpr int kIlTreeThreads = 1024;
__global__ void __launch_bounds__(kIlTreeThreads) il_sum_tree_kernel(View v, int learn_start,
                                                                     double* __restrict__ loss_sum,
                                                                     double* __restrict__ grad_sum, int* fails) {
  __shared__ double part[kIlTreeThreads / 32];
  const int c = blockIdx.x;  // 0: loss, 1 + k: learnable gradient k
  double acc = 0.0;
  for (int p = threadIdx.x; p < v.B; p += blockDim.x)
    acc += !il_row_ok(v, p, c, fails) ? 0.0
           : c == 0                      ? v.loss[p]
                                         : v.grad[static_cast<long>(p) * v.d.nth + learn_start + c - 1];
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = part[threadIdx.x];
    t = warp_sum(t);
    if (threadIdx.x == 0) {
      if (c == 0) *loss_sum = t;
      else grad_sum[c - 1] = t;
    }
  }
}

}  // namespace docp_dev
