// k_assemble.cuh — K1: per-stage linearisation and Schur / stair-
// preconditioner block assembly; plus the right-hand side (gamma) and the
// primal recovery, which share its per-stage data.
//
//   linearize        problem.hpp:202-257 (+ project_pd problem.hpp:157-181)
//   assemble_schur   schur.hpp:114-180
//   assemble_gamma   schur.hpp:187-211
//   recover_primal   sqp.hpp:62-89
//
// One CTA per problem (grid-stride over the active work list); phase A runs
// one thread per stage task, phases B/C one warp per (problem, t) block.
// Every family's cost Hessian is diagonal, so Q_t, R_t and their Cholesky
// factors are stored as diagonals; the formulas below are the reference's
// dense operations specialised to that structure and are value-identical to
// them.
#pragma once

#include "families.cuh"

namespace docp_dev {

constexpr int kAsmThreads = 256;
constexpr int kAsmWarps = kAsmThreads / kWarp;

// ranks that order errors exactly as the reference raises them
constexpr int kNoError = 0x7fffffff;

__device__ inline double* blk_ptr(const View& v, int p) { return v.blocks + static_cast<long>(p) * v.d.blk_stride; }

/// Write entry (e, s) of block b of a region in the device block layout.
__device__ inline void blk_store(double* region, int nx, int b, int e, int s, double val) {
  region[static_cast<long>(b) * nx * nx + blk_off(nx, b, e, s)] = val;
}
__device__ inline double blk_load(const double* region, int nx, int b, int e, int s) {
  return region[static_cast<long>(b) * nx * nx + blk_off(nx, b, e, s)];
}

/// K1. Linearise at Z and assemble -S, Phi^-1 and the factor diagonals.
__global__ void __launch_bounds__(kAsmThreads) assemble_kernel(View v, const int* __restrict__ work,
                                                              const int* __restrict__ n_work, double eps_pd,
                                                              int do_schur) {
  extern __shared__ double sm_asm[];
  __shared__ int s_rank_lin, s_rank_qr, s_rank_chi, s_proj;
  const Dims d = v.d;
  const int nx = d.nx, nu = d.nu, T = d.T, bsz = d.bsz;
  const Family fam = Family::from(v.prob);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int sp = max(bsz, nx * nu);
  double* wbuf = sm_asm + static_cast<long>(warp) * 6 * sp;
  double* sA = wbuf;        // A_t (col-major)
  double* sB = sA + sp;     // B_t
  double* sM = sB + sp;     // chi / T1
  double* sD = sM + sp;     // sym(chi) / P_t
  double* sL = sD + sp;     // chol(chi) / sub_t
  double* sP = sL + sp;     // chi^-1 / P_{t+1}

  for (int w = blockIdx.x; w < *n_work; w += gridDim.x) {
    const int p = work[w];
    const double* th = v.theta + static_cast<long>(p) * d.nth;
    const double* z = v.z + static_cast<long>(p) * d.nz;
    double* qd = v.qd + static_cast<long>(p) * d.nb * nx;
    double* lq = v.lq + static_cast<long>(p) * d.nb * nx;
    double* q = v.q + static_cast<long>(p) * d.nb * nx;
    double* rd = v.rd + static_cast<long>(p) * T * nu;
    double* lr = v.lr + static_cast<long>(p) * T * nu;
    double* r = v.r + static_cast<long>(p) * T * nu;
    double* Am = v.A + static_cast<long>(p) * T * bsz;
    double* Bm = v.Bm + static_cast<long>(p) * T * nx * nu;
    double* Cm = v.C + static_cast<long>(p) * T * nx;
    double* xs = v.xs + static_cast<long>(p) * nx;
    if (tid == 0) {
      s_rank_lin = kNoError;
      s_rank_qr = kNoError;
      s_rank_chi = kNoError;
      s_proj = 0;
    }
    __syncthreads();

    // ---------------- phase A: linearize, one thread per stage task
    const double* wx = fam.w_x(d, th);
    const double* wu = fam.w_u(d, th);
    for (int task = tid; task < 2 * T + 2; task += blockDim.x) {
      if (task <= T) {  // state cost at x_t (problem.hpp:221-230)
        const int t = task;
        const double* x = z + xoff(d, t);
        bool finite = isfinite(diag_cost_value(fam.scale, wx, x, nx));
        bool pass = true, below = false;
        for (int i = 0; i < nx; ++i) {
          const double g = diag_cost_grad(fam.scale, wx[i], x[i]);
          const double h = diag_cost_hess(fam.scale, wx[i]);
          finite = finite && isfinite(g) && isfinite(h);
          pass = pass && (h - eps_pd * 1.0 > 0.0);
          below = below || (h < eps_pd);
        }
        if (!finite) atomicMin(&s_rank_lin, t);
        const bool modified = nx == 1 ? below : !pass;
        if (modified) s_proj = 1;
        for (int i = 0; i < nx; ++i) {
          const double h = diag_cost_hess(fam.scale, wx[i]);
          const double hq = modified ? (h < eps_pd ? eps_pd : h) : h;
          qd[t * nx + i] = hq;
          q[t * nx + i] = diag_cost_grad(fam.scale, wx[i], x[i]) - hq * x[i];
          if (!(hq > 0.0) && !isnan(hq)) atomicMin(&s_rank_qr, t);  // chol_Q (schur.hpp:131-133)
          lq[t * nx + i] = sqrt(hq);
        }
      } else if (task < 2 * T + 1) {  // control cost and dynamics at stage t (problem.hpp:231-252)
        const int t = task - (T + 1);
        const double* x = z + xoff(d, t);
        const double* u = z + uoff(d, t);
        const double* xn = z + xoff(d, t + 1);
        bool finite = isfinite(diag_cost_value(fam.scale, wu, u, nu));
        bool pass = true, below = false;
        for (int i = 0; i < nu; ++i) {
          const double g = diag_cost_grad(fam.scale, wu[i], u[i]);
          const double h = diag_cost_hess(fam.scale, wu[i]);
          finite = finite && isfinite(g) && isfinite(h);
          pass = pass && (h - eps_pd * 1.0 > 0.0);
          below = below || (h < eps_pd);
        }
        if (!finite) atomicMin(&s_rank_lin, T + 1 + 2 * t);
        const bool modified = nu == 1 ? below : !pass;
        if (modified) s_proj = 1;
        for (int i = 0; i < nu; ++i) {
          const double h = diag_cost_hess(fam.scale, wu[i]);
          const double hr = modified ? (h < eps_pd ? eps_pd : h) : h;
          rd[t * nu + i] = hr;
          r[t * nu + i] = diag_cost_grad(fam.scale, wu[i], u[i]) - hr * u[i];
          if (!(hr > 0.0) && !isnan(hr)) atomicMin(&s_rank_qr, T + 1 + t);
          lr[t * nu + i] = sqrt(hr);
        }
        double res[kMaxNx];
        double* jx = Am + static_cast<long>(t) * bsz;
        double* ju = Bm + static_cast<long>(t) * nx * nu;
        fam.dynamics(d, th, xn, x, u, res, jx, ju);
        bool dfin = true;
        for (int i = 0; i < nx; ++i) dfin = dfin && isfinite(res[i]);
        for (int k = 0; k < bsz; ++k) dfin = dfin && isfinite(jx[k]);
        for (int k = 0; k < nx * nu; ++k) dfin = dfin && isfinite(ju[k]);
        if (!dfin) atomicMin(&s_rank_lin, T + 2 + 2 * t);
        for (int i = 0; i < nx; ++i) {  // C_t = A+ x+ + A x + B u - f
          double ax = jx[i] * x[0];
          for (int k = 1; k < nx; ++k) ax = ax + jx[i + k * nx] * x[k];
          double bu = ju[i] * u[0];
          for (int k = 1; k < nu; ++k) bu = bu + ju[i + k * nx] * u[k];
          Cm[t * nx + i] = ((xn[i] + ax) + bu) - res[i];
        }
      } else {  // initial_state (problem.hpp:253-254)
        const double* x_s = fam.x_s(d, th);
        bool fin = true;
        for (int i = 0; i < nx; ++i) {
          xs[i] = x_s[i];
          fin = fin && isfinite(x_s[i]);
        }
        if (!fin) atomicMin(&s_rank_lin, 3 * T + 1);
      }
    }
    __syncthreads();
    const int rank_lin = s_rank_lin, rank_qr = s_rank_qr;
    if (tid == 0) {
      v.pd_proj[p] = s_proj;
      docp_status* st = v.status + p;
      if (rank_lin != kNoError) {
        int where, idx;
        if (rank_lin <= T) {
          where = DOCP_AT_STATE_COST, idx = rank_lin;
        } else if (rank_lin == 3 * T + 1) {
          where = DOCP_AT_INITIAL_STATE, idx = 0;
        } else {
          const int k = rank_lin - (T + 1);
          where = (k & 1) ? DOCP_AT_DYNAMICS : DOCP_AT_CONTROL_COST, idx = k >> 1;
        }
        set_status(st, DOCP_EVALUATION, where, idx);
      } else if (do_schur && rank_qr != kNoError) {
        if (rank_qr <= T)
          set_status(st, DOCP_NUMERICAL, DOCP_AT_CHOL_Q, rank_qr);
        else
          set_status(st, DOCP_NUMERICAL, DOCP_AT_CHOL_R, rank_qr - (T + 1));
      } else {
        set_status(st, DOCP_OK, DOCP_AT_NONE, 0);
      }
    }
    if (!do_schur || rank_lin != kNoError || rank_qr != kNoError) {
      __syncthreads();
      continue;
    }

    // ---------------- phase B: chi_t, phi_t, chol(chi_t), chi_t^-1 (schur.hpp:143-167)
    double* blk = blk_ptr(v, p);
    double* Sd = blk + d.s_diag;
    double* Ss = blk + d.s_sub;
    double* Pd = blk + d.p_diag;
    double* Pu = blk + d.p_sup;
    // stage 0 blocks: -S diag_0 = sym(Q_0^-1), Phi^-1 diag_0 = Q_0
    for (int k = tid; k < bsz; k += blockDim.x) {
      const int i = k % nx, j = k / nx;
      const double l = lq[i];
      const double x = i == j ? (1.0 / l) / l : 0.0;
      blk_store(Sd, nx, 0, i, j, 0.5 * (x + x));
      blk_store(Pd, nx, 0, i, j, i == j ? qd[i] : 0.0);
    }
    for (int t = warp; t < T; t += kAsmWarps) {
      const double* lqt = lq + t * nx;
      const double* lqn = lq + (t + 1) * nx;
      const double* lrt = lr + t * nu;
      for (int k = lane; k < bsz; k += 32) sA[k] = Am[static_cast<long>(t) * bsz + k];
      for (int k = lane; k < nx * nu; k += 32) sB[k] = Bm[static_cast<long>(t) * nx * nu + k];
      __syncwarp();
      for (int k = lane; k < bsz; k += 32) {
        const int i = k % nx, j = k / nx;
        // A Q^-1 A'  (M1(k,j) = (A(j,k)/l_k)/l_k)
        double a = sA[i] * ((sA[j] / lqt[0]) / lqt[0]);
        for (int m = 1; m < nx; ++m) a = a + sA[i + m * nx] * ((sA[j + m * nx] / lqt[m]) / lqt[m]);
        // B R^-1 B'
        double b = sB[i] * ((sB[j] / lrt[0]) / lrt[0]);
        for (int m = 1; m < nu; ++m) b = b + sB[i + m * nx] * ((sB[j + m * nx] / lrt[m]) / lrt[m]);
        // A+ Q+^-1 A+' with A+ = I
        const double c3 = i == j ? (1.0 / lqn[i]) / lqn[i] : 0.0;
        sM[k] = (a + b) + c3;
        // phi_t = A_t Q_t^-1 A+_{t-1}'  (A+_{-1} = A+ = I)
        blk_store(Ss, nx, t, i, j, sA[i + j * nx] * ((1.0 / lqt[j]) / lqt[j]));
      }
      __syncwarp();
      for (int k = lane; k < bsz; k += 32) {
        const int i = k % nx, j = k / nx;
        const double dv = 0.5 * (sM[k] + sM[j + i * nx]);
        sD[k] = dv;
        blk_store(Sd, nx, t + 1, i, j, dv);
        sL[k] = 0.0;
      }
      __syncwarp();
      // Cholesky of chi_t (eigen_lite LLT), rows in parallel
      bool failed = false;
      for (int k = 0; k < nx; ++k) {
        double s = 0.0;
        if (k > 0) {
          s = sL[k] * sL[k];
          for (int j = 1; j < k; ++j) s = s + sL[k + j * nx] * sL[k + j * nx];
        }
        const double piv = sD[k + k * nx] - s;
        if (piv <= 0.0) {
          failed = true;
          break;
        }
        const double lk = sqrt(piv);
        const int i = k + 1 + lane;
        if (lane == 0) sL[k + k * nx] = lk;
        if (i < nx) {
          double tt = 0.0;
          if (k > 0) {
            tt = sL[i] * sL[k];
            for (int j = 1; j < k; ++j) tt = tt + sL[i + j * nx] * sL[k + j * nx];
          }
          sL[i + k * nx] = (sD[i + k * nx] - tt) / lk;
        }
        __syncwarp();
      }
      if (failed) {
        if (lane == 0) atomicMin(&s_rank_chi, t);
        __syncwarp();
        continue;
      }
      // chi_t^-1 = chol.solve(I), one column per lane
      if (lane < nx) {
        double* x = sP + lane * nx;
        for (int i = 0; i < nx; ++i) {
          double s = 0.0;
          if (i > 0) {
            s = sL[i] * x[0];
            for (int j = 1; j < i; ++j) s = s + sL[i + j * nx] * x[j];
          }
          x[i] = ((i == lane ? 1.0 : 0.0) - s) / sL[i + i * nx];
        }
        for (int i = nx - 1; i >= 0; --i) {
          double s = 0.0;
          if (i + 1 < nx) {
            s = sL[i + 1 + i * nx] * x[i + 1];
            for (int j = i + 2; j < nx; ++j) s = s + sL[j + i * nx] * x[j];
          }
          x[i] = (x[i] - s) / sL[i + i * nx];
        }
      }
      __syncwarp();
      for (int k = lane; k < bsz; k += 32) {
        const int i = k % nx, j = k / nx;
        blk_store(Pd, nx, t + 1, i, j, 0.5 * (sP[k] + sP[j + i * nx]));
      }
      __syncwarp();
    }
    __syncthreads();
    if (s_rank_chi != kNoError) {
      if (tid == 0) set_status(v.status + p, DOCP_NUMERICAL, DOCP_AT_CHOL_CHI, s_rank_chi);
      __syncthreads();
      continue;
    }

    // ---------------- phase C: stair off-diagonal (-D_t phi_t') D_{t+1} (schur.hpp:169-179)
    for (int t = warp; t < T; t += kAsmWarps) {
      for (int k = lane; k < bsz; k += 32) {
        const int i = k % nx, j = k / nx;
        sD[k] = blk_load(Pd, nx, t, i, j);
        sL[k] = blk_load(Ss, nx, t, i, j);
        sP[k] = blk_load(Pd, nx, t + 1, i, j);
      }
      __syncwarp();
      for (int k = lane; k < bsz; k += 32) {
        const int i = k % nx, j = k / nx;
        double a = (-sD[i]) * sL[j];
        for (int m = 1; m < nx; ++m) a = a + (-sD[i + m * nx]) * sL[j + m * nx];
        sM[k] = a;
      }
      __syncwarp();
      for (int k = lane; k < bsz; k += 32) {
        const int i = k % nx, j = k / nx;
        double a = sM[i] * sP[j * nx];
        for (int m = 1; m < nx; ++m) a = a + sM[i + m * nx] * sP[m + j * nx];
        blk_store(Pu, nx, t, i, j, a);
      }
      __syncwarp();
    }
    __syncthreads();
  }
}

/// Solve Q_t x = b for the diagonal Cholesky factor l: (b / l) / l.
__device__ inline double diag_solve(double b, double l) { return (b / l) / l; }

/// GAMMA <- -(d + H G^-1 b) (schur.hpp:187-211), one thread per (stage, row).
/// rhs FORWARD: b = flat_b, d = flat_d; ADJOINT: b = -LOSS_GRAD_Z, d = 0.
__global__ void gamma_kernel(View v, const int* __restrict__ work, const int* __restrict__ n_work, int rhs) {
  const Dims d = v.d;
  const int nx = d.nx, nu = d.nu, T = d.T;
  const long total = static_cast<long>(*n_work) * d.nl;
  for (long g = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; g < total;
       g += static_cast<long>(gridDim.x) * blockDim.x) {
    const int p = work[g / d.nl];
    const int row = static_cast<int>(g % d.nl);
    const int blk = row / nx, i = row % nx;
    const double* lq = v.lq + static_cast<long>(p) * d.nb * nx;
    const double* lr = v.lr + static_cast<long>(p) * T * nu;
    const double* lg = v.lgz + static_cast<long>(p) * d.nz;
    auto bx = [&](int t, int k) -> double {
      return rhs == DOCP_RHS_FORWARD ? v.q[(static_cast<long>(p) * d.nb + t) * nx + k] : -lg[xoff(d, t) + k];
    };
    auto bu = [&](int t, int k) -> double {
      return rhs == DOCP_RHS_FORWARD ? v.r[(static_cast<long>(p) * T + t) * nu + k] : -lg[uoff(d, t) + k];
    };
    double out;
    if (blk == 0) {
      const double dd = rhs == DOCP_RHS_FORWARD ? v.xs[static_cast<long>(p) * nx + i] : 0.0;
      out = dd + diag_solve(bx(0, i), lq[i]);
    } else {
      const int t = blk - 1;
      const double* At = v.A + (static_cast<long>(p) * T + t) * d.bsz;
      const double* Bt = v.Bm + (static_cast<long>(p) * T + t) * nx * nu;
      double a = At[i] * diag_solve(bx(t, 0), lq[t * nx]);
      for (int k = 1; k < nx; ++k) a = a + At[i + k * nx] * diag_solve(bx(t, k), lq[t * nx + k]);
      double b = Bt[i] * diag_solve(bu(t, 0), lr[t * nu]);
      for (int k = 1; k < nu; ++k) b = b + Bt[i + k * nx] * diag_solve(bu(t, k), lr[t * nu + k]);
      const double c = diag_solve(bx(t + 1, i), lq[(t + 1) * nx + i]);
      const double dd = rhs == DOCP_RHS_FORWARD ? v.C[(static_cast<long>(p) * T + t) * nx + i] : 0.0;
      out = dd + ((a + b) + c);
    }
    v.gamma[static_cast<long>(p) * d.nl + row] = -out;
  }
}

/// Z_QP <- recover_primal(lambda, b) (sqp.hpp:62-89), one thread per primal entry.
__global__ void recover_kernel(View v, const int* __restrict__ work, const int* __restrict__ n_work,
                               const double* __restrict__ lam_all, int rhs) {
  const Dims d = v.d;
  const int nx = d.nx, nu = d.nu, T = d.T;
  const long total = static_cast<long>(*n_work) * d.nz;
  for (long g = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; g < total;
       g += static_cast<long>(gridDim.x) * blockDim.x) {
    const int p = work[g / d.nz];
    const int e = static_cast<int>(g % d.nz);
    const int t = e / (nx + nu), c = e % (nx + nu);
    const double* lam = lam_all + static_cast<long>(p) * d.nl;
    const double* lg = v.lgz + static_cast<long>(p) * d.nz;
    double rhs_v = rhs == DOCP_RHS_FORWARD ? 0.0 : -lg[e];
    double out;
    if (c < nx) {  // x_t,c = -Q_t^-1 (b + A+_{t-1}' lam_t + A_t' lam_{t+1})
      const int i = c;
      if (rhs == DOCP_RHS_FORWARD) rhs_v = v.q[(static_cast<long>(p) * d.nb + t) * nx + i];
      rhs_v = rhs_v + lam[t * nx + i];
      if (t < T) {
        const double* At = v.A + (static_cast<long>(p) * T + t) * d.bsz;
        const double* l1 = lam + (t + 1) * nx;
        double a = At[i * nx] * l1[0];
        for (int k = 1; k < nx; ++k) a = a + At[k + i * nx] * l1[k];
        rhs_v = rhs_v + a;
      }
      out = -diag_solve(rhs_v, v.lq[(static_cast<long>(p) * d.nb + t) * nx + i]);
    } else {  // u_t,i = -R_t^-1 (b + B_t' lam_{t+1})
      const int i = c - nx;
      if (rhs == DOCP_RHS_FORWARD) rhs_v = v.r[(static_cast<long>(p) * T + t) * nu + i];
      const double* Bt = v.Bm + (static_cast<long>(p) * T + t) * nx * nu;
      const double* l1 = lam + (t + 1) * nx;
      double a = Bt[i * nx] * l1[0];
      for (int k = 1; k < nx; ++k) a = a + Bt[k + i * nx] * l1[k];
      out = -diag_solve(rhs_v + a, v.lr[(static_cast<long>(p) * T + t) * nu + i]);
    }
    v.zqp[static_cast<long>(p) * d.nz + e] = out;
  }
}

}  // namespace docp_dev
