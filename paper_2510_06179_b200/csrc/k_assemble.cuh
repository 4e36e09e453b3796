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

#ifdef DOCP_K1_CLOCK
// phase timing of thread 0 in assemble_kernel_t (A/B builds only: nvcc -DDOCP_K1_CLOCK)
__device__ unsigned long long g_k1_clk[16];
#define K1_CLK(k)                         \
  if (threadIdx.x == 0) {                 \
    const long long t_ = clock64();       \
    k1clk[k] += t_ - k1last;              \
    k1last = t_;                          \
  }
#else
#define K1_CLK(k)
#endif
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

struct AsmShared {
  int rank_lin, rank_qr, rank_chi, proj;
};

/// Phase A for the affine-quadratic family with compile-time block sizes:
/// one thread per ENTRY instead of one per stage task, so the CTA's threads
/// share the work evenly and every store is coalesced. A stage's entries are
/// NX (NU) consecutive lanes of one warp; the per-stage decisions of the
/// reference (project_pd's LLT test, the finiteness checks, problem.hpp:157-
/// 257) are warp-ballots over the stage's lanes, and the first failure is
/// ranked exactly as the per-stage path ranks it. Values and expression
/// order per entry are those of the per-stage path.
template <int NX, int NU>
__device__ void linearize_aq_rows(const View& v, int p, double eps_pd, const Family& fam, const double* z,
                                  const double* th, AsmShared& sh) {
  const Dims d = v.d;
  const int T = d.T, sz = NX + NU;
  const int tid = threadIdx.x, lane = tid & 31;
  const double* wx = th;
  const double* wu = th + NX;
  const double* ath = th + NX + NU;          // A, column-major (affine_quadratic.hpp:27-37)
  const double* bth = ath + NX * NX;         // B
  const double* off = bth + NX * NU;         // b
  double* qd = v.qd + static_cast<long>(p) * d.nb * NX;
  double* lq = v.lq + static_cast<long>(p) * d.nb * NX;
  double* q = v.q + static_cast<long>(p) * d.nb * NX;
  double* rd = v.rd + static_cast<long>(p) * T * NU;
  double* lr = v.lr + static_cast<long>(p) * T * NU;
  double* r = v.r + static_cast<long>(p) * T * NU;
  double* Cm = v.C + static_cast<long>(p) * T * NX;
  double* jx = v.A + a_off(d, p, 0);
  double* ju = v.Bm + b_off(d, p, 0);
  // all lanes of a stage group agree (ballot over the group's lanes)
  auto group_all = [&](bool pred, int n) {
    const unsigned bal = __ballot_sync(0xffffffffu, pred);
    const unsigned gm = (n == 32 ? 0xffffffffu : ((1u << n) - 1u)) << (lane & ~(n - 1));
    return (bal & gm) == gm;
  };
  auto group_any = [&](bool pred, int n) {
    const unsigned bal = __ballot_sync(0xffffffffu, pred);
    const unsigned gm = (n == 32 ? 0xffffffffu : ((1u << n) - 1u)) << (lane & ~(n - 1));
    return (bal & gm) != 0u;
  };
  const int nstate = (T + 1) * NX, nctrl = T * NU, ndyn = T * NX;
  // ---- state cost entries (problem.hpp:221-230)
  for (int base = 0; base < nstate; base += blockDim.x) {
    const int k = base + tid;
    const bool valid = k < nstate;
    const int t = valid ? k / NX : 0, i = k - (k / NX) * NX;
    const double* x = z + t * sz;
    const double h = diag_cost_hess(fam.scale, wx[i]);
    const double g = diag_cost_grad(fam.scale, wx[i], x[i]);
    bool fin = isfinite(g) && isfinite(h);
    if (i == 0) fin = fin && isfinite(diag_cost_value<NX>(fam.scale, wx, x, NX));
    const bool finite = group_all(fin || !valid, NX);
    const bool pass = group_all(h - eps_pd * 1.0 > 0.0, NX);
    const bool below = group_any(h < eps_pd, NX);
    const bool modified = NX == 1 ? below : !pass;
    if (valid) {
      if (!finite && i == 0) atomicMin(&sh.rank_lin, t);
      if (modified) sh.proj = 1;
      const double hq = modified ? (h < eps_pd ? eps_pd : h) : h;
      qd[k] = hq;
      q[k] = g - hq * x[i];
      if (!(hq > 0.0) && !isnan(hq)) atomicMin(&sh.rank_qr, t);  // chol_Q (schur.hpp:131-133)
      lq[k] = sqrt(hq);
    }
  }
  // ---- control cost entries (problem.hpp:231-240)
  for (int base = 0; base < nctrl; base += blockDim.x) {
    const int k = base + tid;
    const bool valid = k < nctrl;
    const int t = valid ? k / NU : 0, i = k - (k / NU) * NU;
    const double* u = z + t * sz + NX;
    const double h = diag_cost_hess(fam.scale, wu[i]);
    const double g = diag_cost_grad(fam.scale, wu[i], u[i]);
    bool fin = isfinite(g) && isfinite(h);
    if (i == 0) fin = fin && isfinite(diag_cost_value<NU>(fam.scale, wu, u, NU));
    const bool finite = group_all(fin || !valid, NU);
    const bool pass = group_all(h - eps_pd * 1.0 > 0.0, NU);
    const bool below = group_any(h < eps_pd, NU);
    const bool modified = NU == 1 ? below : !pass;
    if (valid) {
      if (!finite && i == 0) atomicMin(&sh.rank_lin, T + 1 + 2 * t);
      if (modified) sh.proj = 1;
      const double hr = modified ? (h < eps_pd ? eps_pd : h) : h;
      rd[k] = hr;
      r[k] = g - hr * u[i];
      if (!(hr > 0.0) && !isnan(hr)) atomicMin(&sh.rank_qr, T + 1 + t);
      lr[k] = sqrt(hr);
    }
  }
  // ---- dynamics rows (affine_quadratic.hpp:65-75, problem.hpp:241-252)
  for (int base = 0; base < ndyn; base += blockDim.x) {
    const int k = base + tid;
    const bool valid = k < ndyn;
    const int t = valid ? k / NX : 0, i = k - (k / NX) * NX;
    const double* x = z + t * sz;
    const double* u = x + NX;
    const double* xn = z + (t + 1) * sz;
    double ax = ath[i] * x[0];
#pragma unroll
    for (int c = 1; c < NX; ++c) ax = ax + ath[i + c * NX] * x[c];
    double bu = bth[i] * u[0];
#pragma unroll
    for (int c = 1; c < NU; ++c) bu = bu + bth[i + c * NX] * u[c];
    const double res = ((xn[i] - ax) - bu) - off[i];
    bool fin = isfinite(res);
    if (t == 0) {  // the time-invariant Jacobians, written once: jac_x = -A, jac_u = -B
#pragma unroll
      for (int c = 0; c < NX; ++c) fin = fin && isfinite(-ath[i + c * NX]);
#pragma unroll
      for (int c = 0; c < NU; ++c) fin = fin && isfinite(-bth[i + c * NX]);
      if (valid) {
#pragma unroll
        for (int c = 0; c < NX; ++c) jx[i + c * NX] = -ath[i + c * NX];
#pragma unroll
        for (int c = 0; c < NU; ++c) ju[i + c * NX] = -bth[i + c * NX];
      }
    }
    const bool finite = group_all(fin || !valid, NX);
    if (valid) {
      if (!finite && i == 0) atomicMin(&sh.rank_lin, T + 2 + 2 * t);
      // C_t = A+ x+ + A x + B u - f, with the Jacobians at z (problem.hpp:250-251)
      double cx = (-ath[i]) * x[0];
#pragma unroll
      for (int c = 1; c < NX; ++c) cx = cx + (-ath[i + c * NX]) * x[c];
      double cu = (-bth[i]) * u[0];
#pragma unroll
      for (int c = 1; c < NU; ++c) cu = cu + (-bth[i + c * NX]) * u[c];
      Cm[k] = ((xn[i] + cx) + cu) - res;
    }
  }
  // ---- initial state (problem.hpp:253-254)
  if (tid < 32) {
    const double* x_s = fam.x_s(d, th);
    const bool valid = tid < NX;
    const double xv = valid ? x_s[tid] : 0.0;
    if (valid) v.xs[static_cast<long>(p) * NX + tid] = xv;
    if (!__all_sync(0xffffffffu, !valid || isfinite(xv)) && tid == 0) atomicMin(&sh.rank_lin, 3 * T + 1);
  }
}

/// Phase A of K1 (problem.hpp:202-257): one thread per stage task. Writes the
/// QpData of problem p and the first-error ranks; returns (block-uniform)
/// whether the Schur phases may run. Ends with a __syncthreads. NX, NU > 0
/// fix the block sizes at compile time (same arithmetic). `stage`, when
/// given, is shared memory for nz + nth doubles: z and theta are first
/// copied there with coalesced loads, so the per-stage tasks read on-chip
/// copies instead of issuing dependent global loads.
template <int NX = 0, int NU = 0, bool DR = (NX == 0)>
__device__ bool phase_linearize(const View& v, int p, double eps_pd, int do_schur, AsmShared& sh,
                                double* stage = nullptr) {
  const Dims d = v.d;
  const int nx = NX ? NX : d.nx, nu = NU ? NU : d.nu, T = d.T, bsz = nx * nx;
  const Family fam = Family::from(v.prob);
  const int tid = threadIdx.x;
  const double* th = v.theta + static_cast<long>(p) * d.nth;
  const double* z = v.z + static_cast<long>(p) * d.nz;
  if (stage) {  // made visible by the __syncthreads below
    cta_stage(stage, z, d.nz);
    cta_stage(stage + d.nz, th, d.nth);
    z = stage;
    th = stage + d.nz;
  }
  double* qd = v.qd + static_cast<long>(p) * d.nb * nx;
  double* lq = v.lq + static_cast<long>(p) * d.nb * nx;
  double* q = v.q + static_cast<long>(p) * d.nb * nx;
  double* rd = v.rd + static_cast<long>(p) * T * nu;
  double* lr = v.lr + static_cast<long>(p) * T * nu;
  double* r = v.r + static_cast<long>(p) * T * nu;
  double* Cm = v.C + static_cast<long>(p) * T * nx;
  const bool tv = d.a_stride != 0;  // time-varying Jacobians stored per stage
  double* xs = v.xs + static_cast<long>(p) * nx;
  if (tid == 0) {
    sh.rank_lin = kNoError;
    sh.rank_qr = kNoError;
    sh.rank_chi = kNoError;
    sh.proj = 0;
  }
  __syncthreads();
  const double* wx = fam.w_x(d, th);
  const double* wu = fam.w_u(d, th);
  if constexpr (NX > 0 && NU > 0 && kWarp % NX == 0 && kWarp % NU == 0) {
    if (fam.kind == DOCP_AFFINE_QUADRATIC && !tv) {
      linearize_aq_rows<NX, NU>(v, p, eps_pd, fam, z, th, sh);
      goto tasks_done;
    }
  }
  for (int task = tid; task < 2 * T + 2; task += blockDim.x) {
    if (task <= T) {  // state cost at x_t (problem.hpp:221-230)
      const int t = task;
      const double* x = z + xoff(d, t);
      bool finite = isfinite(diag_cost_value<NX>(fam.scale, wx, x, nx));
      bool pass = true, below = false;
      for (int i = 0; i < nx; ++i) {
        const double g = diag_cost_grad(fam.scale, wx[i], x[i]);
        const double h = diag_cost_hess(fam.scale, wx[i]);
        finite = finite && isfinite(g) && isfinite(h);
        pass = pass && (h - eps_pd * 1.0 > 0.0);
        below = below || (h < eps_pd);
      }
      if (!finite) atomicMin(&sh.rank_lin, t);
      const bool modified = nx == 1 ? below : !pass;
      if (modified) sh.proj = 1;
      for (int i = 0; i < nx; ++i) {
        const double h = diag_cost_hess(fam.scale, wx[i]);
        const double hq = modified ? (h < eps_pd ? eps_pd : h) : h;
        qd[t * nx + i] = hq;
        q[t * nx + i] = diag_cost_grad(fam.scale, wx[i], x[i]) - hq * x[i];
        if (!(hq > 0.0) && !isnan(hq)) atomicMin(&sh.rank_qr, t);  // chol_Q (schur.hpp:131-133)
        lq[t * nx + i] = sqrt(hq);
      }
    } else if (task < 2 * T + 1) {  // control cost and dynamics at stage t (problem.hpp:231-252)
      const int t = task - (T + 1);
      const double* x = z + xoff(d, t);
      const double* u = z + uoff(d, t);
      const double* xn = z + xoff(d, t + 1);
      bool finite = isfinite(diag_cost_value<NU>(fam.scale, wu, u, nu));
      bool pass = true, below = false;
      for (int i = 0; i < nu; ++i) {
        const double g = diag_cost_grad(fam.scale, wu[i], u[i]);
        const double h = diag_cost_hess(fam.scale, wu[i]);
        finite = finite && isfinite(g) && isfinite(h);
        pass = pass && (h - eps_pd * 1.0 > 0.0);
        below = below || (h < eps_pd);
      }
      if (!finite) atomicMin(&sh.rank_lin, T + 1 + 2 * t);
      const bool modified = nu == 1 ? below : !pass;
      if (modified) sh.proj = 1;
      for (int i = 0; i < nu; ++i) {
        const double h = diag_cost_hess(fam.scale, wu[i]);
        const double hr = modified ? (h < eps_pd ? eps_pd : h) : h;
        rd[t * nu + i] = hr;
        r[t * nu + i] = diag_cost_grad(fam.scale, wu[i], u[i]) - hr * u[i];
        if (!(hr > 0.0) && !isnan(hr)) atomicMin(&sh.rank_qr, T + 1 + t);
        lr[t * nu + i] = sqrt(hr);
      }
      double res[NX ? NX : kMaxNx];
      // time-invariant families: one Jacobian copy, written by stage 0
      const bool write_jac = tv || t == 0;
      double* jx = v.A + a_off(d, p, t);
      double* ju = v.Bm + b_off(d, p, t);
      fam.dynamics<NX, NU, DR>(d, th, xn, x, u, res, write_jac ? jx : nullptr, write_jac ? ju : nullptr);
      bool dfin = true;
      for (int i = 0; i < nx; ++i) dfin = dfin && isfinite(res[i]);
      if (write_jac) {
        for (int k = 0; k < bsz; ++k) dfin = dfin && isfinite(jx[k]);
        for (int k = 0; k < nx * nu; ++k) dfin = dfin && isfinite(ju[k]);
      }
      if (!dfin) atomicMin(&sh.rank_lin, T + 2 + 2 * t);
      // affine-quadratic Jacobians straight from theta (-A, -B: affine_quadratic.hpp:71-72)
      const double* ath = th + nx + nu;
      const double* bth = ath + bsz;
      auto JX = [&](int i, int k) { return write_jac ? jx[i + k * nx] : -ath[i + k * nx]; };
      auto JU = [&](int i, int k) { return write_jac ? ju[i + k * nx] : -bth[i + k * nx]; };
      for (int i = 0; i < nx; ++i) {  // C_t = A+ x+ + A x + B u - f
        double ax = JX(i, 0) * x[0];
        for (int k = 1; k < nx; ++k) ax = ax + JX(i, k) * x[k];
        double bu = JU(i, 0) * u[0];
        for (int k = 1; k < nu; ++k) bu = bu + JU(i, k) * u[k];
        Cm[t * nx + i] = ((xn[i] + ax) + bu) - res[i];
      }
    } else {  // initial_state (problem.hpp:253-254)
      const double* x_s = fam.x_s(d, th);
      bool fin = true;
      for (int i = 0; i < nx; ++i) {
        xs[i] = x_s[i];
        fin = fin && isfinite(x_s[i]);
      }
      if (!fin) atomicMin(&sh.rank_lin, 3 * T + 1);
    }
  }
tasks_done:
  __syncthreads();
  const int rank_lin = sh.rank_lin, rank_qr = sh.rank_qr;
  if (tid == 0) {
    v.pd_proj[p] = sh.proj;
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
  return do_schur && rank_lin == kNoError && rank_qr == kNoError;
}

/// Stage-0 blocks: -S diag_0 = sym(Q_0^-1), Phi^-1 diag_0 = Q_0 (schur.hpp:146-147, 171).
__device__ inline void stage0_blocks(const View& v, int p) {
  const Dims d = v.d;
  const int nx = d.nx, bsz = d.bsz;
  double* blk = blk_ptr(v, p);
  const double* lq = v.lq + static_cast<long>(p) * d.nb * nx;
  const double* qd = v.qd + static_cast<long>(p) * d.nb * nx;
  for (int k = threadIdx.x; k < bsz; k += blockDim.x) {
    const int i = k % nx, j = k / nx;
    const double l = lq[i];
    const double x = i == j ? (1.0 / l) / l : 0.0;
    blk_store(blk + d.s_diag, nx, 0, i, j, 0.5 * (x + x));
    blk_store(blk + d.p_diag, nx, 0, i, j, i == j ? qd[i] : 0.0);
  }
}

/// K1 for any (n_x, n_u): phases B/C one warp per (problem, t).
__global__ void __launch_bounds__(kAsmThreads) assemble_kernel(View v, const int* __restrict__ work,
                                                              const int* __restrict__ n_work, double eps_pd,
                                                              int do_schur) {
  extern __shared__ double sm_asm[];
  __shared__ AsmShared sh;
  const Dims d = v.d;
  const int nx = d.nx, nu = d.nu, T = d.T, bsz = d.bsz;
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
    if (!phase_linearize(v, p, eps_pd, do_schur, sh)) {
      __syncthreads();
      continue;
    }
    const double* lq = v.lq + static_cast<long>(p) * d.nb * nx;
    const double* lr = v.lr + static_cast<long>(p) * T * nu;

    // ---------------- phase B: chi_t, phi_t, chol(chi_t), chi_t^-1 (schur.hpp:143-167)
    double* blk = blk_ptr(v, p);
    double* Sd = blk + d.s_diag;
    double* Ss = blk + d.s_sub;
    double* Pd = blk + d.p_diag;
    double* Pu = blk + d.p_sup;
    stage0_blocks(v, p);
    for (int t = warp; t < T; t += kAsmWarps) {
      const double* lqt = lq + t * nx;
      const double* lqn = lq + (t + 1) * nx;
      const double* lrt = lr + t * nu;
      for (int k = lane; k < bsz; k += 32) sA[k] = v.A[a_off(d, p, t) + k];
      for (int k = lane; k < nx * nu; k += 32) sB[k] = v.Bm[b_off(d, p, t) + k];
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
        if (lane == 0) atomicMin(&sh.rank_chi, t);
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
    if (sh.rank_chi != kNoError) {
      if (tid == 0) set_status(v.status + p, DOCP_NUMERICAL, DOCP_AT_CHOL_CHI, sh.rank_chi);
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

constexpr int kAsmGroupThreads = 128;

/// K1 for fixed (NX, NU) (the benchmark shapes): phases B/C run one NX-lane
/// group per (problem, t) block — lane l owns column l of every NX x NX block
/// (row l during the Cholesky), so all 32 lanes of a warp work on 32/NX stages
/// at once. M1 = Q_t^-1 A_t' and M2 = R_t^-1 B_t' are formed once per stage
/// (2 divisions per entry, as the reference's LLT solves), then chi_t, phi_t,
/// chol(chi_t), chi_t^-1 and the stair off-diagonal follow with the same
/// operation order as the runtime-shape kernel (bit-identical results).
///
/// Shared-memory layout: every group matrix (the staged output block too) is
/// column-major with a padded leading dimension (NX + 1 rows, NU + 1 for M2),
/// and consecutive group buffers are skewed by NX doubles mod 16. A 64-bit
/// access is served per half-warp (16 lanes = 16 bank pairs), which holds
/// 16 / NX groups; with this skew their per-lane column walks, row walks and
/// group-uniform (broadcast) accesses hit distinct bank pairs.
template <int NX, int NU>
struct AsmLayout {
  static constexpr int LD = NX + 1;      // column stride of NX-row matrices
  static constexpr int LDU = NU + 1;     // column stride of M2 (NU x NX)
  static constexpr int P2 = NX * LD;     // padded NX x NX
  static constexpr int PB = NU * LD;     // B_t, NX x NU
  static constexpr int PM2 = NX * LDU;   // M2, NU x NX
  // B_t and M2 are dead once chi is formed; the staged output block reuses them
  static constexpr int U = (PB + PM2) > P2 ? (PB + PM2) : P2;
  static constexpr int RAW = 4 * P2 + U;
  static constexpr int SKEW = NX % 16;   // groups of one half-warp on disjoint bank pairs
  static constexpr int GBUF = RAW + ((SKEW - RAW % 16) % 16 + 16) % 16;
};

/// TH threads per CTA (TH / NX stage groups); the launcher picks TH so that the
/// groups divide the horizon's stages into whole rounds where it can.
///
/// FAST = true (PCG mode FAST): the same blocks up to rounding, with the
/// reference's divisions replaced by reciprocals — M1/M2 scale columns by
/// 1/q_k, 1/r_k (q, r the projected cost diagonals), the Cholesky of chi_t
/// takes 1/l_kk = rsqrt(pivot) and keeps it on the factor's diagonal for the
/// triangular solves — and fma accumulation. FAST = false is the
/// reference's arithmetic bit for bit.
/// DR: the instantiation for the drifting family (Family::dynamics' DRIFT
/// branch compiled in; the other families' instantiations leave it out).
template <int NX, int NU, int TH, bool FAST, bool DR = false>
__global__ void __launch_bounds__(TH, NX >= 16 ? 2 : (TH > 128 ? 3 : 4)) assemble_kernel_t(View v, const int* __restrict__ work,
                                                                      const int* __restrict__ n_work, double eps_pd,
                                                                      int do_schur) {
  static_assert(32 % NX == 0, "group size must divide the warp");
  using Lay = AsmLayout<NX, NU>;
  constexpr int B2 = NX * NX;
  constexpr int LD = Lay::LD, LDU = Lay::LDU;
  constexpr int NG = TH / NX;
  extern __shared__ double sm_asm[];
  __shared__ AsmShared sh;
  const Dims d = v.d;
  const int T = d.T;
  const int tid = threadIdx.x;
  const int g = tid / NX, l = tid % NX;
  const unsigned gmask = ((NX == 32 ? 0xffffffffu : ((1u << NX) - 1u))) << ((tid & 31) / NX * NX);
  double* buf = sm_asm + static_cast<long>(g) * Lay::GBUF;
  double* sA = buf;              // A_t            | P_t   (phase C)
  double* sM1 = sA + Lay::P2;    // M1 -> chol L   | sub_t (phase C)
  double* sC = sM1 + Lay::P2;    // chi -> X=chi^-1| T1    (phase C)
  double* sD = sC + Lay::P2;     // sym(chi)       | P_{t+1} (phase C)
  double* sB = sD + Lay::P2;     // B_t            } until chi is formed
  double* sM2 = sB + Lay::PB;    // M2             }
  double* sO = sB;               // output block (logical (i, j) layout; flush permutes)
  // element (i, j) of an NX-row group matrix / of M2
  auto ix = [](int i, int j) { return i + j * LD; };
  auto iu = [](int i, int j) { return i + j * LDU; };
  auto stage = [&](int /*b*/, int i, int j, double val) { sO[ix(i, j)] = val; };
  // coalesced copy of the staged block to block b of a region in the device
  // layout (16-byte stores; offsets o, o + 1 hold entries (e, s), (e + 1, s))
  auto flush = [&](double* region, int b) {
    __syncwarp(gmask);
    double2* dst = reinterpret_cast<double2*>(region + static_cast<long>(b) * B2);
#pragma unroll
    for (int k = l; k < B2 / 2; k += NX) {
      int e, sc;
      blk_entry(NX, b, 2 * k, &e, &sc);
      dst[k] = make_double2(sO[ix(e, sc)], sO[ix(e + 1, sc)]);
    }
    __syncwarp(gmask);
  };

  const bool stage_in = d.nz + d.nth <= NG * Lay::GBUF;
#ifdef DOCP_K1_CLOCK
  long long k1clk[16] = {0}, k1last = clock64();
#endif
  for (int w = blockIdx.x; w < *n_work; w += gridDim.x) {
    const int p = work[w];
    K1_CLK(11);
    // z / theta staged in the group buffers (free until phase B) when they fit
    if (!phase_linearize<NX, NU, DR>(v, p, eps_pd, do_schur, sh, stage_in ? sm_asm : nullptr)) {
      __syncthreads();
      continue;
    }
    K1_CLK(0);
    const double* lq = v.lq + static_cast<long>(p) * d.nb * NX;
    const double* lr = v.lr + static_cast<long>(p) * T * NU;
    const double* qdp = v.qd + static_cast<long>(p) * d.nb * NX;
    const double* rdp = v.rd + static_cast<long>(p) * T * NU;
    double* blk = blk_ptr(v, p);
    double* Sd = blk + d.s_diag;
    double* Ss = blk + d.s_sub;
    double* Pd = blk + d.p_diag;
    double* Pu = blk + d.p_sup;
    stage0_blocks(v, p);

    // Rounds of NG consecutive stages (group g takes stage t0 + g): phase B of
    // every group, a CTA barrier, then phase C of every group with P_t read
    // from the previous group's shared buffer (group 0: the previous round's
    // hand-off in `carry`, or Q_0 at t = 0) and sub_t, P_{t+1} still on-chip.
    double* carry = sm_asm + NG * Lay::GBUF;  // [2][P2]
    for (int t0 = 0; t0 < T; t0 += NG) {
      const int t = t0 + g;
      bool ok = t < T;  // the stage exists and chi_t factorised
      double dq = 0.0;
      // ---------------- phase B (schur.hpp:143-167)
      if (ok) {
        const double* lqt = lq + t * NX;
        const double* lqn = lq + (t + 1) * NX;
        const double* lrt = lr + t * NU;
        const double* At = v.A + a_off(d, p, t);
        const double* Bt = v.Bm + b_off(d, p, t);
        // FAST: the stage's cost diagonals are loaded first, so their latency
        // overlaps the A / B staging below
        double q_t = 0.0, q_n = 0.0, r_t = 0.0;
        if constexpr (FAST) {
          q_t = qdp[t * NX + l];
          q_n = qdp[(t + 1) * NX + l];
          if (l < NU) r_t = rdp[t * NU + l];
        }
#pragma unroll
        for (int k = l; k < B2; k += NX) sA[ix(k % NX, k / NX)] = At[k];
#pragma unroll
        for (int k = l; k < NX * NU; k += NX) sB[ix(k % NX, k / NX)] = Bt[k];
        __syncwarp(gmask);
        K1_CLK(1);
        // M1(k, l) = (A(l,k)/lq_k)/lq_k ; M2(k, l) = (B(l,k)/lr_k)/lr_k
        double c3;
        if constexpr (FAST) {  // lane k scales column k of A (of B) by 1/q_k (1/r_k)
          dq = __drcp_rn(q_t);
          c3 = __drcp_rn(q_n);
#pragma unroll
          for (int j = 0; j < NX; ++j) sM1[ix(l, j)] = sA[ix(j, l)] * dq;
          if (l < NU) {
            const double ir = __drcp_rn(r_t);
#pragma unroll
            for (int j = 0; j < NX; ++j) sM2[iu(l, j)] = sB[ix(j, l)] * ir;
          }
        } else {
#pragma unroll
            for (int k = 0; k < NX; ++k) sM1[ix(k, l)] = (sA[ix(l, k)] / lqt[k]) / lqt[k];
#pragma unroll
            for (int k = 0; k < NU; ++k) sM2[iu(k, l)] = (sB[ix(l, k)] / lrt[k]) / lrt[k];
            c3 = (1.0 / lqn[l]) / lqn[l];
            dq = (1.0 / lqt[l]) / lqt[l];
          }
          __syncwarp(gmask);
          K1_CLK(2);
          // column l of chi = A M1 + B M2 + A+ Q+^-1 A+'  and of phi_t = A Q_t^-1
          // (the lane's columns of M1 and M2 in registers: the stores into sC
          // below would otherwise force their reload for every row)
          double m1[NX], m2[NU];
#pragma unroll
          for (int m = 0; m < NX; ++m) m1[m] = sM1[ix(m, l)];
#pragma unroll
          for (int m = 0; m < NU; ++m) m2[m] = sM2[iu(m, l)];
#pragma unroll
          for (int i = 0; i < NX; ++i) {
            double a = sA[ix(i, 0)] * m1[0];
            double b = sB[ix(i, 0)] * m2[0];
            if constexpr (FAST) {
#pragma unroll
              for (int m = 1; m < NX; ++m) a = fma(sA[ix(i, m)], m1[m], a);
#pragma unroll
              for (int m = 1; m < NU; ++m) b = fma(sB[ix(i, m)], m2[m], b);
            } else {
#pragma unroll
              for (int m = 1; m < NX; ++m) a = a + sA[ix(i, m)] * m1[m];
#pragma unroll
              for (int m = 1; m < NU; ++m) b = b + sB[ix(i, m)] * m2[m];
            }
            sC[ix(i, l)] = (a + b) + (i == l ? c3 : 0.0);
          }
          __syncwarp(gmask);  // B_t / M2 are dead: sO takes their place
          K1_CLK(3);
#pragma unroll
          for (int i = 0; i < NX; ++i) stage(t, i, l, sA[ix(i, l)] * dq);
          flush(Ss, t);
#pragma unroll
          for (int i = 0; i < NX; ++i) {
            const double dv = 0.5 * (sC[ix(i, l)] + sC[ix(l, i)]);
            sD[ix(i, l)] = dv;
            stage(t + 1, i, l, dv);
            sM1[ix(i, l)] = 0.0;  // becomes L
          }
          flush(Sd, t + 1);
          K1_CLK(4);
          // Cholesky of chi_t (eigen_lite LLT): lane l computes row l
          double* sL = sM1;
          bool failed = false;
#pragma unroll
          for (int k = 0; k < NX; ++k) {
            double s = 0.0;
            if (k > 0) {
              s = sL[ix(k, 0)] * sL[ix(k, 0)];
#pragma unroll
              for (int j = 1; j < k; ++j) s = FAST ? fma(sL[ix(k, j)], sL[ix(k, j)], s) : s + sL[ix(k, j)] * sL[ix(k, j)];
            }
            const double piv = sD[ix(k, k)] - s;
            if (piv <= 0.0) {
              failed = true;
              break;
            }
            // FAST: the factor's diagonal holds 1/l_kk (only the solves read it)
            const double lk = FAST ? rsqrt(piv) : sqrt(piv);
            if (l == k) sL[ix(k, k)] = lk;
            if (l > k) {
              double tt = 0.0;
              if (k > 0) {
                tt = sL[ix(l, 0)] * sL[ix(k, 0)];
#pragma unroll
                for (int j = 1; j < k; ++j) tt = FAST ? fma(sL[ix(l, j)], sL[ix(k, j)], tt) : tt + sL[ix(l, j)] * sL[ix(k, j)];
              }
              sL[ix(l, k)] = FAST ? (sD[ix(l, k)] - tt) * lk : (sD[ix(l, k)] - tt) / lk;
            }
            __syncwarp(gmask);
          }
          K1_CLK(5);
          if (failed) {
            if (l == 0) atomicMin(&sh.rank_chi, t);
            __syncwarp(gmask);
            ok = false;
          } else {
          // chi_t^-1 = chol.solve(I): lane l solves column l
          double* sX = sC;
          {
            double x[NX];
#pragma unroll
            for (int i = 0; i < NX; ++i) {
              double s = 0.0;
              if (i > 0) {
                s = sL[ix(i, 0)] * x[0];
#pragma unroll
                for (int j = 1; j < i; ++j) s = FAST ? fma(sL[ix(i, j)], x[j], s) : s + sL[ix(i, j)] * x[j];
              }
              if constexpr (FAST) {
                x[i] = ((i == l ? 1.0 : 0.0) - s) * sL[ix(i, i)];
              } else {
                // a zero numerator (rows above the unit entry of column l)
                // is its own quotient: L(i, i) = sqrt(pivot) > 0, so 0 / L is
                // the same signed zero; skipping the division keeps those
                // lanes off its slow path (taken for zero numerators)
                const double num = (i == l ? 1.0 : 0.0) - s;
                x[i] = num;
                if (num != 0.0) x[i] = num / sL[ix(i, i)];
              }
            }
#pragma unroll
            for (int i = NX - 1; i >= 0; --i) {
              double s = 0.0;
              if (i + 1 < NX) {
                s = sL[ix(i + 1, i)] * x[i + 1];
#pragma unroll
                for (int j = i + 2; j < NX; ++j) s = FAST ? fma(sL[ix(j, i)], x[j], s) : s + sL[ix(j, i)] * x[j];
              }
              if constexpr (FAST) {
                x[i] = (x[i] - s) * sL[ix(i, i)];
              } else {
                const double num = x[i] - s;  // zero numerators as above
                x[i] = num;
                if (num != 0.0) x[i] = num / sL[ix(i, i)];
              }
            }
            __syncwarp(gmask);  // everyone is done reading chi (sC) before it becomes X
#pragma unroll
            for (int i = 0; i < NX; ++i) sX[ix(i, l)] = x[i];
          }
          __syncwarp(gmask);
          K1_CLK(6);
#pragma unroll
          for (int i = 0; i < NX; ++i) {
            const double pv = 0.5 * (sX[ix(i, l)] + sX[ix(l, i)]);
            stage(t + 1, i, l, pv);
            sD[ix(i, l)] = pv;  // P_{t+1} for phase C (sym(chi) is dead after the factorisation)
          }
          flush(Pd, t + 1);
#pragma unroll
          for (int i = 0; i < NX; ++i) sM1[ix(i, l)] = sA[ix(i, l)] * dq;  // sub_t (= the Ss_t block); L is dead
          K1_CLK(7);
        }  // chi_t factorised
      }  // stage exists
      __syncthreads();
      K1_CLK(8);

      // ---------------- phase C: stair off-diagonal (-D_t phi_t') D_{t+1} (schur.hpp:169-179)
      if (ok) {
        const double* Pt;
        if (g > 0) {
          Pt = sm_asm + static_cast<long>(g - 1) * Lay::GBUF + 3 * Lay::P2;  // previous group's P_t
        } else if (t > 0) {
          Pt = carry + ((t0 / NG - 1) & 1) * Lay::P2;
        } else {  // P_0 = Q_0 (stage0_blocks)
          const double* qd0 = v.qd + static_cast<long>(p) * d.nb * NX;
#pragma unroll
          for (int i = 0; i < NX; ++i) sA[ix(i, l)] = i == l ? qd0[l] : 0.0;
          __syncwarp(gmask);
          Pt = sA;
        }
        // T1(i, l) = sum_m (-P_t(i,m)) sub_t(l,m); row l of sub_t and column
        // l of P_{t+1} in registers (the stores in between would force reloads)
        double sub[NX], pn[NX];
#pragma unroll
        for (int m = 0; m < NX; ++m) sub[m] = sM1[ix(l, m)];
#pragma unroll
        for (int i = 0; i < NX; ++i) {
          double a = (-Pt[ix(i, 0)]) * sub[0];
#pragma unroll
          for (int m = 1; m < NX; ++m) a = FAST ? fma(-Pt[ix(i, m)], sub[m], a) : a + (-Pt[ix(i, m)]) * sub[m];
          sC[ix(i, l)] = a;
        }
#pragma unroll
        for (int m = 0; m < NX; ++m) pn[m] = sD[ix(m, l)];
        __syncwarp(gmask);
#pragma unroll
        for (int i = 0; i < NX; ++i) {
          double a = sC[ix(i, 0)] * pn[0];
#pragma unroll
          for (int m = 1; m < NX; ++m) a = FAST ? fma(sC[ix(i, m)], pn[m], a) : a + sC[ix(i, m)] * pn[m];
          stage(t, i, l, a);
        }
        flush(Pu, t);
        if (g == NG - 1) {  // hand P_{t+1} to group 0 of the next round
#pragma unroll
          for (int i = 0; i < NX; ++i) carry[((t0 / NG) & 1) * Lay::P2 + ix(i, l)] = sD[ix(i, l)];
        }
      }
      K1_CLK(9);
      __syncthreads();
      K1_CLK(10);
    }
    if (sh.rank_chi != kNoError) {
      if (tid == 0) set_status(v.status + p, DOCP_NUMERICAL, DOCP_AT_CHOL_CHI, sh.rank_chi);
    }
    __syncthreads();  // sh is re-initialised by the next problem
  }
#ifdef DOCP_K1_CLOCK
  if (threadIdx.x == 0)
    for (int k = 0; k < 12; ++k) atomicAdd(&g_k1_clk[k], static_cast<unsigned long long>(k1clk[k]));
#endif
}

/// Solve Q_t x = b for the diagonal Cholesky factor l: (b / l) / l.
__device__ inline double diag_solve(double b, double l) { return (b / l) / l; }

/// GAMMA <- -(d + H G^-1 b) (schur.hpp:187-211), one CTA per problem: the
/// block solves Q_t^-1 b_x, R_t^-1 b_u are formed once per entry into SMEM
/// (two divisions each, as the reference's LLT solves), then every output row
/// folds them in the reference order. NX, NU > 0 fix the block sizes at
/// compile time (the index arithmetic folds; same floating-point operations).
/// rhs FORWARD: b = flat_b, d = flat_d; ADJOINT: b = -LOSS_GRAD_Z, d = 0.
template <int NX = 0, int NU = 0>
__global__ void __launch_bounds__(128) gamma_kernel(View v, const int* __restrict__ work,
                                                    const int* __restrict__ n_work, int rhs) {
  extern __shared__ double sm_gam[];
  const Dims d = v.d;
  const int nx = NX ? NX : d.nx, nu = NU ? NU : d.nu, T = d.T;
  const int nb = T + 1, nl = nb * nx, nz = nl + T * nu, sz = nx + nu;
  double* sq = sm_gam;              // [T+1][nx]
  double* su = sm_gam + nb * nx;    // [T][nu]
  for (int w = blockIdx.x; w < *n_work; w += gridDim.x) {
    const int p = work[w];
    const double* lq = v.lq + static_cast<long>(p) * nb * nx;
    const double* lr = v.lr + static_cast<long>(p) * T * nu;
    const double* lg = v.lgz + static_cast<long>(p) * nz;
    const double* qp = v.q + static_cast<long>(p) * nb * nx;
    const double* rp = v.r + static_cast<long>(p) * T * nu;
    for (int e = threadIdx.x; e < nb * nx; e += blockDim.x) {
      const int t = e / nx, k = e - t * nx;
      const double b = rhs == DOCP_RHS_FORWARD ? qp[e] : -lg[t * sz + k];
      sq[e] = diag_solve(b, lq[e]);
    }
    for (int e = threadIdx.x; e < T * nu; e += blockDim.x) {
      const int t = e / nu, k = e - t * nu;
      const double b = rhs == DOCP_RHS_FORWARD ? rp[e] : -lg[t * sz + nx + k];
      su[e] = diag_solve(b, lr[e]);
    }
    __syncthreads();
    const double* Cp = v.C + static_cast<long>(p) * T * nx;
    for (int row = threadIdx.x; row < nl; row += blockDim.x) {
      const int blk = row / nx, i = row - blk * nx;
      double out;
      if (blk == 0) {
        const double dd = rhs == DOCP_RHS_FORWARD ? v.xs[static_cast<long>(p) * nx + i] : 0.0;
        out = dd + sq[i];
      } else {
        const int t = blk - 1;
        const double* At = v.A + a_off(d, p, t);
        const double* Bt = v.Bm + b_off(d, p, t);
        const double* s0 = sq + t * nx;
        const double* s1 = su + t * nu;
        double a = At[i] * s0[0];
#pragma unroll
        for (int k = 1; k < nx; ++k) a = a + At[i + k * nx] * s0[k];
        double b = Bt[i] * s1[0];
#pragma unroll
        for (int k = 1; k < nu; ++k) b = b + Bt[i + k * nx] * s1[k];
        const double c = sq[(t + 1) * nx + i];
        const double dd = rhs == DOCP_RHS_FORWARD ? Cp[t * nx + i] : 0.0;
        out = dd + ((a + b) + c);
      }
      v.gamma[static_cast<long>(p) * nl + row] = -out;
    }
    __syncthreads();
  }
}

/// Z_QP <- recover_primal(lambda, b) (sqp.hpp:62-89), one CTA per problem:
/// the problem's multipliers are staged in shared memory with coalesced
/// loads, then one thread per primal entry folds in the reference order.
template <int NX = 0, int NU = 0>
__global__ void __launch_bounds__(128) recover_kernel(View v, const int* __restrict__ work,
                                                      const int* __restrict__ n_work,
                                                      const double* __restrict__ lam_all, int rhs) {
  extern __shared__ double sm_rec[];  // [n_lambda]
  const Dims d = v.d;
  const int nx = NX ? NX : d.nx, nu = NU ? NU : d.nu, T = d.T;
  const int nb = T + 1, nl = nb * nx, nz = nl + T * nu, sz = nx + nu;
  for (int w = blockIdx.x; w < *n_work; w += gridDim.x) {
    const int p = work[w];
    const double* lamg = lam_all + static_cast<long>(p) * nl;
    cta_stage(sm_rec, lamg, nl);
    __syncthreads();
    const double* lam = sm_rec;
    const double* lg = v.lgz + static_cast<long>(p) * nz;
    double* zq = v.zqp + static_cast<long>(p) * nz;
    for (int e = threadIdx.x; e < nz; e += blockDim.x) {
      const int t = e / sz, c = e - t * sz;
      double rhs_v = rhs == DOCP_RHS_FORWARD ? 0.0 : -lg[e];
      double out;
      if (c < nx) {  // x_t,c = -Q_t^-1 (b + A+_{t-1}' lam_t + A_t' lam_{t+1})
        const int i = c;
        if (rhs == DOCP_RHS_FORWARD) rhs_v = v.q[(static_cast<long>(p) * nb + t) * nx + i];
        rhs_v = rhs_v + lam[t * nx + i];
        if (t < T) {
          const double* At = v.A + a_off(d, p, t);
          const double* l1 = lam + (t + 1) * nx;
          double a = At[i * nx] * l1[0];
#pragma unroll
          for (int k = 1; k < nx; ++k) a = a + At[k + i * nx] * l1[k];
          rhs_v = rhs_v + a;
        }
        out = -diag_solve(rhs_v, v.lq[(static_cast<long>(p) * nb + t) * nx + i]);
      } else {  // u_t,i = -R_t^-1 (b + B_t' lam_{t+1})
        const int i = c - nx;
        if (rhs == DOCP_RHS_FORWARD) rhs_v = v.r[(static_cast<long>(p) * T + t) * nu + i];
        const double* Bt = v.Bm + b_off(d, p, t);
        const double* l1 = lam + (t + 1) * nx;
        double a = Bt[i * nx] * l1[0];
#pragma unroll
        for (int k = 1; k < nx; ++k) a = a + Bt[k + i * nx] * l1[k];
        out = -diag_solve(rhs_v + a, v.lr[(static_cast<long>(p) * T + t) * nu + i]);
      }
      zq[e] = out;
    }
    __syncthreads();
  }
}

}  // namespace docp_dev
