// k_pcg.cuh — K2: the fused preconditioned conjugate gradient (pcg.hpp:52-109)
// on (-S) lambda = -gamma with the stair preconditioner Phi^-1.
//
// One CTA per problem; persistent CTAs pull problems from an atomic queue.
// RESIDENT: the problem's whole block record (-S diag + sub, Phi^-1 diag +
// super; symmetric storage, 205,824 B at n_x=8, T=100) is staged into shared
// memory by one TMA bulk copy (cp.async.bulk -> SASS UBLKCP) and re-read from
// SMEM every iteration. STREAMING (records larger than SMEM): the same layout
// is read through the read-only L1/L2 path.
//
// Thread = one BLOCK ROW i (all n_x rows): its lambda_i, r_i, p_i, y_i live
// in registers for the whole solve, and it reads each of its blocks (D_i and
// the off-diagonal block O_i) exactly once per product. O_i serves both
// neighbours: thread i forms its own upper term from O_i and x_{i+1} and the
// lower term of block row i+1 from O_i and x_i, handing the latter over
// through a small SMEM exchange buffer. Only x_{i+1} (8 doubles) and that
// 8-double hand-over cross threads, so SMEM traffic is ~ the block bytes.
// Per iteration: y = (-S) p (btd_matvec, schur.hpp:60-72), v = p'y,
// lambda/r update, r~ = Phi^-1 r (precond_apply, schur.hpp:76-78),
// eta' = r'r~, p update. Dots: warp shuffles + one SMEM stage (FAST) or the
// reference's block-ordered left folds (PARITY, pcg.hpp:37-44). Every product
// keeps the reference's per-row fold order (diag, then sub, then super).
#pragma once

#include "common.cuh"

namespace docp_dev {


template <bool SMEM>
__device__ __forceinline__ double2 ld2(const double* p) {
  if constexpr (SMEM) return *reinterpret_cast<const double2*>(p);
  else return __ldg(reinterpret_cast<const double2*>(p));
}
template <bool SMEM>
__device__ __forceinline__ double ld1(const double* p) {
  if constexpr (SMEM) return *p;
  else return __ldg(p);
}

/// a*b + acc in the chosen arithmetic (PARITY: rounded multiply, then add).
template <bool PAR>
__device__ __forceinline__ double madd(double a, double b, double acc) {
  if constexpr (PAR) return acc + a * b;
  else return fma(a, b, acc);
}

/// Column s of block b (NX rows) from a region in the device block layout.
template <int NX, bool SMEM>
__device__ __forceinline__ void load_col(const double* region, int b, int s, int nx, double* out) {
  if constexpr (NX > 0 && NX % 2 == 0) {
    const double* base = region + static_cast<long>(b) * NX * NX;
#pragma unroll
    for (int k = 0; k < NX / 2; ++k) {
      const double2 c = ld2<SMEM>(base + blk_off(NX, b, 2 * k, s));
      out[2 * k] = c.x;
      out[2 * k + 1] = c.y;
    }
  } else {
    const int n = NX > 0 ? NX : nx;
    const double* base = region + static_cast<long>(b) * n * n;
    for (int e = 0; e < n; ++e) out[e] = ld1<SMEM>(base + blk_off(n, b, e, s));
  }
}

/// Block j of an iterate vector held in SMEM (vec_off layout).
template <int NX>
__device__ __forceinline__ void load_vec(const double* buf, int j, int nx, double* out) {
  if constexpr (NX > 0 && NX % 2 == 0) {
#pragma unroll
    for (int k = 0; k < NX / 2; ++k) {
      const double2 c = *reinterpret_cast<const double2*>(buf + vec_off(NX, j, 2 * k));
      out[2 * k] = c.x;
      out[2 * k + 1] = c.y;
    }
  } else {
    const int n = NX > 0 ? NX : nx;
    for (int e = 0; e < n; ++e) out[e] = buf[j * n + e];
  }
}
template <int NX>
__device__ __forceinline__ void store_vec(double* buf, int j, int nx, const double* in) {
  if constexpr (NX > 0 && NX % 2 == 0) {
#pragma unroll
    for (int k = 0; k < NX / 2; ++k)
      *reinterpret_cast<double2*>(buf + vec_off(NX, j, 2 * k)) = make_double2(in[2 * k], in[2 * k + 1]);
  } else {
    const int n = NX > 0 ? NX : nx;
    for (int e = 0; e < n; ++e) buf[j * n + e] = in[e];
  }
}

/// Block row i of a symmetric block-tridiagonal product, phase 1.
///   own[r] = (D_i x_i)[r]                           (diag term)
/// and, when block row i+1 exists, from the off-diagonal block O_i:
///   S (SWAP=false, O = sub L_i):   up  = L_i' x_{i+1}, out = L_i x_i
///   P (SWAP=true,  O = super U_i): up  = U_i x_{i+1},  out = U_i' x_i
/// `out` is block row i+1's lower term (L_i x_i, resp. U_i' x_i) — handed over.
/// Every entry is a left fold in the reference gemv order.
template <int NX, int NN, bool SWAP, bool PAR, bool SMEM>
__device__ __forceinline__ void btd_phase1_impl(const double* D, const double* O, const double* x, const double* xn,
                                           int i, int nb, int nx, double* own, double* up, double* out) {
  const int n = NX > 0 ? NX : nx;
  double m[NN];
#pragma unroll
  for (int c = 0; c < NN; ++c) {
    if (NX == 0 && c >= n) break;
    load_col<NX, SMEM>(D, i, c, nx, m);
#pragma unroll
    for (int r = 0; r < NN; ++r) {
      if (NX == 0 && r >= n) break;
      own[r] = c == 0 ? m[r] * x[0] : madd<PAR>(m[r], x[c], own[r]);
    }
  }
  if (i + 1 >= nb) return;
  // X dotted with each column, Y accumulated by columns
  const double* X = SWAP ? x : xn;
  const double* Y = SWAP ? xn : x;
  double* dotted = SWAP ? out : up;
  double* accum = SWAP ? up : out;
#pragma unroll
  for (int c = 0; c < NN; ++c) {
    if (NX == 0 && c >= n) break;
    load_col<NX, SMEM>(O, i, c, nx, m);
    double t = m[0] * X[0];
#pragma unroll
    for (int e = 1; e < NN; ++e) {
      if (NX == 0 && e >= n) break;
      t = madd<PAR>(m[e], X[e], t);
    }
    dotted[c] = t;
#pragma unroll
    for (int r = 0; r < NN; ++r) {
      if (NX == 0 && r >= n) break;
      accum[r] = c == 0 ? m[r] * Y[0] : madd<PAR>(m[r], Y[c], accum[r]);
    }
  }
}

template <int NX, int NN, bool SWAP, bool PAR, bool SMEM>
__device__ __noinline__ void btd_phase1_rt(const double* D, const double* O, const double* x, const double* xn, int i,
                                           int nb, int nx, double* own, double* up, double* out) {
  // runtime n_x: the same folds without unrolling (keeps the generic variant small)
  double m[NN];
  for (int c = 0; c < nx; ++c) {
    load_col<NX, SMEM>(D, i, c, nx, m);
    for (int r = 0; r < nx; ++r) own[r] = c == 0 ? m[r] * x[0] : madd<PAR>(m[r], x[c], own[r]);
  }
  if (i + 1 >= nb) return;
  const double* X = SWAP ? x : xn;
  const double* Y = SWAP ? xn : x;
  double* dotted = SWAP ? out : up;
  double* accum = SWAP ? up : out;
  for (int c = 0; c < nx; ++c) {
    load_col<NX, SMEM>(O, i, c, nx, m);
    double t = m[0] * X[0];
    for (int e = 1; e < nx; ++e) t = madd<PAR>(m[e], X[e], t);
    dotted[c] = t;
    for (int r = 0; r < nx; ++r) accum[r] = c == 0 ? m[r] * Y[0] : madd<PAR>(m[r], Y[c], accum[r]);
  }
}

template <int NX, int NN, bool SWAP, bool PAR, bool SMEM>
__device__ __forceinline__ void btd_phase1(const double* D, const double* O, const double* x, const double* xn,
                                           int i, int nb, int nx, double* own, double* up, double* out) {
  if constexpr (NX > 0) btd_phase1_impl<NX, NN, SWAP, PAR, SMEM>(D, O, x, xn, i, nb, nx, own, up, out);
  else btd_phase1_rt<NX, NN, SWAP, PAR, SMEM>(D, O, x, xn, i, nb, nx, own, up, out);
}

/// Dot of the thread's block rows with a block-wide reduction.
/// FAST: fma chains, warp butterflies, one SMEM stage (deterministic and the
/// same value in every warp). PARITY: block_dot of pcg.hpp:37-44 — per-block
/// left folds (local to the owning thread), then a left fold over blocks in
/// index order.
template <int NN, int MAXB, bool PAR>
__device__ __forceinline__ double block_dot(const double (&a)[MAXB][NN], const double (&b)[MAXB][NN],
                                            const int (&bi)[MAXB], int nb, int nx, double* red, double* seg) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  if constexpr (!PAR) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < MAXB; ++k)
      if (bi[k] < nb)
#pragma unroll
        for (int e = 0; e < NN; ++e)
          if (e < nx) s = fma(a[k][e], b[k][e], s);
    s = warp_sum(s);
    if (lane == 0) red[warp] = s;
    __syncthreads();
    const double t = lane < nw ? red[lane] : 0.0;
    return warp_sum(t);
  } else {
#pragma unroll
    for (int k = 0; k < MAXB; ++k)
      if (bi[k] < nb) {
        double s = a[k][0] * b[k][0];
#pragma unroll
        for (int e = 1; e < NN; ++e)
          if (e < nx) s = s + a[k][e] * b[k][e];
        seg[bi[k]] = s;
      }
    __syncthreads();
    double acc = 0.0;
    if (lane == 0)
      for (int i = 0; i < nb; ++i) acc = acc + seg[i];
    return __shfl_sync(0xffffffffu, acc, 0);
  }
}

/// ||a||_2 as Vector::norm() (left fold over all entries; only for the rare
/// eta guard, pcg.hpp:72-79).
template <int NN, int MAXB, bool PAR>
__device__ double block_norm(const double (&a)[MAXB][NN], const int (&bi)[MAXB], int nb, int nx, double* red,
                             double* prod) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  double out;
  if constexpr (!PAR) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < MAXB; ++k)
      if (bi[k] < nb)
        for (int e = 0; e < nx; ++e) s = fma(a[k][e], a[k][e], s);
    s = warp_sum(s);
    if (lane == 0) red[warp] = s;
    __syncthreads();
    out = warp_sum(lane < nw ? red[lane] : 0.0);
  } else {
#pragma unroll
    for (int k = 0; k < MAXB; ++k)
      if (bi[k] < nb)
        for (int e = 0; e < nx; ++e) prod[bi[k] * nx + e] = a[k][e] * a[k][e];
    __syncthreads();
    double acc = 0.0;
    if (lane == 0) {
      acc = prod[0];
      for (int q = 1; q < nb * nx; ++q) acc = acc + prod[q];
    }
    out = __shfl_sync(0xffffffffu, acc, 0);
  }
  __syncthreads();
  return sqrt(out);
}

/// K2. NX in {4, 8, 16}: compile-time block size; NX == 0: any n_x <= 16.
template <int NX, int MAXB, bool PAR, bool RESIDENT>
__global__ void __launch_bounds__(kPcgMaxThreads, (NX == 4 && MAXB == 1 && !PAR) ? 2 : 1) pcg_kernel(View v, const int* __restrict__ work,
                                                            const int* __restrict__ n_work, int* __restrict__ counter,
                                                            double* __restrict__ sol_all, double epsilon,
                                                            int max_iters_cfg) {
  constexpr int NN = NX > 0 ? NX : kMaxNx;
  extern __shared__ __align__(128) double sm_pcg[];
  __shared__ __align__(8) uint64_t s_bar;
  __shared__ int s_work;
  const Dims d = v.d;
  const int nx = NX > 0 ? NX : d.nx;
  const int nl = d.nl, nb = d.nb;
  const int tid = threadIdx.x, NT = blockDim.x;

  double* cur = sm_pcg;
  double* sblk = nullptr;
  if constexpr (RESIDENT) {
    sblk = cur;
    cur += d.blk_stride;
  }
  double* vbuf = cur;  // the neighbour-read vector (lambda, then r / p)
  cur += (nl + 1) & ~1;
  double* xbuf = cur;  // lower-term hand-over
  cur += (nl + 1) & ~1;
  double* red = cur;
  cur += 64;
  double* seg = cur;  // PARITY: per-block dots / norm products (nl doubles)

  if constexpr (RESIDENT) {
    if (tid == 0) mbar_init(&s_bar, 1);
    __syncthreads();
  }
  uint32_t phase = 0;
  const int max_iters = max_iters_cfg > 0 ? max_iters_cfg : 2 * nl;
  const double threshold = epsilon * epsilon;
  int bi[MAXB];
#pragma unroll
  for (int k = 0; k < MAXB; ++k) bi[k] = tid + k * NT;

  for (;;) {
    if (tid == 0) s_work = atomicAdd(counter, 1);
    __syncthreads();
    const int w = s_work;
    if (w >= *n_work) break;
    const int p = work[w];
    if (v.status[p].code != DOCP_OK) {  // failed earlier in this SQP iteration
      __syncthreads();
      continue;
    }
    const double* rec = v.blocks + static_cast<long>(p) * d.blk_stride;
    const double* blk = rec;
    if constexpr (RESIDENT) {
      if (tid == 0) {
        fence_proxy_async();
        const uint32_t bytes = static_cast<uint32_t>((d.p_sup + ((static_cast<long>(d.T) * d.bsz + 1) & ~1L)) * 8);
        mbar_arrive_expect_tx(&s_bar, bytes);
        tma_bulk_g2s(sblk, rec, bytes, &s_bar);
      }
      blk = sblk;
    }
    const double* Sd = blk + d.s_diag;
    const double* Ss = blk + d.s_sub;
    const double* Pd = blk + d.p_diag;
    const double* Pu = blk + d.p_sup;
    const double* gam = v.gamma + static_cast<long>(p) * nl;
    double* sol = sol_all + static_cast<long>(p) * nl;

    double lam[MAXB][NN], r[MAXB][NN], pv[MAXB][NN], y[MAXB][NN];
#pragma unroll
    for (int k = 0; k < MAXB; ++k)
#pragma unroll
      for (int e = 0; e < NN; ++e) {
        lam[k][e] = r[k][e] = pv[k][e] = y[k][e] = 0.0;
        if (bi[k] < nb && e < nx) lam[k][e] = sol[bi[k] * nx + e];
      }
#pragma unroll
    for (int k = 0; k < MAXB; ++k)
      if (bi[k] < nb) store_vec<NX>(vbuf, bi[k], nx, lam[k]);
    if constexpr (RESIDENT) mbar_wait(&s_bar, phase);
    phase ^= 1;
    __syncthreads();

    // out = A x for A in {-S, Phi^-1}; x in registers (xr) and mirrored in vbuf
    auto matvec = [&](bool precond, const double (&xr)[MAXB][NN], double (&out)[MAXB][NN]) {
      double up[MAXB][NN], own[MAXB][NN];
#pragma unroll
      for (int k = 0; k < MAXB; ++k) {
        if (bi[k] >= nb) continue;
        double xn[NN], hand[NN];
        if (bi[k] + 1 < nb) load_vec<NX>(vbuf, bi[k] + 1, nx, xn);
        if (precond)
          btd_phase1<NX, NN, true, PAR, RESIDENT>(Pd, Pu, xr[k], xn, bi[k], nb, nx, own[k], up[k], hand);
        else
          btd_phase1<NX, NN, false, PAR, RESIDENT>(Sd, Ss, xr[k], xn, bi[k], nb, nx, own[k], up[k], hand);
        if (bi[k] + 1 < nb) store_vec<NX>(xbuf, bi[k], nx, hand);
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < MAXB; ++k) {
        if (bi[k] >= nb) continue;
        double low[NN];
        if (bi[k] > 0) load_vec<NX>(xbuf, bi[k] - 1, nx, low);
#pragma unroll
        for (int e = 0; e < NN; ++e) {
          if (e >= nx) break;
          double acc = own[k][e];
          if (bi[k] > 0) acc = acc + low[e];
          if (bi[k] + 1 < nb) acc = acc + up[k][e];
          out[k][e] = acc;
        }
      }
    };

    // r = gamma - (-S) lambda0 ; r~ = Phi^-1 r ; p = r~
    matvec(false, lam, y);
#pragma unroll
    for (int k = 0; k < MAXB; ++k)
      if (bi[k] < nb) {
#pragma unroll
        for (int e = 0; e < NN; ++e)
          if (e < nx) r[k][e] = gam[bi[k] * nx + e] - y[k][e];
      }
    __syncthreads();  // every neighbour read of lambda in vbuf is done
#pragma unroll
    for (int k = 0; k < MAXB; ++k)
      if (bi[k] < nb) store_vec<NX>(vbuf, bi[k], nx, r[k]);
    __syncthreads();
    matvec(true, r, pv);  // r~
    double eta = block_dot<NN, MAXB, PAR>(r, pv, bi, nb, nx, red, seg);
    int status = DOCP_OK, iters = 0;
    if (eta < 0.0) {  // guarded eta (pcg.hpp:72-79)
      const double scale = block_norm<NN, MAXB, PAR>(r, bi, nb, nx, red, seg) *
                           block_norm<NN, MAXB, PAR>(pv, bi, nb, nx, red, seg);
      if (-eta <= 1e-10 * scale + 1e-300) eta = 0.0;
      else status = DOCP_AT_PCG_PRECOND;
    }
#pragma unroll
    for (int k = 0; k < MAXB; ++k)
      if (bi[k] < nb) store_vec<NX>(vbuf, bi[k], nx, pv[k]);

    while (status == DOCP_OK && eta > threshold && iters < max_iters) {
      __syncthreads();
      matvec(false, pv, y);
      const double vv = block_dot<NN, MAXB, PAR>(pv, y, bi, nb, nx, red, seg);
      if (vv <= 0.0) {
        status = DOCP_AT_PCG_CURVATURE;
        break;
      }
      const double alpha = eta / vv;
#pragma unroll
      for (int k = 0; k < MAXB; ++k)
        if (bi[k] < nb) {
#pragma unroll
          for (int e = 0; e < NN; ++e)
            if (e < nx) {
              if constexpr (PAR) {
                lam[k][e] = lam[k][e] + alpha * pv[k][e];
                r[k][e] = r[k][e] - alpha * y[k][e];
              } else {
                lam[k][e] = fma(alpha, pv[k][e], lam[k][e]);
                r[k][e] = fma(-alpha, y[k][e], r[k][e]);
              }
            }
          store_vec<NX>(vbuf, bi[k], nx, r[k]);
        }
      __syncthreads();
      matvec(true, r, y);  // r~ (y reused)
      double eta_next = block_dot<NN, MAXB, PAR>(r, y, bi, nb, nx, red, seg);
      if (eta_next < 0.0) {
        const double scale = block_norm<NN, MAXB, PAR>(r, bi, nb, nx, red, seg) *
                             block_norm<NN, MAXB, PAR>(y, bi, nb, nx, red, seg);
        if (-eta_next <= 1e-10 * scale + 1e-300) {
          eta_next = 0.0;
        } else {
          status = DOCP_AT_PCG_PRECOND;
          break;
        }
      }
      const double beta = eta_next / eta;
#pragma unroll
      for (int k = 0; k < MAXB; ++k)
        if (bi[k] < nb) {
#pragma unroll
          for (int e = 0; e < NN; ++e)
            if (e < nx) {
              if constexpr (PAR) pv[k][e] = y[k][e] + beta * pv[k][e];
              else pv[k][e] = fma(beta, pv[k][e], y[k][e]);
            }
          store_vec<NX>(vbuf, bi[k], nx, pv[k]);
        }
      eta = eta_next;
      ++iters;
    }

#pragma unroll
    for (int k = 0; k < MAXB; ++k)
      if (bi[k] < nb)
#pragma unroll
        for (int e = 0; e < NN; ++e)
          if (e < nx) sol[bi[k] * nx + e] = lam[k][e];
    if (tid == 0) {
      v.pcg_iters[p] = iters;
      v.final_eta[p] = eta;
      v.pcg_conv[p] = status == DOCP_OK && eta <= threshold;
      if (status == DOCP_OK) set_status(v.status + p, DOCP_OK, DOCP_AT_NONE, 0);
      else set_status(v.status + p, DOCP_BREAKDOWN, status, iters);
      atomicAdd(v.pcg_acc, static_cast<unsigned long long>(iters));
      atomicAdd(v.pcg_acc + 1, 1ull);
      atomicAdd(v.pcg_acc + 2, 1ull);  // lifetime solves (docp_pcg_invocations)
    }
    __syncthreads();
  }
}

}  // namespace docp_dev
