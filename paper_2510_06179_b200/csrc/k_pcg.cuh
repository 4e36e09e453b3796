// k_pcg.cuh — K2: the fused preconditioned conjugate gradient (pcg.hpp:52-109)
// on (-S) lambda = -gamma with the stair preconditioner Phi^-1.
//
// One CTA per problem (persistent CTAs pull problems from an atomic work
// queue). In the RESIDENT variant the problem's whole block record (-S diag +
// sub, Phi^-1 diag + super; symmetric storage) is staged into shared memory by
// one TMA bulk copy (cp.async.bulk, SASS UBLKCP) and re-read from SMEM every
// iteration; the STREAMING variant (records larger than SMEM) reads the same
// layout through the read-only L1/L2 path. Thread = one row (block i, row r)
// of the n_x (T+1) system; its lambda, r, p, y entries live in registers for
// the whole solve, p and r are mirrored to SMEM for the neighbour reads of the
// block-tridiagonal products. Per iteration: y = (-S) p (btd_matvec,
// schur.hpp:60-72), v = p'y, lambda/r update, r~ = Phi^-1 r (precond_apply,
// schur.hpp:76-78), eta' = r'r~, p update — the two dots are warp-shuffle +
// SMEM reductions (FAST) or the reference's block-ordered folds (PARITY,
// pcg.hpp:37-44).
#pragma once

#include "common.cuh"

namespace docp_dev {

constexpr int kPcgMaxThreads = 1024;

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

/// acc*1 + a*b in the chosen arithmetic (PARITY: rounded mul then add).
template <bool PAR>
__device__ __forceinline__ double madd(double a, double b, double acc) {
  if constexpr (PAR) return acc + a * b;
  else return fma(a, b, acc);
}

// ---- fixed-NX block accessors (device block layout, common.cuh blk_off)
template <int NX, bool SMEM>
__device__ __forceinline__ void col_load(const double* region, int b, int s, double* out) {
  const double* base = region + static_cast<long>(b) * NX * NX;
#pragma unroll
  for (int k = 0; k < NX / 2; ++k) {
    const double2 c = ld2<SMEM>(base + blk_off(NX, b, 2 * k, s));
    out[2 * k] = c.x;
    out[2 * k + 1] = c.y;
  }
}
template <int NX, bool SMEM>
__device__ __forceinline__ void row_load(const double* region, int b, int e, double* out) {
  const double* base = region + static_cast<long>(b) * NX * NX;
#pragma unroll
  for (int s = 0; s < NX; ++s) out[s] = ld1<SMEM>(base + blk_off(NX, b, e, s));
}
template <int NX>
__device__ __forceinline__ void vec_load(const double* buf, int j, double* out) {
#pragma unroll
  for (int k = 0; k < NX / 2; ++k) {
    const double2 c = *reinterpret_cast<const double2*>(buf + vec_off(NX, j, 2 * k));
    out[2 * k] = c.x;
    out[2 * k + 1] = c.y;
  }
}

/// Row r of block row i of a symmetric block-tridiagonal product
///   y_i = D_i v_i + M_lo v_{i-1} + M_up v_{i+1}   (btd_matvec order, schur.hpp:66-69)
/// D is read by column (exactly symmetric). For -S the stored off-diagonal is
/// the sub block L (M_lo = L_{i-1}: row access; M_up = L_i': column access);
/// for Phi^-1 it is the super block U (M_lo = U_{i-1}': column; M_up = U_i: row).
template <int NX, bool LOWER_ROW, bool PAR, bool SMEM>
__device__ __forceinline__ double btd_row(const double* D, const double* O, const double* vec, int i, int r, int nb) {
  double m[NX], x[NX];
  col_load<NX, SMEM>(D, i, r, m);
  vec_load<NX>(vec, i, x);
  double acc = m[0] * x[0];
#pragma unroll
  for (int c = 1; c < NX; ++c) acc = madd<PAR>(m[c], x[c], acc);
  if (i > 0) {
    if constexpr (LOWER_ROW) row_load<NX, SMEM>(O, i - 1, r, m);
    else col_load<NX, SMEM>(O, i - 1, r, m);
    vec_load<NX>(vec, i - 1, x);
    double t = m[0] * x[0];
#pragma unroll
    for (int c = 1; c < NX; ++c) t = madd<PAR>(m[c], x[c], t);
    acc = acc + t;
  }
  if (i + 1 < nb) {
    if constexpr (LOWER_ROW) col_load<NX, SMEM>(O, i, r, m);
    else row_load<NX, SMEM>(O, i, r, m);
    vec_load<NX>(vec, i + 1, x);
    double t = m[0] * x[0];
#pragma unroll
    for (int c = 1; c < NX; ++c) t = madd<PAR>(m[c], x[c], t);
    acc = acc + t;
  }
  return acc;
}

/// Runtime-NX fallback (plain column-major blocks and vectors).
template <bool LOWER_ROW, bool PAR, bool SMEM>
__device__ __forceinline__ double btd_row_rt(const double* D, const double* O, const double* vec, int i, int r, int nb,
                                             int nx) {
  const long bs = static_cast<long>(nx) * nx;
  const double* Di = D + i * bs;
  double acc = ld1<SMEM>(Di + r * nx) * vec[i * nx];
  for (int c = 1; c < nx; ++c) acc = madd<PAR>(ld1<SMEM>(Di + r * nx + c), vec[i * nx + c], acc);
  if (i > 0) {
    const double* Oi = O + (i - 1) * bs;
    auto el = [&](int c) { return LOWER_ROW ? ld1<SMEM>(Oi + c * nx + r) : ld1<SMEM>(Oi + r * nx + c); };
    double t = el(0) * vec[(i - 1) * nx];
    for (int c = 1; c < nx; ++c) t = madd<PAR>(el(c), vec[(i - 1) * nx + c], t);
    acc = acc + t;
  }
  if (i + 1 < nb) {
    const double* Oi = O + i * bs;
    auto el = [&](int c) { return LOWER_ROW ? ld1<SMEM>(Oi + r * nx + c) : ld1<SMEM>(Oi + c * nx + r); };
    double t = el(0) * vec[(i + 1) * nx];
    for (int c = 1; c < nx; ++c) t = madd<PAR>(el(c), vec[(i + 1) * nx + c], t);
    acc = acc + t;
  }
  return acc;
}

struct PcgSmem {
  double* blocks;  // resident record or nullptr
  double* vbuf;    // p (lambda during the initial residual)
  double* rbuf;    // r
  double* red;     // 2 x 32 warp partials
  double* prod;    // PARITY: per-row products
  double* seg;     // PARITY: per-block dots
};

/// Block-wide dot of per-thread row products. FAST: warp butterflies and a
/// fixed-order cross-warp butterfly (deterministic, identical in every warp).
/// PARITY: block_dot of pcg.hpp:37-44 — per-block left folds, then a left
/// fold over blocks in index order.
template <int MAXR, bool PAR>
__device__ __forceinline__ double block_dot(const double (&a)[MAXR], const double (&b)[MAXR], const int (&row)[MAXR],
                                            int nl, int nx, int nb, double* red, double* prod, double* seg) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  if constexpr (!PAR) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < MAXR; ++k)
      if (row[k] < nl) s = fma(a[k], b[k], s);
    s = warp_sum(s);
    if (lane == 0) red[warp] = s;
    __syncthreads();
    double t = lane < nw ? red[lane] : 0.0;
    return warp_sum(t);
  } else {
#pragma unroll
    for (int k = 0; k < MAXR; ++k)
      if (row[k] < nl) prod[row[k]] = a[k] * b[k];
    __syncthreads();
    for (int i = tid; i < nb; i += blockDim.x) {
      double s = prod[i * nx];
      for (int e = 1; e < nx; ++e) s = s + prod[i * nx + e];
      seg[i] = s;
    }
    __syncthreads();
    double acc = 0.0;
    if (lane == 0)
      for (int i = 0; i < nb; ++i) acc = acc + seg[i];
    return __shfl_sync(0xffffffffu, acc, 0);
  }
}

/// ||a||_2 as Vector::norm(): sqrt of the left fold over all n entries
/// (PARITY) or a tree sum (FAST). Only used by the rare eta guard.
template <int MAXR, bool PAR>
__device__ double block_norm(const double (&a)[MAXR], const int (&row)[MAXR], int nl, double* red, double* prod) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if constexpr (!PAR) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < MAXR; ++k)
      if (row[k] < nl) s = fma(a[k], a[k], s);
    s = warp_sum(s);
    if (lane == 0) red[warp] = s;
    __syncthreads();
    double t = lane < nw ? red[lane] : 0.0;
    t = warp_sum(t);
    __syncthreads();
    return sqrt(t);
  } else {
#pragma unroll
    for (int k = 0; k < MAXR; ++k)
      if (row[k] < nl) prod[row[k]] = a[k] * a[k];
    __syncthreads();
    double acc = 0.0;
    if (lane == 0) {
      acc = prod[0];
      for (int i = 1; i < nl; ++i) acc = acc + prod[i];
    }
    acc = __shfl_sync(0xffffffffu, acc, 0);
    __syncthreads();
    return sqrt(acc);
  }
}

/// K2. NX > 0: fixed block size with the swizzled accessors; NX == 0: any n_x.
template <int NX, int MAXR, bool PAR, bool RESIDENT>
__global__ void __launch_bounds__(kPcgMaxThreads) pcg_kernel(View v, const int* __restrict__ work,
                                                            const int* __restrict__ n_work, int* __restrict__ counter,
                                                            double* __restrict__ sol_all, double epsilon,
                                                            int max_iters_cfg) {
  extern __shared__ __align__(128) double sm_pcg[];
  __shared__ __align__(8) uint64_t s_bar;
  __shared__ int s_work;
  const Dims d = v.d;
  const int nx = NX > 0 ? NX : d.nx;
  const int nl = d.nl, nb = d.nb;
  const int tid = threadIdx.x;
  const int NT = blockDim.x;

  PcgSmem sm;
  double* cur = sm_pcg;
  sm.blocks = nullptr;
  if constexpr (RESIDENT) {
    sm.blocks = cur;
    cur += d.blk_stride;
  }
  sm.vbuf = cur;
  cur += (nl + 1) & ~1;
  sm.rbuf = cur;
  cur += (nl + 1) & ~1;
  sm.red = cur;
  cur += 64;
  sm.prod = cur;
  cur += PAR ? ((nl + 1) & ~1) : 0;
  sm.seg = cur;

  if constexpr (RESIDENT) {
    if (tid == 0) mbar_init(&s_bar, 1);
    __syncthreads();
  }
  uint32_t phase = 0;
  const int max_iters = max_iters_cfg > 0 ? max_iters_cfg : 2 * nl;
  const double threshold = epsilon * epsilon;

  int row[MAXR], bi[MAXR], br[MAXR];
#pragma unroll
  for (int k = 0; k < MAXR; ++k) {
    row[k] = tid + k * NT;
    bi[k] = row[k] / nx;
    br[k] = row[k] - bi[k] * nx;
  }

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
        tma_bulk_g2s(sm.blocks, rec, bytes, &s_bar);
      }
      blk = sm.blocks;
    }
    const double* Sd = blk + d.s_diag;
    const double* Ss = blk + d.s_sub;
    const double* Pd = blk + d.p_diag;
    const double* Pu = blk + d.p_sup;
    const double* gam = v.gamma + static_cast<long>(p) * nl;
    double* sol = sol_all + static_cast<long>(p) * nl;

    double lam[MAXR], r[MAXR], pv[MAXR], y[MAXR];
#pragma unroll
    for (int k = 0; k < MAXR; ++k) {
      lam[k] = 0.0;
      r[k] = 0.0;
      pv[k] = 0.0;
      y[k] = 0.0;
      if (row[k] < nl) {
        lam[k] = sol[row[k]];
        sm.vbuf[NX > 0 ? vec_off(NX, bi[k], br[k]) : row[k]] = lam[k];
      }
    }
    if constexpr (RESIDENT) mbar_wait(&s_bar, phase);
    phase ^= 1;
    __syncthreads();

    auto mv_S = [&](int k) -> double {
      if constexpr (NX > 0) return btd_row<NX, true, PAR, RESIDENT>(Sd, Ss, sm.vbuf, bi[k], br[k], nb);
      else return btd_row_rt<true, PAR, RESIDENT>(Sd, Ss, sm.vbuf, bi[k], br[k], nb, nx);
    };
    auto mv_P = [&](int k) -> double {
      if constexpr (NX > 0) return btd_row<NX, false, PAR, RESIDENT>(Pd, Pu, sm.rbuf, bi[k], br[k], nb);
      else return btd_row_rt<false, PAR, RESIDENT>(Pd, Pu, sm.rbuf, bi[k], br[k], nb, nx);
    };
    auto put_r = [&](int k) { sm.rbuf[NX > 0 ? vec_off(NX, bi[k], br[k]) : row[k]] = r[k]; };
    auto put_p = [&](int k) { sm.vbuf[NX > 0 ? vec_off(NX, bi[k], br[k]) : row[k]] = pv[k]; };

    // r = gamma - (-S) lambda0 ; r~ = Phi^-1 r ; p = r~
#pragma unroll
    for (int k = 0; k < MAXR; ++k)
      if (row[k] < nl) {
        r[k] = gam[row[k]] - mv_S(k);
        put_r(k);
      }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < MAXR; ++k)
      if (row[k] < nl) pv[k] = mv_P(k);  // r~
    double eta = block_dot<MAXR, PAR>(r, pv, row, nl, nx, nb, sm.red, sm.prod, sm.seg);
    int status = DOCP_OK, iters = 0;
    if (eta < 0.0) {  // guarded eta (pcg.hpp:72-79)
      const double scale = block_norm<MAXR, PAR>(r, row, nl, sm.red, sm.prod) *
                           block_norm<MAXR, PAR>(pv, row, nl, sm.red, sm.prod);
      if (-eta <= 1e-10 * scale + 1e-300) eta = 0.0;
      else status = DOCP_AT_PCG_PRECOND;
    }
#pragma unroll
    for (int k = 0; k < MAXR; ++k)
      if (row[k] < nl) put_p(k);

    while (status == DOCP_OK && eta > threshold && iters < max_iters) {
      __syncthreads();
#pragma unroll
      for (int k = 0; k < MAXR; ++k)
        if (row[k] < nl) y[k] = mv_S(k);
      const double vv = block_dot<MAXR, PAR>(pv, y, row, nl, nx, nb, sm.red, sm.prod, sm.seg);
      if (vv <= 0.0) {
        status = DOCP_AT_PCG_CURVATURE;
        break;
      }
      const double alpha = eta / vv;
#pragma unroll
      for (int k = 0; k < MAXR; ++k)
        if (row[k] < nl) {
          if constexpr (PAR) {
            lam[k] = lam[k] + alpha * pv[k];
            r[k] = r[k] - alpha * y[k];
          } else {
            lam[k] = fma(alpha, pv[k], lam[k]);
            r[k] = fma(-alpha, y[k], r[k]);
          }
          put_r(k);
        }
      __syncthreads();
      double rt[MAXR];
#pragma unroll
      for (int k = 0; k < MAXR; ++k) rt[k] = row[k] < nl ? mv_P(k) : 0.0;
      double eta_next = block_dot<MAXR, PAR>(r, rt, row, nl, nx, nb, sm.red, sm.prod, sm.seg);
      if (eta_next < 0.0) {
        const double scale = block_norm<MAXR, PAR>(r, row, nl, sm.red, sm.prod) *
                             block_norm<MAXR, PAR>(rt, row, nl, sm.red, sm.prod);
        if (-eta_next <= 1e-10 * scale + 1e-300) {
          eta_next = 0.0;
        } else {
          status = DOCP_AT_PCG_PRECOND;
          break;
        }
      }
      const double beta = eta_next / eta;
#pragma unroll
      for (int k = 0; k < MAXR; ++k)
        if (row[k] < nl) {
          if constexpr (PAR) pv[k] = rt[k] + beta * pv[k];
          else pv[k] = fma(beta, pv[k], rt[k]);
          put_p(k);
        }
      eta = eta_next;
      ++iters;
    }

#pragma unroll
    for (int k = 0; k < MAXR; ++k)
      if (row[k] < nl) sol[row[k]] = lam[k];
    if (tid == 0) {
      v.pcg_iters[p] = iters;
      v.final_eta[p] = eta;
      v.pcg_conv[p] = status == DOCP_OK && eta <= threshold;
      if (status == DOCP_OK) set_status(v.status + p, DOCP_OK, DOCP_AT_NONE, 0);
      else set_status(v.status + p, DOCP_BREAKDOWN, status, iters);
      atomicAdd(v.pcg_acc, static_cast<unsigned long long>(iters));
      atomicAdd(v.pcg_acc + 1, 1ull);
    }
    __syncthreads();
  }
}

}  // namespace docp_dev
