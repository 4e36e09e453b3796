// k_pcg_h8.cuh — K2 for n_x = 8 (the benchmark shape): two threads per block
// row. Same algorithm, arithmetic and fold orders as pcg_kernel (k_pcg.cuh);
// thread (i, h) owns rows 4h..4h+3 of block row i, so a problem of T = 100
// runs 202 threads (7 warps) with ~100 registers each instead of 101 threads
// at 255, halving the dependent work per thread and doubling the warps that
// hide SMEM and FP64 latency.
//
// Per product A x (A = -S or Phi^-1) thread (i, h) reads:
//   D_i       columns 4h..4h+3          (own rows: dot(column r, x_i))
//   O_i       columns 4h..4h+3          (dots)            } which of the two
//   O_i       rows 4h..4h+3, all columns (accumulations)  } serves `up` / the
//                                                           hand-over depends on A
//   x_i (other half) and x_{i+1} from SMEM; hand-over 4 doubles each way.
// Access orders (column visit j -> 4h + ((j + h) & 3); row chunks 2h + (d ^ h))
// and the NX = 8 layout of common.cuh make every LDS.128 conflict free.
#pragma once

#include "k_pcg.cuh"

namespace docp_dev {

namespace h8 {

/// The 8 entries of column s of block b.
template <bool SMEM>
__device__ __forceinline__ void col8(const double* region, int b, int s, double* m) {
  const double* base = region + static_cast<long>(b) * 64;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double2 c = ld2<SMEM>(base + blk_off(8, b, 2 * k, s));
    m[2 * k] = c.x;
    m[2 * k + 1] = c.y;
  }
}

/// out[q] = dot(column 4h+q of block b, X) for q = 0..3 (left folds).
template <bool PAR, bool SMEM>
__device__ __forceinline__ void col_dots(const double* region, int b, int h, const double* X, double* out) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    double m[8];
    col8<SMEM>(region, b, 4 * h + j, m);
    double a = m[0] * X[0];
#pragma unroll
    for (int e = 1; e < 8; ++e) a = madd<PAR>(m[e], X[e], a);
    out[j] = a;
  }
}

/// Rows 4h..4h+3 of block b: half[c] = (B(4h,c), B(4h+1,c), B(4h+2,c), B(4h+3,c)).
template <bool SMEM>
__device__ __forceinline__ void row_half(const double* region, int b, int h, double2 (&lo)[8], double2 (&hi)[8]) {
  const double* base = region + static_cast<long>(b) * 64;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    lo[c] = ld2<SMEM>(base + blk_off(8, b, 4 * h, c));
    hi[c] = ld2<SMEM>(base + blk_off(8, b, 4 * h + 2, c));
  }
}

/// out[q] = sum_c B(4h+q, c) Y[c] for q = 0..3, c ascending (left folds).
template <bool PAR, bool SMEM>
__device__ __forceinline__ void row_accum(const double* region, int b, int h, const double* Y, double* out) {
  const double* base = region + static_cast<long>(b) * 64;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const double2 lo = ld2<SMEM>(base + blk_off(8, b, 4 * h, c));      // rows 4h, 4h+1
    const double2 hi = ld2<SMEM>(base + blk_off(8, b, 4 * h + 2, c));  // rows 4h+2, 4h+3
    if (c == 0) {
      out[0] = lo.x * Y[0];
      out[1] = lo.y * Y[0];
      out[2] = hi.x * Y[0];
      out[3] = hi.y * Y[0];
    } else {
      out[0] = madd<PAR>(lo.x, Y[c], out[0]);
      out[1] = madd<PAR>(lo.y, Y[c], out[1]);
      out[2] = madd<PAR>(hi.x, Y[c], out[2]);
      out[3] = madd<PAR>(hi.y, Y[c], out[3]);
    }
  }
}

/// Half (rows 4h..4h+3) of block j of an SMEM vector.
__device__ __forceinline__ void load_half(const double* buf, int j, int h, double* out) {
  const double2 a = *reinterpret_cast<const double2*>(buf + vec_off(8, j, 4 * h));
  const double2 b = *reinterpret_cast<const double2*>(buf + vec_off(8, j, 4 * h + 2));
  out[0] = a.x;
  out[1] = a.y;
  out[2] = b.x;
  out[3] = b.y;
}
__device__ __forceinline__ void store_half(double* buf, int j, int h, const double* in) {
  *reinterpret_cast<double2*>(buf + vec_off(8, j, 4 * h)) = make_double2(in[0], in[1]);
  *reinterpret_cast<double2*>(buf + vec_off(8, j, 4 * h + 2)) = make_double2(in[2], in[3]);
}

}  // namespace h8

template <bool PAR, bool RESIDENT, int MAXT>
__global__ void __launch_bounds__(MAXT) pcg_kernel_h8(View v, const int* __restrict__ work,
                                                    const int* __restrict__ n_work, int* __restrict__ counter,
                                                    double* __restrict__ sol_all, double epsilon, int max_iters_cfg) {
  extern __shared__ __align__(128) double sm_pcg[];
  __shared__ __align__(8) uint64_t s_bar;
  __shared__ int s_work;
  const Dims d = v.d;
  const int nl = d.nl, nb = d.nb;
  const int tid = threadIdx.x;
  const int i = tid >> 1, h = tid & 1;
  const bool act = i < nb;
  const int lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;

  double* cur = sm_pcg;
  double* sblk = nullptr;
  if constexpr (RESIDENT) {
    sblk = cur;
    cur += d.blk_stride;
  }
  double* vbuf = cur;
  cur += (nl + 1) & ~1;
  double* xbuf = cur;
  cur += (nl + 1) & ~1;
  double* red = cur;
  cur += 64;
  double* seg = cur;

  if constexpr (RESIDENT) {
    if (tid == 0) mbar_init(&s_bar, 1);
    __syncthreads();
  }
  uint32_t phase = 0;
  const int max_iters = max_iters_cfg > 0 ? max_iters_cfg : 2 * nl;
  const double threshold = epsilon * epsilon;

  // dot of the 4-row halves; PARITY folds each block's 8 products in order
  auto dot = [&](const double* a, const double* b) -> double {
    if constexpr (!PAR) {
      double s = 0.0;
      if (act)
#pragma unroll
        for (int q = 0; q < 4; ++q) s = fma(a[q], b[q], s);
      s = warp_sum(s);
      if (lane == 0) red[warp] = s;
      __syncthreads();
      double t = red[0];  // fixed-order sum of the warp partials, same in every thread
      for (int k = 1; k < nw; ++k) t = t + red[k];
      return t;
    } else {
      if (act)
#pragma unroll
        for (int q = 0; q < 4; ++q) seg[i * 8 + 4 * h + q] = a[q] * b[q];
      __syncthreads();
      if (tid < nb) {
        double s = seg[tid * 8];
#pragma unroll
        for (int e = 1; e < 8; ++e) s = s + seg[tid * 8 + e];
        seg[nl + tid] = s;  // block dot (pcg.hpp:41-42)
      }
      __syncthreads();
      double acc = 0.0;
      if (lane == 0)
        for (int k = 0; k < nb; ++k) acc = acc + seg[nl + k];
      return __shfl_sync(0xffffffffu, acc, 0);
    }
  };
  auto norm = [&](const double* a) -> double {
    __syncthreads();
    double out;
    if constexpr (!PAR) {
      double s = 0.0;
      if (act)
        for (int q = 0; q < 4; ++q) s = fma(a[q], a[q], s);
      s = warp_sum(s);
      if (lane == 0) red[warp] = s;
      __syncthreads();
      out = warp_sum(lane < nw ? red[lane] : 0.0);
    } else {
      if (act)
        for (int q = 0; q < 4; ++q) seg[i * 8 + 4 * h + q] = a[q] * a[q];
      __syncthreads();
      double acc = 0.0;
      if (lane == 0) {
        acc = seg[0];
        for (int k = 1; k < nl; ++k) acc = acc + seg[k];
      }
      out = __shfl_sync(0xffffffffu, acc, 0);
    }
    __syncthreads();
    return sqrt(out);
  };

  for (;;) {
    if (tid == 0) s_work = atomicAdd(counter, 1);
    __syncthreads();
    const int w = s_work;
    if (w >= *n_work) break;
    const int p = work[w];
    if (v.status[p].code != DOCP_OK) {
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

    double lam[4] = {0, 0, 0, 0}, r[4] = {0, 0, 0, 0}, pv[4] = {0, 0, 0, 0}, y[4] = {0, 0, 0, 0};
    if (act) {
#pragma unroll
      for (int q = 0; q < 4; ++q) lam[q] = sol[i * 8 + 4 * h + q];
    }
    if constexpr (RESIDENT) mbar_wait(&s_bar, phase);
    phase ^= 1;
    __syncthreads();

    // out = A x. Phase 1 (no barrier before it): the other half of x_i comes
    // from the partner lane (lane ^ 1) by shuffle; the thread publishes its
    // half of x_i (for block row i-1) and its hand-over (for block row i+1),
    // and forms its diagonal term. One barrier. Phase 2: x_{i+1} and the
    // hand-over from block row i-1 complete the row (diag, sub, super order).
    auto matvec = [&](bool precond, const double* xr, double* out) {
      double other[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) other[q] = __shfl_xor_sync(0xffffffffu, xr[q], 1);
      double xf[8], own[4], hand[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        xf[q] = h ? other[q] : xr[q];
        xf[4 + q] = h ? xr[q] : other[q];
      }
      const double* D = precond ? Pd : Sd;
      const double* O = precond ? Pu : Ss;
      const bool has_next = i + 1 < nb;
      if (act) {
        h8::store_half(vbuf, i, h, xr);
        h8::col_dots<PAR, RESIDENT>(D, i, h, xf, own);
        if (has_next) {
          if (!precond) h8::row_accum<PAR, RESIDENT>(O, i, h, xf, hand);  // L_i x_i
          else h8::col_dots<PAR, RESIDENT>(O, i, h, xf, hand);            // U_i' x_i
          h8::store_half(xbuf, i, h, hand);
        }
      }
      __syncthreads();
      if (act) {
        double up[4], low[4];
        if (has_next) {
          double xn[8];
          h8::load_half(vbuf, i + 1, 0, xn);
          h8::load_half(vbuf, i + 1, 1, xn + 4);
          if (!precond) h8::col_dots<PAR, RESIDENT>(O, i, h, xn, up);  // L_i' x_{i+1}
          else h8::row_accum<PAR, RESIDENT>(O, i, h, xn, up);          // U_i x_{i+1}
        }
        if (i > 0) h8::load_half(xbuf, i - 1, h, low);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          double acc = own[q];
          if (i > 0) acc = acc + low[q];
          if (has_next) acc = acc + up[q];
          out[q] = acc;
        }
      }
    };

    // FAST product: each thread reads only its row half (rows 4h..4h+3) of
    // D_i and O_i — O_i once, kept in registers across the barrier — and
    // forms the transposed product (L_i' x_{i+1}, resp. U_i' x_i) from
    // half-column partial sums exchanged with the partner lane.
    auto matvec_fast = [&](bool precond, const double* xr, double* out) {
      double other[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) other[q] = __shfl_xor_sync(0xffffffffu, xr[q], 1);
      double xf[8];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        xf[q] = h ? other[q] : xr[q];
        xf[4 + q] = h ? xr[q] : other[q];
      }
      const double* D = precond ? Pd : Sd;
      const double* O = precond ? Pu : Ss;
      const bool has_next = act && i + 1 < nb;
      const int bo = has_next ? i : 0;  // O_i exists only below the last block row
      double own[4] = {0, 0, 0, 0}, hand[4] = {0, 0, 0, 0};
      double2 olo[8] = {}, ohi[8] = {};
      if (act) {
        h8::store_half(vbuf, i, h, xr);
        double2 dlo[8], dhi[8];
        h8::row_half<RESIDENT>(D, i, h, dlo, dhi);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          own[0] = fma(dlo[c].x, xf[c], own[0]);
          own[1] = fma(dlo[c].y, xf[c], own[1]);
          own[2] = fma(dhi[c].x, xf[c], own[2]);
          own[3] = fma(dhi[c].y, xf[c], own[3]);
        }
      }
      // D's loads are consumed above; keep the compiler from hoisting O's
      // loads over them (bounds the live registers: O stays resident, D does not)
      asm volatile("" ::: "memory");
      if (has_next) h8::row_half<RESIDENT>(O, bo, h, olo, ohi);
      double part[8];  // half-column partial sums over my rows (P: with x_i)
      if (precond) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          double a = olo[c].x * xr[0];
          a = fma(olo[c].y, xr[1], a);
          a = fma(ohi[c].x, xr[2], a);
          part[c] = fma(ohi[c].y, xr[3], a);
        }
        double recv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) recv[q] = __shfl_xor_sync(0xffffffffu, h ? part[q] : part[4 + q], 1);
#pragma unroll
        for (int q = 0; q < 4; ++q) hand[q] = (h ? part[4 + q] : part[q]) + recv[q];  // U_i' x_i
      } else if (has_next) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {  // L_i x_i, my rows
          hand[0] = fma(olo[c].x, xf[c], hand[0]);
          hand[1] = fma(olo[c].y, xf[c], hand[1]);
          hand[2] = fma(ohi[c].x, xf[c], hand[2]);
          hand[3] = fma(ohi[c].y, xf[c], hand[3]);
        }
      }
      if (has_next) h8::store_half(xbuf, i, h, hand);
      __syncthreads();
      double xn[8];
      if (has_next) {
        h8::load_half(vbuf, i + 1, 0, xn);
        h8::load_half(vbuf, i + 1, 1, xn + 4);
      }
      double up[4] = {0, 0, 0, 0};
      if (!precond) {  // L_i' x_{i+1}: partial sums over my rows of x_{i+1}
        const double* xh = h ? xn + 4 : xn;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          double a = olo[c].x * xh[0];
          a = fma(olo[c].y, xh[1], a);
          a = fma(ohi[c].x, xh[2], a);
          part[c] = fma(ohi[c].y, xh[3], a);
        }
        double recv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) recv[q] = __shfl_xor_sync(0xffffffffu, h ? part[q] : part[4 + q], 1);
#pragma unroll
        for (int q = 0; q < 4; ++q) up[q] = (h ? part[4 + q] : part[q]) + recv[q];
      } else if (has_next) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {  // U_i x_{i+1}, my rows
          up[0] = fma(olo[c].x, xn[c], up[0]);
          up[1] = fma(olo[c].y, xn[c], up[1]);
          up[2] = fma(ohi[c].x, xn[c], up[2]);
          up[3] = fma(ohi[c].y, xn[c], up[3]);
        }
      }
      if (act) {
        double low[4];
        if (i > 0) h8::load_half(xbuf, i - 1, h, low);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          double acc = own[q];
          if (i > 0) acc = acc + low[q];
          if (has_next) acc = acc + up[q];
          out[q] = acc;
        }
      }
    };
    auto mv = [&](bool precond, const double* xr, double* out) {
      if constexpr (PAR) matvec(precond, xr, out);
      else matvec_fast(precond, xr, out);
    };

    mv(false, lam, y);  // y = (-S) lambda0
    if (act)
#pragma unroll
      for (int q = 0; q < 4; ++q) r[q] = gam[i * 8 + 4 * h + q] - y[q];
    __syncthreads();  // every phase-2 read of lambda / its hand-over is done
    mv(true, r, pv);  // r~
    double eta = dot(r, pv);
    int status = DOCP_OK, iters = 0;
    if (eta < 0.0) {
      const double scale = norm(r) * norm(pv);
      if (-eta <= 1e-10 * scale + 1e-300) eta = 0.0;
      else status = DOCP_AT_PCG_PRECOND;
    }

    while (status == DOCP_OK && eta > threshold && iters < max_iters) {
      mv(false, pv, y);
      const double vv = dot(pv, y);
      if (vv <= 0.0) {
        status = DOCP_AT_PCG_CURVATURE;
        break;
      }
      const double alpha = eta / vv;
      if (act) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if constexpr (PAR) {
            lam[q] = lam[q] + alpha * pv[q];
            r[q] = r[q] - alpha * y[q];
          } else {
            lam[q] = fma(alpha, pv[q], lam[q]);
            r[q] = fma(-alpha, y[q], r[q]);
          }
        }
      }
      mv(true, r, y);  // r~ (y reused)
      double eta_next = dot(r, y);
      if (eta_next < 0.0) {
        const double scale = norm(r) * norm(y);
        if (-eta_next <= 1e-10 * scale + 1e-300) {
          eta_next = 0.0;
        } else {
          status = DOCP_AT_PCG_PRECOND;
          break;
        }
      }
      const double beta = eta_next / eta;
      if (act) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if constexpr (PAR) pv[q] = y[q] + beta * pv[q];
          else pv[q] = fma(beta, pv[q], y[q]);
        }
      }
      eta = eta_next;
      ++iters;
    }

    if (act)
#pragma unroll
      for (int q = 0; q < 4; ++q) sol[i * 8 + 4 * h + q] = lam[q];
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
