// k_pcg_h8x.cuh — K2 in the fp32 mode (DOCP_PCG_FP32) for n_x = 8: the FAST
// algorithm of pcg_kernel_h8s (pipelined second dot, Chronopoulos-Gear
// recurrence for (-S) p) on fp32 blocks and fp32 iterates, with the dots
// accumulated in fp64 (the products of two floats are exact in fp64) and the
// scalars alpha, beta, eta in fp64.
//
// Residency: the fp64 record assembled by K1 is read ONCE per solve straight
// from global memory and rounded to fp32 on the way in (no fp32 copy in HBM,
// no TMA staging area):
//   registers  thread (i, h): its shares of the symmetric -S_ii and
//              Phi^-1_ii (18 + 18 floats, as h8s::Sym) and rows 4h..4h+3 of
//              L_i (32 floats);
//   shared     rows 4h..4h+3 of U_i (the Phi^-1 super block), 32 KB per CTA in
//              a thread-major layout (column c of thread t at c * NT + t:
//              every quarter-warp float4 access is conflict free), the
//              vector exchange buffers and the dot partials.
// About 45 KB of shared memory and <= 128 registers per thread, so two
// problems run on every SM: one CTA's record load and dot reductions
// overlap the other's products.
//
// Exit test. eta <= eps^2 with the reference's absolute eps = 1e-12 is below
// fp32 resolution, so in this mode epsilon is RELATIVE: the solve stops at
// eta <= eps^2 * eta_gamma, eta_gamma = gamma' Phi^-1 gamma (the cold-start
// eta; one extra Phi^-1 product per solve). The eta clamp and both breakdown
// checks are the reference's (pcg.hpp:72-93).
#pragma once

#include "k_pcg_h8s.cuh"

namespace docp_dev {

namespace h8x {

struct Sym32 {
  float o[10];     // D_hh upper triangle (h8s::tri)
  float s[4][2];   // D01 rows 0..3, columns 4 + 2h, 5 + 2h
};

__device__ __forceinline__ void load_sym(const double* __restrict__ blk, int b, int h, Sym32& m) {
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = a; c < 4; ++c) m.o[h8s::tri(a, c)] = static_cast<float>(__ldg(blk + blk_off(8, b, 4 * h + a, 4 * h + c)));
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int k = 0; k < 2; ++k) m.s[a][k] = static_cast<float>(__ldg(blk + blk_off(8, b, a, 4 + 2 * h + k)));
}

/// Rows 4h..4h+3 of every column of fp64 block b, rounded to fp32.
__device__ __forceinline__ void load_rows(const double* __restrict__ blk, int b, int h, float4 (&m)[8]) {
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const double2 lo = __ldg(reinterpret_cast<const double2*>(blk + blk_off(8, b, 4 * h, c)));
    const double2 hi = __ldg(reinterpret_cast<const double2*>(blk + blk_off(8, b, 4 * h + 2, c)));
    m[c] = make_float4(static_cast<float>(lo.x), static_cast<float>(lo.y), static_cast<float>(hi.x),
                       static_cast<float>(hi.y));
  }
}

__device__ __forceinline__ float comp(const float4& v, int q) { return q == 0 ? v.x : q == 1 ? v.y : q == 2 ? v.z : v.w; }

/// My 4 rows of D x (as h8s::sym_times, fp32).
__device__ __forceinline__ void sym_times(const Sym32& m, const float* xf, const float* xr, int h, float* out) {
  auto O = [&](int a, int b) { return a <= b ? m.o[h8s::tri(a, b)] : m.o[h8s::tri(b, a)]; };
  float own[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float a = fmaf(O(q, 1), xr[1], O(q, 0) * xr[0]);
    const float b = fmaf(O(q, 3), xr[3], O(q, 2) * xr[2]);
    own[q] = a + b;
  }
  const float xc0 = h ? xf[6] : xf[4], xc1 = h ? xf[7] : xf[5];
  float A[4], Bt[2];
#pragma unroll
  for (int q = 0; q < 4; ++q) A[q] = fmaf(m.s[q][1], xc1, m.s[q][0] * xc0);
#pragma unroll
  for (int k = 0; k < 2; ++k)
    Bt[k] = fmaf(m.s[3][k], xf[3], fmaf(m.s[2][k], xf[2], fmaf(m.s[1][k], xf[1], m.s[0][k] * xf[0])));
  float recv[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float send = h ? A[q] : (q < 2 ? Bt[q] : 0.0f);
    recv[q] = __shfl_xor_sync(0xffffffffu, send, 1);
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float mine = q < 2 ? recv[q] : Bt[q - 2];
    out[q] = h ? own[q] + mine : (own[q] + A[q]) + recv[q];
  }
}

/// My rows of M x (M given by my rows of every column).
__device__ __forceinline__ void rows_times(const float4 (&m)[8], const float* xf, float* out) {
  float a[4], b[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) a[q] = comp(m[0], q) * xf[0], b[q] = comp(m[4], q) * xf[4];
#pragma unroll
  for (int c = 1; c < 4; ++c)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      a[q] = fmaf(comp(m[c], q), xf[c], a[q]);
      b[q] = fmaf(comp(m[4 + c], q), xf[4 + c], b[q]);
    }
#pragma unroll
  for (int q = 0; q < 4; ++q) out[q] = a[q] + b[q];
}

/// My 4 entries of M' x given my rows xm of x (partner completes the sums).
__device__ __forceinline__ void trans_times(const float4 (&m)[8], const float* xm, int h, float* out) {
  float part[8];
#pragma unroll
  for (int c = 0; c < 8; ++c)
    part[c] = fmaf(m[c].w, xm[3], fmaf(m[c].z, xm[2], fmaf(m[c].y, xm[1], m[c].x * xm[0])));
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float send = h ? part[q] : part[4 + q];
    const float recv = __shfl_xor_sync(0xffffffffu, send, 1);
    out[q] = (h ? part[4 + q] : part[q]) + recv;
  }
}

}  // namespace h8x

/// Dynamic shared memory of pcg_kernel_h8x (bytes) for `threads` threads.
__host__ __device__ inline long h8x_smem_bytes(const Dims& d, int threads) {
  return 8L * threads * 16 + 2L * (d.nb + 2) * 8 * 4 + 3L * 16 * 8;
}

template <int MAXT>
__global__ void __launch_bounds__(MAXT, MAXT <= 256 ? 2 : 1) pcg_kernel_h8x(View v, const int* __restrict__ work,
                                                        const int* __restrict__ n_work, int* __restrict__ counter,
                                                        double* __restrict__ sol_all, double epsilon,
                                                        int max_iters_cfg) {
  extern __shared__ __align__(128) unsigned char sm_raw[];
  __shared__ int s_work;
  const Dims d = v.d;
  const int nl = d.nl, nb = d.nb;
  const int tid = threadIdx.x, NT = blockDim.x;
  const int il = tid >> 1, h = tid & 1;
  const int i = il;
  const bool act = i < nb;
  const bool has_next = act && i + 1 < nb;
  const bool has_prev = i > 0;
  const int lane = tid & 31, warp = tid >> 5;
  constexpr int NWS = MAXT / 32;  // warp slots per dot (absent warps' slots stay 0)

  float4* usm = reinterpret_cast<float4*>(sm_raw);                      // [8][NT] my rows of U_i
  float* vbuf = reinterpret_cast<float*>(sm_raw + 8L * NT * 16);        // [nb + 2][8] x_i (slot = row + 1)
  float* xbuf = vbuf + (nb + 2) * 8;                                    // [nb + 2][8] hand-overs
  double* red = reinterpret_cast<double*>(xbuf + (nb + 2) * 8);        // [3][NWS] dot partials

  const int ib = act ? il : nb - 1;
  const int io = has_next ? il : 0;
  const int sv = ib + 1;
  const int my = sv * 8 + 4 * h, nx_ = (sv + 1) * 8 + 4 * h, pv_ = (sv - 1) * 8 + 4 * h;
  const int pp = max(sv - 2, 0) * 8 + 4 * h;  // (-S) hand-over slot, one below (see h8s)
  const int nf = (sv + 1) * 8;

  if (tid < 3 * NWS) red[tid] = 0.0;
  const int max_iters = max_iters_cfg > 0 ? max_iters_cfg : 2 * nl;
  const double eps2 = epsilon * epsilon;

  auto partial = [&](const float* a, const float* b, int slot) {
    double s = static_cast<double>(a[0]) * b[0];
#pragma unroll
    for (int q = 1; q < 4; ++q) s = fma(static_cast<double>(a[q]), static_cast<double>(b[q]), s);
    s = act ? s : 0.0;
    s = warp_sum(s);
    if (lane == 0) red[slot * NWS + warp] = s;
  };
  auto total = [&](int slot) -> double {
    const double2* q = reinterpret_cast<const double2*>(red + slot * NWS);
    const double2 a = q[0], b = q[1], c = q[2], e = q[3];
    const double t8 = ((a.x + a.y) + (b.x + b.y)) + ((c.x + c.y) + (e.x + e.y));
    if constexpr (NWS == 8) {
      return t8;
    } else {
      const double2 f = q[4], g = q[5], k = q[6], m = q[7];
      return t8 + (((f.x + f.y) + (g.x + g.y)) + ((k.x + k.y) + (m.x + m.y)));
    }
  };
  auto dot = [&](const float* a, const float* b) -> double {
    partial(a, b, 0);
    __syncthreads();
    return total(0);
  };
  auto norm = [&](const float* a) -> double {
    __syncthreads();
    partial(a, a, 2);
    __syncthreads();
    return sqrt(total(2));
  };
  auto gather = [&](const float* xr, float* xf) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float o = __shfl_xor_sync(0xffffffffu, xr[q], 1);
      xf[q] = h ? o : xr[q];
      xf[4 + q] = h ? xr[q] : o;
    }
  };
  auto put = [&](float* buf, int o, const float* x) {
    if (act) *reinterpret_cast<float4*>(buf + o) = make_float4(x[0], x[1], x[2], x[3]);
  };
  auto get = [&](const float* buf, int o, float* x) {
    const float4 a = *reinterpret_cast<const float4*>(buf + o);
    x[0] = a.x, x[1] = a.y, x[2] = a.z, x[3] = a.w;
  };
  auto finish = [&](const float* own, const float* low, const float* up, float* out) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float acc = own[q];
      acc = has_prev ? acc + low[q] : acc;
      acc = has_next ? acc + up[q] : acc;
      out[q] = acc;
    }
  };

  h8x::Sym32 sd, pd;
  float4 so[8];  // my rows of L_i

  for (;;) {
    if (tid == 0) s_work = atomicAdd(counter, 1);
    __syncthreads();  // also: the previous problem's reads of usm / vbuf / xbuf are done
    const int w = s_work;
    if (w >= *n_work) break;
    const int pidx = work[w];
    if (v.status[pidx].code != DOCP_OK) {  // failed in an earlier stage (block-uniform)
      __syncthreads();  // every thread has read s_work
      continue;
    }
    const double* rec = v.blocks + static_cast<long>(pidx) * d.blk_stride;
    const double* gam = v.gamma + static_cast<long>(pidx) * nl;
    double* sol = sol_all + static_cast<long>(pidx) * nl;
    float lam[4] = {0, 0, 0, 0}, g[4] = {0, 0, 0, 0};
    if (act) {
      const double2 l0 = *reinterpret_cast<const double2*>(sol + i * 8 + 4 * h);
      const double2 l1 = *reinterpret_cast<const double2*>(sol + i * 8 + 4 * h + 2);
      const double2 g0 = __ldg(reinterpret_cast<const double2*>(gam + i * 8 + 4 * h));
      const double2 g1 = __ldg(reinterpret_cast<const double2*>(gam + i * 8 + 4 * h + 2));
      lam[0] = static_cast<float>(l0.x), lam[1] = static_cast<float>(l0.y);
      lam[2] = static_cast<float>(l1.x), lam[3] = static_cast<float>(l1.y);
      g[0] = static_cast<float>(g0.x), g[1] = static_cast<float>(g0.y);
      g[2] = static_cast<float>(g1.x), g[3] = static_cast<float>(g1.y);
    }
    // the record, once: fp64 -> fp32
    h8x::load_sym(rec + d.s_diag + static_cast<long>(ib) * 64, ib, h, sd);
    h8x::load_sym(rec + d.p_diag + static_cast<long>(ib) * 64, ib, h, pd);
    h8x::load_rows(rec + d.s_sub + static_cast<long>(io) * 64, io, h, so);
    {
      float4 uu[8];
      h8x::load_rows(rec + d.p_sup + static_cast<long>(io) * 64, io, h, uu);
#pragma unroll
      for (int c = 0; c < 8; ++c) usm[c * NT + tid] = uu[c];
    }
    __syncthreads();

    auto matvec_s_dot = [&](const float* xr, float* out, const float* a, const float* b, int slot) {
      float xf[8], own[4], hand[4], low[4], up[4], xn[4];
      gather(xr, xf);
      put(vbuf, my, xr);
      h8x::sym_times(sd, xf, xr, h, own);
      h8x::rows_times(so, xf, hand);  // L_i x_i
      put(xbuf, pv_, hand);           // slot i (h8s: never a slot the Phi^-1 product still reads)
      partial(a, b, slot);
      __syncthreads();
      get(vbuf, nx_, xn);
      h8x::trans_times(so, xn, h, up);  // L_i' x_{i+1}
      get(xbuf, pp, low);
      finish(own, low, up, out);
    };
    auto matvec_p = [&](const float* xr, float* out) {
      float xf[8], own[4], hand[4], low[4], up[4], xn[8];
      gather(xr, xf);
      put(vbuf, my, xr);
      h8x::sym_times(pd, xf, xr, h, own);
      __syncthreads();
      get(vbuf, nf, xn);
      get(vbuf, nf + 4, xn + 4);
      {
        float4 uu[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) uu[c] = usm[c * NT + tid];
        h8x::trans_times(uu, xr, h, hand);  // U_i' x_i
        h8x::rows_times(uu, xn, up);       // U_i x_{i+1}
      }
      put(xbuf, my, hand);
      __syncthreads();
      get(xbuf, pv_, low);
      finish(own, low, up, out);
    };

    float r[4] = {0, 0, 0, 0}, pv[4], y[4], rt[4], sr[4];
    // eta_gamma = gamma' Phi^-1 gamma: the scale of the relative exit test
    matvec_p(g, rt);
    const double eta_g = dot(g, rt);
    const double threshold = eps2 * eta_g;
    matvec_s_dot(lam, y, r, r, 2);  // y = (-S) lambda0 (slot 2: unread)
#pragma unroll
    for (int q = 0; q < 4; ++q) r[q] = act ? g[q] - y[q] : 0.0f;
    __syncthreads();  // every phase-2 read of lambda / its hand-over is done
    matvec_p(r, rt);
    matvec_s_dot(rt, sr, r, rt, 1);
    double eta = total(1);
    int status = DOCP_OK, iters = 0;
    if (eta < 0.0) {
      const double scale = norm(r) * norm(rt);
      if (-eta <= 1e-10 * scale + 1e-300) eta = 0.0;
      else status = DOCP_AT_PCG_PRECOND;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) pv[q] = rt[q], y[q] = sr[q];

    while (status == DOCP_OK && eta > threshold && iters < max_iters) {
      const double vv = dot(pv, y);
      if (vv <= 0.0) {
        status = DOCP_AT_PCG_CURVATURE;
        break;
      }
      const float alpha = static_cast<float>(eta / vv);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        lam[q] = fmaf(alpha, pv[q], lam[q]);
        r[q] = fmaf(-alpha, y[q], r[q]);
      }
      matvec_p(r, rt);
      matvec_s_dot(rt, sr, r, rt, 1);
      double eta_next = total(1);
      if (eta_next < 0.0) {
        const double scale = norm(r) * norm(rt);
        if (-eta_next <= 1e-10 * scale + 1e-300) {
          eta_next = 0.0;
        } else {
          status = DOCP_AT_PCG_PRECOND;
          break;
        }
      }
      const float beta = static_cast<float>(eta_next / eta);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        pv[q] = fmaf(beta, pv[q], rt[q]);
        y[q] = fmaf(beta, y[q], sr[q]);
      }
      eta = eta_next;
      ++iters;
    }

    if (act) {
      *reinterpret_cast<double2*>(sol + i * 8 + 4 * h) = make_double2(lam[0], lam[1]);
      *reinterpret_cast<double2*>(sol + i * 8 + 4 * h + 2) = make_double2(lam[2], lam[3]);
    }
    if (tid == 0) {
      v.pcg_iters[pidx] = iters;
      v.final_eta[pidx] = eta;
      v.pcg_conv[pidx] = status == DOCP_OK && eta <= threshold;
      if (status == DOCP_OK) set_status(v.status + pidx, DOCP_OK, DOCP_AT_NONE, 0);
      else set_status(v.status + pidx, DOCP_BREAKDOWN, status, iters);
      atomicAdd(v.pcg_acc, static_cast<unsigned long long>(iters));
      atomicAdd(v.pcg_acc + 1, 1ull);
      atomicAdd(v.pcg_acc + 2, 1ull);
    }
  }
}

}  // namespace docp_dev
