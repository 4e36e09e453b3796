// k_pcg_h16f.cuh — K2 FAST mode for n_x = 16 (the paper's 16-state presets):
// four threads per block row, thread (i, q) owning rows 4q..4q+3.
//
// Same algorithm and checks as pcg_kernel_h8f (pcg.hpp:52-109), FAST
// arithmetic. Layout (common.cuh blk_off, n_x = 16): column-major 16 x 16
// blocks whose 16-byte chunks are XOR-permuted by the block's parity, so the
// chunk holding rows 4q + 2j, 4q + 2j + 1 of column c of block b sits at
//     b * 256 + 16 c + 4 q + 2 (j ^ (b & 1))
// and a quarter-warp (two block rows x four q) reads eight distinct banks.
// x_i is gathered across the quad by shuffles; transposed products are quad
// reduce-scatters of column partial sums (xor 2, then xor 1). The off-diagonal
// rows stay in registers across the product's barrier.
//
// CL > 1: the block rows are split over a thread-block cluster exactly as in
// pcg_kernel_h8f (halo rows through distributed shared memory, cluster-wide
// dots) so records larger than one SM's shared memory stay on-chip.
#pragma once

#include "k_pcg_h8f.cuh"

namespace docp_dev {

namespace h16f {

/// Quad reduce-scatter of 16 column partial sums: lane q of the quad receives
/// the sums of columns 4q..4q+3.
__device__ __forceinline__ void reduce_scatter(const double* part, int q, double* out) {
  const bool hi = (q >> 1) & 1;
  double s1[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double send = hi ? part[k] : part[8 + k];
    const double recv = __shfl_xor_sync(0xffffffffu, send, 2);
    s1[k] = (hi ? part[8 + k] : part[k]) + recv;
  }
  const bool odd = q & 1;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double send = odd ? s1[k] : s1[4 + k];
    const double recv = __shfl_xor_sync(0xffffffffu, send, 1);
    out[k] = (odd ? s1[4 + k] : s1[k]) + recv;
  }
}

/// Rows 4q..4q+3 of the 16 columns of the block at `blk` (per-thread offsets o[j]).
__device__ __forceinline__ void load_rows(const double* blk, const int (&o)[2], double2 (&d)[16][2]) {
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    d[c][0] = *reinterpret_cast<const double2*>(blk + o[0] + 16 * c);
    d[c][1] = *reinterpret_cast<const double2*>(blk + o[1] + 16 * c);
  }
}

}  // namespace h16f

/// Block rows per CTA / dynamic shared memory (doubles) of pcg_kernel_h16f<*, CL>.
__host__ __device__ inline int h16f_rows(const Dims& d, int cl) { return (d.nb + cl - 1) / cl; }
__host__ __device__ inline long h16f_smem_doubles(const Dims& d, int cl) {
  const long R = h16f_rows(d, cl);
  return 4 * R * 256 + 2 * (R + 2) * 16 + 3L * cl * 8;
}

template <int MAXT, int CL>
__global__ void __launch_bounds__(MAXT, 1) pcg_kernel_h16f(View v, const int* __restrict__ work,
                                                         const int* __restrict__ n_work, int* __restrict__ counter,
                                                         double* __restrict__ sol_all, double epsilon,
                                                         int max_iters_cfg) {
  extern __shared__ __align__(128) double sm_pcg[];
  __shared__ __align__(8) uint64_t s_bar[2];  // [0]: -S blocks, [1]: Phi^-1 blocks
  __shared__ int s_work;
  const Dims d = v.d;
  const int nl = d.nl, nb = d.nb;
  const int tid = threadIdx.x;
  const int crank = CL == 1 ? 0 : static_cast<int>(cooperative_groups::this_cluster().block_rank());
  const int R = h16f_rows(d, CL);
  const int row0 = crank * R;
  const int nrows = max(0, min(R, nb - row0));
  const int nsub = max(0, min(R, nb - 1 - row0));
  const int il = tid >> 2, q = tid & 3;
  const int i = row0 + il;
  const bool act = il < nrows;
  const bool has_next = act && i + 1 < nb;
  const bool has_prev = i > 0;
  const int lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int qbase = lane & ~3;

  double* sSd = sm_pcg;
  double* sSs = sSd + R * 256;
  double* sPd = sSs + R * 256;
  double* sPu = sPd + R * 256;
  double* vbuf = sPu + R * 256;        // [R + 2] slots of 16 (halo slots 0, R + 1)
  double* xbuf = vbuf + (R + 2) * 16;
  double* red = xbuf + (R + 2) * 16;   // [3][CL][8]

  const int m = i & 1;
  const int o[2] = {4 * q + 2 * m, 4 * q + 2 * (1 - m)};

  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
  }
  __syncthreads();
  uint32_t phase = 0;
  const int max_iters = max_iters_cfg > 0 ? max_iters_cfg : 2 * nl;
  const double threshold = epsilon * epsilon;

  auto partial = [&](const double* a, const double* b, int slot) {
    double s = fma(a[3], b[3], fma(a[2], b[2], fma(a[1], b[1], a[0] * b[0])));
    s = act ? s : 0.0;
    s = warp_sum(s);
    if (lane == 0) {
      const int at = (slot * CL + crank) * 8 + warp;
      if constexpr (CL == 1) {
        red[at] = s;
      } else {
#pragma unroll
        for (int c = 0; c < CL; ++c) cooperative_groups::this_cluster().map_shared_rank(red, c)[at] = s;
      }
    }
  };
  auto total = [&](int slot) -> double {
    double t = red[slot * CL * 8];
    for (int k = 1; k < CL * 8; ++k)
      if ((k & 7) < nw) t = t + red[slot * CL * 8 + k];
    return t;
  };
  auto dot = [&](const double* a, const double* b) -> double {
    partial(a, b, 0);
    h8f_sync<CL>();
    return total(0);
  };
  auto norm = [&](const double* a) -> double {
    h8f_sync<CL>();
    partial(a, a, 2);
    h8f_sync<CL>();
    return sqrt(total(2));
  };

  for (;;) {
    if (tid == 0 && crank == 0) {
      const int wk = atomicAdd(counter, 1);
      if constexpr (CL == 1) {
        s_work = wk;
      } else {
#pragma unroll
        for (int c = 0; c < CL; ++c) *cooperative_groups::this_cluster().map_shared_rank(&s_work, c) = wk;
      }
    }
    h8f_sync<CL>();
    const int w = s_work;
    if (w >= *n_work) break;
    const int pidx = work[w];
    if (v.status[pidx].code != DOCP_OK) {
      h8f_sync<CL>();
      continue;
    }
    const double* rec = v.blocks + static_cast<long>(pidx) * d.blk_stride;
    if (tid == 0) {
      fence_proxy_async();
      const uint32_t bd = static_cast<uint32_t>(nrows) * 2048u, bo = static_cast<uint32_t>(nsub) * 2048u;
      mbar_arrive_expect_tx(&s_bar[0], bd + bo);
      mbar_arrive_expect_tx(&s_bar[1], bd + bo);
      if (bd) tma_bulk_g2s(sSd, rec + d.s_diag + row0 * 256, bd, &s_bar[0]);
      if (bo) tma_bulk_g2s(sSs, rec + d.s_sub + row0 * 256, bo, &s_bar[0]);
      if (bd) tma_bulk_g2s(sPd, rec + d.p_diag + row0 * 256, bd, &s_bar[1]);
      if (bo) tma_bulk_g2s(sPu, rec + d.p_sup + row0 * 256, bo, &s_bar[1]);
    }
    const double* gam = v.gamma + static_cast<long>(pidx) * nl;
    double* sol = sol_all + static_cast<long>(pidx) * nl;
    const int ib = act ? il : max(0, nrows - 1);
    const int io = has_next ? il : 0;
    const double* SdI = sSd + ib * 256;
    const double* PdI = sPd + ib * 256;
    const double* SsI = sSs + io * 256;
    const double* PuI = sPu + io * 256;
    // vector slots (vec_off, n_x = 16): chunk k of slot j at j * 16 + 2 (k ^ (j & 1))
    auto voff = [](int j, int k) { return j * 16 + 2 * (k ^ (j & 1)); };
    const int sv = (act ? il : max(0, nrows - 1)) + 1;
    const int my0 = voff(sv, 2 * q), my1 = voff(sv, 2 * q + 1);
    const int nx0 = voff(sv + 1, 2 * q), nx1 = voff(sv + 1, 2 * q + 1);
    const int pv0 = voff(sv - 1, 2 * q), pv1 = voff(sv - 1, 2 * q + 1);
    const bool to_prev = CL > 1 && act && il == 0 && crank > 0;
    const bool to_next = CL > 1 && act && il == R - 1 && crank < CL - 1;
    const int hx0 = voff(R + 1, 2 * q), hx1 = voff(R + 1, 2 * q + 1);
    const int hh0 = voff(0, 2 * q), hh1 = voff(0, 2 * q + 1);

    double lam[4] = {0, 0, 0, 0}, r[4], pv[4], y[4];
    if (act) {
      const double2 a = *reinterpret_cast<const double2*>(sol + i * 16 + 4 * q);
      const double2 b = *reinterpret_cast<const double2*>(sol + i * 16 + 4 * q + 2);
      lam[0] = a.x, lam[1] = a.y, lam[2] = b.x, lam[3] = b.y;
    }
    mbar_wait(&s_bar[0], phase);

    auto put = [&](double* buf, int a0, int a1, const double* x) {
      if (act) {
        *reinterpret_cast<double2*>(buf + a0) = make_double2(x[0], x[1]);
        *reinterpret_cast<double2*>(buf + a1) = make_double2(x[2], x[3]);
      }
    };
    auto put_remote = [&](double* buf, int rank, int a0, int a1, const double* x) {
      double* rb = cooperative_groups::this_cluster().map_shared_rank(buf, rank);
      *reinterpret_cast<double2*>(rb + a0) = make_double2(x[0], x[1]);
      *reinterpret_cast<double2*>(rb + a1) = make_double2(x[2], x[3]);
    };
    auto get = [&](const double* buf, int a0, int a1, double* x) {
      const double2 a = *reinterpret_cast<const double2*>(buf + a0);
      const double2 b = *reinterpret_cast<const double2*>(buf + a1);
      x[0] = a.x, x[1] = a.y, x[2] = b.x, x[3] = b.y;
    };
    // my 4 rows of M x (xf: all 16 entries), two 8-column partial sums
    auto rows_times = [&](const double2 (&mm)[16][2], const double* xf, double* out) {
      double a[4], b[4];
      a[0] = mm[0][0].x * xf[0], a[1] = mm[0][0].y * xf[0], a[2] = mm[0][1].x * xf[0], a[3] = mm[0][1].y * xf[0];
      b[0] = mm[8][0].x * xf[8], b[1] = mm[8][0].y * xf[8], b[2] = mm[8][1].x * xf[8], b[3] = mm[8][1].y * xf[8];
#pragma unroll
      for (int c = 1; c < 8; ++c) {
        a[0] = fma(mm[c][0].x, xf[c], a[0]);
        a[1] = fma(mm[c][0].y, xf[c], a[1]);
        a[2] = fma(mm[c][1].x, xf[c], a[2]);
        a[3] = fma(mm[c][1].y, xf[c], a[3]);
        b[0] = fma(mm[8 + c][0].x, xf[8 + c], b[0]);
        b[1] = fma(mm[8 + c][0].y, xf[8 + c], b[1]);
        b[2] = fma(mm[8 + c][1].x, xf[8 + c], b[2]);
        b[3] = fma(mm[8 + c][1].y, xf[8 + c], b[3]);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) out[k] = a[k] + b[k];
    };
    // my 4 entries of M' x from my rows xm of x
    auto trans_times = [&](const double2 (&mm)[16][2], const double* xm, double* out) {
      double part[16];
#pragma unroll
      for (int c = 0; c < 16; ++c)
        part[c] = fma(mm[c][1].y, xm[3], fma(mm[c][1].x, xm[2], fma(mm[c][0].y, xm[1], mm[c][0].x * xm[0])));
      h16f::reduce_scatter(part, q, out);
    };

    auto matvec = [&](bool precond, const double* xr, double* out) {
      double xf[16];
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int e = 0; e < 4; ++e) xf[4 * k + e] = __shfl_sync(0xffffffffu, xr[e], qbase + k);
      put(vbuf, my0, my1, xr);
      if constexpr (CL > 1)
        if (to_prev) put_remote(vbuf, crank - 1, hx0, hx1, xr);
      double own[4];
      {
        double2 dd[16][2];
        h16f::load_rows(precond ? PdI : SdI, o, dd);
        rows_times(dd, xf, own);
      }
      asm volatile("" ::: "memory");  // D is consumed: bound the live registers before O
      double2 oo[16][2];
      h16f::load_rows(precond ? PuI : SsI, o, oo);
      double hand[4];
      if (precond) trans_times(oo, xr, hand);  // U_i' x_i
      else rows_times(oo, xf, hand);            // L_i x_i
      put(xbuf, my0, my1, hand);
      if constexpr (CL > 1)
        if (to_next) put_remote(xbuf, crank + 1, hh0, hh1, hand);
      h8f_sync<CL>();
      double up[4], low[4];
      if (!precond) {  // L_i' x_{i+1}
        double xn[4];
        get(vbuf, nx0, nx1, xn);
        trans_times(oo, xn, up);
      } else {  // U_i x_{i+1}
        double xn[16];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const double2 t = *reinterpret_cast<const double2*>(vbuf + voff(sv + 1, k));
          xn[2 * k] = t.x;
          xn[2 * k + 1] = t.y;
        }
        rows_times(oo, xn, up);
      }
      get(xbuf, pv0, pv1, low);
#pragma unroll
      for (int k = 0; k < 4; ++k) {  // diag, then sub (i > 0), then super (i < nb - 1)
        double acc = own[k];
        acc = has_prev ? acc + low[k] : acc;
        acc = has_next ? acc + up[k] : acc;
        out[k] = acc;
      }
    };

    matvec(false, lam, y);  // y = (-S) lambda0
    if (act) {
      const double2 a = *reinterpret_cast<const double2*>(gam + i * 16 + 4 * q);
      const double2 b = *reinterpret_cast<const double2*>(gam + i * 16 + 4 * q + 2);
      r[0] = a.x - y[0], r[1] = a.y - y[1], r[2] = b.x - y[2], r[3] = b.y - y[3];
    } else {
      r[0] = r[1] = r[2] = r[3] = 0.0;
    }
    h8f_sync<CL>();
    mbar_wait(&s_bar[1], phase);
    phase ^= 1;
    matvec(true, r, pv);  // r~
    double eta = dot(r, pv);
    int status = DOCP_OK, iters = 0;
    if (eta < 0.0) {
      const double scale = norm(r) * norm(pv);
      if (-eta <= 1e-10 * scale + 1e-300) eta = 0.0;
      else status = DOCP_AT_PCG_PRECOND;
    }

    while (status == DOCP_OK && eta > threshold && iters < max_iters) {
      matvec(false, pv, y);
      const double vv = dot(pv, y);
      if (vv <= 0.0) {
        status = DOCP_AT_PCG_CURVATURE;
        break;
      }
      const double alpha = eta / vv;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        lam[k] = fma(alpha, pv[k], lam[k]);
        r[k] = fma(-alpha, y[k], r[k]);
      }
      matvec(true, r, y);  // r~ (y reused)
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
#pragma unroll
      for (int k = 0; k < 4; ++k) pv[k] = fma(beta, pv[k], y[k]);
      eta = eta_next;
      ++iters;
    }

    if (act) {
      *reinterpret_cast<double2*>(sol + i * 16 + 4 * q) = make_double2(lam[0], lam[1]);
      *reinterpret_cast<double2*>(sol + i * 16 + 4 * q + 2) = make_double2(lam[2], lam[3]);
    }
    if (tid == 0 && crank == 0) {
      v.pcg_iters[pidx] = iters;
      v.final_eta[pidx] = eta;
      v.pcg_conv[pidx] = status == DOCP_OK && eta <= threshold;
      if (status == DOCP_OK) set_status(v.status + pidx, DOCP_OK, DOCP_AT_NONE, 0);
      else set_status(v.status + pidx, DOCP_BREAKDOWN, status, iters);
      atomicAdd(v.pcg_acc, static_cast<unsigned long long>(iters));
      atomicAdd(v.pcg_acc + 1, 1ull);
      atomicAdd(v.pcg_acc + 2, 1ull);  // lifetime solves (docp_pcg_invocations)
    }
    h8f_sync<CL>();
  }
}

}  // namespace docp_dev
