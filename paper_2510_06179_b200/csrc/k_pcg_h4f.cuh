// k_pcg_h4f.cuh — K2 FAST mode for n_x = 4 (the cart-pole / double-integrator
// shapes): one thread per block row, owning all four rows, so x_i never
// crosses lanes and every transposed product is complete in the thread.
//
// Same algorithm and checks as pcg_kernel (pcg.hpp:52-109), FAST arithmetic,
// with the instruction diet of pcg_kernel_h8f: the n_x = 4 block layout
// (common.cuh blk_off: column s' = s ^ (b & 3), chunk' = chunk ^ ((b >> 2) & 1))
// puts the chunk holding rows 2j, 2j+1 of logical column s of block b at
//     b * 16 + 4 (s ^ p) + 2 (j ^ m),   p = b & 3, m = (b >> 2) & 1,
// so eight per-thread offsets replace the swizzle arithmetic (and a
// quarter-warp's eight consecutive block rows read eight distinct banks);
// block rows are padded to the thread count and masked with selects; the
// off-diagonal block stays in registers across the product's barrier.
#pragma once

#include "k_pcg.cuh"

namespace docp_dev {

/// Dynamic shared memory of pcg_kernel_h4f (doubles): the four regions
/// (n_b blocks each), vbuf / xbuf with halo slots, dot partials.
__host__ __device__ inline long h4f_smem_doubles(const Dims& d) { return 4L * d.nb * 16 + 2L * (d.nb + 2) * 4 + 24; }

template <int MAXT>
__global__ void __launch_bounds__(MAXT, 2) pcg_kernel_h4f(View v, const int* __restrict__ work,
                                                        const int* __restrict__ n_work, int* __restrict__ counter,
                                                        double* __restrict__ sol_all, double epsilon,
                                                        int max_iters_cfg) {
  extern __shared__ __align__(128) double sm_pcg[];
  __shared__ __align__(8) uint64_t s_bar[2];  // [0]: -S blocks, [1]: Phi^-1 blocks
  __shared__ int s_work;
  const Dims d = v.d;
  const int nl = d.nl, nb = d.nb;
  const int tid = threadIdx.x;
  const int i = tid;
  const bool act = i < nb;
  const bool has_next = act && i + 1 < nb;
  const bool has_prev = i > 0;
  const int lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;

  double* sSd = sm_pcg;
  double* sSs = sSd + nb * 16;
  double* sPd = sSs + nb * 16;
  double* sPu = sPd + nb * 16;
  double* vbuf = sPu + nb * 16;       // [nb + 2] slots of 4 (slot = row + 1)
  double* xbuf = vbuf + (nb + 2) * 4;
  double* red = xbuf + (nb + 2) * 4;  // [3][8]

  const int ib = act ? i : nb - 1;    // rows past the last one reuse its block (masked)
  const int p = ib & 3, m = (ib >> 2) & 1;
  int o[4][2];
#pragma unroll
  for (int s = 0; s < 4; ++s)
#pragma unroll
    for (int j = 0; j < 2; ++j) o[s][j] = 4 * (s ^ p) + 2 * (j ^ m);
  // vector slots (vec_off, n_x = 4): chunk k of slot j at 4 j + 2 (k ^ ((j >> 2) & 1))
  auto voff = [](int j, int k) { return 4 * j + 2 * (k ^ ((j >> 2) & 1)); };
  const int sv = ib + 1;
  const int my0 = voff(sv, 0), my1 = voff(sv, 1), nx0 = voff(sv + 1, 0), nx1 = voff(sv + 1, 1);
  const int pv0 = voff(sv - 1, 0), pv1 = voff(sv - 1, 1);

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
    if (lane == 0) red[slot * 8 + warp] = s;
  };
  auto total = [&](int slot) -> double {
    double t = red[slot * 8];
    for (int k = 1; k < nw; ++k) t = t + red[slot * 8 + k];
    return t;
  };
  auto dot = [&](const double* a, const double* b) -> double {
    partial(a, b, 0);
    __syncthreads();
    return total(0);
  };
  auto norm = [&](const double* a) -> double {
    __syncthreads();
    partial(a, a, 2);
    __syncthreads();
    return sqrt(total(2));
  };
  auto load = [&](const double* blk, double2 (&mm)[4][2]) {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      mm[s][0] = *reinterpret_cast<const double2*>(blk + o[s][0]);
      mm[s][1] = *reinterpret_cast<const double2*>(blk + o[s][1]);
    }
  };
  auto rows_times = [&](const double2 (&mm)[4][2], const double* x, double* out) {  // M x
    out[0] = fma(mm[3][0].x, x[3], fma(mm[2][0].x, x[2], fma(mm[1][0].x, x[1], mm[0][0].x * x[0])));
    out[1] = fma(mm[3][0].y, x[3], fma(mm[2][0].y, x[2], fma(mm[1][0].y, x[1], mm[0][0].y * x[0])));
    out[2] = fma(mm[3][1].x, x[3], fma(mm[2][1].x, x[2], fma(mm[1][1].x, x[1], mm[0][1].x * x[0])));
    out[3] = fma(mm[3][1].y, x[3], fma(mm[2][1].y, x[2], fma(mm[1][1].y, x[1], mm[0][1].y * x[0])));
  };
  auto trans_times = [&](const double2 (&mm)[4][2], const double* x, double* out) {  // M' x
#pragma unroll
    for (int s = 0; s < 4; ++s)
      out[s] = fma(mm[s][1].y, x[3], fma(mm[s][1].x, x[2], fma(mm[s][0].y, x[1], mm[s][0].x * x[0])));
  };
  auto put = [&](double* buf, const double* x) {
    if (act) {
      *reinterpret_cast<double2*>(buf + my0) = make_double2(x[0], x[1]);
      *reinterpret_cast<double2*>(buf + my1) = make_double2(x[2], x[3]);
    }
  };
  auto get = [&](const double* buf, int a0, int a1, double* x) {
    const double2 a = *reinterpret_cast<const double2*>(buf + a0);
    const double2 b = *reinterpret_cast<const double2*>(buf + a1);
    x[0] = a.x, x[1] = a.y, x[2] = b.x, x[3] = b.y;
  };

  for (;;) {
    if (tid == 0) s_work = atomicAdd(counter, 1);
    __syncthreads();
    const int w = s_work;
    if (w >= *n_work) break;
    const int pidx = work[w];
    if (v.status[pidx].code != DOCP_OK) {
      __syncthreads();
      continue;
    }
    const double* rec = v.blocks + static_cast<long>(pidx) * d.blk_stride;
    if (tid == 0) {
      fence_proxy_async();
      const uint32_t bd = static_cast<uint32_t>(nb) * 128u, bo = static_cast<uint32_t>(nb - 1) * 128u;
      mbar_arrive_expect_tx(&s_bar[0], bd + bo);
      mbar_arrive_expect_tx(&s_bar[1], bd + bo);
      tma_bulk_g2s(sSd, rec + d.s_diag, bd, &s_bar[0]);
      if (bo) tma_bulk_g2s(sSs, rec + d.s_sub, bo, &s_bar[0]);
      tma_bulk_g2s(sPd, rec + d.p_diag, bd, &s_bar[1]);
      if (bo) tma_bulk_g2s(sPu, rec + d.p_sup, bo, &s_bar[1]);
    }
    const double* gam = v.gamma + static_cast<long>(pidx) * nl;
    double* sol = sol_all + static_cast<long>(pidx) * nl;
    const int io = has_next ? i : 0;
    const double* SdI = sSd + ib * 16;
    const double* PdI = sPd + ib * 16;
    const double* SsI = sSs + io * 16;
    const double* PuI = sPu + io * 16;

    double lam[4] = {0, 0, 0, 0}, r[4], pv[4], y[4];
    if (act) {
      const double2 a = *reinterpret_cast<const double2*>(sol + i * 4);
      const double2 b = *reinterpret_cast<const double2*>(sol + i * 4 + 2);
      lam[0] = a.x, lam[1] = a.y, lam[2] = b.x, lam[3] = b.y;
    }
    mbar_wait(&s_bar[0], phase);

    // out = A x, A = -S (D = S_ii, O = L_i) or Phi^-1 (D = P_ii, O = U_i)
    auto matvec = [&](bool precond, const double* x, double* out) {
      put(vbuf, x);
      double own[4];
      {
        double2 dd[4][2];
        load(precond ? PdI : SdI, dd);
        rows_times(dd, x, own);
      }
      double2 oo[4][2];
      load(precond ? PuI : SsI, oo);
      double hand[4];
      if (precond) trans_times(oo, x, hand);  // U_i' x_i
      else rows_times(oo, x, hand);            // L_i x_i
      put(xbuf, hand);
      __syncthreads();
      double xn[4], up[4], low[4];
      get(vbuf, nx0, nx1, xn);
      if (precond) rows_times(oo, xn, up);  // U_i x_{i+1}
      else trans_times(oo, xn, up);         // L_i' x_{i+1}
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
      const double2 a = *reinterpret_cast<const double2*>(gam + i * 4);
      const double2 b = *reinterpret_cast<const double2*>(gam + i * 4 + 2);
      r[0] = a.x - y[0], r[1] = a.y - y[1], r[2] = b.x - y[2], r[3] = b.y - y[3];
    } else {
      r[0] = r[1] = r[2] = r[3] = 0.0;
    }
    __syncthreads();  // every phase-2 read of lambda / its hand-over is done
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
      *reinterpret_cast<double2*>(sol + i * 4) = make_double2(lam[0], lam[1]);
      *reinterpret_cast<double2*>(sol + i * 4 + 2) = make_double2(lam[2], lam[3]);
    }
    if (tid == 0) {
      v.pcg_iters[pidx] = iters;
      v.final_eta[pidx] = eta;
      v.pcg_conv[pidx] = status == DOCP_OK && eta <= threshold;
      if (status == DOCP_OK) set_status(v.status + pidx, DOCP_OK, DOCP_AT_NONE, 0);
      else set_status(v.status + pidx, DOCP_BREAKDOWN, status, iters);
      atomicAdd(v.pcg_acc, static_cast<unsigned long long>(iters));
      atomicAdd(v.pcg_acc + 1, 1ull);
      atomicAdd(v.pcg_acc + 2, 1ull);  // lifetime solves (docp_pcg_invocations)
    }
    __syncthreads();
  }
}

}  // namespace docp_dev
