// k_pcg_h8f.cuh — K2 FAST mode for n_x = 8 with resident blocks: the
// instruction-lean form of pcg_kernel_h8 (same algorithm, pcg.hpp:52-109,
// same exit test / eta clamp / breakdown checks; FAST arithmetic).
//
// What changes against pcg_kernel_h8<FAST>:
//  * block addressing is hoisted: for thread (i, h) the chunk holding rows
//    4h + 2j, 4h + 2j + 1 of logical column c of a block lies at
//        block + 8c + r(c) + 2 (j ^ m),   r(c) = +-8p + 4(h or 1-h)
//    (p = i & 1, m = (i >> 1) & 1; common.cuh blk_off), so eight per-thread
//    offsets and compile-time immediates replace the per-load swizzle math
//    (the j ^ m term is what keeps a quarter-warp's four blocks on distinct
//    banks, so it stays in the per-thread offsets);
//  * no branches on the row: the CTA's block rows are padded to the thread
//    count (vector buffers sized to match), rows past the last one compute
//    on whatever their addresses hold and are masked out of every result
//    (selects, not multiplies, so garbage NaNs cannot leak);
//  * every 8-term accumulation runs as two 4-term partial sums (ILP).
// Vector rows keep the conflict-free vec_off layout, with per-thread offsets.
//
// CL > 1 (long horizons, T > 113): a thread-block cluster of CL CTAs solves
// one problem; CTA c holds block rows [cR, cR + R) of every region in its own
// shared memory (four TMA bulk copies), so the blocks stay on-chip however
// long the horizon. Neighbour rows across a CTA boundary exchange x and the
// hand-over through distributed shared memory (halo rows of vbuf / xbuf),
// dot products gather every warp's partial in every CTA, and the barriers
// become cluster barriers. CL = 1 is the single-CTA kernel.
#pragma once

#include <cooperative_groups.h>

#include "k_pcg.cuh"

namespace docp_dev {

namespace h8f {

__device__ __forceinline__ double sel(bool c, double a, double b) { return c ? a : b; }

/// Per-thread chunk offsets (in doubles, relative to a block): [k][j] for
/// the column class k = (c >= 4) * 2 + (c & 1) and row pair j.
struct Bases {
  int o[4][2];
};

/// Rows 4h..4h+3 of all 8 columns of the block at `blk`: d[c][j] = rows
/// 4h + 2j, 4h + 2j + 1 of column c.
__device__ __forceinline__ void load_rows(const double* blk, const Bases& bs, double2 (&d)[8][2]) {
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int k = (c >= 4) * 2 + (c & 1);
    d[c][0] = *reinterpret_cast<const double2*>(blk + bs.o[k][0] + 8 * c);
    d[c][1] = *reinterpret_cast<const double2*>(blk + bs.o[k][1] + 8 * c);
  }
}

}  // namespace h8f

/// Block rows per CTA for a cluster of cl CTAs.
__host__ __device__ inline int h8f_rows(const Dims& d, int cl) { return (d.nb + cl - 1) / cl; }

/// Dynamic shared memory of pcg_kernel_h8f<*, CL> (doubles): four regions of
/// R blocks, vbuf / xbuf with two halo rows (a second pair for CL > 1, whose
/// (-S) product follows the Phi^-1 product with no barrier between), and
/// 3 x CL x 8 dot partials. Where the second pair does not fit (dbuf =
/// false: the longest horizons of a cluster size) the kernel puts a cluster
/// barrier between the two products instead; it tells from its dynamic shared
/// memory size which layout it was launched with.
__host__ __device__ inline long h8f_smem_doubles(const Dims& d, int cl, bool dbuf = true) {
  const long R = h8f_rows(d, cl);
  return 4 * R * 64 + (cl > 1 && dbuf ? 4 : 2) * (R + 2) * 8 + 3L * cl * 8;
}

template <int CL>
__device__ __forceinline__ void h8f_sync() {
  if constexpr (CL == 1) __syncthreads();
  else cooperative_groups::this_cluster().sync();
}

template <int MAXT, int CL>
__global__ void __launch_bounds__(MAXT, 1) pcg_kernel_h8f(View v, const int* __restrict__ work,
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
  const int R = h8f_rows(d, CL);               // block rows per CTA
  const int row0 = crank * R;                  // first global block row of this CTA
  const int nrows = max(0, min(R, nb - row0));  // block rows this CTA owns
  const int nsub = max(0, min(R, nb - 1 - row0));  // ... that have an off-diagonal block
  const int il = tid >> 1, h = tid & 1;
  const int i = row0 + il;                     // global block row
  const bool act = il < nrows;
  const bool has_next = act && i + 1 < nb;
  const bool has_prev = i > 0;
  const int lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;

  double* sSd = sm_pcg;            // [R] blocks
  double* sSs = sSd + R * 64;      // [R]
  double* sPd = sSs + R * 64;      // [R]
  double* sPu = sPd + R * 64;      // [R]
  double* vbuf = sPu + R * 64;     // [R + 2] x_i halves; slot = local row + 1, slots 0 / R+1 are halos
  double* xbuf = vbuf + (R + 2) * 8;  // [R + 2] hand-overs
  // second pair for matvec_s_dot (CL > 1): it runs right after the Phi^-1
  // product, whose phase-2 reads of the neighbours' slots (and of the halos
  // the neighbour CTAs wrote) must not race with this product's phase-1 writes
  uint32_t dyn_bytes;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn_bytes));
  const bool dbuf = CL > 1 && dyn_bytes >= h8f_smem_doubles(d, CL, true) * 8;
  double* vbuf2 = dbuf ? xbuf + (R + 2) * 8 : vbuf;
  double* xbuf2 = dbuf ? vbuf2 + (R + 2) * 8 : xbuf;
  double* red = dbuf ? xbuf2 + (R + 2) * 8 : xbuf + (R + 2) * 8;  // [3][CL][8] dot partials

  const int p = i & 1, m = (i >> 1) & 1;
  h8f::Bases bs;
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int j = 0; j < 2; ++j)
      bs.o[k][j] = ((k & 1) ? -8 * p : 8 * p) + 4 * ((k >> 1) ? 1 - h : h) + 2 * (j ^ m);

  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
  }
  __syncthreads();
  uint32_t phase = 0;
  const int max_iters = max_iters_cfg > 0 ? max_iters_cfg : 2 * nl;
  const double threshold = epsilon * epsilon;

  // block-wide (cluster-wide) dots: warp tree, every warp's partial stored in
  // every CTA of the cluster, one barrier, then the same fixed-order sum in
  // every thread. `slot` selects one of three partial areas so that dots
  // without a barrier between them never overwrite partials still being read.
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
    if (tid == 0) {  // this CTA's rows of the four regions
      fence_proxy_async();
      const uint32_t bd = static_cast<uint32_t>(nrows) * 512u, bo = static_cast<uint32_t>(nsub) * 512u;
      // -S first on its own barrier: the first product only needs those blocks,
      // so it starts while the Phi^-1 half is still in flight
      mbar_arrive_expect_tx(&s_bar[0], bd + bo);
      mbar_arrive_expect_tx(&s_bar[1], bd + bo);
      if (bd) tma_bulk_g2s(sSd, rec + d.s_diag + row0 * 64, bd, &s_bar[0]);
      if (bo) tma_bulk_g2s(sSs, rec + d.s_sub + row0 * 64, bo, &s_bar[0]);
      if (bd) tma_bulk_g2s(sPd, rec + d.p_diag + row0 * 64, bd, &s_bar[1]);
      if (bo) tma_bulk_g2s(sPu, rec + d.p_sup + row0 * 64, bo, &s_bar[1]);
    }
    const double* gam = v.gamma + static_cast<long>(pidx) * nl;
    double* sol = sol_all + static_cast<long>(pidx) * nl;
    // this thread's blocks (rows past the last one reuse a valid block; masked below)
    const int ib = act ? il : max(0, nrows - 1);
    const int io = has_next ? il : 0;
    const double* SdI = sSd + ib * 64;
    const double* PdI = sPd + ib * 64;
    const double* SsI = sSs + io * 64;
    const double* PuI = sPu + io * 64;
    // vector slots in the vec_off layout (common.cuh): chunk k of slot j sits at
    // j * 8 + 2 (k ^ ((j >> 1) & 3)); per-thread offsets of the chunks used
    // (rows past the last one use its offsets; they never store)
    auto voff = [](int j, int k) { return j * 8 + 2 * (k ^ ((j >> 1) & 3)); };
    const int sv = (act ? il : max(0, nrows - 1)) + 1;  // my slot
    const int my0 = voff(sv, 2 * h), my1 = voff(sv, 2 * h + 1);            // my half of row i
    const int nx0 = voff(sv + 1, 2 * h), nx1 = voff(sv + 1, 2 * h + 1);    // ... of row i + 1
    const int pv0 = voff(sv - 1, 2 * h), pv1 = voff(sv - 1, 2 * h + 1);    // ... of row i - 1
    const int nf0 = voff(sv + 1, 0), nf1 = voff(sv + 1, 1), nf2 = voff(sv + 1, 2), nf3 = voff(sv + 1, 3);
    // halo targets in the neighbours: my x half -> slot R+1 of CTA c-1 (first row),
    // my hand-over -> slot 0 of CTA c+1 (last row)
    const bool to_prev = CL > 1 && act && il == 0 && crank > 0;
    const bool to_next = CL > 1 && act && il == R - 1 && crank < CL - 1;
    const int hx0 = voff(R + 1, 2 * h), hx1 = voff(R + 1, 2 * h + 1);
    const int hh0 = voff(0, 2 * h), hh1 = voff(0, 2 * h + 1);

    double lam[4] = {0, 0, 0, 0}, r[4], pv[4], y[4];
    if (act) {
      const double2 a = *reinterpret_cast<const double2*>(sol + i * 8 + 4 * h);
      const double2 b = *reinterpret_cast<const double2*>(sol + i * 8 + 4 * h + 2);
      lam[0] = a.x, lam[1] = a.y, lam[2] = b.x, lam[3] = b.y;
    }
    mbar_wait(&s_bar[0], phase);

    // ---- building blocks of a product A x (A = -S: D = S_ii, O = L_i = S_{i+1,i};
    //      A = Phi^-1: D = P_ii, O = U_i = P_{i,i+1}); 4-term partial sums for ILP
    auto gather = [&](const double* xr, double* xf) {  // x_i in logical order
      double other[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) other[q] = __shfl_xor_sync(0xffffffffu, xr[q], 1);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        xf[q] = h8f::sel(h, other[q], xr[q]);
        xf[4 + q] = h8f::sel(h, xr[q], other[q]);
      }
    };
    auto rows_times = [&](const double2 (&m)[8][2], const double* xf, double* out) {  // my rows of M x
      double a[4], b[4];
      a[0] = m[0][0].x * xf[0], a[1] = m[0][0].y * xf[0], a[2] = m[0][1].x * xf[0], a[3] = m[0][1].y * xf[0];
      b[0] = m[4][0].x * xf[4], b[1] = m[4][0].y * xf[4], b[2] = m[4][1].x * xf[4], b[3] = m[4][1].y * xf[4];
#pragma unroll
      for (int c = 1; c < 4; ++c) {
        a[0] = fma(m[c][0].x, xf[c], a[0]);
        a[1] = fma(m[c][0].y, xf[c], a[1]);
        a[2] = fma(m[c][1].x, xf[c], a[2]);
        a[3] = fma(m[c][1].y, xf[c], a[3]);
        b[0] = fma(m[4 + c][0].x, xf[4 + c], b[0]);
        b[1] = fma(m[4 + c][0].y, xf[4 + c], b[1]);
        b[2] = fma(m[4 + c][1].x, xf[4 + c], b[2]);
        b[3] = fma(m[4 + c][1].y, xf[4 + c], b[3]);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) out[q] = a[q] + b[q];
    };
    // my 4 entries of M' x given my rows xm of x: half-column partial sums
    // over my rows, the partner lane completes the sums of my columns
    auto trans_times = [&](const double2 (&m)[8][2], const double* xm, double* out) {
      double part[8];
#pragma unroll
      for (int c = 0; c < 8; ++c)
        part[c] = fma(m[c][1].y, xm[3], fma(m[c][1].x, xm[2], fma(m[c][0].y, xm[1], m[c][0].x * xm[0])));
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double send = h8f::sel(h, part[q], part[4 + q]);
        const double recv = __shfl_xor_sync(0xffffffffu, send, 1);
        out[q] = h8f::sel(h, part[4 + q], part[q]) + recv;
      }
    };
    auto put = [&](double* buf, int o0, int o1, const double* x) {
      if (act) {
        *reinterpret_cast<double2*>(buf + o0) = make_double2(x[0], x[1]);
        *reinterpret_cast<double2*>(buf + o1) = make_double2(x[2], x[3]);
      }
    };
    auto get = [&](const double* buf, int o0, int o1, double* x) {
      const double2 a = *reinterpret_cast<const double2*>(buf + o0);
      const double2 b = *reinterpret_cast<const double2*>(buf + o1);
      x[0] = a.x, x[1] = a.y, x[2] = b.x, x[3] = b.y;
    };
    // phase 1 for vector x (buffers vb, xb): publishes x_i and the hand-over
    // for block row i+1, returns D_i x_i
    auto phase1 = [&](bool precond, const double2 (&dd)[8][2], const double2 (&oo)[8][2], const double* xr,
                      double* vb, double* xb, double* own) {
      double xf[8];
      gather(xr, xf);
      put(vb, my0, my1, xr);
      if constexpr (CL > 1)
        if (to_prev) {
          double* rv = cooperative_groups::this_cluster().map_shared_rank(vb, crank - 1);
          *reinterpret_cast<double2*>(rv + hx0) = make_double2(xr[0], xr[1]);
          *reinterpret_cast<double2*>(rv + hx1) = make_double2(xr[2], xr[3]);
        }
      rows_times(dd, xf, own);
      double hand[4];
      if (precond) trans_times(oo, xr, hand);  // U_i' x_i
      else rows_times(oo, xf, hand);            // L_i x_i
      put(xb, my0, my1, hand);
      if constexpr (CL > 1)
        if (to_next) {
          double* rx = cooperative_groups::this_cluster().map_shared_rank(xb, crank + 1);
          *reinterpret_cast<double2*>(rx + hh0) = make_double2(hand[0], hand[1]);
          *reinterpret_cast<double2*>(rx + hh1) = make_double2(hand[2], hand[3]);
        }
    };
    // phase 2 (after the barrier): the sub term (hand-over of row i-1) and the super term
    auto phase2 = [&](bool precond, const double2 (&oo)[8][2], const double* vb, const double* xb, double* low,
                      double* up) {
      if (!precond) {  // L_i' x_{i+1}
        double xn[4];
        get(vb, nx0, nx1, xn);
        trans_times(oo, xn, up);
      } else {  // U_i x_{i+1}
        double xn[8];
        get(vb, nf0, nf1, xn);
        get(vb, nf2, nf3, xn + 4);
        rows_times(oo, xn, up);
      }
      get(xb, pv0, pv1, low);
    };
    auto finish = [&](const double* own, const double* low, const double* up, double* out) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {  // diag, then sub (i > 0), then super (i < nb - 1)
        double acc = own[q];
        acc = has_prev ? acc + low[q] : acc;
        acc = has_next ? acc + up[q] : acc;
        out[q] = acc;
      }
    };

    auto matvec = [&](bool precond, const double* xr, double* out) {
      double2 dd[8][2], oo[8][2];
      h8f::load_rows(precond ? PdI : SdI, bs, dd);
      h8f::load_rows(precond ? PuI : SsI, bs, oo);
      double own[4], low[4], up[4];
      phase1(precond, dd, oo, xr, vbuf, xbuf, own);
      h8f_sync<CL>();
      phase2(precond, oo, vbuf, xbuf, low, up);
      finish(own, low, up, out);
    };
    // (-S) x with the partials of the dot a'b published before the product's
    // (cluster) barrier, which then serves both
    auto matvec_s_dot = [&](const double* xr, double* out, const double* a, const double* b, int slot) {
      double2 dd[8][2], oo[8][2];
      h8f::load_rows(SdI, bs, dd);
      h8f::load_rows(SsI, bs, oo);
      double own[4], low[4], up[4];
      if (!dbuf) h8f_sync<CL>();  // the Phi^-1 product's phase-2 reads of vbuf / xbuf are done
      phase1(false, dd, oo, xr, vbuf2, xbuf2, own);
      partial(a, b, slot);
      h8f_sync<CL>();
      phase2(false, oo, vbuf2, xbuf2, low, up);
      finish(own, low, up, out);
    };

    matvec(false, lam, y);  // y = (-S) lambda0
    if (act) {
      const double2 a = *reinterpret_cast<const double2*>(gam + i * 8 + 4 * h);
      const double2 b = *reinterpret_cast<const double2*>(gam + i * 8 + 4 * h + 2);
      r[0] = a.x - y[0], r[1] = a.y - y[1], r[2] = b.x - y[2], r[3] = b.y - y[3];
    } else {
      r[0] = r[1] = r[2] = r[3] = 0.0;
    }
    h8f_sync<CL>();  // every phase-2 read of lambda / its hand-over is done
    mbar_wait(&s_bar[1], phase);
    phase ^= 1;
    matvec(true, r, pv);  // r~
    int status = DOCP_OK, iters = 0;
    double finals_eta = 0.0;
    if constexpr (CL == 1) {  // the single-CTA form folds exactly as pcg_kernel_h8r
    double eta = dot(r, pv);
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
      for (int q = 0; q < 4; ++q) {
        lam[q] = fma(alpha, pv[q], lam[q]);
        r[q] = fma(-alpha, y[q], r[q]);
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
      for (int q = 0; q < 4; ++q) pv[q] = fma(beta, pv[q], y[q]);
      eta = eta_next;
      ++iters;
    }

    finals_eta = eta;
    } else {
    // Clusters: the second dot is pipelined as in pcg_kernel_h8s: w = (-S) r~
    // is formed while eta' = r'r~ reduces (one cluster barrier fewer per
    // iteration), p = r~ + beta p, y = w + beta y (Chronopoulos-Gear's s).
    double rt[4], sr[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) rt[q] = pv[q];
    matvec_s_dot(rt, sr, r, rt, 1);
    double eta = total(1);
    if (eta < 0.0) {
      const double scale = norm(r) * norm(rt);
      if (-eta <= 1e-10 * scale + 1e-300) eta = 0.0;
      else status = DOCP_AT_PCG_PRECOND;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) y[q] = sr[q];
    while (status == DOCP_OK && eta > threshold && iters < max_iters) {
      const double vv = dot(pv, y);
      if (vv <= 0.0) {
        status = DOCP_AT_PCG_CURVATURE;
        break;
      }
      const double alpha = eta / vv;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        lam[q] = fma(alpha, pv[q], lam[q]);
        r[q] = fma(-alpha, y[q], r[q]);
      }
      matvec(true, r, rt);               // r~
      matvec_s_dot(rt, sr, r, rt, 1);    // (-S) r~ while eta' = r'r~ reduces
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
      const double beta = eta_next / eta;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        pv[q] = fma(beta, pv[q], rt[q]);
        y[q] = fma(beta, y[q], sr[q]);
      }
      eta = eta_next;
      ++iters;
    }
    finals_eta = eta;
    }

    if (act) {
      *reinterpret_cast<double2*>(sol + i * 8 + 4 * h) = make_double2(lam[0], lam[1]);
      *reinterpret_cast<double2*>(sol + i * 8 + 4 * h + 2) = make_double2(lam[2], lam[3]);
    }
    if (tid == 0 && crank == 0) {
      v.pcg_iters[pidx] = iters;
      v.final_eta[pidx] = finals_eta;
      v.pcg_conv[pidx] = status == DOCP_OK && finals_eta <= threshold;
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
