// k_pcg_h8s.cuh — K2 FAST mode for n_x = 8, single CTA: pcg_kernel_h8r with
// BOTH symmetric diagonal blocks (-S_ii and Phi^-1_ii) held in registers in
// packed form, so the preconditioner product reads only the super-diagonal
// blocks from shared memory.
//
// -S diag and Phi^-1 diag are symmetric by construction (schur.hpp:145-164:
// sym(Q_0^-1), sym(chi_t), sym(chi_t^-1), and Q_0), so the two threads of a
// block row split the 36 distinct entries: thread h keeps the upper triangle
// of its own 4 x 4 diagonal sub-block (10 values) and columns 4+2h, 5+2h of
// the upper-right 4 x 4 sub-block (8 values). Its product
//   y_{R_h} = D_hh x_h                       (own sub-block, symmetric)
//   y_top  += D01[:, c_h] x[c_h]             (h = 0 keeps it, h = 1 sends it)
//   y[c_h] += D01[:, c_h]' x_top             (h = 1 keeps it, h = 0 sends it)
// is 32 fmas per thread, as for the full block, plus one 4-value partner
// exchange. 18 doubles per block instead of 32 leave room for Phi^-1_ii next
// to -S_ii and L_i; the Phi^-1 half read from shared memory per iteration
// drops from (2T+1) to T blocks. FAST arithmetic (a different fold order
// from h8r / h8f; same iteration counts, <= 1e-9 relative).
//
// Requires exactly symmetric diagonal blocks: used for systems assembled on
// the device (docp_batch::sym_blocks); uploaded systems use pcg_kernel_h8r.
#pragma once

#include "k_pcg_h8r.cuh"

namespace docp_dev {

namespace h8s {

/// Packed upper triangle of a 4 x 4 symmetric block: (a, b), a <= b.
__host__ __device__ constexpr int tri(int a, int b) { return a * 4 - a * (a - 1) / 2 + (b - a); }

/// Thread h's share of a symmetric 8 x 8 block (see the header comment).
struct Sym {
  double o[10];  // D_hh upper triangle
  double s[4][2];  // D01 rows 0..3, columns 4+2h, 5+2h
};

/// Loads thread h's share of symmetric block b (block index b for the swizzle) at blk.
__device__ __forceinline__ void load_sym(const double* blk, int b, int h, Sym& m) {
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = a; c < 4; ++c) m.o[tri(a, c)] = blk[blk_off(8, b, 4 * h + a, 4 * h + c)];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int k = 0; k < 2; ++k) m.s[a][k] = blk[blk_off(8, b, a, 4 + 2 * h + k)];
}

/// My 4 rows of D x (xf: x in logical order, xr: my half).
__device__ __forceinline__ void sym_times(const Sym& m, const double* xf, const double* xr, int h, double* out) {
  auto O = [&](int a, int b) { return a <= b ? m.o[tri(a, b)] : m.o[tri(b, a)]; };
  double own[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const double a = fma(O(q, 1), xr[1], O(q, 0) * xr[0]);
    const double b = fma(O(q, 3), xr[3], O(q, 2) * xr[2]);
    own[q] = a + b;
  }
  const double xc0 = h ? xf[6] : xf[4], xc1 = h ? xf[7] : xf[5];
  double A[4], Bt[2];
#pragma unroll
  for (int q = 0; q < 4; ++q) A[q] = fma(m.s[q][1], xc1, m.s[q][0] * xc0);
#pragma unroll
  for (int k = 0; k < 2; ++k)
    Bt[k] = fma(m.s[3][k], xf[3], fma(m.s[2][k], xf[2], fma(m.s[1][k], xf[1], m.s[0][k] * xf[0])));
  double recv[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const double send = h ? A[q] : (q < 2 ? Bt[q] : 0.0);
    recv[q] = __shfl_xor_sync(0xffffffffu, send, 1);
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const double mine = q < 2 ? recv[q] : Bt[q - 2];  // h = 1: rows 4,5 from the partner, 6,7 own
    out[q] = h ? own[q] + mine : (own[q] + A[q]) + recv[q];
  }
}

}  // namespace h8s

/// Dynamic shared memory of pcg_kernel_h8s (doubles). PREFETCH: Phi^-1 of the
/// current problem plus a staging area for the next problem's -S; otherwise
/// one record-sized region that takes -S, then Phi^-1, of the current problem.
template <int MAXT, bool PREFETCH, bool SD_SMEM = false, int CL = 1>
__host__ __device__ inline long h8s_smem_doubles(const Dims& d) {
  constexpr int NWS = MAXT <= 256 ? 8 : 16;
  const long R = (d.nb + CL - 1) / CL;  // block rows per CTA
  return (PREFETCH ? 4L : SD_SMEM ? 3L : 2L) * R * 64 + (R + 2) * 8 + (R + 2 + (CL > 1)) * 8 + 3L * NWS * CL;
}

/// MAXT = 256: 255 registers per thread; with PREFETCH = false (T <= 127) the
/// -S and Phi^-1 halves of a record that does not fit twice in shared memory
/// are loaded one after the other into the same region. pcg_kernel_h8s_wide
/// (below) extends that to T <= 191.
#ifdef DOCP_H8S_CLOCK
__device__ unsigned long long g_h8s_clk[16];
#define H8S_CLK(k)                        \
  if (tid == 0) {                         \
    const long long t_ = clock64();       \
    clk[k] += t_ - t_last;                \
    t_last = t_;                          \
  }
#else
#define H8S_CLK(k)
#endif

/// PD_SMEM: the Phi^-1 diagonal blocks are read from shared memory every
/// iteration (rows 4h..4h+3, as U_i) instead of being held in registers:
/// 36 registers fewer, for the wide form whose 9-12 warps cap every thread
/// at 168 registers (an SMSP then holds three warps).
/// SD_SMEM (with PD_SMEM, no prefetch): the -S diagonal blocks stay in a
/// third shared-memory region as well, so only L_i's rows stay in registers:
/// the > 8-warp forms (168 registers per thread) then run without spilling
/// where three regions fit (T <= 134).
/// CL > 1 (long horizons, FAST, no prefetch): a thread-block cluster of CL
/// CTAs solves one problem, CTA c holding block rows [cR, cR + R) of every
/// region with this kernel's register residency. Neighbour rows across a CTA
/// boundary exchange x and the hand-overs through distributed shared memory
/// (halo slots: vbuf R + 1 <- the next CTA's first row; xbuf 1 and 0 <- the
/// previous CTA's last row, for the Phi^-1 and the (-S) products), every
/// warp's dot partial goes to every CTA, and the product and dot barriers
/// become cluster barriers.
template <int MAXT, bool PREFETCH, bool PD_SMEM = false, bool SD_SMEM = false, int CL = 1>
__device__ __forceinline__ void h8s_body(View v, const int* __restrict__ work, const int* __restrict__ n_work,
                                         int* __restrict__ counter, double* __restrict__ sol_all, double epsilon,
                                         int max_iters_cfg) {
  extern __shared__ __align__(128) double sm_pcg[];
  __shared__ __align__(8) uint64_t s_bar[2];  // [0]: staged -S blocks, [1]: Phi^-1 blocks
  __shared__ int s_next, s_pidx;
  const Dims d = v.d;
  const int nl = d.nl, nb = d.nb;
  const int tid = threadIdx.x;
  static_assert(CL == 1 || (!PREFETCH && !SD_SMEM), "the cluster form is a no-prefetch form");
  const int crank = CL == 1 ? 0 : static_cast<int>(cooperative_groups::this_cluster().block_rank());
  const int R = CL == 1 ? nb : (nb + CL - 1) / CL;  // block rows per CTA
  const int row0 = crank * R;                        // first global block row of this CTA
  const int nrows = CL == 1 ? nb : max(0, min(R, nb - row0));
  const int nsub = CL == 1 ? nb - 1 : max(0, min(R, nb - 1 - row0));
  const int il = tid >> 1, h = tid & 1;
  const int i = row0 + il;  // global block row
  const bool act = il < nrows;
  const bool has_next = act && i + 1 < nb;
  const bool has_prev = i > 0;
  const int lane = tid & 31, warp = tid >> 5;
  const int nwk = *n_work;
#ifdef DOCP_H8S_CLOCK
  long long clk[16] = {0}, t_last = clock64();
#endif

  constexpr int NWS = MAXT <= 256 ? 8 : 16;  // warp slots per dot
  static_assert(!SD_SMEM || (PD_SMEM && !PREFETCH), "SD_SMEM is a no-prefetch, PD_SMEM form");
  double* sPd = sm_pcg;            // [R] Phi^-1 diagonal blocks (current problem)
  double* sPu = sPd + R * 64;      // [R] Phi^-1 super blocks
  double* sSr = sPu + R * 64;      // SD_SMEM: [R] -S diagonal blocks, resident
  // -S diagonal / sub blocks: the next problem's (staging) or, without the
  // prefetch, the current problem's in the same region as Phi^-1 (SD_SMEM:
  // the diagonal ones straight into their resident region)
  double* sNd = PREFETCH ? sPu + R * 64 : SD_SMEM ? sSr : sPd;
  double* sNs = SD_SMEM ? sPd : sNd + R * 64;
  double* vbuf = sPu + (PREFETCH ? 3 : SD_SMEM ? 2 : 1) * R * 64;  // [R + 2] x_i halves (slot = row + 1)
  double* xbuf = vbuf + (R + 2) * 8;  // hand-overs (CL > 1: one more halo slot in front)
  double* red = xbuf + (R + 2 + (CL > 1)) * 8;  // [3][CL][NWS] dot partials

  const int p = i & 1, m = (i >> 1) & 1;
  h8f::Bases bs;
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int j = 0; j < 2; ++j)
      bs.o[k][j] = ((k & 1) ? -8 * p : 8 * p) + 4 * ((k >> 1) ? 1 - h : h) + 2 * (j ^ m);

  // local block of this row (inactive rows: the last one)
  const int ib = CL == 1 ? (act ? il : nb - 1) : (act ? il : max(0, nrows - 1));
  const int gb = row0 + ib;                      // its global index (the record's swizzle)
  const int io = has_next ? il : 0;
  const double* PdI = sPd + ib * 64;
  const double* PuI = sPu + io * 64;
  const double* NdI = sNd + ib * 64;
  const double* NsI = sNs + io * 64;
  auto voff = [](int j, int k) { return j * 8 + 2 * (k ^ ((j >> 1) & 3)); };
  const int sv = ib + 1;
  const int my0 = voff(sv, 2 * h), my1 = voff(sv, 2 * h + 1);
  const int nx0 = voff(sv + 1, 2 * h), nx1 = voff(sv + 1, 2 * h + 1);
  const int pv0 = voff(sv - 1, 2 * h), pv1 = voff(sv - 1, 2 * h + 1);
  // the (-S) product's hand-over goes one slot lower than the Phi^-1 one (row
  // i writes slot i, reads slot i - 1): matvec_s_dot follows matvec_p with no
  // barrier between, and this way the only slot it overwrites is the one this
  // same thread has just read (row 0 reads slot 0, masked by has_prev)
  const int pp0 = voff(max(sv - 2, 0), 2 * h), pp1 = voff(max(sv - 2, 0), 2 * h + 1);
  const int nf0 = voff(sv + 1, 0), nf1 = voff(sv + 1, 1), nf2 = voff(sv + 1, 2), nf3 = voff(sv + 1, 3);
  // hand-over slots: CL > 1 shifts them one up so that the (-S) product's
  // (one slot lower) has a halo slot for row 0 too
  constexpr int XS = CL > 1 ? 1 : 0;
  const int xmy0 = CL == 1 ? my0 : voff(sv + XS, 2 * h), xmy1 = CL == 1 ? my1 : voff(sv + XS, 2 * h + 1);
  const int xpv0 = CL == 1 ? pv0 : voff(sv - 1 + XS, 2 * h), xpv1 = CL == 1 ? pv1 : voff(sv - 1 + XS, 2 * h + 1);
  const int xpp0 = CL == 1 ? pp0 : voff(max(sv - 2 + XS, 0), 2 * h);
  const int xpp1 = CL == 1 ? pp1 : voff(max(sv - 2 + XS, 0), 2 * h + 1);
  // halos: my x half -> slot sv + R of the previous CTA (my first row), my
  // hand-overs -> slot (their slot) - R of the next CTA (my last row)
  const bool to_prev = CL > 1 && act && il == 0 && crank > 0;
  const bool to_next = CL > 1 && act && il == R - 1 && crank < CL - 1;
  const uint32_t bd = static_cast<uint32_t>(CL == 1 ? nb : nrows) * 512u;
  const uint32_t bo = static_cast<uint32_t>(CL == 1 ? nb - 1 : nsub) * 512u;

  // next work item and its problem index (tid 0 only). Problems that failed
  // earlier are skipped at the start of their turn (all threads read the
  // status there), which keeps tid 0's chain to one atomic and one load.
  auto grab = [&]() {
    const int w = atomicAdd(counter, 1);
    s_next = w;
    s_pidx = w < nwk ? work[w] : 0;
  };
  auto stage_s = [&](int pi) {  // -S blocks of problem pi (this CTA's rows) -> staging area
    const double* rec = v.blocks + static_cast<long>(pi) * d.blk_stride;
    if constexpr (CL > 1) rec += static_cast<long>(row0) * 64;
    mbar_arrive_expect_tx(&s_bar[0], bd + bo);
    if (CL == 1 || bd) tma_bulk_g2s(sNd, rec + d.s_diag, bd, &s_bar[0]);
    if (bo) tma_bulk_g2s(sNs, rec + d.s_sub, bo, &s_bar[0]);
  };

  if constexpr (CL == 1) {
    if (tid < 3 * NWS) red[tid] = 0.0;
  } else {
    for (int k = tid; k < 3 * NWS * CL; k += blockDim.x) red[k] = 0.0;
  }
  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    if constexpr (CL == 1) {
      grab();
      if (PREFETCH && s_next < nwk) stage_s(s_pidx);
    }
  }
  __syncthreads();
  if constexpr (CL > 1) h8f_sync<CL>();  // every CTA of the cluster running (and its red zeroed) before any remote access
  uint32_t phase = 0, ph1 = 0;  // parities of s_bar[0] (staging) and s_bar[1] (Phi^-1)
  const int max_iters = max_iters_cfg > 0 ? max_iters_cfg : 2 * nl;
  const double threshold = epsilon * epsilon;

  auto partial = [&](const double* a, const double* b, int slot) {
    double s = fma(a[3], b[3], fma(a[2], b[2], fma(a[1], b[1], a[0] * b[0])));
    s = act ? s : 0.0;
    s = warp_sum(s);
    if (lane == 0) {
      if constexpr (CL == 1) {
        red[slot * NWS + warp] = s;
      } else {
        const int at = (slot * CL + crank) * NWS + warp;
#pragma unroll
        for (int c = 0; c < CL; ++c) cooperative_groups::this_cluster().map_shared_rank(red, c)[at] = s;
      }
    }
  };
  // pairwise over the 8 warp slots (slots of absent warps hold 0): depth 3
  auto total1 = [&](const double* base) -> double {
    const double2* q = reinterpret_cast<const double2*>(base);
    const double2 a = q[0], b = q[1], c = q[2], e = q[3];
    const double t8 = ((a.x + a.y) + (b.x + b.y)) + ((c.x + c.y) + (e.x + e.y));
    if constexpr (NWS == 8) {
      return t8;
    } else {
      const double2 f = q[4], g = q[5], k = q[6], m = q[7];
      return t8 + (((f.x + f.y) + (g.x + g.y)) + ((k.x + k.y) + (m.x + m.y)));
    }
  };
  // CL > 1: the CTAs' partial sums in rank order (every CTA the same bits)
  auto total = [&](int slot) -> double {
    double t = total1(red + slot * CL * NWS);
#pragma unroll
    for (int c = 1; c < CL; ++c) t = t + total1(red + (slot * CL + c) * NWS);
    return t;
  };
  auto dot = [&](const double* a, const double* b) -> double {
    partial(a, b, 0);
    H8S_CLK(6);
    h8f_sync<CL>();
    H8S_CLK(7);
    const double t = total(0);
    H8S_CLK(8);
    return t;
  };
  auto norm = [&](const double* a) -> double {
    h8f_sync<CL>();
    partial(a, a, 2);
    h8f_sync<CL>();
    return sqrt(total(2));
  };
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
  auto rows_times = [&](const double2 (&mm)[8][2], const double* xf, double* out) {  // my rows of M x
    double a[4], b[4];
    a[0] = mm[0][0].x * xf[0], a[1] = mm[0][0].y * xf[0], a[2] = mm[0][1].x * xf[0], a[3] = mm[0][1].y * xf[0];
    b[0] = mm[4][0].x * xf[4], b[1] = mm[4][0].y * xf[4], b[2] = mm[4][1].x * xf[4], b[3] = mm[4][1].y * xf[4];
#pragma unroll
    for (int c = 1; c < 4; ++c) {
      a[0] = fma(mm[c][0].x, xf[c], a[0]);
      a[1] = fma(mm[c][0].y, xf[c], a[1]);
      a[2] = fma(mm[c][1].x, xf[c], a[2]);
      a[3] = fma(mm[c][1].y, xf[c], a[3]);
      b[0] = fma(mm[4 + c][0].x, xf[4 + c], b[0]);
      b[1] = fma(mm[4 + c][0].y, xf[4 + c], b[1]);
      b[2] = fma(mm[4 + c][1].x, xf[4 + c], b[2]);
      b[3] = fma(mm[4 + c][1].y, xf[4 + c], b[3]);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) out[q] = a[q] + b[q];
  };
  auto trans_times = [&](const double2 (&mm)[8][2], const double* xm, double* out) {  // my 4 entries of M' x
    double part[8];
#pragma unroll
    for (int c = 0; c < 8; ++c)
      part[c] = fma(mm[c][1].y, xm[3], fma(mm[c][1].x, xm[2], fma(mm[c][0].y, xm[1], mm[c][0].x * xm[0])));
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
  // CL > 1: my x half into the previous CTA's halo slot sv + R (first row)
  auto put_halo_x = [&](const double* x) {
    if constexpr (CL > 1)
      if (to_prev) {
        double* rv = cooperative_groups::this_cluster().map_shared_rank(vbuf, crank - 1);
        *reinterpret_cast<double2*>(rv + voff(sv + R, 2 * h)) = make_double2(x[0], x[1]);
        *reinterpret_cast<double2*>(rv + voff(sv + R, 2 * h + 1)) = make_double2(x[2], x[3]);
      }
  };
  // ... and my hand-over into the next CTA's slot `slot` (last row)
  auto put_halo_hand = [&](const double* x, int slot) {
    if constexpr (CL > 1)
      if (to_next) {
        double* rx = cooperative_groups::this_cluster().map_shared_rank(xbuf, crank + 1);
        *reinterpret_cast<double2*>(rx + voff(slot, 2 * h)) = make_double2(x[0], x[1]);
        *reinterpret_cast<double2*>(rx + voff(slot, 2 * h + 1)) = make_double2(x[2], x[3]);
      }
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

  h8s::Sym sd, pd;  // my shares of -S_ii and Phi^-1_ii, resident for the whole solve
  double2 so[8][2];  // my rows of L_i

  for (;;) {
    if constexpr (CL > 1) {  // the cluster's next problem, taken by CTA 0 for all
      if (tid == 0 && crank == 0) {
        const int wk = atomicAdd(counter, 1);
        const int pk = wk < nwk ? work[wk] : 0;
#pragma unroll
        for (int c = 0; c < CL; ++c) {
          *cooperative_groups::this_cluster().map_shared_rank(&s_next, c) = wk;
          *cooperative_groups::this_cluster().map_shared_rank(&s_pidx, c) = pk;
        }
      }
      h8f_sync<CL>();
    }
    const int w = s_next;
    if (w >= nwk) break;
    const int pidx = s_pidx;
    // this problem's warm start and right-hand side, issued before the
    // staging wait so their latency overlaps it
    const double* gam = v.gamma + static_cast<long>(pidx) * nl;
    double* sol = sol_all + static_cast<long>(pidx) * nl;
    double2 l01 = make_double2(0.0, 0.0), l23 = l01, g01 = l01, g23 = l01;
    if (act) {
      l01 = *reinterpret_cast<const double2*>(sol + i * 8 + 4 * h);
      l23 = *reinterpret_cast<const double2*>(sol + i * 8 + 4 * h + 2);
      g01 = *reinterpret_cast<const double2*>(gam + i * 8 + 4 * h);
      g23 = *reinterpret_cast<const double2*>(gam + i * 8 + 4 * h + 2);
    }
    const bool runnable = v.status[pidx].code == DOCP_OK;  // failed in an earlier stage: skip
    if constexpr (!PREFETCH) {
      if (!runnable) {  // block-uniform
        if constexpr (CL > 1) {
          h8f_sync<CL>();  // s_next / s_pidx read in every CTA
        } else {
          __syncthreads();  // s_next / s_pidx read by every thread
          if (tid == 0) grab();
          __syncthreads();
        }
        continue;
      }
      if (tid == 0) {  // this problem's -S into the record region (free since the last barrier)
        fence_proxy_async();
        stage_s(pidx);
      }
    }
    mbar_wait(&s_bar[0], phase);
    if constexpr (!SD_SMEM) h8s::load_sym(NdI, gb, h, sd);
    h8f::load_rows(NsI, bs, so);
    __syncthreads();  // staging area consumed; s_next / s_pidx read; Phi^-1 reads of the previous problem done
    phase ^= 1;
    if constexpr (PREFETCH) {
      if (!runnable) {  // block-uniform; s_bar[1] is not armed for a skipped problem
        if (tid == 0) {
          fence_proxy_async();
          grab();
          if (s_next < nwk) stage_s(s_pidx);
        }
        __syncthreads();
        continue;
      }
    }
    if (tid == 0) {
      fence_proxy_async();
      const double* rec = v.blocks + static_cast<long>(pidx) * d.blk_stride;
      if constexpr (CL > 1) rec += static_cast<long>(row0) * 64;
      mbar_arrive_expect_tx(&s_bar[1], bd + bo);
      if (CL == 1 || bd) tma_bulk_g2s(sPd, rec + d.p_diag, bd, &s_bar[1]);
      if (bo) tma_bulk_g2s(sPu, rec + d.p_sup, bo, &s_bar[1]);
      if constexpr (CL == 1) {
        grab();  // s_next / s_pidx: read after the end-of-problem barrier
        if (PREFETCH && s_next < nwk) stage_s(s_pidx);
      }
    }

    double lam[4] = {l01.x, l01.y, l23.x, l23.y}, r[4] = {0, 0, 0, 0}, pv[4], y[4];

    // out = (-S) x from the register-resident blocks; the partials of the dot
    // a'b are published with the product's exchange (one barrier for both)
    auto matvec_s_dot = [&](const double* xr, double* out, const double* a, const double* b, int slot) {
      double xf[8], own[4], hand[4], low[4], up[4], xn[4];
      gather(xr, xf);
      put(vbuf, my0, my1, xr);
      put_halo_x(xr);
      H8S_CLK(12);
      if constexpr (SD_SMEM) {
        double2 dd[8][2];
        h8f::load_rows(NdI, bs, dd);
        rows_times(dd, xf, own);
      } else {
        h8s::sym_times(sd, xf, xr, h, own);
      }
      H8S_CLK(13);
      rows_times(so, xf, hand);  // L_i x_i
      put(xbuf, xpv0, xpv1, hand);  // slot i (see pp0 above)
      put_halo_hand(hand, sv - 1 + XS - R);
      H8S_CLK(14);
      partial(a, b, slot);
      H8S_CLK(0);
      h8f_sync<CL>();
      H8S_CLK(1);
      get(vbuf, nx0, nx1, xn);
      trans_times(so, xn, up);   // L_i' x_{i+1}
      get(xbuf, xpp0, xpp1, low);
      finish(own, low, up, out);
    };
    // out = Phi^-1 x from shared memory. Two exchanges (x_{i+1}, then the
    // U_i' x_i hand-over) so that each thread reads its half of U_i once for
    // both U_i' x_i and U_i x_{i+1}: shared-memory traffic is what bounds this
    // phase, one barrier is cheaper than a second pass over U_i.
    auto matvec_p = [&](const double* xr, double* out) {
      double xf[8], own[4], hand[4], low[4], up[4], xn[8];
      gather(xr, xf);
      put(vbuf, my0, my1, xr);
      put_halo_x(xr);
      if constexpr (PD_SMEM) {
        double2 dd[8][2];
        h8f::load_rows(PdI, bs, dd);
        rows_times(dd, xf, own);
      } else {
        h8s::sym_times(pd, xf, xr, h, own);
      }
      H8S_CLK(3);
      h8f_sync<CL>();
      H8S_CLK(1);
      get(vbuf, nf0, nf1, xn);
      get(vbuf, nf2, nf3, xn + 4);
      {
        double2 oo[8][2];
        h8f::load_rows(PuI, bs, oo);
        trans_times(oo, xr, hand);  // U_i' x_i
        rows_times(oo, xn, up);     // U_i x_{i+1}
      }
      put(xbuf, xmy0, xmy1, hand);
      put_halo_hand(hand, sv + XS - R);
      H8S_CLK(4);
      h8f_sync<CL>();
      H8S_CLK(1);
      get(xbuf, xpv0, xpv1, low);
      finish(own, low, up, out);
    };

    matvec_s_dot(lam, y, r, r, 2);  // y = (-S) lambda0 (slot 2: an unread dummy dot)
    if (act) {
      r[0] = g01.x - y[0], r[1] = g01.y - y[1], r[2] = g23.x - y[2], r[3] = g23.y - y[3];
    } else {
      r[0] = r[1] = r[2] = r[3] = 0.0;
    }
    h8f_sync<CL>();  // every phase-2 read of lambda / its hand-over is done
    mbar_wait(&s_bar[1], ph1);
    ph1 ^= 1;
    if constexpr (!PD_SMEM) h8s::load_sym(PdI, gb, h, pd);
    double rt[4], sr[4];  // r~ and (-S) r~
    matvec_p(r, rt);                 // r~ = Phi^-1 r
    // Pipelined second dot: sr = (-S) r~ is formed while eta = r'r~ reduces
    // (its partials ride on the product's barrier); p = r~ + beta p and
    // y = (-S) p = sr + beta y then need no product of their own. y is the
    // recurrence of Chronopoulos-Gear's s; v = p'y stays a direct dot.
    matvec_s_dot(rt, sr, r, rt, 1);
    double eta = total(1);
    int status = DOCP_OK, iters = 0;
    if (eta < 0.0) {
      const double scale = norm(r) * norm(rt);
      if (-eta <= 1e-10 * scale + 1e-300) eta = 0.0;
      else status = DOCP_AT_PCG_PRECOND;
    }
    double inv_eta = 1.0 / eta;  // beta = eta' / eta as eta' * (1 / eta), the division off the critical path
#pragma unroll
    for (int q = 0; q < 4; ++q) pv[q] = rt[q], y[q] = sr[q];

    H8S_CLK(11);
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
      H8S_CLK(9);
      matvec_p(r, rt);                 // r~
      H8S_CLK(5);
      matvec_s_dot(rt, sr, r, rt, 1);   // sr = (-S) r~ while eta' = r'r~ reduces
      H8S_CLK(2);
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
      const double beta = eta_next * inv_eta;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        pv[q] = fma(beta, pv[q], rt[q]);
        y[q] = fma(beta, y[q], sr[q]);
      }
      eta = eta_next;
      inv_eta = 1.0 / eta;
      ++iters;
      H8S_CLK(10);
    }

    if (act) {
      *reinterpret_cast<double2*>(sol + i * 8 + 4 * h) = make_double2(lam[0], lam[1]);
      *reinterpret_cast<double2*>(sol + i * 8 + 4 * h + 2) = make_double2(lam[2], lam[3]);
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
    // s_next is published; Phi^-1 / vectors (and, CL > 1, the halos) free for the next problem
    if constexpr (CL > 1) h8f_sync<CL>();
    else __syncthreads();
  }
#ifdef DOCP_H8S_CLOCK
  if (tid == 0)
    for (int k = 0; k < 16; ++k) atomicAdd(&g_h8s_clk[k], static_cast<unsigned long long>(clk[k]));
#endif
}

template <int MAXT, bool PREFETCH>
__global__ void __launch_bounds__(MAXT, 1) pcg_kernel_h8s(View v, const int* __restrict__ work,
                                                        const int* __restrict__ n_work, int* __restrict__ counter,
                                                        double* __restrict__ sol_all, double epsilon,
                                                        int max_iters_cfg) {
  h8s_body<MAXT, PREFETCH>(v, work, n_work, counter, sol_all, epsilon, max_iters_cfg);
}

/// Long horizons (T > 191): a cluster of CL CTAs of <= 8 warps each, the
/// blocks register- and shared-memory-resident across them.
template <int CL>
__global__ void __launch_bounds__(256, 1) pcg_kernel_h8s_cl(View v, const int* __restrict__ work,
                                                           const int* __restrict__ n_work, int* __restrict__ counter,
                                                           double* __restrict__ sol_all, double epsilon,
                                                           int max_iters_cfg) {
  h8s_body<256, false, false, false, CL>(v, work, n_work, counter, sol_all, epsilon, max_iters_cfg);
}

/// Up to 384 threads (T <= 191): 9-12 warps, so an SMSP holds three of them
/// and its quarter of the register file (16K) caps every thread at 168
/// registers (some spilling).
__global__ void __maxnreg__(168)
    pcg_kernel_h8s_wide(View v, const int* __restrict__ work, const int* __restrict__ n_work,
                        int* __restrict__ counter, double* __restrict__ sol_all, double epsilon, int max_iters_cfg) {
  h8s_body<384, false, true>(v, work, n_work, counter, sol_all, epsilon, max_iters_cfg);
}

/// The same with -S_ii in shared memory too (T <= 134): no spills at 168.
__global__ void __maxnreg__(168)
    pcg_kernel_h8s_wide_sd(View v, const int* __restrict__ work, const int* __restrict__ n_work,
                           int* __restrict__ counter, double* __restrict__ sol_all, double epsilon, int max_iters_cfg) {
  h8s_body<384, false, true, true>(v, work, n_work, counter, sol_all, epsilon, max_iters_cfg);
}

}  // namespace docp_dev
