// k_pcg_h8p.cuh — K2 PARITY mode for n_x = 8 on device-assembled systems:
// the reference's arithmetic bit for bit (btd_matvec's diag -> sub -> super
// accumulation with every block product a left fold seeded with its first
// term, schur.hpp:60-72; block_dot's per-block folds summed in block-index
// order, pcg.hpp:37-44; separately rounded products, no FMA) with the data
// residency of pcg_kernel_h8s (k_pcg_h8s.cuh):
//
//   registers  thread (i, h), h = 0, 1 the two threads of block row i:
//              its share of the symmetric -S_ii and Phi^-1_ii (18 + 18
//              doubles, SymP below) and two 4 x 4 quarters of L_i (32);
//   shared     Phi^-1 super blocks U_i (TMA at the problem's start), the next
//              problem's -S blocks (TMA prefetch), vector exchange buffers,
//              the block dots.
//
// A left fold is sequential, but it can be cut anywhere and continued by
// another thread with the partial sum, bit for bit. Every product below is
// split that way between the two threads of a row:
//   * off-diagonal blocks: with W = L_i (for -S) or U_i' (for Phi^-1) the
//     row needs hand_r = sum_c W(r, c) x_i[c] (the sub term of row i + 1)
//     and up_r = sum_c W(c, r) x_{i+1}[c] (its own super term). Thread 0
//     holds the quarters W00, W11, thread 1 W10, W01 (Wab = rows 4a..4a+3,
//     columns 4b..4b+3), so each thread folds the first half (c < 4) of four
//     outputs, the partners swap partial sums, and each folds the second half
//     of the other four: both threads do the same work in the same code;
//   * symmetric diagonal blocks: thread h keeps its D_hh triangle and rows
//     2h, 2h + 1 of D01; the partner sends the products (thread 1 -> 0) and
//     the two-term partial sums (thread 0 -> 1) the other's rows need.
// block_dot: each block's 8-term fold is cut between the two threads, the
// 101 block dots go to shared memory, and lane 0 of every warp folds them in
// index order (a sequential chain of T + 1 additions, the one part of the
// iteration that cannot be parallelised without changing the bits).
#pragma once

#include "k_pcg_h8s.cuh"

namespace docp_dev {

namespace h8p {

/// Thread h's share of a symmetric 8 x 8 block D: the upper triangle of D_hh
/// (packed as h8s::tri) and rows 2h, 2h + 1 of D01 = D(0..3, 4..7).
struct SymP {
  double t[10];
  double s[2][4];  // s[a][j] = D(2h + a, 4 + j)
};

__device__ __forceinline__ void load_symp(const double* blk, int b, int h, SymP& m) {
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = a; c < 4; ++c) m.t[h8s::tri(a, c)] = blk[blk_off(8, b, 4 * h + a, 4 * h + c)];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int j = 0; j < 4; ++j) m.s[a][j] = blk[blk_off(8, b, 2 * h + a, 4 + j)];
}

/// The two quarters of W (= L_i, the stored -S sub block) thread h keeps:
/// f[a][b] = W(4h + a, b), g[a][b] = W(4(1 - h) + a, 4 + b).
struct Quarters {
  double f[4][4];
  double g[4][4];
};

__device__ __forceinline__ void load_quarters(const double* blk, int b, int h, Quarters& w) {
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const double2 u = *reinterpret_cast<const double2*>(blk + blk_off(8, b, 4 * h + 2 * j, c));
      w.f[2 * j][c] = u.x, w.f[2 * j + 1][c] = u.y;
      const double2 v = *reinterpret_cast<const double2*>(blk + blk_off(8, b, 4 * (1 - h) + 2 * j, 4 + c));
      w.g[2 * j][c] = v.x, w.g[2 * j + 1][c] = v.y;
    }
}

__device__ __forceinline__ double sel(bool c, double a, double b) { return c ? a : b; }

/// Phase 1 of a product for thread h: own[q] = (D x_i) rows 4h + q (exact
/// folds) and hs[q] = hand-over rows 4(1 - h) + q (the second halves of
/// hand_r = sum_c W(r, c) x_i[c]), given hf[q] = the first halves of rows
/// 4h + q this thread folded. One 12-round partner exchange serves both.
__device__ __forceinline__ void phase1_fold(const SymP& m, const double* xf, int h, const double* hf,
                                            const double (&g)[4][4], double* own, double* hs) {
  auto T = [&](int a, int b) { return a <= b ? m.t[h8s::tri(a, b)] : m.t[h8s::tri(b, a)]; };
  // products D01(a, j) x: thread 0 -> (rows 0, 1: columns 0, 1 of rows 4 + j),
  // thread 1 -> rows 2, 3 of D01 times x[4 + j] (thread 0's rows 2, 3)
  double A[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) A[k] = m.s[k >> 2][k & 3] * (h ? xf[4 + (k & 3)] : xf[k >> 2]);
  double recv[12];
#pragma unroll
  for (int k = 0; k < 12; ++k) {
    double snd;
    if (k < 4) snd = h ? A[k] : A[k] + A[4 + k];  // t0: D(4+k, 0) x0 + D(4+k, 1) x1
    else if (k < 8) snd = h ? A[k] : hf[k - 4];
    else snd = h ? hf[k - 8] : 0.0;
    recv[k] = __shfl_xor_sync(0xffffffffu, snd, 1);
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    // t0 row q: sum_c<4 D00(q, c) x_c, then D01(q, .) x_{4..7};
    // t1 row 4 + q: (t0's two-term partial) + D01(2, q) x2 + D01(3, q) x3, then D11(q, .) x_{4..7}
    double acc = h ? recv[q] : T(q, 0) * xf[0] + T(q, 1) * xf[1];
    acc = acc + sel(h, m.s[0][q], T(q, 2)) * xf[2];
    acc = acc + sel(h, m.s[1][q], T(q, 3)) * xf[3];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double term;
      if (q < 2) term = sel(h, T(q, j), m.s[q][j]) * xf[4 + j];
      else term = h ? T(q, j) * xf[4 + j] : recv[(q - 2) * 4 + j];
      acc = acc + term;
    }
    own[q] = acc;
  }
  // hand-over second halves: partner's first half + W(., 4..7) x_{4..7}
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    double acc = h ? recv[4 + q] : recv[8 + q];
#pragma unroll
    for (int c = 0; c < 4; ++c) acc = acc + g[q][c] * xf[4 + c];
    hs[q] = acc;
  }
}

/// First halves hf[q] = sum_{c < 4} f[q][c] x[c] (left fold).
__device__ __forceinline__ void first_halves(const double (&f)[4][4], const double* xf, double* hf) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    double acc = f[q][0] * xf[0];
#pragma unroll
    for (int c = 1; c < 4; ++c) acc = acc + f[q][c] * xf[c];
    hf[q] = acc;
  }
}

/// Phase 2: up[q] = sum_c W(c, 4h + q) x_{i+1}[c] given the coefficient
/// quarters c1[c][q] (first half, outputs this thread starts: 4h + q) and
/// c2[c][q] (second half, outputs 4(1 - h) + q it finishes).
template <class C1, class C2>
__device__ __forceinline__ void up_fold(C1 c1, C2 c2, const double* xn, double* up) {
  double u[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    double acc = c1(0, q) * xn[0];
#pragma unroll
    for (int c = 1; c < 4; ++c) acc = acc + c1(c, q) * xn[c];
    u[q] = acc;
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    double acc = __shfl_xor_sync(0xffffffffu, u[q], 1);
#pragma unroll
    for (int c = 0; c < 4; ++c) acc = acc + c2(c, q) * xn[4 + c];
    u[q] = acc;
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) up[q] = __shfl_xor_sync(0xffffffffu, u[q], 1);
}

}  // namespace h8p

/// Dynamic shared memory of pcg_kernel_h8p (doubles): as h8s, plus the block
/// dots (nb, even) and nothing else; the rare eta < 0 path folds the norms
/// in the vector buffers.
/// Block-dot slots: nb rounded up to 16, plus two blocks of 16, all past nb
/// zero (the fold warp reads whole 16-blocks one block ahead, unguarded).
__host__ __device__ inline long h8p_seg_doubles(int nb) { return ((nb + 15) & ~15) + 32; }

template <bool PREFETCH>
__host__ __device__ inline long h8p_smem_doubles(const Dims& d) {
  return (PREFETCH ? 4L : 2L) * d.nb * 64 + 2L * (d.nb + 2) * 8 + h8p_seg_doubles(d.nb);
}

#ifdef DOCP_H8P_CLOCK
// phase timing of thread 0 (A/B builds only: nvcc -DDOCP_H8P_CLOCK)
__device__ unsigned long long g_h8p_clk[16];
#define H8P_CLK(k)                        \
  if (tid == 0) {                         \
    const long long t_ = clock64();       \
    clk[k] += t_ - t_last;                \
    t_last = t_;                          \
  }
#else
#define H8P_CLK(k)
#endif

/// CW: a CTA whose last warp holds no block rows (T <= 111; launched with the
/// rows' warps plus that one, so short horizons run fewer warps) folds
/// the block dots there (one extra barrier per dot, the fold from registers).
constexpr int CW_WARP = 7;  // at most 7 warps of block rows (T <= 111), the fold warp after them
/// SDS: -S_ii stays in shared memory for the solve (a fourth region instead
/// of the next problem's prefetch): the (-S) diagonal product reads full rows
/// there (no partner exchange, no packed share in registers), at the price of
/// exposing the record load at each problem's start.
template <int MAXT, bool PREFETCH, bool CW = false, bool SDS = false>
__device__ __forceinline__ void h8p_body(View v, const int* __restrict__ work, const int* __restrict__ n_work,
                                         int* __restrict__ counter, double* __restrict__ sol_all, double epsilon,
                                         int max_iters_cfg) {
  extern __shared__ __align__(128) double sm_pcg[];
  __shared__ __align__(8) uint64_t s_bar[2];  // [0]: staged -S blocks, [1]: Phi^-1 blocks
  __shared__ int s_next, s_pidx;
  __shared__ double s_dot;
  const Dims d = v.d;
  const int nl = d.nl, nb = d.nb;
  const int tid = threadIdx.x;
  const int R = nb;
  const int il = tid >> 1, h = tid & 1;
  const int i = il;
  const bool act = i < nb;
  const bool has_next = act && i + 1 < nb;
  const bool has_prev = i > 0;
  const int lane = tid & 31, warp = tid >> 5;
  const int nwk = *n_work;
#ifdef DOCP_H8P_CLOCK
  long long clk[12] = {0}, t_last = clock64();
#endif

  static_assert(!(SDS && PREFETCH), "SDS keeps -S of the current problem where the prefetch would land");
  double* sPd = SDS ? sm_pcg + 2 * R * 64 : sm_pcg;  // [R] Phi^-1 diagonal blocks
  double* sPu = sPd + R * 64;                        // [R] Phi^-1 super blocks
  double* sNd = SDS ? sm_pcg : (PREFETCH ? sPu + R * 64 : sPd);  // -S diagonal blocks (staging, or resident: SDS)
  double* sNs = sNd + R * 64;
  double* vbuf = (SDS || PREFETCH) ? sm_pcg + 4 * R * 64 : sPu + R * 64;  // [R + 2] x_i (slot = row + 1)
  double* xbuf = vbuf + (R + 2) * 8;                 // [R + 2] hand-overs
  double* seg = xbuf + (R + 2) * 8;                  // [h8p_seg_doubles] block dots, zero past nb

  const int ib = act ? il : nb - 1;
  const int io = has_next ? il : 0;
  const double* PuI = sPu + io * 64;
  auto voff = [](int j, int k) { return j * 8 + 2 * (k ^ ((j >> 1) & 3)); };
  const int sv = ib + 1;
  const int my0 = voff(sv, 2 * h), my1 = voff(sv, 2 * h + 1);                // my half of row i
  const int ho0 = voff(sv + 1, 2 * (1 - h)), ho1 = voff(sv + 1, 2 * (1 - h) + 1);  // hand-over I write (row i+1)
  const int nf0 = voff(sv + 1, 0), nf1 = voff(sv + 1, 1), nf2 = voff(sv + 1, 2), nf3 = voff(sv + 1, 3);
  const uint32_t bd = static_cast<uint32_t>(nb) * 512u, bo = static_cast<uint32_t>(nb - 1) * 512u;
  // U_i chunk offsets: within each access family only the column's low two
  // bits (q or c) and the row pair j vary, and blk_off (common.cuh) maps them
  // to disjoint bit fields, so offset = base ^ (8 q + 2 j) with one base per
  // family: phase 1 rows 2j.. of column 4h + q (bf) and rows 4 + 2j.. of
  // column 4(1-h) + q (bg); phase 2 rows 4h + 2j.. of column c (b1) and rows
  // 4(1-h) + 2j.. of column 4 + c (b2)
  const int bf = blk_off(8, io, 0, 4 * h), bg = blk_off(8, io, 4, 4 * (1 - h));
  const int b1 = blk_off(8, io, 4 * h, 0), b2 = blk_off(8, io, 4 * (1 - h), 4);
  // Phi^-1_ii: column 4h + q, rows 2k.. at bdg ^ (8 q + 2 k) (same identity, block ib)
  const double* PdI = sPd + ib * 64;
  const double* SdI = sNd + ib * 64;  // SDS: -S_ii resident (same tile offsets as Phi^-1_ii)
  const int bdg = blk_off(8, ib, 0, 4 * h);
  auto grab = [&]() {
    const int w = atomicAdd(counter, 1);
    s_next = w;
    s_pidx = w < nwk ? work[w] : 0;
  };
  auto stage_s = [&](int pi) {
    const double* rec = v.blocks + static_cast<long>(pi) * d.blk_stride;
    mbar_arrive_expect_tx(&s_bar[0], bd + bo);
    tma_bulk_g2s(sNd, rec + d.s_diag, bd, &s_bar[0]);
    if (bo) tma_bulk_g2s(sNs, rec + d.s_sub, bo, &s_bar[0]);
  };

  for (int k = nb + tid; k < h8p_seg_doubles(nb); k += blockDim.x) seg[k] = 0.0;
  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    grab();
    if (PREFETCH && s_next < nwk) stage_s(s_pidx);
  }
  __syncthreads();
  uint32_t phase = 0, ph1 = 0;
  const int max_iters = max_iters_cfg > 0 ? max_iters_cfg : 2 * nl;
  const double threshold = epsilon * epsilon;

  auto gather = [&](const double* xr, double* xf) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double o = __shfl_xor_sync(0xffffffffu, xr[q], 1);
      xf[q] = h ? o : xr[q];
      xf[4 + q] = h ? xr[q] : o;
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
  auto finish = [&](const double* own, const double* low, const double* up, double* out) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {  // diag, then sub (i > 0), then super (i < nb - 1): btd_matvec's order
      double acc = own[q];
      acc = has_prev ? acc + low[q] : acc;
      acc = has_next ? acc + up[q] : acc;
      out[q] = acc;
    }
  };
  // The block dots in index order from 0.0 (pcg.hpp:37-44), by one lane:
  // whole blocks of 16, zero-padded at the end in shared memory (exact: a
  // fold seeded with +0.0 is never -0.0, so acc + 0.0 = acc), two LDS.128 per
  // four entries, one block loaded ahead: no predicate, select or branch
  // inside a block of the dependent chain (a per-group exit test costs more
  // than the padding adds)
  auto fold_seg = [&]() -> double {
    const double2* sg = reinterpret_cast<const double2*>(seg);
    const int nblk = (nb + 15) >> 4;
    double2 A[8], Bv[8];
    double acc = 0.0;
#pragma unroll
    for (int t = 0; t < 8; ++t) A[t] = sg[t];
    for (int k = 0; k < nblk; k += 2) {
#pragma unroll
      for (int t = 0; t < 8; ++t) Bv[t] = sg[8 * (k + 1) + t];
#pragma unroll
      for (int t = 0; t < 8; ++t) acc = (acc + A[t].x) + A[t].y;
      if (k + 1 >= nblk) break;
#pragma unroll
      for (int t = 0; t < 8; ++t) A[t] = sg[8 * (k + 2) + t];
#pragma unroll
      for (int t = 0; t < 8; ++t) acc = (acc + Bv[t].x) + Bv[t].y;
    }
    return acc;
  };
  // block_dot (pcg.hpp:37-44): the 8-term fold of block i is cut after its
  // 4th term (thread 0 -> thread 1); the block dots are then folded by the
  // spare warp's lane 0 (CW) or by lane 0 of every warp (no second barrier)
  auto dot = [&](const double* a, const double* b) -> double {
    double s = a[0] * b[0];
    s = s + a[1] * b[1];
    s = s + a[2] * b[2];
    s = s + a[3] * b[3];
    const double lo = __shfl_xor_sync(0xffffffffu, s, 1);
    double t = lo + a[0] * b[0];
    t = t + a[1] * b[1];
    t = t + a[2] * b[2];
    t = t + a[3] * b[3];
    if (act && h) seg[i] = t;
    H8P_CLK(6);
    __syncthreads();
    H8P_CLK(7);
    if constexpr (CW) {
      // warp 7 holds no block rows: its lane 0 folds the block dots with all
      // of them in flight at once (its registers are free), the others wait
      if (warp == static_cast<int>(blockDim.x >> 5) - 1) {  // the last warp holds no block rows
        if (lane == 0) {
#ifdef DOCP_H8P_CLOCK
          const long long tc0 = clock64();
#endif
          const double acc = fold_seg();
          s_dot = acc;
#ifdef DOCP_H8P_CLOCK
          atomicAdd(&g_h8p_clk[12], static_cast<unsigned long long>(clock64() - tc0));
          atomicAdd(&g_h8p_clk[13], 1ull);
#endif
        }
      }
      __syncthreads();
      const double tot = s_dot;
      H8P_CLK(8);
      return tot;
    }
    double acc = 0.0;
    if (lane == 0) {
      acc = fold_seg();
    }
    const double tot = __shfl_sync(0xffffffffu, acc, 0);
    H8P_CLK(8);
    return tot;
  };
  // ||a|| as the reference's eta guard computes it (Vector::norm: the squares
  // folded over the whole vector in index order, seeded with the first);
  // only on the rare eta < 0 path; uses the vector buffers as scratch
  auto norm = [&](const double* a) -> double {
    __syncthreads();
    if (act)
#pragma unroll
      for (int q = 0; q < 4; ++q) vbuf[i * 8 + 4 * h + q] = a[q] * a[q];
    __syncthreads();
    double acc = 0.0;
    if (lane == 0) {
      acc = vbuf[0];
      for (int k = 1; k < nl; ++k) acc = acc + vbuf[k];
    }
    acc = __shfl_sync(0xffffffffu, acc, 0);
    __syncthreads();
    return sqrt(acc);
  };

  h8p::SymP sd;      // -S_ii share, resident for the whole solve (Phi^-1_ii is read from shared memory)
  h8p::Quarters lq;  // quarters of L_i

  for (;;) {
    const int w = s_next;
    if (w >= nwk) break;
    const int pidx = s_pidx;
    const double* gam = v.gamma + static_cast<long>(pidx) * nl;
    double* sol = sol_all + static_cast<long>(pidx) * nl;
    double2 l01 = make_double2(0.0, 0.0), l23 = l01, g01 = l01, g23 = l01;
    if (act) {
      l01 = *reinterpret_cast<const double2*>(sol + i * 8 + 4 * h);
      l23 = *reinterpret_cast<const double2*>(sol + i * 8 + 4 * h + 2);
      g01 = *reinterpret_cast<const double2*>(gam + i * 8 + 4 * h);
      g23 = *reinterpret_cast<const double2*>(gam + i * 8 + 4 * h + 2);
    }
    const bool runnable = v.status[pidx].code == DOCP_OK;
    if constexpr (!PREFETCH) {
      if (!runnable) {
        __syncthreads();
        if (tid == 0) grab();
        __syncthreads();
        continue;
      }
      if (tid == 0) {
        fence_proxy_async();
        stage_s(pidx);
        if constexpr (SDS) {  // Phi^-1 has its own regions: load it now too
          const double* rec = v.blocks + static_cast<long>(pidx) * d.blk_stride;
          mbar_arrive_expect_tx(&s_bar[1], bd + bo);
          tma_bulk_g2s(sPd, rec + d.p_diag, bd, &s_bar[1]);
          if (bo) tma_bulk_g2s(sPu, rec + d.p_sup, bo, &s_bar[1]);
        }
      }
    }
    mbar_wait(&s_bar[0], phase);
    if constexpr (!SDS) h8p::load_symp(sNd + ib * 64, ib, h, sd);
    h8p::load_quarters(sNs + io * 64, io, h, lq);
    __syncthreads();  // staging area consumed; s_next / s_pidx read; previous Phi^-1 reads done
    phase ^= 1;
    if constexpr (PREFETCH) {
      if (!runnable) {
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
      if constexpr (!SDS) {
        fence_proxy_async();
        const double* rec = v.blocks + static_cast<long>(pidx) * d.blk_stride;
        mbar_arrive_expect_tx(&s_bar[1], bd + bo);
        tma_bulk_g2s(sPd, rec + d.p_diag, bd, &s_bar[1]);
        if (bo) tma_bulk_g2s(sPu, rec + d.p_sup, bo, &s_bar[1]);
      }
      grab();
      if (PREFETCH && s_next < nwk) stage_s(s_pidx);
    }

    // lambda lives in its global row (sol, L1/L2-resident) between updates:
    // lambda += alpha p is off the critical path, and registers are the
    // binding resource of this kernel
    double r[4], pv[4], y[4], rt[4];
    double2* lam_g = reinterpret_cast<double2*>(sol + ib * 8 + 4 * h);

    // y = (-S) x: L_i's quarters in registers
    auto matvec_s = [&](const double* xr, double* out) {
      double xf[8], own[4], hf[4], hs[4], low[4], up[4], xn[8];
      gather(xr, xf);
      put(vbuf, my0, my1, xr);
      h8p::first_halves(lq.f, xf, hf);
      if constexpr (SDS) {
        // own rows of -S_ii x from shared memory (row 4h + q = column 4h + q): full folds
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          double col[8];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const double2 a = *reinterpret_cast<const double2*>(SdI + (bdg ^ (8 * q + 2 * k)));
            col[2 * k] = a.x, col[2 * k + 1] = a.y;
          }
          double acc = col[0] * xf[0];
#pragma unroll
          for (int c = 1; c < 8; ++c) acc = acc + col[c] * xf[c];
          own[q] = acc;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {  // hand-over second halves after the partner's first halves
          double acc = __shfl_xor_sync(0xffffffffu, hf[q], 1);
#pragma unroll
          for (int c = 0; c < 4; ++c) acc = acc + lq.g[q][c] * xf[4 + c];
          hs[q] = acc;
        }
      } else {
        h8p::phase1_fold(sd, xf, h, hf, lq.g, own, hs);
      }
      put(xbuf, ho0, ho1, hs);
      H8P_CLK(0);
      __syncthreads();
      H8P_CLK(1);
      get(vbuf, nf0, nf1, xn);
      get(vbuf, nf2, nf3, xn + 4);
      {
        // up: outputs 4h + q start with W(c<4, 4h + q) (t0: f[c][q], t1: g[c][q])
        // and outputs 4(1-h) + q end with W(4 + c, 4(1-h) + q) (t0: g[c][q], t1: f[c][q])
        h8p::up_fold([&](int c, int q) { return h8p::sel(h, lq.g[c][q], lq.f[c][q]); },
                     [&](int c, int q) { return h8p::sel(h, lq.f[c][q], lq.g[c][q]); }, xn, up);
      }
      get(xbuf, my0, my1, low);
      finish(own, low, up, out);
    };
    // y = Phi^-1 x: U_i read from shared memory (W = U_i')
    // y = Phi^-1 x: the diagonal rows and U_i from shared memory (W = U_i'),
    // U_i's two quarters read ONCE per product: phase 1 exchanges x, then
    // both the hand-over (W's rows) and the super term (W's columns) are
    // folded from the same registers, and a second barrier hands the
    // hand-over on (each thread's quarters serve the hand-over's first and
    // second halves as f, g, and the super term's as f, g for h = 0 and as
    // g, f for h = 1).
    auto matvec_p = [&](const double* xr, double* out) {
      double xf[8], own[4], hs[4], low[4], up[4];
      gather(xr, xf);
      put(vbuf, my0, my1, xr);
      // own rows of Phi^-1_ii x (row 4h + q = column 4h + q, symmetric): full folds
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        double col[8];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const double2 a = *reinterpret_cast<const double2*>(PdI + (bdg ^ (8 * q + 2 * k)));
          col[2 * k] = a.x, col[2 * k + 1] = a.y;
        }
        double acc = col[0] * xf[0];
#pragma unroll
        for (int c = 1; c < 8; ++c) acc = acc + col[c] * xf[c];
        own[q] = acc;
      }
      H8P_CLK(4);
      __syncthreads();  // x_{i+1} published
      H8P_CLK(1);
      {
        double f[4][4], g[4][4];  // f[q][c] = U(c, 4h + q), g[q][c] = U(4 + c, 4(1-h) + q)
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const double2 a = *reinterpret_cast<const double2*>(PuI + (bf ^ (8 * q + 2 * j)));
            f[q][2 * j] = a.x, f[q][2 * j + 1] = a.y;
            const double2 b = *reinterpret_cast<const double2*>(PuI + (bg ^ (8 * q + 2 * j)));
            g[q][2 * j] = b.x, g[q][2 * j + 1] = b.y;
          }
        double hf[4];
        h8p::first_halves(f, xf, hf);
#pragma unroll
        for (int q = 0; q < 4; ++q) {  // hand-over second halves after the partner's first halves
          double acc = __shfl_xor_sync(0xffffffffu, hf[q], 1);
#pragma unroll
          for (int c = 0; c < 4; ++c) acc = acc + g[q][c] * xf[4 + c];
          hs[q] = acc;
        }
        double xn[8];
        get(vbuf, nf0, nf1, xn);
        get(vbuf, nf2, nf3, xn + 4);
        // up_r = sum_c U(r, c) x_{i+1}[c]: first halves from U(4h + q, c < 4), second from U(4(1-h) + q, 4 + c)
        h8p::up_fold([&](int c, int q) { return h8p::sel(h, g[c][q], f[c][q]); },
                     [&](int c, int q) { return h8p::sel(h, f[c][q], g[c][q]); }, xn, up);
      }
      put(xbuf, ho0, ho1, hs);
      __syncthreads();  // hand-overs published
      get(xbuf, my0, my1, low);
      finish(own, low, up, out);
    };

    {
      const double lam0[4] = {l01.x, l01.y, l23.x, l23.y};
      matvec_s(lam0, y);  // y = (-S) lambda0
    }
    if (act) {
      r[0] = g01.x - y[0], r[1] = g01.y - y[1], r[2] = g23.x - y[2], r[3] = g23.y - y[3];
    } else {
      r[0] = r[1] = r[2] = r[3] = 0.0;
    }
    __syncthreads();  // every phase-2 read of lambda / its hand-over is done
    mbar_wait(&s_bar[1], ph1);
    ph1 ^= 1;
    matvec_p(r, rt);  // r~ = Phi^-1 r
    double eta = dot(r, rt);
    int status = DOCP_OK, iters = 0;
    if (eta < 0.0) {
      const double scale = norm(r) * norm(rt);
      if (-eta <= 1e-10 * scale + 1e-300) eta = 0.0;
      else status = DOCP_AT_PCG_PRECOND;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) pv[q] = rt[q];

    H8P_CLK(11);
    while (status == DOCP_OK && eta > threshold && iters < max_iters) {
      H8P_CLK(9);
      matvec_s(pv, y);
      H8P_CLK(2);
      // this row's lambda, in flight while the dot reduces
      const double2 la = lam_g[0], lb = lam_g[1];
      const double vv = dot(pv, y);
      if (vv <= 0.0) {
        status = DOCP_AT_PCG_CURVATURE;
        break;
      }
      const double alpha = eta / vv;
      if (act) {
        lam_g[0] = make_double2(la.x + alpha * pv[0], la.y + alpha * pv[1]);
        lam_g[1] = make_double2(lb.x + alpha * pv[2], lb.y + alpha * pv[3]);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) r[q] = r[q] - alpha * y[q];
      H8P_CLK(9);
      matvec_p(r, rt);
      H8P_CLK(3);
      double eta_next = dot(r, rt);
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
      for (int q = 0; q < 4; ++q) pv[q] = rt[q] + beta * pv[q];
      eta = eta_next;
      ++iters;
    }

    H8P_CLK(10);
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
    __syncthreads();
  }
#ifdef DOCP_H8P_CLOCK
  if (tid == 0)
    for (int k = 0; k < 12; ++k) atomicAdd(&g_h8p_clk[k], static_cast<unsigned long long>(clk[k]));
#endif
}

template <int MAXT, bool PREFETCH, bool CW = false, bool SDS = false>
__global__ void __launch_bounds__(MAXT, 1) pcg_kernel_h8p(View v, const int* __restrict__ work,
                                                        const int* __restrict__ n_work, int* __restrict__ counter,
                                                        double* __restrict__ sol_all, double epsilon,
                                                        int max_iters_cfg) {
  h8p_body<MAXT, PREFETCH, CW, SDS>(v, work, n_work, counter, sol_all, epsilon, max_iters_cfg);
}

}  // namespace docp_dev
