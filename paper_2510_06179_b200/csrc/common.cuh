// common.cuh — shared definitions of the B200 DiffMPC hot path.
//
// Arithmetic: the library is compiled with --fmad=false, so a*b+c is a
// rounded multiply followed by a rounded add — the operation order of the
// reference (eigen_lite convention). The FAST PCG mode opts
// back into fused multiply-adds explicitly with fma().
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "docp_cuda.h"

namespace docp_dev {

constexpr int kMaxNx = 16;
constexpr int kMaxNu = 16;
constexpr int kWarp = 32;
constexpr int kPcgMaxThreads = 256;  // K2: one thread per block row (MAXB block rows per thread beyond)

/// Problem dimensions and per-problem strides (in doubles) of every field.
struct Dims {
  int nx, nu, T;
  int nl;   // n_x (T+1)
  int nz;   // n_x (T+1) + n_u T
  int nth;  // theta size
  int nb;   // T + 1 blocks
  int bsz;  // n_x * n_x
  // block region offsets inside one problem's block record (doubles)
  long s_diag, s_sub, p_diag, p_sup, blk_stride;
  // stage Jacobian storage A_t [nx*nx], B_t [nx*nu]: families whose Jacobians
  // do not depend on t or z (affine-quadratic: A_t = -A, B_t = -B) keep one
  // copy per problem (stride 0 over t)
  long a_per, a_stride, b_per, b_stride;
};

/// A_t / B_t of problem p (column-major).
__host__ __device__ inline long a_off(const Dims& d, int p, int t) { return p * d.a_per + t * d.a_stride; }
__host__ __device__ inline long b_off(const Dims& d, int p, int t) { return p * d.b_per + t * d.b_stride; }

__host__ __device__ inline int xoff(const Dims& d, int t) { return t * (d.nx + d.nu); }  // trajectory.hpp:72-74
__host__ __device__ inline int uoff(const Dims& d, int t) { return t * (d.nx + d.nu) + d.nx; }

/// Device block layout (DESIGN.md §HBM layout). A block is stored column
/// by column (physical column s', NX doubles each); the 16-byte chunks of a
/// column and the columns are permuted per block index b so that the PCG
/// kernels' shared-memory reads are bank-conflict free (each quarter-warp
/// LDS.128 touches 8 distinct 4-bank groups):
///   NX = 8: s' = s ^ (b & 1),   chunk' = chunk ^ ((b >> 1) & 1) ^ (2 * ((s >> 2) & 1))
///           (pcg_kernel_h8: two threads per block row reading row halves
///            (chunks 2h, 2h+1 of every column) or column halves)
///   NX = 4: s' = s ^ (b & 3),   chunk' = chunk ^ ((b >> 2) & 1)
///           (pcg_kernel: one thread per block row)
///   NX = 16: chunk' = chunk ^ (b & 1)
///           (pcg_kernel_h16f: four threads per block row, rows 4q..4q+3)
///   other : plain column-major.
__host__ __device__ inline int blk_off(int nx, int b, int e, int s) {
  if (nx == 8) {
    const int sp = s ^ (b & 1);
    const int ch = (e >> 1) ^ ((b >> 1) & 1) ^ (((s >> 2) & 1) << 1);
    return sp * 8 + ((ch << 1) | (e & 1));
  }
  if (nx == 4) {
    const int sp = s ^ (b & 3);
    return sp * 4 + ((((e >> 1) ^ ((b >> 2) & 1)) << 1) | (e & 1));
  }
  if (nx == 16) return s * 16 + ((((e >> 1) ^ (b & 1)) << 1) | (e & 1));
  return s * nx + e;
}

/// Inverse of blk_off: the entry (e, s) stored at offset o of block b.
__host__ __device__ inline void blk_entry(int nx, int b, int o, int* e, int* s) {
  if (nx == 8) {
    const int ss = (o >> 3) ^ (b & 1);
    const int ch = ((o >> 1) & 3) ^ ((b >> 1) & 1) ^ (((ss >> 2) & 1) << 1);
    *s = ss;
    *e = (ch << 1) | (o & 1);
    return;
  }
  if (nx == 4) {
    *s = (o >> 2) ^ (b & 3);
    *e = ((((o >> 1) & 1) ^ ((b >> 2) & 1)) << 1) | (o & 1);
    return;
  }
  if (nx == 16) {
    *s = o >> 4;
    *e = ((((o >> 1) & 7) ^ (b & 1)) << 1) | (o & 1);
    return;
  }
  *s = o / nx;
  *e = o % nx;
}

/// Iterate-vector layout in shared memory (block j, entry e): conflict-free
/// LDS.128/STS.128 by 8 consecutive block rows.
__host__ __device__ inline int vec_off(int nx, int j, int e) {
  if (nx == 8) return j * 8 + ((((e >> 1) ^ ((j >> 1) & 3)) << 1) | (e & 1));
  if (nx == 4) return j * 4 + ((((e >> 1) ^ ((j >> 2) & 1)) << 1) | (e & 1));
  if (nx == 16) return j * 16 + ((((e >> 1) ^ (j & 1)) << 1) | (e & 1));
  return j * nx + e;
}

inline Dims make_dims(const docp_problem& p) {
  Dims d;
  d.nx = p.n_x;
  d.nu = p.n_u;
  d.T = p.horizon;
  d.nl = d.nx * (d.T + 1);
  d.nz = d.nl + d.nu * d.T;
  d.nth = p.family == DOCP_DRIFT        ? 36  // docp_drift::NTH
          : p.family == DOCP_CARTPOLE    ? 9
          : p.family == DOCP_ATTITUDE ? 12  // reference 9 + the instance inertia
                                      : d.nx + d.nu + d.nx * d.nx + d.nx * d.nu + 2 * d.nx;
  d.nb = d.T + 1;
  d.bsz = d.nx * d.nx;
  auto up2 = [](long n) { return (n + 1) & ~1L; };  // 16-byte multiples for bulk copies
  long diag = up2(static_cast<long>(d.nb) * d.bsz), off = up2(static_cast<long>(d.T) * d.bsz);
  d.s_diag = 0;
  d.s_sub = d.s_diag + diag;
  d.p_diag = d.s_sub + off;
  d.p_sup = d.p_diag + diag;
  d.blk_stride = (d.p_sup + off + 31) & ~31L;  // 256-byte aligned records
  const bool tv = p.family != DOCP_AFFINE_QUADRATIC;
  d.a_stride = tv ? d.bsz : 0;
  d.b_stride = tv ? static_cast<long>(d.nx) * d.nu : 0;
  d.a_per = tv ? static_cast<long>(d.T) * d.bsz : d.bsz;
  d.b_per = tv ? static_cast<long>(d.T) * d.nx * d.nu : static_cast<long>(d.nx) * d.nu;
  return d;
}

/// Everything a kernel needs about a resident batch, passed by value.
struct View {
  Dims d;
  int B;
  docp_problem prob;
  double *theta, *z, *lam, *lt, *lgz, *grad, *gamma, *zqp;
  // QpData: diagonal Hessians (every family's Hessian is diagonal; problem.hpp:157-181)
  double *qd, *lq, *q;      // [B][T+1][nx]  projected Q diag, its Cholesky diag, gradient q
  double *rd, *lr, *r;      // [B][T][nu]
  double *A, *Bm, *C, *xs;  // [B][T][nx*nx], [B][T][nx*nu] col-major, [B][T][nx], [B][nx]
  double* blocks;           // [B][blk_stride] device block layout
  docp_status* status;
  int *sqp_iters, *converged, *pcg_iters, *pcg_conv, *pcg_hist, *pd_proj, *accepted;
  double *kkt, *final_eta, *step_sizes, *mu, *alpha, *loss;
  unsigned long long* pcg_acc;  // [0] iterations, [1] solves (roofline accounting), [2] lifetime solves
  int max_hist;
};

/// Rollout record of one batch: every step's solution (for the backward
/// re-linearisation), the chained states and controls, per-instance flags.
struct RolloutRec {
  double *z, *lam;     // [H][B][n_z], [H][B][n_lambda]
  double *x, *u;       // [H+1][B][n_x], [H][B][n_u]
  double *xbar, *ex;   // [B][n_x] backward state cotangent, env VJP in x
  double *gtot;        // [B][n_theta] accumulated gradient
  double* reward;      // [B]
  int* alive;          // [B] rollout (and then backward) still running
  docp_status* rstat;  // [B] first truncation
  int H;
};

// ------------------------------------------------------------ status helpers
__device__ inline void set_status(docp_status* st, int code, int where, int index) {
  st->code = code;
  st->where = where;
  st->index = index;
  st->step = 0;
}

// ------------------------------------------------------------ PTX wrappers
__device__ inline uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ inline void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ inline void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ inline void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "DOCP_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra DOCP_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

/// TMA bulk copy global -> shared (SASS UBLKCP); completion is counted on bar.
__device__ inline void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__device__ inline void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

/// Coalesced global -> shared staging by the whole CTA: src[e] goes to
/// dst[map(e)]. Each thread issues U loads before their stores, so U loads
/// are in flight per thread; a plain copy loop leaves one, since the
/// compiler cannot move a load above the previous store through the generic
/// shared-memory pointer.
template <int U = 8, class Map>
__device__ __forceinline__ void cta_stage(double* dst, const double* __restrict__ src, int n, Map map) {
  for (int e0 = threadIdx.x; e0 < n; e0 += U * blockDim.x) {
    double t[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int e = e0 + k * blockDim.x;
      t[k] = e < n ? src[e] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int e = e0 + k * blockDim.x;
      if (e < n) dst[map(e)] = t[k];
    }
  }
}
template <int U = 8>
__device__ __forceinline__ void cta_stage(double* dst, const double* __restrict__ src, int n) {
  cta_stage<U>(dst, src, n, [](int e) { return e; });
}

__device__ inline double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ inline double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

}  // namespace docp_dev
