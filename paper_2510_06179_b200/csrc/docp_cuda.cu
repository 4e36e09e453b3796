// docp_cuda.cu — host driver and C ABI (include/docp_cuda.h) of the
// B200-native DiffMPC hot path: a batch object holding every problem's state
// in HBM, the SQP loop (sqp.hpp:213-261) and the backward pass
// (backward.hpp:27-50) driven from C++, and the five kernels K1–K4 (+K5's
// reduction for the gradient sum; the NCCL exchange is done by the caller).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <mutex>
#include <set>

#include "batch.cuh"
#include "families.cuh"
#include "k_assemble.cuh"
#include "k_rollout.cuh"
#include "k_step.cuh"

using namespace docp_dev;
using namespace docp_host;

namespace docp_host {

thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};
// PCG solves are counted on the device (one per problem the kernel actually
// solves, pcg.hpp:57); docp_pcg_invocations sums the live batches' counters
// and those of destroyed batches.
std::mutex g_batches_mu;
std::set<docp_batch*> g_batches;
uint64_t g_retired_solves = 0;

uint64_t batch_solves(docp_batch* b) {
  unsigned long long n = 0;
  if (cudaStreamSynchronize(b->stream) != cudaSuccess) return 0;
  if (cudaMemcpy(&n, b->v.pcg_acc + 2, sizeof n, cudaMemcpyDeviceToHost) != cudaSuccess) return 0;
  return n;
}

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

}  // namespace docp_host

namespace {

template <class T>
int dalloc(docp_batch* b, T** out, size_t count) {
  void* p = nullptr;
  CUDA_TRY(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
  CUDA_TRY(cudaMemset(p, 0, std::max<size_t>(count, 1) * sizeof(T)));
  b->allocs.push_back(p);
  *out = static_cast<T*>(p);
  return DOCP_OK;
}

int ensure_hist(docp_batch* b, int n) {
  if (n <= b->max_hist) return DOCP_OK;
  int rc;
  ++b->layout_gen;
  if ((rc = dalloc(b, &b->v.pcg_hist, static_cast<size_t>(b->B) * n))) return rc;
  if ((rc = dalloc(b, &b->v.step_sizes, static_cast<size_t>(b->B) * n))) return rc;
  b->max_hist = n;
  b->v.max_hist = n;
  return DOCP_OK;
}

// ---------------------------------------------------------------- kernels of the driver
__global__ void init_solve_kernel(View v, int* __restrict__ list, int* __restrict__ count) {
  // one warp per problem: coalesced finiteness scan of z0 and lambda0 (sqp.hpp:217-224)
  const Dims d = v.d;
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < v.B; p += warps) {
    const double* z = v.z + static_cast<long>(p) * d.nz;
    const double* l = v.lam + static_cast<long>(p) * d.nl;
    bool fin = true;  // & (not &&): the loads are independent and stay in flight together
    for (int e = lane; e < d.nz; e += 32) fin &= static_cast<bool>(isfinite(z[e]));
    for (int e = lane; e < d.nl; e += 32) fin &= static_cast<bool>(isfinite(l[e]));
    fin = __all_sync(0xffffffffu, fin);
    if (lane == 0) {
      v.mu[p] = 1.0;
      v.sqp_iters[p] = 0;
      v.converged[p] = 0;
      v.kkt[p] = 0.0;
      if (fin) {
        set_status(v.status + p, DOCP_OK, DOCP_AT_NONE, 0);
        list[atomicAdd(count, 1)] = p;
      } else {
        set_status(v.status + p, DOCP_DIMENSION, DOCP_AT_INITIAL_GUESS, 0);
      }
    }
  }
}

/// Next active list: problems still OK and not converged (order is
/// irrelevant: problems are independent).
__global__ void compact_kernel(View v, const int* __restrict__ in, const int* __restrict__ n_in,
                               int* __restrict__ out, int* __restrict__ n_out) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < *n_in; k += gridDim.x * blockDim.x) {
    const int p = in[k];
    if (v.status[p].code == DOCP_OK && !v.converged[p]) out[atomicAdd(n_out, 1)] = p;
  }
}

/// Problems whose status is OK (the finalize / backward set).
__global__ void ok_list_kernel(View v, int* __restrict__ out, int* __restrict__ n_out) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < v.B; p += gridDim.x * blockDim.x)
    if (v.status[p].code == DOCP_OK) out[atomicAdd(n_out, 1)] = p;
}

__global__ void iota_kernel(int* out, int n, int* count) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) out[k] = k;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    count[0] = n;
    count[4] = 0;           // IL epochs: failed demonstrations since the last docp_il_failures
    count[5] = 0x7fffffff;  // ... and the first of them
  }
}

__global__ void reset_status_kernel(View v) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < v.B; p += gridDim.x * blockDim.x)
    set_status(v.status + p, DOCP_OK, DOCP_AT_NONE, 0);
}

// ---------------------------------------------------------------- launch helpers
template <int NX, int NU, int TH, bool DR = false>
int launch_assemble_th(docp_batch* b, const int* list, const int* count, int n_hint, double eps_pd, int do_schur,
                       bool fast) {
  constexpr int NG = TH / NX;
  // NG group buffers + the two-block P_t hand-off between rounds
  const size_t smem = (static_cast<size_t>(NG) * AsmLayout<NX, NU>::GBUF + 2 * AsmLayout<NX, NU>::P2) * sizeof(double);
  auto kern = fast ? assemble_kernel_t<NX, NU, TH, true, DR> : assemble_kernel_t<NX, NU, TH, false, DR>;
  if (do_schur) b->sym_blocks = true;
  CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int per_sm = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TH, smem));
  const int grid = std::max(1, std::min(n_hint, std::max(1, per_sm) * b->num_sms));
  ProfScope ps(b, DOCP_PROF_ASSEMBLE);
  kern<<<grid, TH, smem, b->stream>>>(b->v, list, count, eps_pd, do_schur);
  LAUNCH_CHECK();
  return DOCP_OK;
}

/// 128 threads: 16 groups of 8 lanes (n_x = 8). A 160-thread variant (whole
/// rounds at T = 100) measured 3% slower: occupancy fell from 16 to 15 warps/SM.
template <int NX, int NU, bool DR = false>
int launch_assemble_t(docp_batch* b, const int* list, const int* count, int n_hint, double eps_pd, int do_schur,
                      bool fast) {
  return launch_assemble_th<NX, NU, kAsmGroupThreads, DR>(b, list, count, n_hint, eps_pd, do_schur, fast);
}

/// K1. fast (PCG mode FAST): reciprocal / fma arithmetic in the compile-time
/// shapes (assemble_kernel_t<..., true>); the runtime-shape kernel is always
/// the reference's arithmetic.
int launch_assemble(docp_batch* b, const int* list, const int* count, int n_hint, double eps_pd, int do_schur,
                    bool fast = false) {
  const int nx = b->d.nx, nu = b->d.nu;
  // the drifting family runs its own instantiation (the model's dual-number
  // Jacobians need ~255 registers; the other families' kernels leave it out)
  if (b->prob.family == DOCP_DRIFT) {
    if (nx == 8 && nu == 2) return launch_assemble_t<8, 2, true>(b, list, count, n_hint, eps_pd, do_schur, fast);
  } else if (nx == 8 && nu == 4) {
    return launch_assemble_t<8, 4>(b, list, count, n_hint, eps_pd, do_schur, fast);
  }
  const bool shaped = b->prob.family != DOCP_DRIFT;
  if (shaped && nx == 8 && nu == 2) return launch_assemble_t<8, 2>(b, list, count, n_hint, eps_pd, do_schur, fast);
  if (nx == 4 && nu == 2) return launch_assemble_t<4, 2>(b, list, count, n_hint, eps_pd, do_schur, fast);
  if (nx == 4 && nu == 1) return launch_assemble_t<4, 1>(b, list, count, n_hint, eps_pd, do_schur, fast);
  if (nx == 16 && nu == 8) return launch_assemble_t<16, 8>(b, list, count, n_hint, eps_pd, do_schur, fast);
  const int sp = std::max(b->d.bsz, b->d.nx * b->d.nu);
  const size_t smem = static_cast<size_t>(kAsmWarps) * 6 * sp * sizeof(double);
  if (do_schur) b->sym_blocks = true;
  CUDA_TRY(cudaFuncSetAttribute(assemble_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  const int grid = std::max(1, std::min(n_hint, b->num_sms * 8));
  ProfScope ps(b, DOCP_PROF_ASSEMBLE);
  assemble_kernel<<<grid, kAsmThreads, smem, b->stream>>>(b->v, list, count, eps_pd, do_schur);
  LAUNCH_CHECK();
  return DOCP_OK;
}

/// One CTA per problem (grid-stride over the work list), the grid sized to
/// the resident CTAs of the whole GPU.
template <class K, class... A>
int launch_per_problem(docp_batch* b, K kern, int threads, size_t smem, int n_hint, A... args) {
  CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int per_sm = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
  if (per_sm < 1) return fail(DOCP_UNSUPPORTED, "kernel does not fit on an SM (smem %zu)", smem);
  kern<<<std::max(1, std::min(n_hint, per_sm * b->num_sms)), threads, smem, b->stream>>>(b->v, args...);
  LAUNCH_CHECK();
  return DOCP_OK;
}

/// Compile-time block sizes for the shipped configurations, runtime otherwise.
#define DOCP_DISPATCH_NXNU(nx, nu, CALL)                        \
  do {                                                          \
    if ((nx) == 8 && (nu) == 4) { constexpr int NX = 8, NU = 4; CALL; } \
    if ((nx) == 8 && (nu) == 2) { constexpr int NX = 8, NU = 2; CALL; } \
    if ((nx) == 4 && (nu) == 1) { constexpr int NX = 4, NU = 1; CALL; } \
    if ((nx) == 4 && (nu) == 2) { constexpr int NX = 4, NU = 2; CALL; } \
    { constexpr int NX = 0, NU = 0; CALL; }                     \
  } while (0)

int launch_gamma(docp_batch* b, const int* list, const int* count, int n_hint, int rhs) {
  ProfScope ps(b, DOCP_PROF_GAMMA);
  const size_t smem = (static_cast<size_t>(b->d.nb) * b->d.nx + static_cast<size_t>(b->d.T) * b->d.nu) * 8;
  DOCP_DISPATCH_NXNU(b->d.nx, b->d.nu,
                     return launch_per_problem(b, gamma_kernel<NX, NU>, 128, smem, n_hint, list, count, rhs));
}

int launch_recover(docp_batch* b, const int* list, const int* count, int n_hint, const double* lam, int rhs) {
  ProfScope ps(b, DOCP_PROF_RECOVER);
  const size_t smem = static_cast<size_t>(b->d.nl) * 8;
  DOCP_DISPATCH_NXNU(b->d.nx, b->d.nu,
                     return launch_per_problem(b, recover_kernel<NX, NU>, 128, smem, n_hint, list, count, lam, rhs));
}

int launch_vjp(docp_batch* b, const int* list, const int* count, int n_hint) {
  ProfScope ps(b, DOCP_PROF_VJP);
  size_t smem = (2 * static_cast<size_t>(b->d.nz) + 2 * static_cast<size_t>(b->d.nl)) * 8;
  const int staged = smem <= 96 * 1024;  // long horizons read the vectors in place
  if (!staged) smem = 0;
  DOCP_DISPATCH_NXNU(b->d.nx, b->d.nu,
                     return launch_per_problem(b, vjp_kernel<NX, NU>, 128, smem, n_hint, list, count, staged));
}

size_t pcg_smem(const Dims& d, bool resident) {
  auto up2 = [](long n) { return (n + 1) & ~1L; };
  long dbl = 3 * up2(d.nl) + up2(d.nb) + 64;  // vbuf, xbuf, products + block dots, reduction
  if (resident) dbl += d.blk_stride;
  return static_cast<size_t>(dbl) * sizeof(double);
}

PcgPlan plan_pcg(const docp_batch* b) {
  PcgPlan pl{};
  int max_optin = 0;
  cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, b->device);
  const size_t static_smem = 64;
  pl.resident = pcg_smem(b->d, true) + static_smem <= static_cast<size_t>(max_optin);
  pl.smem = pcg_smem(b->d, pl.resident);
  const int nb = b->d.nb;  // one thread per block row (MAXB block rows beyond 256)
  pl.threads = std::min(kPcgMaxThreads, (nb + 31) / 32 * 32);
  const int need = (nb + pl.threads - 1) / pl.threads;
  pl.maxr = need <= 1 ? 1 : need <= 2 ? 2 : 0;
  return pl;
}

int launch_pcg(docp_batch* b, const docp_pcg_config& cfg, const int* list, const int* count, int n_hint,
               double* sol) {
  if (!(cfg.epsilon > 0.0 && cfg.max_iters >= 0)) return fail(DOCP_DIMENSION, "pcg: invalid config");
  if (cfg.mode == DOCP_PCG_FP32) {
    if (b->d.nx != 8) return fail(DOCP_UNSUPPORTED, "pcg fp32 mode: n_x = 8 only (n_x = %d)", b->d.nx);
    return launch_pcg_fp32_nx8(b, list, count, n_hint, sol, cfg.epsilon, cfg.max_iters);
  }
  if (cfg.mode != DOCP_PCG_FAST && cfg.mode != DOCP_PCG_PARITY) return fail(DOCP_INVALID, "pcg: unknown mode %d", cfg.mode);
  const bool par = cfg.mode == DOCP_PCG_PARITY;
  const PcgPlan pl = plan_pcg(b);
  switch (b->d.nx) {
    case 4: return launch_pcg_nx4(b, pl, par, list, count, n_hint, sol, cfg.epsilon, cfg.max_iters);
    case 8: return launch_pcg_nx8(b, pl, par, list, count, n_hint, sol, cfg.epsilon, cfg.max_iters);
    case 16: return launch_pcg_nx16(b, pl, par, list, count, n_hint, sol, cfg.epsilon, cfg.max_iters);
    case 6: return launch_pcg_nx6(b, pl, par, list, count, n_hint, sol, cfg.epsilon, cfg.max_iters);
    case 9: return launch_pcg_nx9(b, pl, par, list, count, n_hint, sol, cfg.epsilon, cfg.max_iters);
    default: return launch_pcg_nxrt(b, pl, par, list, count, n_hint, sol, cfg.epsilon, cfg.max_iters);
  }
}

int launch_step(docp_batch* b, const docp_sqp_config& cfg, const int* list, const int* count, int n_hint, int iter,
                int is_loop) {
  StepCfg sc{};
  sc.n_alpha = cfg.n_step_candidates;
  for (int i = 0; i < sc.n_alpha; ++i) sc.alphas[i] = cfg.step_candidates[i];
  sc.eta_armijo = cfg.eta_armijo;
  sc.rho_penalty = cfg.rho_penalty;
  sc.mu_floor = cfg.mu_floor_denominator;
  sc.conv_tol = cfg.convergence_tol;
  sc.iter = iter;
  sc.max_iters = cfg.max_sqp_iters;
  sc.is_loop = is_loop;
  int max_optin = 0;
  CUDA_TRY(cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, b->device));
  const bool stage = (step_smem_doubles(b->d, sc.n_alpha, true) * sizeof(double) + 1024) <= static_cast<size_t>(max_optin);
  const size_t smem = static_cast<size_t>(step_smem_doubles(b->d, sc.n_alpha, stage)) * sizeof(double);
  if (smem + 1024 > static_cast<size_t>(max_optin)) return fail(DOCP_UNSUPPORTED, "line search: horizon too long");
  const int nx = b->d.nx, nu = b->d.nu;
  auto kern = stage ? step_kernel<0, 0, true> : step_kernel<0, 0, false>;
  if (b->prob.family == DOCP_DRIFT) {  // the drifting family's instantiation (Family::dynamics' DRIFT branch)
    if (nx == 8 && nu == 2) kern = stage ? step_kernel<8, 2, true, true> : step_kernel<8, 2, false, true>;
  } else if (nx == 8 && nu == 4) kern = stage ? step_kernel<8, 4, true> : step_kernel<8, 4, false>;
  else if (nx == 8 && nu == 2) kern = stage ? step_kernel<8, 2, true> : step_kernel<8, 2, false>;
  else if (nx == 4 && nu == 2) kern = step_kernel<4, 2, true>;
  else if (nx == 4 && nu == 1) kern = step_kernel<4, 1, true>;
  if (!stage && ((nx == 4 && nu == 2) || (nx == 4 && nu == 1))) kern = step_kernel<0, 0, false>;
  CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int per_sm = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kStepThreads, smem));
  const int grid = std::max(1, std::min(n_hint, std::max(1, per_sm) * b->num_sms));
  ProfScope ps(b, DOCP_PROF_STEP);
  kern<<<grid, kStepThreads, smem, b->stream>>>(b->v, list, count, sc);
  LAUNCH_CHECK();
  return DOCP_OK;
}

int launch_kkt(docp_batch* b, const int* list, const int* count, int n_hint) {
  const Dims& d = b->d;
  const size_t smem =
      static_cast<size_t>((d.T + 1) * (d.nx + d.nu + 1) + (d.T + 1) * (d.nx + 1) + d.nth) * sizeof(double);
  int max_optin = 0;
  CUDA_TRY(cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, b->device));
  if (smem + 1024 > static_cast<size_t>(max_optin)) return fail(DOCP_UNSUPPORTED, "kkt_residual: horizon too long");
  auto kern = kkt_kernel<0, 0>;
  const int nx = b->d.nx, nu = b->d.nu;
  if (b->prob.family == DOCP_DRIFT) {  // the drifting family's instantiation (Family::dynamics' DRIFT branch)
    if (nx == 8 && nu == 2) kern = kkt_kernel<8, 2, true>;
  } else if (nx == 8 && nu == 4) kern = kkt_kernel<8, 4>;
  else if (nx == 8 && nu == 2) kern = kkt_kernel<8, 2>;
  else if (nx == 4 && nu == 2) kern = kkt_kernel<4, 2>;
  else if (nx == 4 && nu == 1) kern = kkt_kernel<4, 1>;
  CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int per_sm = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kKktThreads, smem));
  const int grid = std::max(1, std::min(n_hint, std::max(1, per_sm) * b->num_sms));
  ProfScope ps(b, DOCP_PROF_KKT);
  kern<<<grid, kKktThreads, smem, b->stream>>>(b->v, list, count);
  LAUNCH_CHECK();
  return DOCP_OK;
}

int read_count(docp_batch* b, const int* dev_count, int* out) {
  CUDA_TRY(cudaMemcpyAsync(b->h_count, dev_count, sizeof(int), cudaMemcpyDeviceToHost, b->stream));
  CUDA_TRY(cudaStreamSynchronize(b->stream));
  *out = *b->h_count;
  return DOCP_OK;
}

int validate_sqp(const docp_sqp_config* cfg) {  // sqp.hpp:23-33
  if (!cfg) return fail(DOCP_INVALID, "null config");
  if (cfg->n_step_candidates < 1) return fail(DOCP_DIMENSION, "sqp: empty step candidate list");
  if (cfg->n_step_candidates > DOCP_MAX_STEP_CANDIDATES)
    return fail(DOCP_UNSUPPORTED, "sqp: at most %d step candidates", DOCP_MAX_STEP_CANDIDATES);
  for (int i = 0; i < cfg->n_step_candidates; ++i) {
    const double a = cfg->step_candidates[i];
    const bool in_range = a > 0.0 && a <= 1.0;
    const bool decreasing = i == 0 || a < cfg->step_candidates[i - 1];
    if (!(in_range && decreasing))
      return fail(DOCP_DIMENSION, "sqp: step candidates must be strictly decreasing in (0,1]");
  }
  if (!(cfg->eta_armijo > 0.0 && cfg->eta_armijo < 1.0)) return fail(DOCP_DIMENSION, "sqp: eta out of range");
  return DOCP_OK;
}

double* field_base(docp_batch* b, int f, size_t* per, size_t* elem) {
  const Dims& d = b->d;
  *elem = sizeof(double);
  switch (f) {
    case DOCP_F_THETA: *per = d.nth; return b->v.theta;
    case DOCP_F_Z: *per = d.nz; return b->v.z;
    case DOCP_F_LAMBDA: *per = d.nl; return b->v.lam;
    case DOCP_F_LAMBDA_TILDE: *per = d.nl; return b->v.lt;
    case DOCP_F_LOSS_GRAD_Z: *per = d.nz; return b->v.lgz;
    case DOCP_F_GRAD_THETA: *per = d.nth; return b->v.grad;
    case DOCP_F_GAMMA: *per = d.nl; return b->v.gamma;
    case DOCP_F_Z_QP: *per = d.nz; return b->v.zqp;
    case DOCP_F_KKT: *per = 1; return b->v.kkt;
    case DOCP_F_FINAL_ETA: *per = 1; return b->v.final_eta;
    case DOCP_F_STEP_SIZES: *per = b->max_hist; return b->v.step_sizes;
    case DOCP_F_MU: *per = 1; return b->v.mu;
    case DOCP_F_ALPHA: *per = 1; return b->v.alpha;
    case DOCP_F_LOSS: *per = 1; return b->v.loss;
    case DOCP_F_REWARD: *per = 1; return b->roll.reward;
    default: break;
  }
  *elem = sizeof(int);
  switch (f) {
    case DOCP_F_STATUS: *per = 1; *elem = sizeof(docp_status); return reinterpret_cast<double*>(b->v.status);
    case DOCP_F_ROLLOUT_STATUS:
      *per = 1;
      *elem = sizeof(docp_status);
      return reinterpret_cast<double*>(b->roll.rstat);
    case DOCP_F_SQP_ITERS: *per = 1; return reinterpret_cast<double*>(b->v.sqp_iters);
    case DOCP_F_CONVERGED: *per = 1; return reinterpret_cast<double*>(b->v.converged);
    case DOCP_F_PCG_ITERS: *per = 1; return reinterpret_cast<double*>(b->v.pcg_iters);
    case DOCP_F_PCG_CONVERGED: *per = 1; return reinterpret_cast<double*>(b->v.pcg_conv);
    case DOCP_F_PCG_HISTORY: *per = b->max_hist; return reinterpret_cast<double*>(b->v.pcg_hist);
    case DOCP_F_PD_PROJECTED: *per = 1; return reinterpret_cast<double*>(b->v.pd_proj);
    case DOCP_F_ACCEPTED: *per = 1; return reinterpret_cast<double*>(b->v.accepted);
    default: return nullptr;
  }
}

int check_problem(const docp_problem* p) {
  if (!p) return fail(DOCP_INVALID, "null problem");
  if (p->family != DOCP_AFFINE_QUADRATIC && p->family != DOCP_CARTPOLE && p->family != DOCP_ATTITUDE &&
      p->family != DOCP_DRIFT)
    return fail(DOCP_UNSUPPORTED, "unknown problem family %d", p->family);
  if (p->n_x < 1 || p->n_u < 1 || p->horizon < 1) return fail(DOCP_DIMENSION, "dimensions must be positive");
  if (p->n_x > kMaxNx || p->n_u > kMaxNu)
    return fail(DOCP_UNSUPPORTED, "n_x, n_u must be <= %d (got %d, %d)", kMaxNx, p->n_x, p->n_u);
  if (p->family == DOCP_CARTPOLE && (p->n_x != 4 || p->n_u != 1))
    return fail(DOCP_DIMENSION, "cart-pole has n_x = 4, n_u = 1");
  if (p->family == DOCP_ATTITUDE && (p->n_x != 3 || p->n_u != 3))
    return fail(DOCP_DIMENSION, "attitude has n_x = n_u = 3");
  if (p->family == DOCP_DRIFT && (p->n_x != 8 || p->n_u != 2))
    return fail(DOCP_DIMENSION, "drift has n_x = 8, n_u = 2");
  return DOCP_OK;
}

}  // namespace

// ================================================================== C ABI
extern "C" {

int docp_abi_version(void) { return DOCP_ABI_VERSION; }

int docp_theta_size(const docp_problem* p) {
  if (check_problem(p)) return -1;
  return make_dims(*p).nth;
}

int docp_batch_create(const docp_problem* problem, int32_t batch_size, int32_t device, docp_batch** out) {
  if (!out) return fail(DOCP_INVALID, "null out");
  *out = nullptr;
  int rc = check_problem(problem);
  if (rc) return rc;
  if (batch_size < 1) return fail(DOCP_DIMENSION, "batch size must be >= 1");
  CUDA_TRY(cudaSetDevice(device));
  auto* b = new docp_batch;
  b->prob = *problem;
  b->d = make_dims(*problem);
  b->B = batch_size;
  b->device = device;
  cudaDeviceGetAttribute(&b->num_sms, cudaDevAttrMultiProcessorCount, device);
  const Dims& d = b->d;
  const size_t B = static_cast<size_t>(batch_size);
  View& v = b->v;
  v.d = d;
  v.B = batch_size;
  v.prob = *problem;
#define A(ptr, n)                                  \
  if ((rc = dalloc(b, &ptr, (n)))) {               \
    delete b;                                      \
    return rc;                                     \
  }
  A(v.theta, B * d.nth);
  A(v.z, B * d.nz);
  A(v.lam, B * d.nl);
  A(v.lt, B * d.nl);
  A(v.lgz, B * d.nz);
  A(v.grad, B * d.nth);
  A(v.gamma, B * d.nl);
  A(v.zqp, B * d.nz);
  A(v.qd, B * d.nb * d.nx);
  A(v.lq, B * d.nb * d.nx);
  A(v.q, B * d.nb * d.nx);
  A(v.rd, B * d.T * d.nu);
  A(v.lr, B * d.T * d.nu);
  A(v.r, B * d.T * d.nu);
  A(v.A, B * d.a_per);
  A(v.Bm, B * d.b_per);
  A(v.C, B * d.T * d.nx);
  A(v.xs, B * d.nx);
  A(v.blocks, B * d.blk_stride);
  A(v.status, B);
  A(v.sqp_iters, B);
  A(v.converged, B);
  A(v.pcg_iters, B);
  A(v.pcg_conv, B);
  A(v.pd_proj, B);
  A(v.accepted, B);
  A(v.kkt, B);
  A(v.final_eta, B);
  A(v.mu, B);
  A(v.alpha, B);
  A(v.loss, B);
  A(b->all_list, B);
  A(b->list[0], B);
  A(b->list[1], B);
  A(b->counts, 8);
  A(v.pcg_acc, 3);
  A(b->roll.reward, B);
  A(b->roll.alive, B);
  A(b->roll.rstat, B);
  A(b->roll.xbar, B * d.nx);
  A(b->roll.ex, B * d.nx);
  A(b->roll.gtot, B * d.nth);
#undef A
  if ((rc = ensure_hist(b, 20))) {
    delete b;
    return rc;
  }
  if (cudaMallocHost(&b->h_count, sizeof(int)) != cudaSuccess) {
    delete b;
    return fail(DOCP_CUDA_ERROR, "cudaMallocHost failed");
  }
  iota_kernel<<<grid_for(batch_size, 256, 4096), 256, 0, b->stream>>>(b->all_list, batch_size, b->counts);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(b->stream) != cudaSuccess) {
    delete b;
    return fail(DOCP_CUDA_ERROR, "batch init failed");
  }
  {
    std::lock_guard<std::mutex> lk(g_batches_mu);
    g_batches.insert(b);
  }
  *out = b;
  return DOCP_OK;
}

void docp_batch_destroy(docp_batch* b) {
  if (!b) return;
  {
    std::lock_guard<std::mutex> lk(g_batches_mu);
    if (g_batches.erase(b)) g_retired_solves += batch_solves(b);
  }
  delete b;
}

int docp_batch_set_stream(docp_batch* b, void* stream) {
  if (!b) return fail(DOCP_INVALID, "null batch");
  b->stream = static_cast<cudaStream_t>(stream);
  return DOCP_OK;
}

int docp_batch_sync(docp_batch* b) {
  if (!b) return fail(DOCP_INVALID, "null batch");
  CUDA_TRY(cudaStreamSynchronize(b->stream));
  return DOCP_OK;
}

int32_t docp_batch_size(const docp_batch* b) { return b ? b->B : 0; }

int docp_batch_field_ptr(docp_batch* b, int32_t field, void** ptr, size_t* bytes) {
  if (!b || !ptr) return fail(DOCP_INVALID, "null argument");
  size_t per = 0, elem = 0;
  double* base = field_base(b, field, &per, &elem);
  if (!base) return fail(DOCP_INVALID, "unknown field %d", field);
  *ptr = base;
  if (bytes) *bytes = per * elem * static_cast<size_t>(b->B);
  return DOCP_OK;
}

int docp_batch_upload(docp_batch* b, int32_t field, const void* src, int32_t on_device) {
  void* dst;
  size_t bytes;
  int rc = docp_batch_field_ptr(b, field, &dst, &bytes);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, b->stream));
  if (!on_device) CUDA_TRY(cudaStreamSynchronize(b->stream));
  return DOCP_OK;
}

int docp_batch_download(docp_batch* b, int32_t field, void* dst, int32_t on_device) {
  void* src;
  size_t bytes;
  int rc = docp_batch_field_ptr(b, field, &src, &bytes);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, b->stream));
  if (!on_device) CUDA_TRY(cudaStreamSynchronize(b->stream));
  return DOCP_OK;
}

int docp_batch_upload_schur(docp_batch* b, const double* s_diag, const double* s_sub, const double* p_diag,
                            const double* p_super) {
  if (b) b->sym_blocks = false;
  if (!b) return fail(DOCP_INVALID, "null batch");
  const Dims& d = b->d;
  const int nx = d.nx;
  std::vector<double> rec(static_cast<size_t>(b->B) * d.blk_stride, 0.0);
  for (int p = 0; p < b->B; ++p) {
    double* r = rec.data() + static_cast<size_t>(p) * d.blk_stride;
    auto put = [&](const double* src, long region, int nblk) {
      for (int k = 0; k < nblk; ++k)
        for (int s = 0; s < nx; ++s)
          for (int e = 0; e < nx; ++e)
            r[region + static_cast<long>(k) * d.bsz + blk_off(nx, k, e, s)] =
                src[(static_cast<size_t>(p) * nblk + k) * d.bsz + e + s * nx];
    };
    put(s_diag, d.s_diag, d.nb);
    put(s_sub, d.s_sub, d.T);
    put(p_diag, d.p_diag, d.nb);
    put(p_super, d.p_sup, d.T);
  }
  CUDA_TRY(cudaMemcpyAsync(b->v.blocks, rec.data(), rec.size() * sizeof(double), cudaMemcpyHostToDevice, b->stream));
  CUDA_TRY(cudaStreamSynchronize(b->stream));
  return DOCP_OK;
}

int docp_batch_download_schur(docp_batch* b, double* s_diag, double* s_sub, double* p_diag, double* p_super) {
  if (!b) return fail(DOCP_INVALID, "null batch");
  const Dims& d = b->d;
  const int nx = d.nx;
  std::vector<double> rec(static_cast<size_t>(b->B) * d.blk_stride);
  CUDA_TRY(cudaMemcpyAsync(rec.data(), b->v.blocks, rec.size() * sizeof(double), cudaMemcpyDeviceToHost, b->stream));
  CUDA_TRY(cudaStreamSynchronize(b->stream));
  for (int p = 0; p < b->B; ++p) {
    const double* r = rec.data() + static_cast<size_t>(p) * d.blk_stride;
    auto get = [&](double* dst, long region, int nblk) {
      if (!dst) return;
      for (int k = 0; k < nblk; ++k)
        for (int s = 0; s < nx; ++s)
          for (int e = 0; e < nx; ++e)
            dst[(static_cast<size_t>(p) * nblk + k) * d.bsz + e + s * nx] =
                r[region + static_cast<long>(k) * d.bsz + blk_off(nx, k, e, s)];
    };
    get(s_diag, d.s_diag, d.nb);
    get(s_sub, d.s_sub, d.T);
    get(p_diag, d.p_diag, d.nb);
    get(p_super, d.p_sup, d.T);
  }
  return DOCP_OK;
}

int docp_batch_download_qp(docp_batch* b, double* Q, double* q, double* R, double* r, double* A, double* Bm,
                           double* C, double* x_s) {
  if (!b) return fail(DOCP_INVALID, "null batch");
  const Dims& d = b->d;
  const size_t B = static_cast<size_t>(b->B);
  auto fetch = [&](const double* src, size_t n, std::vector<double>& out) -> int {
    out.resize(n);
    CUDA_TRY(cudaMemcpy(out.data(), src, n * sizeof(double), cudaMemcpyDeviceToHost));
    return DOCP_OK;
  };
  std::vector<double> qd, rd, tmp;
  int rc;
  if ((rc = fetch(b->v.qd, B * d.nb * d.nx, qd)) || (rc = fetch(b->v.rd, B * d.T * d.nu, rd))) return rc;
  if (Q) {
    std::fill(Q, Q + B * d.nb * d.bsz, 0.0);
    for (size_t k = 0; k < B * d.nb; ++k)
      for (int i = 0; i < d.nx; ++i) Q[k * d.bsz + i + i * d.nx] = qd[k * d.nx + i];
  }
  if (R) {
    const size_t b2 = static_cast<size_t>(d.nu) * d.nu;
    std::fill(R, R + B * d.T * b2, 0.0);
    for (size_t k = 0; k < B * d.T; ++k)
      for (int i = 0; i < d.nu; ++i) R[k * b2 + i + i * d.nu] = rd[k * d.nu + i];
  }
  auto copy = [&](double* dst, const double* src, size_t n) -> int {
    if (dst) CUDA_TRY(cudaMemcpy(dst, src, n * sizeof(double), cudaMemcpyDeviceToHost));
    return DOCP_OK;
  };
  if ((rc = copy(q, b->v.q, B * d.nb * d.nx)) || (rc = copy(r, b->v.r, B * d.T * d.nu)) ||
      (rc = copy(C, b->v.C, B * d.T * d.nx)) || (rc = copy(x_s, b->v.xs, B * d.nx)))
    return rc;
  std::vector<double> a, bm;
  if ((rc = fetch(b->v.A, B * d.a_per, a)) || (rc = fetch(b->v.Bm, B * d.b_per, bm))) return rc;
  const size_t bu = static_cast<size_t>(d.nx) * d.nu;
  for (int p = 0; p < b->B; ++p)
    for (int t = 0; t < d.T; ++t) {
      if (A) std::copy_n(a.data() + a_off(d, p, t), d.bsz, A + (static_cast<size_t>(p) * d.T + t) * d.bsz);
      if (Bm) std::copy_n(bm.data() + b_off(d, p, t), bu, Bm + (static_cast<size_t>(p) * d.T + t) * bu);
    }
  return DOCP_OK;
}

// ---------------------------------------------------------------- primitives
int docp_linearize(docp_batch* b, double eps_pd) {
  if (!b) return fail(DOCP_INVALID, "null batch");
  b->last_eps_pd = eps_pd;
  return launch_assemble(b, b->all_list, b->counts, b->B, eps_pd, 0);
}

int docp_assemble_schur(docp_batch* b) {
  if (!b) return fail(DOCP_INVALID, "null batch");
  // The kernel rebuilds the (deterministic) QP data at the last
  // linearization point (Z, THETA, eps_pd) and assembles from it.
  return launch_assemble(b, b->all_list, b->counts, b->B, b->last_eps_pd, 1);
}

int docp_assemble_gamma(docp_batch* b, int32_t rhs) {
  if (!b) return fail(DOCP_INVALID, "null batch");
  if (rhs != DOCP_RHS_FORWARD && rhs != DOCP_RHS_ADJOINT) return fail(DOCP_INVALID, "bad rhs");
  return launch_gamma(b, b->all_list, b->counts, b->B, rhs);
}

int docp_pcg_solve(docp_batch* b, const docp_pcg_config* cfg, int32_t field) {
  if (!b || !cfg) return fail(DOCP_INVALID, "null argument");
  double* sol = field == DOCP_F_LAMBDA ? b->v.lam : field == DOCP_F_LAMBDA_TILDE ? b->v.lt : nullptr;
  if (!sol) return fail(DOCP_INVALID, "pcg solution field must be LAMBDA or LAMBDA_TILDE");
  reset_status_kernel<<<grid_for(b->B, 256, 4096), 256, 0, b->stream>>>(b->v);
  LAUNCH_CHECK();
  return launch_pcg(b, *cfg, b->all_list, b->counts, b->B, sol);
}

int docp_recover_primal(docp_batch* b, int32_t field, int32_t rhs) {
  if (!b) return fail(DOCP_INVALID, "null batch");
  const double* lam = field == DOCP_F_LAMBDA ? b->v.lam : field == DOCP_F_LAMBDA_TILDE ? b->v.lt : nullptr;
  if (!lam) return fail(DOCP_INVALID, "lambda field must be LAMBDA or LAMBDA_TILDE");
  return launch_recover(b, b->all_list, b->counts, b->B, lam, rhs);
}

int docp_line_search(docp_batch* b, const docp_sqp_config* cfg) {
  if (!b) return fail(DOCP_INVALID, "null batch");
  int rc = validate_sqp(cfg);
  if (rc) return rc;
  return launch_step(b, *cfg, b->all_list, b->counts, b->B, 0, 0);
}

int docp_kkt_residual(docp_batch* b) {
  if (!b) return fail(DOCP_INVALID, "null batch");
  return launch_kkt(b, b->all_list, b->counts, b->B);
}

extern "C++" {
namespace {
/// Runs `body` (stream work only, no host synchronisation) through a cached
/// CUDA graph when the batch has its own stream and is not profiling: the
/// first call with a given key captures and instantiates, later calls replay.
template <class F>
int run_graph(docp_batch* b, docp_batch::GraphCache& gc, std::vector<char> key, F&& body) {
  if (!b->stream || b->profiling || std::getenv("DOCP_NO_GRAPHS")) return body();
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  CUDA_TRY(cudaStreamIsCapturing(b->stream, &cs));
  if (cs != cudaStreamCaptureStatusNone) return body();  // inside an enclosing capture (a rollout graph)
  const char* gen = reinterpret_cast<const char*>(&b->layout_gen);
  key.insert(key.end(), gen, gen + sizeof b->layout_gen);
  if (!(gc.exec && gc.key == key)) {
    if (gc.exec) {
      cudaGraphExecDestroy(gc.exec);
      gc.exec = nullptr;
    }
    const uint64_t l0 = g_launches.load();
    CUDA_TRY(cudaStreamBeginCapture(b->stream, cudaStreamCaptureModeThreadLocal));
    const int rc = body();
    cudaGraph_t graph = nullptr;
    const cudaError_t e = cudaStreamEndCapture(b->stream, &graph);
    if (rc) {
      if (graph) cudaGraphDestroy(graph);
      return rc;
    }
    CUDA_TRY(e);
    const cudaError_t ei = cudaGraphInstantiate(&gc.exec, graph, 0);
    cudaGraphDestroy(graph);
    CUDA_TRY(ei);
    gc.key = key;
    gc.launches = g_launches.load() - l0;
    g_launches.fetch_sub(gc.launches);  // counted when the graph runs
  }
  CUDA_TRY(cudaGraphLaunch(gc.exec, b->stream));
  g_launches.fetch_add(gc.launches);
  return DOCP_OK;
}

template <class T>
void key_add(std::vector<char>& k, const T& v) {
  const char* p = reinterpret_cast<const char*>(&v);
  k.insert(k.end(), p, p + sizeof v);
}
}  // namespace
}  // extern "C++"

static int sqp_solve_body(docp_batch* b, const docp_sqp_config* cfg);

int docp_sqp_solve(docp_batch* b, const docp_sqp_config* cfg) {  // sqp.hpp:213-261
  if (!b) return fail(DOCP_INVALID, "null batch");
  int rc = validate_sqp(cfg);
  if (rc) return rc;
  if ((rc = ensure_hist(b, std::max(1, cfg->max_sqp_iters)))) return rc;
  // Up to 4 SQP iterations the host never waits on the device (below), so
  // the whole solve is one cached CUDA graph when the batch has its own
  // stream: a small-batch call (C1: B = 1, one SQP step) costs one graph
  // launch instead of ~15 kernel launches.
  if (cfg->max_sqp_iters <= 4) {
    std::vector<char> key;
    key_add(key, *cfg);
    return run_graph(b, b->graph_solve, key, [&]() { return sqp_solve_body(b, cfg); });
  }
  return sqp_solve_body(b, cfg);
}

static int sqp_solve_body(docp_batch* b, const docp_sqp_config* cfg) {
  int rc;
  int cur = 0;
  CUDA_TRY(cudaMemsetAsync(b->counts + 1, 0, 2 * sizeof(int), b->stream));
  init_solve_kernel<<<grid_for(static_cast<long>(b->B) * 32, 256, b->num_sms * 8), 256, 0, b->stream>>>(b->v, b->list[0], b->counts + 1);
  LAUNCH_CHECK();
  // The loop is enqueued without waiting on the device: every kernel reads
  // the active count from device memory and exits early when it is zero, so
  // iterations after global convergence cost a few empty launches. The host
  // reads the count back only at iterations 4, 8, 16, ... to stop early
  // (one synchronisation for the benchmark's max_sqp_iters = 5).
  int n_bound = b->B;  // upper bound of the active count, sizes the grids
  // The affine-quadratic family's Q_t, R_t (diagonal cost Hessians, then
  // project_pd), A_t and B_t depend on theta only, never on z
  // (affine_quadratic.hpp:39-81, quadratic_cost.hpp:9-20), so the -S / Phi^-1
  // blocks assembled at the first iteration are, bit for bit, the ones every
  // later re-linearisation of this solve would assemble (same theta, same
  // eps_pd, same arithmetic). Later iterations and the final refresh re-run
  // the linearisation (q_t, r_t, C_t, the evaluation checks) and keep the
  // blocks; a Cholesky that fails on them failed at the first iteration.
  const bool keep_blocks = b->prob.family == DOCP_AFFINE_QUADRATIC && !std::getenv("DOCP_REASSEMBLE");
  int ran = 0;
  for (int iter = 0; iter < cfg->max_sqp_iters && n_bound > 0; ++iter, ++ran) {
    const int* list = b->list[cur];
    const int* cnt = b->counts + 1 + cur;
    const int schur = iter == 0 || !keep_blocks;
    if ((rc = launch_assemble(b, list, cnt, n_bound, cfg->eps_pd, schur, cfg->pcg.mode != DOCP_PCG_PARITY))) return rc;
    if ((rc = launch_gamma(b, list, cnt, n_bound, DOCP_RHS_FORWARD))) return rc;
    if ((rc = launch_pcg(b, cfg->pcg, list, cnt, n_bound, b->v.lam))) return rc;
    if ((rc = launch_recover(b, list, cnt, n_bound, b->v.lam, DOCP_RHS_FORWARD))) return rc;
    if ((rc = launch_step(b, *cfg, list, cnt, n_bound, iter, 1))) return rc;
    const int nxt = cur ^ 1;
    CUDA_TRY(cudaMemsetAsync(b->counts + 1 + nxt, 0, sizeof(int), b->stream));
    compact_kernel<<<grid_for(n_bound, 256, 4096), 256, 0, b->stream>>>(b->v, list, cnt, b->list[nxt],
                                                                         b->counts + 1 + nxt);
    LAUNCH_CHECK();
    cur = nxt;
    const int done = iter + 1;
    if (done < cfg->max_sqp_iters && done >= 4 && (done & (done - 1)) == 0)
      if ((rc = read_count(b, b->counts + 1 + cur, &n_bound))) return rc;
  }
  // refresh QP / Schur at the returned trajectory, KKT diagnostic (sqp.hpp:254-259)
  CUDA_TRY(cudaMemsetAsync(b->counts + 1 + (cur ^ 1), 0, sizeof(int), b->stream));
  int* fin = b->list[cur ^ 1];
  int* fin_cnt = b->counts + 1 + (cur ^ 1);
  ok_list_kernel<<<grid_for(b->B, 256, 4096), 256, 0, b->stream>>>(b->v, fin, fin_cnt);
  LAUNCH_CHECK();
  // every problem of fin was in the first iteration's list (init_solve lists
  // exactly the OK problems; statuses never return to OK)
  const int schur = !(keep_blocks && ran > 0);
  if ((rc = launch_assemble(b, fin, fin_cnt, b->B, cfg->eps_pd, schur, cfg->pcg.mode != DOCP_PCG_PARITY))) return rc;
  if ((rc = launch_kkt(b, fin, fin_cnt, b->B))) return rc;
  return DOCP_OK;
}

static int backward_vjp_body(docp_batch* b, const docp_pcg_config* cfg);

int docp_backward_vjp(docp_batch* b, const docp_pcg_config* cfg) {  // backward.hpp:27-50
  if (!b || !cfg) return fail(DOCP_INVALID, "null argument");
  std::vector<char> key;
  key_add(key, *cfg);
  return run_graph(b, b->graph_vjp, key, [&]() { return backward_vjp_body(b, cfg); });
}

static int backward_vjp_body(docp_batch* b, const docp_pcg_config* cfg) {
  int rc;
  CUDA_TRY(cudaMemsetAsync(b->counts + 1, 0, sizeof(int), b->stream));
  ok_list_kernel<<<grid_for(b->B, 256, 4096), 256, 0, b->stream>>>(b->v, b->list[0], b->counts + 1);
  LAUNCH_CHECK();
  const int* list = b->list[0];
  const int* cnt = b->counts + 1;
  if ((rc = launch_gamma(b, list, cnt, b->B, DOCP_RHS_ADJOINT))) return rc;
  if ((rc = launch_pcg(b, *cfg, list, cnt, b->B, b->v.lt))) return rc;
  if ((rc = launch_recover(b, list, cnt, b->B, b->v.lt, DOCP_RHS_ADJOINT))) return rc;
  return launch_vjp(b, list, cnt, b->B);
}

// ---------------------------------------------------------------- rollouts (batch.hpp:172-258)
namespace {
int ensure_rollout(docp_batch* b, int H) {
  if (H <= b->roll_cap) return DOCP_OK;
  const Dims& d = b->d;
  const size_t B = static_cast<size_t>(b->B), h = static_cast<size_t>(H);
  int rc;
  ++b->layout_gen;
  if ((rc = dalloc(b, &b->roll.z, h * B * d.nz)) || (rc = dalloc(b, &b->roll.lam, h * B * d.nl)) ||
      (rc = dalloc(b, &b->roll.x, (h + 1) * B * d.nx)) || (rc = dalloc(b, &b->roll.u, h * B * d.nu)))
    return rc;
  b->roll_cap = H;
  return DOCP_OK;
}
}  // namespace



int docp_rollout(docp_batch* b, const docp_sqp_config* cfg, const double* x_init, int32_t x_init_on_device,
                 int32_t H) {
  if (!b || !cfg || !x_init) return fail(DOCP_INVALID, "null argument");
  if (b->prob.family == DOCP_CARTPOLE || b->prob.family == DOCP_DRIFT)
    return fail(DOCP_UNSUPPORTED, "rollout: environments exist for the affine and attitude tasks");
  if (H < 1) return fail(DOCP_DIMENSION, "rollout: episode length must be >= 1");
  int rc = validate_sqp(cfg);
  if (rc) return rc;
  if ((rc = ensure_rollout(b, H))) return rc;
  if ((rc = ensure_hist(b, std::max(1, cfg->max_sqp_iters)))) return rc;
  b->roll.H = H;
  b->roll_eps_pd = cfg->eps_pd;
  // the initial states go to the record's x_0 slot first (outside any graph)
  CUDA_TRY(cudaMemcpyAsync(b->roll.x, x_init, sizeof(double) * b->B * b->d.nx,
                           x_init_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, b->stream));
  auto body = [&]() -> int {
    const int g = grid_for(static_cast<long>(b->B) * 32, 256, b->num_sms * 8);
    rollout_init_kernel<<<g, 256, 0, b->stream>>>(b->v, b->roll, b->roll.x);
    LAUNCH_CHECK();
    int r;
    for (int t = 0; t < H; ++t) {
      rollout_pre_kernel<<<g, 256, 0, b->stream>>>(b->v, b->roll, t);
      LAUNCH_CHECK();
      if ((r = docp_sqp_solve(b, cfg))) return r;
      rollout_post_kernel<<<g, 256, 0, b->stream>>>(b->v, b->roll, t);
      LAUNCH_CHECK();
    }
    return DOCP_OK;
  };
  // the SQP loop reads the active count back from iteration 4 on: only
  // shorter solves are free of host synchronisation and can be captured
  if (cfg->max_sqp_iters > 4) return body();
  std::vector<char> key;
  key_add(key, H);
  key_add(key, *cfg);
  return run_graph(b, b->graph_fwd, key, body);
}

int docp_rollout_backward(docp_batch* b, const docp_pcg_config* cfg) {
  if (!b || !cfg) return fail(DOCP_INVALID, "null argument");
  const int H = b->roll.H;
  if (H < 1 || b->roll_cap < H) return fail(DOCP_INVALID, "rollout_backward: no rollout recorded");
  auto body = [&]() -> int {
    const int g = grid_for(static_cast<long>(b->B) * 32, 256, b->num_sms * 8);
    rollout_back_init_kernel<<<grid_for(static_cast<long>(b->B) * b->d.nth, 256, b->num_sms * 8), 256, 0,
                               b->stream>>>(b->v, b->roll);
    LAUNCH_CHECK();
    int rc;
    for (int t = H - 1; t >= 0; --t) {
      CUDA_TRY(cudaMemsetAsync(b->counts + 1, 0, sizeof(int), b->stream));
      rollout_back_pre_kernel<<<g, 256, 0, b->stream>>>(b->v, b->roll, t, b->list[0], b->counts + 1);
      LAUNCH_CHECK();
      // the step's cached matrices: re-linearised at its recorded solution
      if ((rc = launch_assemble(b, b->list[0], b->counts + 1, b->B, b->roll_eps_pd, 1, cfg->mode != DOCP_PCG_PARITY)))
        return rc;
      if ((rc = docp_backward_vjp(b, cfg))) return rc;
      rollout_back_post_kernel<<<grid_for(b->B, 128, b->num_sms * 4), 128, 0, b->stream>>>(b->v, b->roll, t);
      LAUNCH_CHECK();
    }
    rollout_back_fini_kernel<<<grid_for(static_cast<long>(b->B) * b->d.nth, 256, b->num_sms * 8), 256, 0,
                               b->stream>>>(b->v, b->roll);
    LAUNCH_CHECK();
    return DOCP_OK;
  };
  std::vector<char> key;
  key_add(key, H);
  key_add(key, *cfg);
  key_add(key, b->roll_eps_pd);
  return run_graph(b, b->graph_bwd, key, body);
}

int docp_il_epoch(docp_batch* b, const docp_sqp_config* cfg, const double* weights, int32_t learn_start,
                  int32_t learn_size, const double* demos, double den, double* loss_sum, double* grad_sum) {
  if (!b || !cfg || !weights || !demos || !loss_sum || !grad_sum) return fail(DOCP_INVALID, "null argument");
  if (learn_start < 0 || learn_size < 0 || learn_start + learn_size > b->d.nth)
    return fail(DOCP_DIMENSION, "learnable segment out of range");
  int rc;
  il_setup_kernel<<<grid_for(static_cast<long>(b->B) * (learn_size + b->d.nz), 256, b->num_sms * 16), 256, 0,
                    b->stream>>>(b->v, weights, learn_start, learn_size, demos);
  LAUNCH_CHECK();
  if ((rc = docp_sqp_solve(b, cfg))) return rc;
  {
    auto kl = cfg->pcg.mode != DOCP_PCG_PARITY ? il_loss_kernel<true> : il_loss_kernel<false>;
    kl<<<grid_for(static_cast<long>(b->B) * 32, kIlLossThreads, b->num_sms * 8), kIlLossThreads, 0, b->stream>>>(
        b->v, demos, den);
  }
  LAUNCH_CHECK();
  if ((rc = docp_backward_vjp(b, &cfg->pcg))) return rc;
  if (cfg->pcg.mode != DOCP_PCG_PARITY) {
    il_sum_tree_kernel<<<1 + learn_size, kIlTreeThreads, 0, b->stream>>>(b->v, learn_start, loss_sum, grad_sum,
                                                                        b->counts + 4);
  } else {
    const int cols = 1 + learn_size;
    const int ctas = (cols + kIlSumCols - 1) / kIlSumCols;
    const int ncol = std::min(kIlSumCols, cols);
    // two staging buffers in 192 KB of shared memory
    const int rows = std::max(1, std::min(b->B, (96 * 1024 / 8) / ncol - 1));
    const size_t smem = 2 * static_cast<size_t>(rows | 1) * ncol * sizeof(double);
    CUDA_TRY(cudaFuncSetAttribute(il_sum_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    il_sum_kernel<<<ctas, kIlSumThreads, smem, b->stream>>>(b->v, learn_start, learn_size, rows, loss_sum, grad_sum,
                                                            b->counts + 4);
  }
  LAUNCH_CHECK();
  return DOCP_OK;
}

int docp_il_failures(docp_batch* b, int32_t* n_failed, int32_t* first_failed) {
  if (!b || !n_failed || !first_failed) return fail(DOCP_INVALID, "null argument");
  int h[2];
  CUDA_TRY(cudaMemcpyAsync(h, b->counts + 4, sizeof h, cudaMemcpyDeviceToHost, b->stream));
  CUDA_TRY(cudaStreamSynchronize(b->stream));
  *n_failed = h[0];
  *first_failed = h[0] ? h[1] : -1;
  const int reset[2] = {0, 0x7fffffff};
  CUDA_TRY(cudaMemcpyAsync(b->counts + 4, reset, sizeof reset, cudaMemcpyHostToDevice, b->stream));
  CUDA_TRY(cudaStreamSynchronize(b->stream));
  return DOCP_OK;
}

int docp_profile_begin(docp_batch* b) {
  if (!b) return fail(DOCP_INVALID, "null batch");
  CUDA_TRY(cudaStreamSynchronize(b->stream));
  for (auto& v : b->prof) v.clear();
  b->prof_seq.clear();
  b->pool_used = 0;
  CUDA_TRY(cudaMemsetAsync(b->v.pcg_acc, 0, 2 * sizeof(unsigned long long), b->stream));
  b->profiling = true;
  return DOCP_OK;
}

int docp_profile_end(docp_batch* b, docp_profile* out) {
  if (!b || !out) return fail(DOCP_INVALID, "null argument");
  b->profiling = false;
  CUDA_TRY(cudaStreamSynchronize(b->stream));
  std::memset(out, 0, sizeof *out);
  for (int k = 0; k < DOCP_PROF_KINDS; ++k) {
    out->launches[k] = static_cast<int32_t>(b->prof[k].size());
    double ms = 0.0;
    for (auto& ev : b->prof[k]) {
      float t = 0.f;
      CUDA_TRY(cudaEventElapsedTime(&t, ev.first, ev.second));
      ms += t;
    }
    out->ms[k] = ms;
  }
  if (!b->prof_seq.empty()) {
    float span = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&span, b->prof_seq.front().start, b->prof_seq.back().stop));
    out->span_ms = span;
    out->max_gap_after = out->max_gap_before = -1;
    for (size_t k = 1; k < b->prof_seq.size(); ++k) {
      float g = 0.f;
      CUDA_TRY(cudaEventElapsedTime(&g, b->prof_seq[k - 1].stop, b->prof_seq[k].start));
      out->gap_ms += g;
      if (g > out->max_gap_ms) {
        out->max_gap_ms = g;
        out->max_gap_after = b->prof_seq[k - 1].kind;
        out->max_gap_before = b->prof_seq[k].kind;
      }
    }
  }
  unsigned long long acc[2];
  CUDA_TRY(cudaMemcpy(acc, b->v.pcg_acc, sizeof acc, cudaMemcpyDeviceToHost));
  out->pcg_iterations = acc[0];
  out->pcg_solves = acc[1];
  const Dims& d = b->d;
  const double b_it = 16.0 * d.bsz * (2.0 * d.T + 1.0);  // symmetric -S + Phi^-1, fp64
  out->pcg_bytes_per_iteration = b_it;
  out->pcg_algorithmic_bytes =
      (static_cast<double>(acc[0]) + static_cast<double>(acc[1])) * b_it + static_cast<double>(acc[1]) * 24.0 * d.nl;
  return DOCP_OK;
}

uint64_t docp_pcg_invocations(void) {
  std::lock_guard<std::mutex> lk(g_batches_mu);
  uint64_t n = g_retired_solves;
  for (docp_batch* b : g_batches) n += batch_solves(b);
  return n;
}
uint64_t docp_kernel_launches(void) { return g_launches.load(); }
const char* docp_last_error(void) { return g_last_error.c_str(); }

int docp_format_status(const docp_status* s, char* buf, int32_t cap) {
  if (!s || !buf || cap <= 0) return 0;
  if (s->step > 0) {  // RolloutTruncation wrapping a solve failure (batch.hpp:186-191)
    docp_status inner = *s;
    inner.step = 0;
    const int n = snprintf(buf, cap, "rollout: solve failed at step %d: ", s->step - 1);
    if (n < 0 || n >= cap) return n;
    return n + docp_format_status(&inner, buf + n, cap - n);
  }
  const int i = s->index;
  switch (s->where) {  // messages of common.hpp / problem.hpp / schur.hpp / pcg.hpp / sqp.hpp
    case DOCP_AT_NONE: return snprintf(buf, cap, "ok");
    case DOCP_AT_STATE_COST: return snprintf(buf, cap, "state_cost returned non-finite values at stage %d", i);
    case DOCP_AT_CONTROL_COST: return snprintf(buf, cap, "control_cost returned non-finite values at stage %d", i);
    case DOCP_AT_DYNAMICS: return snprintf(buf, cap, "dynamics_residual returned non-finite values at stage %d", i);
    case DOCP_AT_INITIAL_STATE: return snprintf(buf, cap, "initial_state returned non-finite values at stage %d", i);
    case DOCP_AT_CHOL_Q: return snprintf(buf, cap, "assemble_schur: Cholesky of Q failed at stage %d", i);
    case DOCP_AT_CHOL_R: return snprintf(buf, cap, "assemble_schur: Cholesky of R failed at stage %d", i);
    case DOCP_AT_CHOL_CHI: return snprintf(buf, cap, "assemble_schur: Cholesky of chi failed at stage %d", i);
    case DOCP_AT_PCG_CURVATURE:
      return snprintf(buf, cap, "pcg: p'Sp <= 0 (loss of positive definiteness) at iteration %d", i);
    case DOCP_AT_PCG_PRECOND: return snprintf(buf, cap, "pcg: preconditioner lost definiteness at iteration %d", i);
    case DOCP_AT_MERIT_STATE: return snprintf(buf, cap, "merit: non-finite state cost at stage %d", i);
    case DOCP_AT_MERIT_CONTROL: return snprintf(buf, cap, "merit: non-finite control cost at stage %d", i);
    case DOCP_AT_SQP_ITERATE: return snprintf(buf, cap, "sqp: non-finite iterate at iteration %d", i);
    case DOCP_AT_INITIAL_GUESS: return snprintf(buf, cap, "sqp: initial guess must be finite");
    case DOCP_AT_ROLLOUT_ENV:
      return snprintf(buf, cap, "rollout: environment produced a non-finite state at step %d", i);
    default: return snprintf(buf, cap, "error %d at %d", s->code, i);
  }
}

int docp_describe(const docp_problem* p, char* buf, int32_t cap) {
  if (check_problem(p) || !buf) return -1;
  const Dims d = make_dims(*p);
  int dev = 0, max_optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const bool res = pcg_smem(d, true) + 64 <= static_cast<size_t>(max_optin);
  const int cl = d.nx == 16 ? h16f_cluster_for(d, dev) : h8f_cluster_for(d, dev);
  const char* fk = d.nx == 16 ? "pcg_kernel_h16f" : "pcg_kernel_h8f";
  char fast[128];
  const int s8 = d.nx == 8 ? h8s_variant_for(d, dev) : 0;
  if (h4f_fits(d, dev)) snprintf(fast, sizeof fast, "pcg_kernel_h4f(resident)");
  else if (s8 >= 2) snprintf(fast, sizeof fast, "pcg_kernel_h8s<%d,no-prefetch%s>(resident); uploaded systems %s",
                             s8 == 2 ? 256 : 384, s8 == 4 ? ",-S in smem" : "",
                             cl == 2 ? "pcg_kernel_h8f(cluster2)" : "pcg_kernel_h8f");
  else if (d.nx == 8 && s8 == 0 && h8s_cluster_preferred(d, dev))
    snprintf(fast, sizeof fast, "pcg_kernel_h8s_cl(cluster%d,resident); uploaded systems pcg_kernel_h8f",
             h8s_cluster_for(d, dev));
  else if (cl == 1) snprintf(fast, sizeof fast, "%s(resident)",
                           d.nx == 8 ? "pcg_kernel_h8s; uploaded systems pcg_kernel_h8r" : fk);
  else if (cl > 1) snprintf(fast, sizeof fast, "%s(cluster%d,resident)", fk, cl);
  else snprintf(fast, sizeof fast, "%s", d.nx == 8 ? (2 * d.nb <= 512 ? "pcg_kernel_h8" : "pcg_kernel<8>")
                                                   : d.nx == 4 ? "pcg_kernel<4>" : (d.nx == 6 || d.nx == 9) ? "pcg_kernel<NX=6|9>" : "pcg_kernel<runtime>");
  const int p8 = d.nx == 8 ? h8p_variant_for(d, dev) : 0;
  const char* parity = p8 == 1   ? "pcg_kernel_h8p<-S resident>; uploaded systems pcg_kernel_h8"
                       : p8 == 2 ? "pcg_kernel_h8p<no-prefetch>; uploaded systems pcg_kernel_h8"
                       : d.nx == 8 ? (2 * d.nb <= 512 ? "pcg_kernel_h8" : "pcg_kernel<8>")
                                   : d.nx == 4 ? "pcg_kernel<4>" : (d.nx == 6 || d.nx == 9) ? "pcg_kernel<NX=6|9>" : "pcg_kernel<runtime>";
  return snprintf(buf, cap, "nx=%d layout=%s record=%ld B parity=%s(%s) fast=%s", d.nx,
                  d.nx == 8 ? "swizzle8" : d.nx == 4 ? "swizzle4" : "colmajor", d.blk_stride * 8, parity,
                  res ? "resident" : "streaming", fast);

}

}  // extern "C"

#ifdef DOCP_K1_CLOCK
/// A/B builds only: cycles of assemble_kernel_t's thread 0 per phase, summed over launches (then reset).
extern "C" int docp_k1_clock(unsigned long long* out) {
  if (cudaMemcpyFromSymbol(out, docp_dev::g_k1_clk, 16 * sizeof(unsigned long long)) != cudaSuccess) return 1;
  static const unsigned long long zero[16] = {0};
  return cudaMemcpyToSymbol(docp_dev::g_k1_clk, zero, sizeof zero) != cudaSuccess;
}
#endif
