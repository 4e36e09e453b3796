// pcg_nx8.cu — K2 instantiations for n_x = 8 (separate translation unit for build parallelism)
#include <cstdlib>
#include <cstring>

#include "k_pcg_h8.cuh"
#include "k_pcg_h8f.cuh"
#include "pcg_launch.cuh"

namespace docp_host {

template <bool PAR, bool RES>
int launch_h8(docp_batch* b, const PcgPlan& pl, const int* list, const int* count, int n_hint, double* sol, double eps,
              int max_iters) {
  // <= 256 threads (T <= 127) leaves room for 255 registers per thread
  auto kern = 2 * b->d.nb <= 256 ? pcg_kernel_h8<PAR, RES, 256> : pcg_kernel_h8<PAR, RES, 512>;
  const int threads = (2 * b->d.nb + 31) / 32 * 32;
  CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(pl.smem)));
  int per_sm = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, pl.smem));
  if (per_sm < 1) return fail(DOCP_UNSUPPORTED, "pcg: kernel does not fit on an SM (smem %zu)", pl.smem);
  const int grid = std::max(1, std::min(n_hint, per_sm * b->num_sms));
  CUDA_TRY(cudaMemsetAsync(b->counts + 3, 0, sizeof(int), b->stream));
  ProfScope ps(b, DOCP_PROF_PCG);
  kern<<<grid, threads, pl.smem, b->stream>>>(b->v, list, count, b->counts + 3, sol, eps, max_iters);
  LAUNCH_CHECK();
  return DOCP_OK;
}

/// FAST with resident blocks: the instruction-lean pcg_kernel_h8f.
int launch_h8f(docp_batch* b, const PcgPlan&, const int* list, const int* count, int n_hint, double* sol,
               double eps, int max_iters) {
  auto kern = pcg_kernel_h8f<256>;
  const size_t smem = h8f_smem_doubles(b->d) * sizeof(double);
  const int threads = (2 * b->d.nb + 31) / 32 * 32;
  CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int per_sm = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
  if (per_sm < 1) return fail(DOCP_UNSUPPORTED, "pcg: kernel does not fit on an SM (smem %zu)", smem);
  const int grid = std::max(1, std::min(n_hint, per_sm * b->num_sms));
  CUDA_TRY(cudaMemsetAsync(b->counts + 3, 0, sizeof(int), b->stream));
  ProfScope ps(b, DOCP_PROF_PCG);
  kern<<<grid, threads, smem, b->stream>>>(b->v, list, count, b->counts + 3, sol, eps, max_iters);
  LAUNCH_CHECK();
  return DOCP_OK;
}

/// Kernel variant override for A/B measurements: DOCP_PCG_VARIANT=h8 keeps
/// FAST solves on pcg_kernel_h8.
static bool force_h8() {
  const char* e = std::getenv("DOCP_PCG_VARIANT");
  return e && std::strcmp(e, "h8") == 0;
}

/// n_x = 8: FAST + resident blocks -> pcg_kernel_h8f; otherwise two threads
/// per block row (pcg_kernel_h8) up to T = 255, one thread per block row
/// (pcg_kernel) beyond.
DOCP_PCG_LAUNCHER(launch_pcg_nx8) {
  if (!par && pl.resident && 2 * b->d.nb <= 256 && !force_h8())
    return launch_h8f(b, pl, list, count, n_hint, sol, eps, max_iters);
  if (2 * b->d.nb <= 512) {
    if (par) return pl.resident ? launch_h8<true, true>(b, pl, list, count, n_hint, sol, eps, max_iters)
                                : launch_h8<true, false>(b, pl, list, count, n_hint, sol, eps, max_iters);
    return pl.resident ? launch_h8<false, true>(b, pl, list, count, n_hint, sol, eps, max_iters)
                       : launch_h8<false, false>(b, pl, list, count, n_hint, sol, eps, max_iters);
  }
  return launch_pcg_nx<8>(b, pl, par, list, count, n_hint, sol, eps, max_iters);
}

}  // namespace docp_host
