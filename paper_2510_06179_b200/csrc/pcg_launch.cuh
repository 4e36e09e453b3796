// pcg_launch.cuh — host launchers of the K2 template variants (included by
// one translation unit per block size).
#pragma once

#include "batch.cuh"
#include "k_pcg.cuh"

namespace docp_host {
using namespace docp_dev;

template <int NX, int MAXB, bool PAR, bool RES>
int launch_pcg_t(docp_batch* b, const PcgPlan& pl, const int* list, const int* count, int n_hint, double* sol,
                 double eps, int max_iters) {
  auto kern = pcg_kernel<NX, MAXB, PAR, RES>;
  CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(pl.smem)));
  int per_sm = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, pl.threads, pl.smem));
  if (per_sm < 1) return fail(DOCP_UNSUPPORTED, "pcg: kernel does not fit on an SM (smem %zu)", pl.smem);
  const int grid = std::max(1, std::min(n_hint, per_sm * b->num_sms));
  CUDA_TRY(cudaMemsetAsync(b->counts + 3, 0, sizeof(int), b->stream));
  ProfScope ps(b, DOCP_PROF_PCG);
  kern<<<grid, pl.threads, pl.smem, b->stream>>>(b->v, list, count, b->counts + 3, sol, eps, max_iters);
  LAUNCH_CHECK();
  return DOCP_OK;
}

template <int NX, bool PAR, bool RES>
int launch_pcg_r(docp_batch* b, const PcgPlan& pl, const int* list, const int* count, int n_hint, double* sol,
                 double eps, int max_iters) {
  switch (pl.maxr) {
    case 1: return launch_pcg_t<NX, 1, PAR, RES>(b, pl, list, count, n_hint, sol, eps, max_iters);
    case 2: return launch_pcg_t<NX, 2, PAR, RES>(b, pl, list, count, n_hint, sol, eps, max_iters);
    default:
      return fail(DOCP_UNSUPPORTED,
                  "pcg: horizon %d too long for the one-thread-per-block-row kernel (T <= 511; FAST n_x = 8 / 16 "
                  "runs longer horizons on thread-block clusters)",
                  b->d.T);
  }
}

template <int NX>
int launch_pcg_nx(docp_batch* b, const PcgPlan& pl, bool par, const int* list, const int* count, int n_hint,
                  double* sol, double eps, int max_iters) {
  if (par) {
    return pl.resident ? launch_pcg_r<NX, true, true>(b, pl, list, count, n_hint, sol, eps, max_iters)
                       : launch_pcg_r<NX, true, false>(b, pl, list, count, n_hint, sol, eps, max_iters);
  }
  return pl.resident ? launch_pcg_r<NX, false, true>(b, pl, list, count, n_hint, sol, eps, max_iters)
                     : launch_pcg_r<NX, false, false>(b, pl, list, count, n_hint, sol, eps, max_iters);
}


}  // namespace docp_host
