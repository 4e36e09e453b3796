// pcg_nx4.cu — K2 for n_x = 4 (separate translation unit for build parallelism)
#include <cstdlib>
#include <cstring>

#include "k_pcg_h4f.cuh"
#include "pcg_launch.cuh"

namespace docp_host {

constexpr int kH4fMaxThreads = 256;

/// Whether FAST n_x = 4 solves of this shape run pcg_kernel_h4f (one CTA per
/// problem, blocks resident; DOCP_PCG_VARIANT=generic keeps pcg_kernel<4>).
bool h4f_fits(const Dims& d, int device) {
  if (d.nx != 4 || d.nb > kH4fMaxThreads) return false;
  const char* e = std::getenv("DOCP_PCG_VARIANT");
  if (e && std::strcmp(e, "generic") == 0) return false;
  int max_optin = 0;
  cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  return h4f_smem_doubles(d) * 8 + 64 <= static_cast<long>(max_optin);
}

static int launch_h4f(docp_batch* b, const int* list, const int* count, int n_hint, double* sol, double eps,
                      int max_iters) {
  auto kern = pcg_kernel_h4f<kH4fMaxThreads>;
  const size_t smem = h4f_smem_doubles(b->d) * sizeof(double);
  const int threads = (b->d.nb + 31) / 32 * 32;
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

/// n_x = 4: FAST -> pcg_kernel_h4f while T < 256 and the blocks fit on-chip;
/// PARITY (or longer horizons): the one-thread-per-block-row pcg_kernel<4>.
DOCP_PCG_LAUNCHER(launch_pcg_nx4) {
  if (!par && h4f_fits(b->d, b->device)) return launch_h4f(b, list, count, n_hint, sol, eps, max_iters);
  return launch_pcg_nx<4>(b, pl, par, list, count, n_hint, sol, eps, max_iters);
}

}  // namespace docp_host
