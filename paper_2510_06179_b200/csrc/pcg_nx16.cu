// pcg_nx16.cu — K2 for n_x = 16 (separate translation unit for build parallelism)
#include "k_pcg_h16f.cuh"
#include "pcg_launch.cuh"

namespace docp_host {

/// FAST: pcg_kernel_h16f on a cluster of CL CTAs (CL = 1: one CTA per problem).
template <int CL>
int launch_h16f_cl(docp_batch* b, const int* list, const int* count, int n_hint, double* sol, double eps,
                   int max_iters) {
  auto kern = pcg_kernel_h16f<256, CL>;
  const size_t smem = h16f_smem_doubles(b->d, CL) * sizeof(double);
  const int threads = (4 * h16f_rows(b->d, CL) + 31) / 32 * 32;
  CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  cudaLaunchConfig_t lc{};
  cudaLaunchAttribute attr[1];
  lc.blockDim = dim3(threads);
  lc.dynamicSmemBytes = smem;
  lc.stream = b->stream;
  int groups = 0;
  if (CL == 1) {
    int per_sm = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
    groups = per_sm * b->num_sms;
  } else {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    lc.attrs = attr;
    lc.numAttrs = 1;
    lc.gridDim = dim3(CL * b->num_sms);
    CUDA_TRY(cudaOccupancyMaxActiveClusters(&groups, kern, &lc));
  }
  if (groups < 1) return fail(DOCP_UNSUPPORTED, "pcg: kernel does not fit (cluster %d, smem %zu)", CL, smem);
  lc.gridDim = dim3(CL * std::max(1, std::min(n_hint, groups)));
  CUDA_TRY(cudaMemsetAsync(b->counts + 3, 0, sizeof(int), b->stream));
  ProfScope ps(b, DOCP_PROF_PCG);
  CUDA_TRY(cudaLaunchKernelEx(&lc, kern, b->v, list, count, b->counts + 3, sol, eps, max_iters));
  LAUNCH_CHECK();
  return DOCP_OK;
}

int h16f_cluster_for(const Dims& d, int device) {
  if (d.nx != 16) return 0;
  int max_optin = 0;
  cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  for (int cl : {1, 2, 4, 8}) {
    if (cl > 1 && (cl - 1) * h16f_rows(d, cl) >= d.nb) break;  // every CTA must own a row
    if (h16f_rows(d, cl) <= 64 && h16f_smem_doubles(d, cl) * 8 + 64 <= static_cast<long>(max_optin)) return cl;
  }
  return 0;
}

/// n_x = 16: FAST -> pcg_kernel_h16f on the smallest cluster that keeps the
/// blocks on-chip; PARITY (or no fitting cluster): the runtime-shape kernel.
DOCP_PCG_LAUNCHER(launch_pcg_nx16) {
  if (!par) {
    switch (h16f_cluster_for(b->d, b->device)) {
      case 1: return launch_h16f_cl<1>(b, list, count, n_hint, sol, eps, max_iters);
      case 2: return launch_h16f_cl<2>(b, list, count, n_hint, sol, eps, max_iters);
      case 4: return launch_h16f_cl<4>(b, list, count, n_hint, sol, eps, max_iters);
      case 8: return launch_h16f_cl<8>(b, list, count, n_hint, sol, eps, max_iters);
      default: break;
    }
  }
  return launch_pcg_nx<0>(b, pl, par, list, count, n_hint, sol, eps, max_iters);
}

}  // namespace docp_host
