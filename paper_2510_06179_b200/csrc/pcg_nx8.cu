// pcg_nx8.cu — K2 instantiations for n_x = 8 (separate translation unit for build parallelism)
#include <cstdlib>
#include <cstring>

#include "k_pcg_h8.cuh"
#include "k_pcg_h8f.cuh"
#include "k_pcg_h8p.cuh"
#include "k_pcg_h8r.cuh"
#include "k_pcg_h8s.cuh"
#include "k_pcg_h8x.cuh"
#include "pcg_launch.cuh"

namespace docp_host {

static bool force_variant(const char* name);

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

/// FAST: the instruction-lean pcg_kernel_h8f, on a cluster of cl CTAs
/// (cl = 1: one CTA per problem; cl > 1: the problem's block rows split over
/// the cluster's shared memories).
template <int CL>
int launch_h8f_cl(docp_batch* b, const int* list, const int* count, int n_hint, double* sol, double eps,
                  int max_iters) {
  auto kern = pcg_kernel_h8f<256, CL>;
  int max_optin = 0;
  cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, b->device);
  size_t smem = h8f_smem_doubles(b->d, CL, true) * sizeof(double);
  if (smem + 64 > static_cast<size_t>(max_optin)) smem = h8f_smem_doubles(b->d, CL, false) * sizeof(double);
  const int threads = (2 * h8f_rows(b->d, CL) + 31) / 32 * 32;
  CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  cudaLaunchConfig_t lc{};
  cudaLaunchAttribute attr[1];
  lc.blockDim = dim3(threads);
  lc.dynamicSmemBytes = smem;
  lc.stream = b->stream;
  int groups = 0;  // concurrently resident clusters (CTAs for CL = 1)
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

/// FAST, device-assembled systems beyond one SM (T > 191): pcg_kernel_h8s_cl
/// on a cluster of CL CTAs (h8s's register residency, rows split over the
/// cluster). Returns -1 (nothing launched) when the shape does not fit.
template <int CL>
static int launch_h8s_cl(docp_batch* b, const int* list, const int* count, int n_hint, double* sol, double eps,
                         int max_iters) {
  auto kern = pcg_kernel_h8s_cl<CL>;
  const int R = (b->d.nb + CL - 1) / CL;
  const int threads = (2 * R + 31) / 32 * 32;
  if (threads > 256) return -1;
  const size_t smem = h8s_smem_doubles<256, false, false, CL>(b->d) * sizeof(double);
  int max_optin = 0;
  cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, b->device);
  if (smem + 256 > static_cast<size_t>(max_optin)) return -1;
  CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  cudaLaunchConfig_t lc{};
  cudaLaunchAttribute attr[1];
  lc.blockDim = dim3(threads);
  lc.dynamicSmemBytes = smem;
  lc.stream = b->stream;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  lc.gridDim = dim3(CL * b->num_sms);
  int groups = 0;
  CUDA_TRY(cudaOccupancyMaxActiveClusters(&groups, kern, &lc));
  if (groups < 1) return -1;
  lc.gridDim = dim3(CL * std::max(1, std::min(n_hint, groups)));
  CUDA_TRY(cudaMemsetAsync(b->counts + 3, 0, sizeof(int), b->stream));
  ProfScope ps(b, DOCP_PROF_PCG);
  CUDA_TRY(cudaLaunchKernelEx(&lc, kern, b->v, list, count, b->counts + 3, sol, eps, max_iters));
  LAUNCH_CHECK();
  return DOCP_OK;
}

/// Smallest cluster (2 .. 8) for pcg_kernel_h8s_cl: <= 128 block rows (8
/// warps) per CTA, every CTA owning a row, two record regions per CTA in
/// shared memory; 0 if none.
int h8s_cluster_for(const Dims& d, int device) {
  if (d.nx != 8) return 0;
  int max_optin = 0;
  cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  for (int cl = 2; cl <= 8; ++cl) {
    const int R = (d.nb + cl - 1) / cl;
    if ((cl - 1) * R >= d.nb) break;
    if (R > 128) continue;
    const long doubles = 2L * R * 64 + (R + 2) * 8 + (R + 3) * 8 + 3L * 8 * cl;
    if (doubles * 8 + 256 <= static_cast<long>(max_optin)) return cl;
  }
  return 0;
}

/// Whether long-horizon FAST solves of device-assembled systems take the
/// register-resident cluster form over the shared-memory one (h8f): when it
/// needs fewer CTAs per problem, or at two (measured at B = 4,096: T = 200
/// 111K vs 104K problems/s, T = 240 103K vs 69K, T = 320 60K vs 46K; at an
/// equal cluster of 3 or 4 h8f is within +-5 %, ahead at T = 256).
bool h8s_cluster_preferred(const Dims& d, int device) {
  const int cs = h8s_cluster_for(d, device);
  if (cs == 0) return false;
  const int cf = h8f_cluster_for(d, device);
  return cf == 0 || cs < cf || cs == 2;
}

/// FAST, one CTA per problem: pcg_kernel_h8r (-S in registers, next
/// problem's -S prefetched into shared memory).
static int launch_h8r(docp_batch* b, const int* list, const int* count, int n_hint, double* sol, double eps,
                      int max_iters) {
  auto kern = pcg_kernel_h8r<256>;
  const size_t smem = h8r_smem_doubles(b->d) * sizeof(double);
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

/// FAST, one CTA per problem, device-assembled (symmetric) diagonal blocks:
/// pcg_kernel_h8s (both diagonal blocks in registers). Returns -1 (nothing
/// launched) when the variant does not fit this shape.
template <int MAXT, bool PREFETCH, bool SD = false>
static int launch_h8s(docp_batch* b, const int* list, const int* count, int n_hint, double* sol, double eps,
                      int max_iters) {
  auto kern = MAXT == 384 ? (SD ? pcg_kernel_h8s_wide_sd : pcg_kernel_h8s_wide) : pcg_kernel_h8s<MAXT, PREFETCH>;
  const int threads = (2 * b->d.nb + 31) / 32 * 32;
  if (threads > MAXT) return -1;
  const size_t smem = h8s_smem_doubles<MAXT, PREFETCH, SD>(b->d) * sizeof(double);
  int max_optin = 0;
  cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, b->device);
  if (smem + 256 > static_cast<size_t>(max_optin)) return -1;
  CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int per_sm = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
  if (per_sm < 1) return -1;
  const int grid = std::max(1, std::min(n_hint, per_sm * b->num_sms));
  CUDA_TRY(cudaMemsetAsync(b->counts + 3, 0, sizeof(int), b->stream));
  ProfScope ps(b, DOCP_PROF_PCG);
  kern<<<grid, threads, smem, b->stream>>>(b->v, list, count, b->counts + 3, sol, eps, max_iters);
  LAUNCH_CHECK();
  return DOCP_OK;
}

/// PARITY, one CTA per problem, device-assembled (symmetric) diagonal
/// blocks: pcg_kernel_h8p (the reference's arithmetic with h8s's residency).
/// Returns -1 (nothing launched) when the variant does not fit this shape.
/// SDS: -S_ii resident in shared memory instead of the next problem's
/// prefetch (where four record regions fit, T <= 111: C3 243K -> 250K
/// problems/s, the (-S) diagonal product without the partner exchange
/// outweighs the exposed record load).
template <bool PREFETCH>
static int launch_h8p(docp_batch* b, const int* list, const int* count, int n_hint, double* sol, double eps,
                      int max_iters, bool sds = false) {
  // a spare eighth warp folds the block dots (T <= 111; DOCP_PCG_VARIANT=h8p_nocw: every warp does)
  const bool cw = 2 * b->d.nb <= 32 * CW_WARP && !force_variant("h8p_nocw");
  sds = sds && !PREFETCH;
  auto kern = cw ? pcg_kernel_h8p<256, PREFETCH, true> : pcg_kernel_h8p<256, PREFETCH, false>;
  if constexpr (!PREFETCH)
    if (sds) kern = cw ? pcg_kernel_h8p<256, false, true, true> : pcg_kernel_h8p<256, false, false, true>;
  // CW: the block rows' warps plus the fold warp (short horizons launch fewer warps)
  const int threads = (2 * b->d.nb + 31) / 32 * 32 + (cw ? 32 : 0);
  if (threads > 256) return -1;
  const size_t smem = (sds ? h8p_smem_doubles<true>(b->d) : h8p_smem_doubles<PREFETCH>(b->d)) * sizeof(double);
  int max_optin = 0;
  cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, b->device);
  if (smem + 256 > static_cast<size_t>(max_optin)) return -1;
  CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int per_sm = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
  if (per_sm < 1) return -1;
  const int grid = std::max(1, std::min(n_hint, per_sm * b->num_sms));
  CUDA_TRY(cudaMemsetAsync(b->counts + 3, 0, sizeof(int), b->stream));
  ProfScope ps(b, DOCP_PROF_PCG);
  kern<<<grid, threads, smem, b->stream>>>(b->v, list, count, b->counts + 3, sol, eps, max_iters);
  LAUNCH_CHECK();
  return DOCP_OK;
}

/// fp32 mode (n_x = 8): pcg_kernel_h8x, two CTAs per SM up to T = 127, one
/// beyond (T <= 255).
int launch_pcg_fp32_nx8(docp_batch* b, const int* list, const int* count, int n_hint, double* sol, double eps,
                        int max_iters) {
  const int threads = (2 * b->d.nb + 31) / 32 * 32;
  if (threads > 512) return fail(DOCP_UNSUPPORTED, "pcg fp32 mode: horizon %d too long (T <= 255)", b->d.T);
  auto kern = threads <= 256 ? pcg_kernel_h8x<256> : pcg_kernel_h8x<512>;
  const size_t smem = h8x_smem_bytes(b->d, threads);
  CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int per_sm = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
  if (per_sm < 1) return fail(DOCP_UNSUPPORTED, "pcg fp32 mode: kernel does not fit on an SM (smem %zu)", smem);
  const int grid = std::max(1, std::min(n_hint, per_sm * b->num_sms));
  CUDA_TRY(cudaMemsetAsync(b->counts + 3, 0, sizeof(int), b->stream));
  ProfScope ps(b, DOCP_PROF_PCG);
  kern<<<grid, threads, smem, b->stream>>>(b->v, list, count, b->counts + 3, sol, eps, max_iters);
  LAUNCH_CHECK();
  return DOCP_OK;
}

/// The h8p variant for this shape (0: none): 1 = prefetching (T <= 112),
/// 2 = no prefetch (T <= 127).
int h8p_variant_for(const Dims& d, int device) {
  if (d.nx != 8) return 0;
  int max_optin = 0;
  cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  const int threads = (2 * d.nb + 31) / 32 * 32;
  if (threads > 256) return 0;
  if (h8p_smem_doubles<true>(d) * 8 + 256 <= static_cast<long>(max_optin)) return 1;
  if (h8p_smem_doubles<false>(d) * 8 + 256 <= static_cast<long>(max_optin)) return 2;
  return 0;
}

/// The h8s variant for this shape (0: none): 1 = prefetching, 256 threads
/// (T <= 113); 2 = no prefetch, 256 threads (T <= 127); 3 = no prefetch, up
/// to 384 threads at 168 registers (T <= 191).
int h8s_variant_for(const Dims& d, int device) {
  if (d.nx != 8) return 0;
  int max_optin = 0;
  cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  const int threads = (2 * d.nb + 31) / 32 * 32;
  if (threads <= 256 && h8s_smem_doubles<256, true>(d) * 8 + 256 <= static_cast<long>(max_optin)) return 1;
  if (threads <= 256 && h8s_smem_doubles<256, false>(d) * 8 + 256 <= static_cast<long>(max_optin)) return 2;
  if (threads <= 384 && h8s_smem_doubles<384, false, true>(d) * 8 + 256 <= static_cast<long>(max_optin) &&
      !std::getenv("DOCP_H8S_NO_SD"))
    return 4;
  if (threads <= 384 && h8s_smem_doubles<384, false>(d) * 8 + 256 <= static_cast<long>(max_optin)) return 3;
  return 0;
}

/// Smallest cluster (1 .. 8) whose per-CTA share of the blocks fits in
/// shared memory with at most 128 block rows per CTA; 0 if none.
int h8f_cluster_for(const Dims& d, int device) {
  if (d.nx != 8) return 0;
  int max_optin = 0;
  cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  int min_cl = 1;  // DOCP_H8F_CLUSTER=c: A/B override, smallest cluster size tried
  if (const char* e = std::getenv("DOCP_H8F_CLUSTER")) min_cl = std::atoi(e);
  for (int cl : {1, 2, 3, 4, 5, 6, 7, 8}) {
    if (cl > 1 && (cl - 1) * h8f_rows(d, cl) >= d.nb) break;  // every CTA must own a row
    if (cl < min_cl) continue;
    if (h8f_rows(d, cl) <= 128 && h8f_smem_doubles(d, cl, false) * 8 + 64 <= static_cast<long>(max_optin)) return cl;
  }
  return 0;
}
static int h8f_cluster(const docp_batch* b) { return h8f_cluster_for(b->d, b->device); }

/// Kernel variant override for A/B measurements: DOCP_PCG_VARIANT=h8 keeps
/// FAST solves on pcg_kernel_h8.
static bool force_variant(const char* name) {
  const char* e = std::getenv("DOCP_PCG_VARIANT");
  return e && std::strcmp(e, name) == 0;
}
static bool force_h8() { return force_variant("h8"); }

/// n_x = 8: FAST -> pcg_kernel_h8f on the smallest cluster that keeps the
/// blocks on-chip; PARITY (or no fitting cluster): two threads per block row
/// (pcg_kernel_h8) up to T = 255, one thread per block row (pcg_kernel) beyond.
DOCP_PCG_LAUNCHER(launch_pcg_nx8) {
  if (par && b->sym_blocks && !force_h8()) {
    int rc = -1;
    int var = h8p_variant_for(b->d, b->device);
    // where the prefetch form fits, the resident -S form runs instead (A/B:
    // DOCP_PCG_VARIANT=h8p_pf the prefetch form, h8p_np the plain no-prefetch one)
    if (var == 1 && force_variant("h8p_pf")) rc = launch_h8p<true>(b, list, count, n_hint, sol, eps, max_iters);
    else if (var == 1) rc = launch_h8p<false>(b, list, count, n_hint, sol, eps, max_iters, !force_variant("h8p_np"));
    else if (var == 2) rc = launch_h8p<false>(b, list, count, n_hint, sol, eps, max_iters);
    if (rc != -1) return rc;
  }
  if (!par && !force_h8() && b->sym_blocks && !force_variant("h8r") && !force_variant("h8f")) {
    int rc = -1;
    int var = h8s_variant_for(b->d, b->device);
    if (var == 1 && force_variant("h8s_np")) var = 2;  // A/B: the no-prefetch form on a short horizon
    switch (var) {
      case 1: rc = launch_h8s<256, true>(b, list, count, n_hint, sol, eps, max_iters); break;
      case 2: rc = launch_h8s<256, false>(b, list, count, n_hint, sol, eps, max_iters); break;
      case 3: rc = launch_h8s<384, false>(b, list, count, n_hint, sol, eps, max_iters); break;
      case 4: rc = launch_h8s<384, false, true>(b, list, count, n_hint, sol, eps, max_iters); break;
      default: break;
    }
    if (rc != -1) return rc;
    // beyond one SM: the same residency on a thread-block cluster (DOCP_PCG_VARIANT=h8f: the
    // shared-memory cluster form instead)
    if (var == 0 && !force_variant("h8f_cl") && h8s_cluster_preferred(b->d, b->device)) {
      switch (h8s_cluster_for(b->d, b->device)) {
        case 2: rc = launch_h8s_cl<2>(b, list, count, n_hint, sol, eps, max_iters); break;
        case 3: rc = launch_h8s_cl<3>(b, list, count, n_hint, sol, eps, max_iters); break;
        case 4: rc = launch_h8s_cl<4>(b, list, count, n_hint, sol, eps, max_iters); break;
        case 5: rc = launch_h8s_cl<5>(b, list, count, n_hint, sol, eps, max_iters); break;
        case 6: rc = launch_h8s_cl<6>(b, list, count, n_hint, sol, eps, max_iters); break;
        case 7: rc = launch_h8s_cl<7>(b, list, count, n_hint, sol, eps, max_iters); break;
        case 8: rc = launch_h8s_cl<8>(b, list, count, n_hint, sol, eps, max_iters); break;
        default: break;
      }
      if (rc != -1) return rc;
    }
  }
  if (!par && !force_h8()) {
    switch (h8f_cluster(b)) {
      case 1:
        if (force_variant("h8f")) return launch_h8f_cl<1>(b, list, count, n_hint, sol, eps, max_iters);
        return launch_h8r(b, list, count, n_hint, sol, eps, max_iters);
      case 2: return launch_h8f_cl<2>(b, list, count, n_hint, sol, eps, max_iters);
      case 3: return launch_h8f_cl<3>(b, list, count, n_hint, sol, eps, max_iters);
      case 4: return launch_h8f_cl<4>(b, list, count, n_hint, sol, eps, max_iters);
      case 5: return launch_h8f_cl<5>(b, list, count, n_hint, sol, eps, max_iters);
      case 6: return launch_h8f_cl<6>(b, list, count, n_hint, sol, eps, max_iters);
      case 7: return launch_h8f_cl<7>(b, list, count, n_hint, sol, eps, max_iters);
      case 8: return launch_h8f_cl<8>(b, list, count, n_hint, sol, eps, max_iters);
      default: break;
    }
  }
  if (2 * b->d.nb <= 512) {
    if (par) return pl.resident ? launch_h8<true, true>(b, pl, list, count, n_hint, sol, eps, max_iters)
                                : launch_h8<true, false>(b, pl, list, count, n_hint, sol, eps, max_iters);
    return pl.resident ? launch_h8<false, true>(b, pl, list, count, n_hint, sol, eps, max_iters)
                       : launch_h8<false, false>(b, pl, list, count, n_hint, sol, eps, max_iters);
  }
  return launch_pcg_nx<8>(b, pl, par, list, count, n_hint, sol, eps, max_iters);
}

}  // namespace docp_host

#ifdef DOCP_H8P_CLOCK
/// A/B builds only: cycles of pcg_kernel_h8p's thread 0 per phase, summed over launches (then reset).
extern "C" int docp_h8p_clock(unsigned long long* out) {
  if (cudaMemcpyFromSymbol(out, docp_dev::g_h8p_clk, 16 * sizeof(unsigned long long)) != cudaSuccess) return 1;
  static const unsigned long long zero[16] = {0};
  return cudaMemcpyToSymbol(docp_dev::g_h8p_clk, zero, sizeof zero) != cudaSuccess;
}
#endif

#ifdef DOCP_H8S_CLOCK
/// A/B builds only: cycles of pcg_kernel_h8s's thread 0 per phase, summed over launches (then reset).
extern "C" int docp_h8s_clock(unsigned long long* out) {
  if (cudaMemcpyFromSymbol(out, docp_dev::g_h8s_clk, 16 * sizeof(unsigned long long)) != cudaSuccess) return 1;
  static const unsigned long long zero[16] = {0};
  return cudaMemcpyToSymbol(docp_dev::g_h8s_clk, zero, sizeof zero) != cudaSuccess;
}
#endif
