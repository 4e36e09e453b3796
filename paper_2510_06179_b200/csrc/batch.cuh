// batch.cuh — the device-resident batch object and the host launch helpers
// shared by the translation units of libdocp_cuda.so.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"

namespace docp_host {

extern std::atomic<uint64_t> g_launches;
int fail(int code, const char* fmt, ...);

}  // namespace docp_host

#define CUDA_TRY(expr)                                                                                   \
  do {                                                                                                   \
    cudaError_t e_ = (expr);                                                                             \
    if (e_ != cudaSuccess) return docp_host::fail(DOCP_CUDA_ERROR, "%s: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)

#define LAUNCH_CHECK()                                                                                   \
  do {                                                                                                   \
    docp_host::g_launches.fetch_add(1, std::memory_order_relaxed);                                       \
    cudaError_t e_ = cudaGetLastError();                                                                 \
    if (e_ != cudaSuccess) return docp_host::fail(DOCP_CUDA_ERROR, "kernel launch: %s", cudaGetErrorString(e_)); \
  } while (0)

struct docp_batch {
  docp_problem prob{};
  docp_dev::Dims d{};
  int B = 0;
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  docp_dev::View v{};
  // work lists: all problems, and two ping-pong active lists
  int* all_list = nullptr;
  int* list[2] = {nullptr, nullptr};
  int* counts = nullptr;  // [0] all, [1] list0, [2] list1, [3] pcg queue counter
  int* h_count = nullptr; // pinned
  std::vector<void*> allocs;
  int max_hist = 0;
  double last_eps_pd = 1e-6;
  // the stored diagonal blocks are exactly symmetric (assembled on the device,
  // schur.hpp:145-164); uploaded systems may not be (pcg_kernel_h8s needs it)
  bool sym_blocks = false;
  // rollout record (docp_rollout / docp_rollout_backward), grown on demand
  docp_dev::RolloutRec roll{};
  int roll_cap = -1;  // episode steps the record holds
  double roll_eps_pd = 1e-6;
  // CUDA graphs of whole rollouts, replayed while their arguments and the
  // batch's buffers (layout_gen) are unchanged
  struct GraphCache {
    cudaGraphExec_t exec = nullptr;
    std::vector<char> key;
    uint64_t launches = 0;
  };
  GraphCache graph_fwd, graph_bwd;  // rollouts
  GraphCache graph_solve, graph_vjp;  // sqp_solve (<= 4 iterations), backward_vjp
  uint64_t layout_gen = 0;  // bumped whenever a device buffer is reallocated
  // profiling: CUDA events around every launch, per kernel kind, on the batch stream
  bool profiling = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof[DOCP_PROF_KINDS];
  struct ProfRec {
    int kind;
    cudaEvent_t start, stop;
  };
  std::vector<ProfRec> prof_seq;  // every profiled launch in stream order
  std::vector<cudaEvent_t> event_pool;
  size_t pool_used = 0;

  ~docp_batch() {
    if (graph_fwd.exec) cudaGraphExecDestroy(graph_fwd.exec);
    if (graph_bwd.exec) cudaGraphExecDestroy(graph_bwd.exec);
    if (graph_solve.exec) cudaGraphExecDestroy(graph_solve.exec);
    if (graph_vjp.exec) cudaGraphExecDestroy(graph_vjp.exec);
    for (cudaEvent_t e : event_pool) cudaEventDestroy(e);
    for (void* p : allocs) cudaFree(p);
    if (h_count) cudaFreeHost(h_count);
  }
};

namespace docp_host {

inline int grid_for(long items, int threads, int cap_blocks = 1 << 20) {
  long g = (items + threads - 1) / threads;
  return static_cast<int>(std::max<long>(1, std::min<long>(g, cap_blocks)));
}

inline cudaEvent_t pool_event(docp_batch* b) {
  if (b->pool_used == b->event_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    b->event_pool.push_back(e);
  }
  return b->event_pool[b->pool_used++];
}

/// RAII scope recording a (start, stop) event pair around one launch.
struct ProfScope {
  docp_batch* b;
  int kind;
  cudaEvent_t stop = nullptr;
  ProfScope(docp_batch* bb, int k) : b(bb), kind(k) {
    if (!b->profiling) return;
    cudaEvent_t start = pool_event(b);
    stop = pool_event(b);
    cudaEventRecord(start, b->stream);
    b->prof[kind].emplace_back(start, stop);
    b->prof_seq.push_back({kind, start, stop});
  }
  ~ProfScope() {
    if (stop) cudaEventRecord(stop, b->stream);
  }
};

struct PcgPlan {
  bool resident;
  int threads;
  int maxr;
  size_t smem;
};

// per-block-size PCG launchers (pcg_nx*.cu, compiled in parallel)
#define DOCP_PCG_LAUNCHER(name)                                                                                \
  int name(docp_batch* b, const PcgPlan& pl, bool par, const int* list, const int* count, int n_hint, double* sol, \
           double eps, int max_iters)
DOCP_PCG_LAUNCHER(launch_pcg_nx4);
/// Whether FAST n_x = 4 solves of this shape run pcg_kernel_h4f.
bool h4f_fits(const docp_dev::Dims& d, int device);
DOCP_PCG_LAUNCHER(launch_pcg_nx16);
int h16f_cluster_for(const docp_dev::Dims& d, int device);
/// Cluster size pcg_kernel_h8f uses for this batch's shape (0: not used).
int h8f_cluster_for(const docp_dev::Dims& d, int device);
/// pcg_kernel_h8s variant for a device-assembled system (0: none; 1: T <= 113; 2: T <= 127; 3: T <= 191).
int h8s_variant_for(const docp_dev::Dims& d, int device);
int h8s_cluster_for(const docp_dev::Dims& d, int device);
bool h8s_cluster_preferred(const docp_dev::Dims& d, int device);
/// pcg_kernel_h8p (PARITY) variant for a device-assembled system (0: none; 1: prefetching; 2: no prefetch).
int h8p_variant_for(const docp_dev::Dims& d, int device);
DOCP_PCG_LAUNCHER(launch_pcg_nx8);
/// The fp32 mode's K2 (pcg_kernel_h8x, n_x = 8).
int launch_pcg_fp32_nx8(docp_batch* b, const int* list, const int* count, int n_hint, double* sol, double eps,
                        int max_iters);
DOCP_PCG_LAUNCHER(launch_pcg_nxrt);
DOCP_PCG_LAUNCHER(launch_pcg_nx6);
DOCP_PCG_LAUNCHER(launch_pcg_nx9);

}  // namespace docp_host
