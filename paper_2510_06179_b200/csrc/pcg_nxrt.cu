// pcg_nxrt.cu — K2 instantiations for n_x (any, runtime loops) (separate translation unit for build parallelism)
#include "pcg_launch.cuh"

namespace docp_host {
DOCP_PCG_LAUNCHER(launch_pcg_nxrt) { return launch_pcg_nx<0>(b, pl, par, list, count, n_hint, sol, eps, max_iters); }
}  // namespace docp_host
