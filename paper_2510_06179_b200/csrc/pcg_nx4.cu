// pcg_nx4.cu — K2 instantiations for n_x = 4 (separate translation unit for build parallelism)
#include "pcg_launch.cuh"

namespace docp_host {
DOCP_PCG_LAUNCHER(launch_pcg_nx4) { return launch_pcg_nx<4>(b, pl, par, list, count, n_hint, sol, eps, max_iters); }
}  // namespace docp_host
