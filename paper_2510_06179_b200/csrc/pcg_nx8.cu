// pcg_nx8.cu — K2 instantiations for n_x = 8 (separate translation unit for build parallelism)
#include "pcg_launch.cuh"

namespace docp_host {
DOCP_PCG_LAUNCHER(launch_pcg_nx8) { return launch_pcg_nx<8>(b, pl, par, list, count, n_hint, sol, eps, max_iters); }
}  // namespace docp_host
