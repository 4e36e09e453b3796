// pcg_nxct.cu — K2 instantiations of the one-thread-per-block-row kernel
// (k_pcg.cuh) at compile-time n_x for the shapes between the specialised
// ones: n_x = 6 and 9 (the drifting shape of SURVEY.md §8(d) C4), where the
// runtime-n_x kernel's loops cannot unroll (separate translation unit for
// build parallelism).
#include "pcg_launch.cuh"

namespace docp_host {
DOCP_PCG_LAUNCHER(launch_pcg_nx6) { return launch_pcg_nx<6>(b, pl, par, list, count, n_hint, sol, eps, max_iters); }
DOCP_PCG_LAUNCHER(launch_pcg_nx9) { return launch_pcg_nx<9>(b, pl, par, list, count, n_hint, sol, eps, max_iters); }
}  // namespace docp_host
