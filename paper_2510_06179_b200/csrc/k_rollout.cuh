// k_rollout.cuh — closed-loop MPC rollouts on the device:
// the per-step glue of docp::rollout / rollout_backward (batch.hpp:172-258)
// with the benchmark tasks' environments: each instance steps its own
// dynamics x' = phi(x, u) (explicit step of the family; the affine family's
// x' = A x + B u + b) with reward R(x', u) = -(w_r |x'|^2 + |u|^2), w_r = 1
// for the affine task (make_affine_env, train.hpp:195-213) and 0.1 for the
// attitude task (make_attitude_rl_task, train.hpp:239-263).
// The solves themselves are the batched K1-K4 path; these kernels only move
// states between steps, apply the environment, and chain the cotangents. One
// warp per instance; lane 0 does the n_x-sized arithmetic in the reference's
// expression order, all lanes copy trajectories.
#pragma once

#include "families.cuh"

namespace docp_dev {

__device__ inline int xs_off(const Dims& d, const Family& fam) {
  return fam.kind == DOCP_AFFINE_QUADRATIC ? d.nx + d.nu + d.nx * d.nx + d.nx * d.nu + d.nx : d.nx + d.nu;
}
/// Reward weight on |x'|^2 of the family's RL task.
__device__ inline double reward_wx(const Family& fam) { return fam.kind == DOCP_ATTITUDE ? 0.1 : 1.0; }
/// x' = phi(x, u): the explicit step, as -f(x' = 0, x, u) (exact: the
/// residual is 0 - phi, every family's phi(x,u) is evaluated as in its step).
__device__ inline void env_step(const Dims& d, const Family& fam, const double* th, const double* x, const double* u,
                                double* xn) {
  double zero[kMaxNx], res[kMaxNx];
  for (int i = 0; i < d.nx; ++i) zero[i] = 0.0;
  fam.dynamics<0, 0, false>(d, th, zero, x, u, res, nullptr, nullptr);
  for (int i = 0; i < d.nx; ++i) xn[i] = -res[i];
}

/// Step 0: x_0 = x_init, zero warm starts, everything alive.
__global__ void rollout_init_kernel(View v, RolloutRec rr, const double* __restrict__ x_init) {
  const Dims d = v.d;
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < v.B; p += warps) {
    for (int e = lane; e < d.nz; e += 32) v.z[static_cast<long>(p) * d.nz + e] = 0.0;
    for (int e = lane; e < d.nl; e += 32) v.lam[static_cast<long>(p) * d.nl + e] = 0.0;
    if (x_init != rr.x)  // (docp_rollout stages x_init in the record already)
      for (int e = lane; e < d.nx; e += 32) rr.x[static_cast<long>(p) * d.nx + e] = x_init[static_cast<long>(p) * d.nx + e];
    if (lane == 0) {
      rr.reward[p] = 0.0;
      rr.alive[p] = 1;
      set_status(rr.rstat + p, DOCP_OK, DOCP_AT_NONE, 0);
    }
  }
}

/// Before the step-t solve: THETA's initial-state segment <- x_t
/// (step_theta.set_segment, batch.hpp:183). Truncated instances get a
/// non-finite initial guess so every kernel of the solve skips them.
__global__ void rollout_pre_kernel(View v, RolloutRec rr, int t) {
  const Dims d = v.d;
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int xs = xs_off(d, Family::from(v.prob));
  for (int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < v.B; p += warps) {
    const double* xt = rr.x + (static_cast<long>(t) * v.B + p) * d.nx;
    if (rr.alive[p]) {
      for (int e = lane; e < d.nx; e += 32) v.theta[static_cast<long>(p) * d.nth + xs + e] = xt[e];
    } else if (lane == 0) {
      v.z[static_cast<long>(p) * d.nz] = __longlong_as_double(0x7ff8000000000000ll);  // NaN
    }
  }
}

/// After the step-t solve (batch.hpp:185-208): truncate on a failed solve,
/// apply u_0, step the environment, accumulate the reward, record the step.
__global__ void rollout_post_kernel(View v, RolloutRec rr, int t) {
  const Dims d = v.d;
  const int nx = d.nx, nu = d.nu;
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < v.B; p += warps) {
    if (!rr.alive[p]) continue;
    const docp_status st = v.status[p];
    if (st.code != DOCP_OK) {  // RolloutTruncation "rollout: solve failed at step t: ..."
      if (lane == 0) {
        rr.rstat[p] = st;
        rr.rstat[p].step = t + 1;
        rr.alive[p] = 0;
      }
      continue;
    }
    const double* z = v.z + static_cast<long>(p) * d.nz;
    const double* x = rr.x + (static_cast<long>(t) * v.B + p) * nx;
    double* xn = rr.x + (static_cast<long>(t + 1) * v.B + p) * nx;
    double* u = rr.u + (static_cast<long>(t) * v.B + p) * nu;
    if (lane == 0) {
      const Family fam = Family::from(v.prob);
      const double* th = v.theta + static_cast<long>(p) * d.nth;
      double uu[kMaxNu], xv[kMaxNx];
      for (int i = 0; i < nu; ++i) uu[i] = z[uoff(d, 0) + i];  // policy_first_control (sqp.hpp:264-266)
      env_step(d, fam, th, x, uu, xv);
      bool fin = true;
      double sx = 0.0;
      for (int i = 0; i < nx; ++i) {
        xn[i] = xv[i];
        fin = fin && isfinite(xv[i]);
        sx = i == 0 ? xv[i] * xv[i] : sx + xv[i] * xv[i];
      }
      double su = uu[0] * uu[0];
      for (int i = 1; i < nu; ++i) su = su + uu[i] * uu[i];
      for (int i = 0; i < nu; ++i) u[i] = uu[i];
      if (!fin) {
        set_status(rr.rstat + p, DOCP_DIVERGENCE, DOCP_AT_ROLLOUT_ENV, t);
        rr.alive[p] = 0;
      } else {
        rr.reward[p] = rr.reward[p] + (-(reward_wx(fam) * sx + su));
      }
    }
    // record the step's solution (warm_z / warm_lambda stay in Z, LAMBDA)
    double* rz = rr.z + (static_cast<long>(t) * v.B + p) * d.nz;
    double* rl = rr.lam + (static_cast<long>(t) * v.B + p) * d.nl;
    const double* lam = v.lam + static_cast<long>(p) * d.nl;
    for (int e = lane; e < d.nz; e += 32) rz[e] = z[e];
    for (int e = lane; e < d.nl; e += 32) rl[e] = lam[e];
  }
}

/// Backward, before step t's adjoint solve (batch.hpp:235-248): reward and
/// environment cotangents, the loss gradient on u_0, and the step's
/// linearisation point (THETA's initial state, Z, LAMBDA) restored.
/// Instances that are not alive get a failing status and are not listed.
__global__ void rollout_back_pre_kernel(View v, RolloutRec rr, int t, int* __restrict__ list,
                                        int* __restrict__ count) {
  const Dims d = v.d;
  const int nx = d.nx, nu = d.nu;
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const Family fam = Family::from(v.prob);
  const int xs = xs_off(d, fam);
  for (int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < v.B; p += warps) {
    if (!rr.alive[p]) {
      if (lane == 0) set_status(v.status + p, DOCP_DIVERGENCE, DOCP_AT_ROLLOUT_ENV, -1);
      continue;
    }
    const double* x = rr.x + (static_cast<long>(t) * v.B + p) * nx;
    const double* xn = rr.x + (static_cast<long>(t + 1) * v.B + p) * nx;
    const double* u = rr.u + (static_cast<long>(t) * v.B + p) * nu;
    double* lg = v.lgz + static_cast<long>(p) * d.nz;
    double* th = v.theta + static_cast<long>(p) * d.nth;
    for (int e = lane; e < d.nz; e += 32) lg[e] = 0.0;
    for (int e = lane; e < nx; e += 32) th[xs + e] = x[e];
    const double* rz = rr.z + (static_cast<long>(t) * v.B + p) * d.nz;
    const double* rl = rr.lam + (static_cast<long>(t) * v.B + p) * d.nl;
    for (int e = lane; e < d.nz; e += 32) v.z[static_cast<long>(p) * d.nz + e] = rz[e];
    for (int e = lane; e < d.nl; e += 32) v.lam[static_cast<long>(p) * d.nl + e] = rl[e];
    __syncwarp();
    if (lane == 0) {
      // step_vjp: the step's Jacobians (dphi/dx, dphi/du) = -(jac_x, jac_u) of the residual
      double jx[kMaxNx * kMaxNx], ju[kMaxNx * kMaxNu], res[kMaxNx];
      fam.dynamics<0, 0, false>(d, th, xn, x, u, res, jx, ju);
      double* xbar = rr.xbar + static_cast<long>(p) * nx;
      double* ex = rr.ex + static_cast<long>(p) * nx;
      const double rx = fam.kind == DOCP_ATTITUDE ? -0.2 : -2.0;  // reward_grad (train.hpp:208-211, 254-257)
      double cot[kMaxNx];
      for (int i = 0; i < nx; ++i) cot[i] = xbar[i] + (rx * xn[i]);  // xbar + r_x
      for (int k = 0; k < nx; ++k) {  // e_x = jac_x' cot
        double s = (-jx[k * nx]) * cot[0];
        for (int i = 1; i < nx; ++i) s = s + (-jx[i + k * nx]) * cot[i];
        ex[k] = s;
      }
      for (int k = 0; k < nu; ++k) {  // ubar = r_u + jac_u' cot
        double s = (-ju[k * nx]) * cot[0];
        for (int i = 1; i < nx; ++i) s = s + (-ju[i + k * nx]) * cot[i];
        lg[uoff(d, 0) + k] = (-2.0 * u[k]) + s;
      }
      list[atomicAdd(count, 1)] = p;
      set_status(v.status + p, DOCP_OK, DOCP_AT_NONE, 0);
    }
  }
}

/// Backward, after step t's adjoint solve: the policy's x-cotangent from the
/// initial-state segment, the rest accumulated (batch.hpp:249-254).
__global__ void rollout_back_post_kernel(View v, RolloutRec rr, int t) {
  const Dims d = v.d;
  const int nx = d.nx;
  const int xs = xs_off(d, Family::from(v.prob));
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < v.B; p += gridDim.x * blockDim.x) {
    if (!rr.alive[p]) continue;
    const docp_status st = v.status[p];
    if (st.code != DOCP_OK) {  // the reference's rollout_backward would throw
      rr.rstat[p] = st;
      rr.alive[p] = 0;
      continue;
    }
    const double* g = v.grad + static_cast<long>(p) * d.nth;
    double* gt = rr.gtot + static_cast<long>(p) * d.nth;
    double* xbar = rr.xbar + static_cast<long>(p) * nx;
    const double* ex = rr.ex + static_cast<long>(p) * nx;
    for (int k = 0; k < d.nth; ++k)
      if (k < xs || k >= xs + nx) gt[k] = gt[k] + g[k];
      else gt[k] = gt[k] + 0.0;  // the segment is zeroed before the sum
    for (int i = 0; i < nx; ++i) xbar[i] = ex[i] + g[xs + i];
  }
}

/// Backward start (zero cotangents and sums, lambda~ = 0) and end (the
/// initial-state segment of the gradient = xbar; GRAD_THETA <- the sums).
__global__ void rollout_back_init_kernel(View v, RolloutRec rr) {
  const Dims d = v.d;
  for (long g = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; g < static_cast<long>(v.B) * d.nth;
       g += static_cast<long>(gridDim.x) * blockDim.x)
    rr.gtot[g] = 0.0;
  for (long g = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; g < static_cast<long>(v.B) * d.nx;
       g += static_cast<long>(gridDim.x) * blockDim.x)
    rr.xbar[g] = 0.0;
  for (long g = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; g < static_cast<long>(v.B) * d.nl;
       g += static_cast<long>(gridDim.x) * blockDim.x)
    v.lt[g] = 0.0;
}

__global__ void rollout_back_fini_kernel(View v, RolloutRec rr) {
  const Dims d = v.d;
  const int xs = xs_off(d, Family::from(v.prob));
  for (long g = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; g < static_cast<long>(v.B) * d.nth;
       g += static_cast<long>(gridDim.x) * blockDim.x) {
    const int p = static_cast<int>(g / d.nth), k = static_cast<int>(g % d.nth);
    double val = rr.gtot[g];
    if (k >= xs && k < xs + d.nx) val = rr.xbar[static_cast<long>(p) * d.nx + (k - xs)];
    v.grad[g] = rr.alive[p] ? val : 0.0;
  }
}

}  // namespace docp_dev
