// families.cuh — device problem families (the OcpDefinition callbacks of
// the reference, which cannot cross to the GPU as std::function).
//
// Every expression keeps the reference's evaluation order so that, compiled
// with --fmad=false, stage values are bit-identical to the reference headers
// (cart-pole's sin/cos aside: crmath.cuh's are correctly rounded; glibc's
// misround ~0.1% of arguments by one ulp).
#pragma once

#include "common.cuh"
#include "crmath.cuh"
#include "docp_drift_model.h"

namespace docp_dev {

/// Diagonal quadratic stage cost  scale * v' diag(w) v
/// (affine_quadratic.hpp:47-64, quadratic_cost.hpp:9-20). Returns the value;
/// grad_i = ((2 scale) w_i) v_i and hess = diag((2 scale) w_i).
template <int N = 0>
__device__ inline double diag_cost_value(double scale, const double* w, const double* v, int n_rt) {
  const int n = N ? N : n_rt;
  double acc = v[0] * (w[0] * v[0]);
#pragma unroll
  for (int i = 1; i < n; ++i) acc = acc + v[i] * (w[i] * v[i]);
  return scale * acc;
}
__device__ inline double diag_cost_grad(double scale, double w, double v) { return ((2.0 * scale) * w) * v; }
__device__ inline double diag_cost_hess(double scale, double w) { return (2.0 * scale) * w; }

/// The drifting family's residual and Jacobians, out of line: its dual-number
/// evaluation needs a large stack frame that must not inflate the kernels
/// (step, KKT, linearize) for the families that never call it.
__device__ __noinline__ void drift_dynamics(const double* th, double dt, const double* xn, const double* x,
                                            const double* u, double* res, double* jx, double* ju) {
  double xn_[docp_drift::NX], jxx[docp_drift::NX * docp_drift::NX], juu[docp_drift::NX * docp_drift::NU];
  docp_drift::step(th, dt, x, u, xn_, jx ? jxx : nullptr, ju ? juu : nullptr);
  for (int i = 0; i < docp_drift::NX; ++i) res[i] = xn[i] - xn_[i];
  if (jx)
    for (int k = 0; k < docp_drift::NX * docp_drift::NX; ++k) jx[k] = -jxx[k];
  if (ju)
    for (int k = 0; k < docp_drift::NX * docp_drift::NU; ++k) ju[k] = -juu[k];
}

struct Family {
  int kind;
  double scale;
  double cart_mass, pole_mass, length, gravity, dt;

  __host__ __device__ static Family from(const docp_problem& p) {
    Family f;
    f.kind = p.family;
    f.scale = p.family == DOCP_AFFINE_QUADRATIC ? p.cost_scale : 0.5;  // quadratic_cost scale 0.5
    f.cart_mass = p.cart_mass;
    f.pole_mass = p.pole_mass;
    f.length = p.length;
    f.gravity = p.gravity;
    f.dt = p.dt;
    return f;
  }

  __device__ const double* w_x(const Dims&, const double* th) const { return th; }
  __device__ const double* w_u(const Dims& d, const double* th) const { return th + d.nx; }
  /// initial_state(theta)
  __device__ const double* x_s(const Dims& d, const double* th) const {
    if (kind != DOCP_AFFINE_QUADRATIC) return th + d.nx + d.nu;  // [w_x | w_u | x_0 (| ...)]
    return th + d.nx + d.nu + d.nx * d.nx + d.nx * d.nu + d.nx;
  }

  /// Dynamics residual f = x+ - phi(x, u) and its Jacobians (jac_x_next = I).
  /// res[nx]; jx[nx*nx], ju[nx*nu] column-major (may be null). NX, NU > 0
  /// fix the sizes at compile time (same arithmetic, unrolled).
  /// DRIFT: whether the drifting family's branch is compiled in. Only the
  /// runtime-shape kernels (NX = 0) carry it; the launchers route DOCP_DRIFT
  /// to them, so the compile-time-shape kernels of the other families keep
  /// their register budgets (the model's dual-number Jacobians need ~255).
  template <int NX = 0, int NU = 0, bool DRIFT = (NX == 0)>
  __device__ void dynamics(const Dims& d, const double* th, const double* xn, const double* x, const double* u,
                           double* res, double* jx, double* ju) const {
    const int nx = NX ? NX : d.nx, nu = NU ? NU : d.nu;
    if (kind == DOCP_AFFINE_QUADRATIC) {  // affine_quadratic.hpp:65-75
      const double* a = th + nx + nu;
      const double* b = a + nx * nx;
      const double* off = b + nx * nu;
#pragma unroll
      for (int i = 0; i < nx; ++i) {
        double ax = a[i] * x[0];
#pragma unroll
        for (int k = 1; k < nx; ++k) ax = ax + a[i + k * nx] * x[k];
        double bu = b[i] * u[0];
#pragma unroll
        for (int k = 1; k < nu; ++k) bu = bu + b[i + k * nx] * u[k];
        res[i] = ((xn[i] - ax) - bu) - off[i];
      }
      if (jx)
        for (int k = 0; k < nx * nx; ++k) jx[k] = -a[k];
      if (ju)
        for (int k = 0; k < nx * nu; ++k) ju[k] = -b[k];
      return;
    }
    if constexpr (DRIFT) {
      if (kind == DOCP_DRIFT) {  // make_explicit_dynamics(docp_drift::step): the shared model definition
        drift_dynamics(th, dt, xn, x, u, res, jx, ju);
        return;
      }
    }
    if (kind == DOCP_ATTITUDE) {  // make_explicit_dynamics(attitude_step), attitude.hpp:16-42
      const double* in = th + 9;   // AttitudeParams::inertia (THETA tail)
      double jw[3], h[3], ji[3], xn_[3];
      for (int i = 0; i < 3; ++i) jw[i] = in[i] * x[i];
      h[0] = jw[1] * x[2] - jw[2] * x[1];  // jw.cross(w)
      h[1] = jw[2] * x[0] - jw[0] * x[2];
      h[2] = jw[0] * x[1] - jw[1] * x[0];
      for (int i = 0; i < 3; ++i) ji[i] = 1.0 / in[i];
      for (int i = 0; i < 3; ++i) xn_[i] = x[i] + dt * (ji[i] * (h[i] + u[i]));
      for (int i = 0; i < 3; ++i) res[i] = xn[i] - xn_[i];
      if (jx) {  // jac_x = I + (dt j_inv) .* (skew(jw) - skew(w) diag(J)), negated
        double sj[9], sw[9];  // row-major skew matrices (attitude.hpp:16-20)
        auto skew = [](const double* v, double* m) {
          m[0] = 0.0, m[1] = -v[2], m[2] = v[1];
          m[3] = v[2], m[4] = 0.0, m[5] = -v[0];
          m[6] = -v[1], m[7] = v[0], m[8] = 0.0;
        };
        skew(jw, sj);
        skew(x, sw);
        for (int i = 0; i < 3; ++i)
          for (int k = 0; k < 3; ++k) {
            const double dh = sj[3 * i + k] - sw[3 * i + k] * in[k];
            jx[i + 3 * k] = -((i == k ? 1.0 : 0.0) + (dt * ji[i]) * dh);
          }
      }
      if (ju)
        for (int i = 0; i < 3; ++i)
          for (int k = 0; k < 3; ++k) ju[i + 3 * k] = -(dt * (i == k ? ji[i] : 0.0));
      return;
    }
    // cart-pole: make_explicit_dynamics(cartpole_step), cartpole.hpp:28-78
    double sn, c;  // correctly rounded (crmath.cuh): glibc-equivalent except at its rare misroundings
    crmath::sincos_cr(x[2], &sn, &c);
    const double mp = pole_mass;
    const double len = length;
    const double g = gravity;
    const double big_m = cart_mass + pole_mass;
    const double dd = big_m + mp * (1.0 - c * c);
    const double xd1 = (-mp * len * sn * x[3] * x[3] + mp * g * sn * c) / (dd * len);
    const double xd3 = (-mp * len * sn * x[3] + mp * g * sn * c + u[0]) / dd;
    res[0] = xn[0] - (x[0] + dt * x[1]);
    res[1] = xn[1] - (x[1] + dt * xd1);
    res[2] = xn[2] - (x[2] + dt * x[3]);
    res[3] = xn[3] - (x[3] + dt * xd3);
    if (jx) {
      const double d_d3 = 2.0 * mp * sn * c;
      const double n2 = -mp * len * sn * x[3] * x[3] + mp * g * sn * c;
      const double n2_d3 = -mp * len * c * x[3] * x[3] + mp * g * (c * c - sn * sn);
      const double n2_d4 = -2.0 * mp * len * sn * x[3];
      const double n4 = -mp * len * sn * x[3] + mp * g * sn * c + u[0];
      const double n4_d3 = -mp * len * c * x[3] + mp * g * (c * c - sn * sn);
      const double n4_d4 = -mp * len * sn;
      double J[16];
      for (int k = 0; k < 16; ++k) J[k] = 0.0;
      J[0 + 1 * 4] = 1.0;
      J[1 + 2 * 4] = (n2_d3 * dd - n2 * d_d3) / (dd * dd * len);
      J[1 + 3 * 4] = n2_d4 / (dd * len);
      J[2 + 3 * 4] = 1.0;
      J[3 + 2 * 4] = (n4_d3 * dd - n4 * d_d3) / (dd * dd);
      J[3 + 3 * 4] = n4_d4 / dd;
      for (int j = 0; j < 4; ++j)
        for (int i = 0; i < 4; ++i) jx[i + j * 4] = -((i == j ? 1.0 : 0.0) + dt * J[i + j * 4]);
    }
    if (ju) {
      ju[0] = -(dt * 0.0);
      ju[1] = -(dt * 0.0);
      ju[2] = -(dt * 0.0);
      ju[3] = -(dt * (1.0 / dd));
    }
  }
};

}  // namespace docp_dev
