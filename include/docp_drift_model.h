/* docp_drift_model.h — the drifting family (DOCP_DRIFT) of SURVEY.md §8(f)5:
 * a dynamic bicycle model with coupled-slip brush (Fiala) tires in path
 * coordinates, augmented with its controls and
 * discretised by Heun's (explicit trapezoidal) rule in 4 sub-steps. The rear
 * wheel speed is taken quasi-static (the drive torque sets the rear tire's
 * longitudinal force; its coupled-slip effect is the friction-circle limit
 * on the lateral force): with the paper's tire stiffnesses the wheel-speed
 * mode (~ r_w^2 C_r / (V I_w) ~ 250 / s) is far too stiff for an explicit
 * step, and the reference's OCP form (make_explicit_dynamics, A+ = I) has no
 * implicit one.
 *
 * The reference ships NO implementation of this model (PAPER.md gives the
 * states, parameters and cost, not the tire equations; SURVEY.md §8(d) C4:
 * "parity unpinned"). This header is therefore the model's single
 * definition: it is compiled into the GPU path (csrc/families.cuh, device)
 * and into the reference-solver harness (oracle/ref_driver.cpp, host), so the
 * parity tests pin the SOLVER (the reference's sqp_solve / backward_vjp on
 * these callbacks) bit for bit; the model itself is not reference-backed.
 * Every function uses only +, -, *, / and sqrt (IEEE correctly rounded on
 * both sides; the library is built with --fmad=false, the harness with
 * -ffp-contract=off) and its own sin/cos, so host and device agree bitwise.
 *
 *   state  X = (r, V, beta, dphi, e, s, delta, F_x)   n_x = 8
 *          yaw rate, speed, sideslip, heading error, lateral error, path
 *          distance, steering angle, rear drive force (kN; torque / r_w)
 *   control u = (d delta / dt, d F_x / dt)                     n_u = 2
 *   OCP state: the deviation xbar = X - X_ref from a reference drift state,
 *          so the diagonal quadratic cost of the reference (quadratic_cost.hpp)
 *          tracks X_ref: c = 1/2 xbar' diag(w_x) xbar, 1/2 u' diag(w_u) u.
 *   theta  [w_x (8) | w_u (2) | xbar_0 (8) | X_ref (8) | a, b, m, I_z, r_w,
 *          C_f, C_r, mu_f, mu_r, kappa (10)]                    n_theta = 36
 *          dtheta covers the cost weights and xbar_0 (the reference's
 *          make_quadratic_cost_theta_vjp); the vehicle parameters are
 *          per-instance (domain-randomised) data with zero gradient.
 */
#ifndef DOCP_DRIFT_MODEL_H
#define DOCP_DRIFT_MODEL_H

#include <math.h>

#ifdef __CUDACC__
#define DOCP_HD __host__ __device__ __forceinline__
#else
#define DOCP_HD inline
#endif

namespace docp_drift {

constexpr int NX = 8, NU = 2, NP = 10;
constexpr int NTH = NX + NU + NX + NX + NP;
constexpr int TH_XREF = NX + NU + NX, TH_PARAMS = TH_XREF + NX;
enum { P_A, P_B, P_M, P_IZ, P_RW, P_CF, P_CR, P_MUF, P_MUR, P_KAPPA };
constexpr double kGravity = 9.81;

/* ---- forward-mode dual numbers: value and N partials */
template <int N>
struct Dual {
  double v;
  double d[N];
};

template <int N>
DOCP_HD Dual<N> cst(double c) {
  Dual<N> r;
  r.v = c;
  for (int k = 0; k < N; ++k) r.d[k] = 0.0;
  return r;
}
template <int N>
DOCP_HD Dual<N> operator+(const Dual<N>& a, const Dual<N>& b) {
  Dual<N> r;
  r.v = a.v + b.v;
  for (int k = 0; k < N; ++k) r.d[k] = a.d[k] + b.d[k];
  return r;
}
template <int N>
DOCP_HD Dual<N> operator-(const Dual<N>& a, const Dual<N>& b) {
  Dual<N> r;
  r.v = a.v - b.v;
  for (int k = 0; k < N; ++k) r.d[k] = a.d[k] - b.d[k];
  return r;
}
template <int N>
DOCP_HD Dual<N> operator-(const Dual<N>& a) {
  Dual<N> r;
  r.v = -a.v;
  for (int k = 0; k < N; ++k) r.d[k] = -a.d[k];
  return r;
}
template <int N>
DOCP_HD Dual<N> operator*(const Dual<N>& a, const Dual<N>& b) {
  Dual<N> r;
  r.v = a.v * b.v;
  for (int k = 0; k < N; ++k) r.d[k] = a.d[k] * b.v + a.v * b.d[k];
  return r;
}
template <int N>
DOCP_HD Dual<N> operator/(const Dual<N>& a, const Dual<N>& b) {
  Dual<N> r;
  r.v = a.v / b.v;
  const double ib = 1.0 / b.v;
  for (int k = 0; k < N; ++k) r.d[k] = (a.d[k] - r.v * b.d[k]) * ib;
  return r;
}
template <int N>
DOCP_HD Dual<N> operator+(const Dual<N>& a, double c) {
  Dual<N> r = a;
  r.v = a.v + c;
  return r;
}
template <int N>
DOCP_HD Dual<N> operator+(double c, const Dual<N>& a) {
  return a + c;
}
template <int N>
DOCP_HD Dual<N> operator-(const Dual<N>& a, double c) {
  Dual<N> r = a;
  r.v = a.v - c;
  return r;
}
template <int N>
DOCP_HD Dual<N> operator-(double c, const Dual<N>& a) {
  Dual<N> r;
  r.v = c - a.v;
  for (int k = 0; k < N; ++k) r.d[k] = -a.d[k];
  return r;
}
template <int N>
DOCP_HD Dual<N> operator*(const Dual<N>& a, double c) {
  Dual<N> r;
  r.v = a.v * c;
  for (int k = 0; k < N; ++k) r.d[k] = a.d[k] * c;
  return r;
}
template <int N>
DOCP_HD Dual<N> operator*(double c, const Dual<N>& a) {
  return a * c;
}
template <int N>
DOCP_HD Dual<N> operator/(double c, const Dual<N>& a) {
  return cst<N>(c) / a;
}
template <int N>
DOCP_HD Dual<N> operator/(const Dual<N>& a, double c) {
  Dual<N> r;
  r.v = a.v / c;
  for (int k = 0; k < N; ++k) r.d[k] = a.d[k] / c;
  return r;
}

/* ---- deterministic sin / cos: two-term Cody-Waite reduction by pi/2,
 * Taylor to degree 17 / 18 on |r| <= pi/4 (a few ulp for the moderate
 * angles of this model; identical bits on host and device since only +, -,
 * * and rint are used) */
DOCP_HD void sincos_det(double x, double* s, double* c) {
  const double k = rint(x * 0.63661977236758134308);
  const double r = (x - k * 1.57079632673412561417) - k * 6.07710050650619224932e-11;
  const double r2 = r * r;
  double ps = 1.0 / 355687428096000.0;  // 1/17!
  ps = -1.0 / 1307674368000.0 + r2 * ps;
  ps = 1.0 / 6227020800.0 + r2 * ps;
  ps = -1.0 / 39916800.0 + r2 * ps;
  ps = 1.0 / 362880.0 + r2 * ps;
  ps = -1.0 / 5040.0 + r2 * ps;
  ps = 1.0 / 120.0 + r2 * ps;
  ps = -1.0 / 6.0 + r2 * ps;
  const double sr = r + (r * r2) * ps;
  double pc = 1.0 / 6402373705728000.0;  // 1/18!
  pc = -1.0 / 20922789888000.0 + r2 * pc;
  pc = 1.0 / 87178291200.0 + r2 * pc;
  pc = -1.0 / 479001600.0 + r2 * pc;
  pc = 1.0 / 3628800.0 + r2 * pc;
  pc = -1.0 / 40320.0 + r2 * pc;
  pc = 1.0 / 720.0 + r2 * pc;
  pc = -1.0 / 24.0 + r2 * pc;
  pc = 0.5 + r2 * pc;
  const double cr = 1.0 - r2 * pc;
  const long q = static_cast<long>(k) & 3;
  *s = q == 0 ? sr : q == 1 ? cr : q == 2 ? -sr : -cr;
  *c = q == 0 ? cr : q == 1 ? -sr : q == 2 ? -cr : sr;
}

template <int N>
DOCP_HD void sincos_d(const Dual<N>& x, Dual<N>* s, Dual<N>* c) {
  double sv, cv;
  sincos_det(x.v, &sv, &cv);
  s->v = sv;
  c->v = cv;
  for (int k = 0; k < N; ++k) {
    s->d[k] = cv * x.d[k];
    c->d[k] = -(sv * x.d[k]);
  }
}
DOCP_HD void sincos_d(double x, double* s, double* c) { sincos_det(x, s, c); }

template <int N>
DOCP_HD Dual<N> sqrt_d(const Dual<N>& a) {  // a.v > 0
  Dual<N> r;
  r.v = sqrt(a.v);
  const double h = 0.5 / r.v;
  for (int k = 0; k < N; ++k) r.d[k] = a.d[k] * h;
  return r;
}
DOCP_HD double sqrt_d(double a) { return sqrt(a); }

template <int N>
DOCP_HD double val(const Dual<N>& a) {
  return a.v;
}
DOCP_HD double val(double a) { return a; }
template <class S>
struct Lift {
  static DOCP_HD S of(double c) { return S(c); }
};
template <int N>
struct Lift<Dual<N>> {
  static DOCP_HD Dual<N> of(double c) { return cst<N>(c); }
};
template <class S>
DOCP_HD S lift(double c) {
  return Lift<S>::of(c);
}

template <class S>
DOCP_HD S as_s(double c) {
  return lift<S>(c);
}
template <class S>
DOCP_HD S as_s(const S& x) {
  return x;
}

/* ---- Fiala brush tire (Svendenius 2007) with the coupled-slip friction
 * limit of the driven axle (friction circle: F_y,max = sqrt((mu F_z)^2 -
 * F_x^2)): lateral force for slip tan(alpha) = z, sliding beyond
 * z_sl = 3 F_y,max / C. */
template <class S, class M>
DOCP_HD S fiala_lateral(double C, const M& Fmax, const S& z) {
  const M zsl = (3.0 * Fmax) / C;
  const double zv = val(z);
  if (zv < val(zsl) && zv > -val(zsl)) {
    const S az = zv < 0.0 ? -z : z;
    const M k2 = (C * C) / (3.0 * Fmax);
    const M k3 = (C * C * C) / (27.0 * (Fmax * Fmax));
    return (k2 * (az * z) - C * z) - k3 * ((z * z) * z);
  }
  return as_s<S>(zv < 0.0 ? Fmax : -Fmax);
}

/// Continuous dynamics f(X, u) (the bicycle in path coordinates).
template <class S>
DOCP_HD void rhs(const S* X, const S* u, const double* P, S* f) {
  const double a = P[P_A], b = P[P_B], m = P[P_M], Iz = P[P_IZ];
  const double kap = P[P_KAPPA];
  const S& r = X[0];
  const S& V = X[1];
  const S& e = X[4];
  S sb, cb, sd, cd, sp, cp;
  sincos_d(X[2], &sb, &cb);  // beta
  sincos_d(X[6], &sd, &cd);  // delta
  sincos_d(X[3], &sp, &cp);  // dphi
  const S Vx = V * cb, Vy = V * sb;
  const S zf = (Vy + a * r) / Vx;
  const S td = sd / cd;
  const S tan_af = (zf - td) / (1.0 + zf * td);  // tan(atan(zf) - delta)
  const S tan_ar = (Vy - b * r) / Vx;
  const double Fzf = m * kGravity * b / (a + b), Fzr = m * kGravity * a / (a + b);
  const double muzf = P[P_MUF] * Fzf, muzr = P[P_MUR] * Fzr;
  const S Fxr = 1000.0 * X[7];  // quasi-static rear wheel: the drive force (kN) is the tire's longitudinal force
  const S Fyf = fiala_lateral(P[P_CF], muzf, tan_af);
  const S Fmax_r = sqrt_d(muzr * muzr - Fxr * Fxr);  // coupled slip: the friction circle's lateral share
  const S Fyr = fiala_lateral(P[P_CR], Fmax_r, tan_ar);
  const S c_db = cd * cb + sd * sb;  // cos(delta - beta)
  const S s_db = sd * cb - cd * sb;  // sin(delta - beta)
  const S c_pb = cp * cb - sp * sb;  // cos(dphi + beta)
  const S s_pb = sp * cb + cp * sb;  // sin(dphi + beta)
  const S sdot = (V * c_pb) / (1.0 - kap * e);
  f[0] = ((a * Fyf) * cd - b * Fyr) / Iz;
  f[1] = ((Fxr * cb + Fyr * sb) - Fyf * s_db) / m;
  f[2] = ((Fyf * c_db - Fxr * sb) + Fyr * cb) / (m * V) - r;
  f[3] = r - kap * sdot;
  f[4] = V * s_pb;
  f[5] = sdot;
  f[6] = u[0];
  f[7] = u[1];
}

/// One step of length dt: kSub Heun (explicit trapezoidal) sub-steps (the
/// lateral tire dynamics, ~ (C_f + C_r) / (m V) ~ 25 / s, are stiff for one
/// explicit step of 0.1 s).
constexpr int kSub = 4;
template <class S>
DOCP_HD void heun(const S* X, const S* u, const double* P, double dt, S* Xn) {
  const double h = dt / kSub;
  S x[NX];
  for (int i = 0; i < NX; ++i) x[i] = X[i];
  for (int k = 0; k < kSub; ++k) {
    S f1[NX], xt[NX], f2[NX];
    rhs(x, u, P, f1);
    for (int i = 0; i < NX; ++i) xt[i] = x[i] + h * f1[i];
    rhs(xt, u, P, f2);
    for (int i = 0; i < NX; ++i) x[i] = x[i] + (0.5 * h) * (f1[i] + f2[i]);
  }
  for (int i = 0; i < NX; ++i) Xn[i] = x[i];
}

/// The OCP's explicit step in deviation coordinates,
///   phi(xbar, u) = heun(xbar + X_ref, u) - X_ref,
/// and its Jacobians d phi / d xbar (NX x NX) and d phi / d u (NX x NU),
/// column-major (either may be null). th: the instance's theta.
DOCP_HD void step(const double* th, double dt, const double* xbar, const double* u, double* xn, double* jx,
                  double* ju) {
  const double* xref = th + TH_XREF;
  const double* P = th + TH_PARAMS;
  if (!jx && !ju) {
    double X[NX], Xn[NX];
    for (int i = 0; i < NX; ++i) X[i] = xbar[i] + xref[i];
    heun(X, u, P, dt, Xn);
    for (int i = 0; i < NX; ++i) xn[i] = Xn[i] - xref[i];
    return;
  }
  // The Jacobian in KJ-column passes (directional derivatives; KJ = 1 measured
  // fastest on the B200: C4 linearisation 500 -> 329 ms per epoch): every
  // partial is the same sequence of operations whatever the chunking, so the
  // bits do not depend on KJ; small duals keep the device evaluation in
  // registers instead of local memory.
#ifndef DOCP_DRIFT_KJ
#define DOCP_DRIFT_KJ 1
#endif
  constexpr int KJ = DOCP_DRIFT_KJ;
  typedef Dual<KJ> D;
  for (int c0 = 0; c0 < NX + NU; c0 += KJ) {
    D X[NX], U[NU], Xn[NX];
    for (int i = 0; i < NX; ++i) {
      X[i] = cst<KJ>(xbar[i] + xref[i]);
      if (i >= c0 && i < c0 + KJ) X[i].d[i - c0] = 1.0;
    }
    for (int j = 0; j < NU; ++j) {
      U[j] = cst<KJ>(u[j]);
      if (NX + j >= c0 && NX + j < c0 + KJ) U[j].d[NX + j - c0] = 1.0;
    }
    heun(X, U, P, dt, Xn);
    for (int i = 0; i < NX; ++i) {
      if (c0 == 0) xn[i] = Xn[i].v - xref[i];
      for (int k = 0; k < KJ; ++k) {
        const int col = c0 + k;
        if (col < NX) {
          if (jx) jx[i + col * NX] = Xn[i].d[k];
        } else if (ju) {
          ju[i + (col - NX) * NX] = Xn[i].d[k];
        }
      }
    }
  }
}

}  // namespace docp_drift

#endif
