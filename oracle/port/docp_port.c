/* docp_port.c — plain-C restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE / ORACLE: the checker for the CUDA path, never the
 * thing measured or shipped (see docp_port.h). Each function cites the
 * reference routine it restates; arithmetic follows the eigen_lite
 * convention (left folds seeded with the first term, products evaluated
 * before they are added, no FMA: build with -ffp-contract=off).
 */
#include "docp_port.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ utils */

static int fail(port_status* st, int code, int iteration, const char* fmt, ...) {
  if (st) {
    va_list ap;
    va_start(ap, fmt);
    st->code = code;
    st->iteration = iteration;
    vsnprintf(st->message, sizeof st->message, fmt, ap);
    va_end(ap);
  }
  return code;
}

static void ok(port_status* st) {
  if (st) {
    st->code = PORT_OK;
    st->iteration = 0;
    st->message[0] = 0;
  }
}

/* A(i,k) of a column-major m-row matrix */
#define M_(A, m, i, k) ((A)[(i) + (k) * (m)])

/* y = A x, A m x n (eigen_lite product: fold over k seeded with k = 0) */
static void gemv(const double* A, int m, int n, const double* x, double* y) {
  for (int i = 0; i < m; ++i) {
    double acc = 0.0;
    if (n > 0) {
      acc = M_(A, m, i, 0) * x[0];
      for (int k = 1; k < n; ++k) acc = acc + M_(A, m, i, k) * x[k];
    }
    y[i] = acc;
  }
}

/* y = A' x, A m x n, y has n entries */
static void gemv_t(const double* A, int m, int n, const double* x, double* y) {
  for (int i = 0; i < n; ++i) {
    double acc = 0.0;
    if (m > 0) {
      acc = M_(A, m, 0, i) * x[0];
      for (int k = 1; k < m; ++k) acc = acc + M_(A, m, k, i) * x[k];
    }
    y[i] = acc;
  }
}

/* C = A B (A m x k, B k x n), opA/opB: transpose flags */
static void gemm(const double* A, int tA, const double* B, int tB, int m, int k, int n, double* C) {
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < m; ++i) {
      double acc = 0.0;
      for (int l = 0; l < k; ++l) {
        double a = tA ? A[l + i * k] : A[i + l * m];
        double b = tB ? B[j + l * n] : B[l + j * k];
        acc = (l == 0) ? a * b : acc + a * b;
      }
      C[i + j * m] = acc;
    }
}

static double dotv(const double* a, const double* b, int n) {
  if (n == 0) return 0.0;
  double acc = a[0] * b[0];
  for (int k = 1; k < n; ++k) acc = acc + a[k] * b[k];
  return acc;
}

static double normv(const double* a, int n) { return sqrt(dotv(a, a, n)); }

static double abs_sum(const double* a, int n) {
  if (n == 0) return 0.0;
  double acc = fabs(a[0]);
  for (int k = 1; k < n; ++k) acc = acc + fabs(a[k]);
  return acc;
}

static int all_finite(const double* a, int n) {
  for (int k = 0; k < n; ++k)
    if (!isfinite(a[k])) return 0;
  return 1;
}

/* 0.5 * (M + M') in place, n x n */
static void symmetrize(double* M, int n) {
  double* t = (double*)malloc(sizeof(double) * (size_t)(n * n));
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) t[i + j * n] = 0.5 * (M[i + j * n] + M[j + i * n]);
  memcpy(M, t, sizeof(double) * (size_t)(n * n));
  free(t);
}

/* eigen_lite LLT: returns 0 on success, 1 when a pivot is <= 0. */
static int llt(const double* A, int n, double* L) {
  memset(L, 0, sizeof(double) * (size_t)(n * n));
  for (int k = 0; k < n; ++k) {
    double s = 0.0;
    if (k > 0) {
      s = M_(L, n, k, 0) * M_(L, n, k, 0);
      for (int j = 1; j < k; ++j) s = s + M_(L, n, k, j) * M_(L, n, k, j);
    }
    double x = M_(A, n, k, k) - s;
    if (x <= 0.0) return 1;
    x = sqrt(x);
    M_(L, n, k, k) = x;
    for (int i = k + 1; i < n; ++i) {
      double t = 0.0;
      if (k > 0) {
        t = M_(L, n, i, 0) * M_(L, n, k, 0);
        for (int j = 1; j < k; ++j) t = t + M_(L, n, i, j) * M_(L, n, k, j);
      }
      M_(L, n, i, k) = (M_(A, n, i, k) - t) / x;
    }
  }
  return 0;
}

/* In-place LLT solve of ncol right-hand sides (column-major n x ncol). */
static void llt_solve(const double* L, int n, double* b, int ncol) {
  for (int c = 0; c < ncol; ++c) {
    double* x = b + (size_t)c * n;
    for (int i = 0; i < n; ++i) {
      double s = 0.0;
      if (i > 0) {
        s = M_(L, n, i, 0) * x[0];
        for (int j = 1; j < i; ++j) s = s + M_(L, n, i, j) * x[j];
      }
      x[i] = (x[i] - s) / M_(L, n, i, i);
    }
    for (int i = n - 1; i >= 0; --i) {
      double s = 0.0;
      if (i + 1 < n) {
        s = M_(L, n, i + 1, i) * x[i + 1];
        for (int j = i + 2; j < n; ++j) s = s + M_(L, n, j, i) * x[j];
      }
      x[i] = (x[i] - s) / M_(L, n, i, i);
    }
  }
}

/* ------------------------------------------------------------------ solver state */

struct port_solver {
  port_problem p;
  int nx, nu, T, nlam, nz, ntheta;
  /* QpData (problem.hpp:103-151) */
  double *Q, *q, *R, *r, *Ap, *A, *B, *C, *xs;
  int pd_projected;
  /* SchurSystem (schur.hpp:84-95) */
  double *Sd, *Ssub, *Ssup, *Pd, *Psub, *Psup, *LQ, *LR;
  /* SolveResult z / lambda (sqp.hpp:40-52) */
  double *z, *lam;
  /* scratch */
  double* w;
};

int port_theta_size(const port_problem* p) {
  if (p->family == PORT_AFFINE_QUADRATIC)
    return p->nx + p->nu + p->nx * p->nx + p->nx * p->nu + p->nx + p->nx;
  if (p->family == PORT_CARTPOLE) return 4 + 1 + 4;
  return -1;
}

port_solver* port_create(const port_problem* prob) {
  if (prob->nx < 1 || prob->nu < 1 || prob->horizon < 1) return NULL;
  if (prob->family == PORT_CARTPOLE && (prob->nx != 4 || prob->nu != 1)) return NULL;
  if (prob->family != PORT_CARTPOLE && prob->family != PORT_AFFINE_QUADRATIC) return NULL;
  port_solver* s = (port_solver*)calloc(1, sizeof *s);
  s->p = *prob;
  s->nx = prob->nx;
  s->nu = prob->nu;
  s->T = prob->horizon;
  s->nlam = s->nx * (s->T + 1);
  s->nz = s->nx * (s->T + 1) + s->nu * s->T;
  s->ntheta = port_theta_size(prob);
  const size_t nx = (size_t)s->nx, nu = (size_t)s->nu, T = (size_t)s->T;
#define ALLOC(f, n) s->f = (double*)calloc((n) + 1, sizeof(double))
  ALLOC(Q, (T + 1) * nx * nx);
  ALLOC(q, (T + 1) * nx);
  ALLOC(R, T * nu * nu);
  ALLOC(r, T * nu);
  ALLOC(Ap, T * nx * nx);
  ALLOC(A, T * nx * nx);
  ALLOC(B, T * nx * nu);
  ALLOC(C, T * nx);
  ALLOC(xs, nx);
  ALLOC(Sd, (T + 1) * nx * nx);
  ALLOC(Ssub, T * nx * nx);
  ALLOC(Ssup, T * nx * nx);
  ALLOC(Pd, (T + 1) * nx * nx);
  ALLOC(Psub, T * nx * nx);
  ALLOC(Psup, T * nx * nx);
  ALLOC(LQ, (T + 1) * nx * nx);
  ALLOC(LR, T * nu * nu);
  ALLOC(z, (size_t)s->nz);
  ALLOC(lam, (size_t)s->nlam);
  ALLOC(w, 16 * (size_t)(s->nz + s->nlam) + 64 * (nx + nu) * (nx + nu));
#undef ALLOC
  return s;
}

void port_destroy(port_solver* s) {
  if (!s) return;
  double* ptrs[] = {s->Q,  s->q,    s->R,    s->r,  s->Ap,   s->A,    s->B,  s->C,  s->xs, s->Sd,
                    s->Ssub, s->Ssup, s->Pd, s->Psub, s->Psup, s->LQ, s->LR, s->z, s->lam, s->w};
  for (size_t i = 0; i < sizeof ptrs / sizeof ptrs[0]; ++i) free(ptrs[i]);
  free(s);
}

static int xoff(const port_solver* s, int t) { return t * (s->nx + s->nu); }            /* trajectory.hpp:72-74 */
static int uoff(const port_solver* s, int t) { return t * (s->nx + s->nu) + s->nx; }

/* ------------------------------------------------------------------ family callbacks */

/* Diagonal quadratic stage cost scale * v' diag(w) v
 * (affine_quadratic.hpp:47-64, quadratic_cost.hpp:9-20). hess is dense n x n. */
static void diag_cost(double scale, const double* w, const double* v, int n, double* value, double* grad,
                      double* hess) {
  double wv[64];
  for (int i = 0; i < n; ++i) wv[i] = w[i] * v[i];
  *value = scale * dotv(v, wv, n);
  const double s2 = 2.0 * scale;
  if (grad)
    for (int i = 0; i < n; ++i) grad[i] = (s2 * w[i]) * v[i];
  if (hess) {
    memset(hess, 0, sizeof(double) * (size_t)(n * n));
    for (int i = 0; i < n; ++i) hess[i + i * n] = s2 * w[i];
  }
}

static double cost_scale(const port_solver* s) {
  return s->p.family == PORT_CARTPOLE ? 0.5 : s->p.cost_scale;
}

static void state_cost(const port_solver* s, const double* theta, const double* x, double* value, double* grad,
                       double* hess) {
  diag_cost(cost_scale(s), theta + 0, x, s->nx, value, grad, hess);
}

static void control_cost(const port_solver* s, const double* theta, const double* u, double* value,
                         double* grad, double* hess) {
  diag_cost(cost_scale(s), theta + s->nx, u, s->nu, value, grad, hess);
}

static const double* initial_state(const port_solver* s, const double* theta) {
  if (s->p.family == PORT_CARTPOLE) return theta + 5;
  return theta + s->nx + s->nu + s->nx * s->nx + s->nx * s->nu + s->nx;
}

/* cartpole.hpp:28-42 */
static void cartpole_xdot(const port_problem* p, const double* x, const double* u, double* xdot) {
  const double sn = sin(x[2]);
  const double c = cos(x[2]);
  const double mp = p->pole_mass;
  const double len = p->length;
  const double big_m = p->cart_mass + p->pole_mass;
  const double d = big_m + mp * (1.0 - c * c);
  xdot[0] = x[1];
  xdot[1] = (-mp * len * sn * x[3] * x[3] + mp * p->gravity * sn * c) / (d * len);
  xdot[2] = x[3];
  xdot[3] = (-mp * len * sn * x[3] + mp * p->gravity * sn * c + u[0]) / d;
}

/* Dynamics residual f = x+ - phi(x,u) with Jacobians (jac_x_next = I).
 * affine_quadratic.hpp:65-75; problem.hpp:80-97 with cartpole.hpp:44-78. */
static void dynamics(const port_solver* s, const double* theta, const double* xn, const double* x,
                     const double* u, double* res, double* jac_x, double* jac_u) {
  const int nx = s->nx, nu = s->nu;
  if (s->p.family == PORT_AFFINE_QUADRATIC) {
    const double* a = theta + nx + nu;
    const double* b = a + nx * nx;
    const double* off = b + nx * nu;
    double ax[64], bu[64];
    gemv(a, nx, nx, x, ax);
    gemv(b, nx, nu, u, bu);
    for (int i = 0; i < nx; ++i) res[i] = ((xn[i] - ax[i]) - bu[i]) - off[i];
    for (int k = 0; k < nx * nx; ++k) jac_x[k] = -a[k];
    for (int k = 0; k < nx * nu; ++k) jac_u[k] = -b[k];
    return;
  }
  /* cart-pole explicit Euler step (cartpole.hpp:44-78) */
  const port_problem* p = &s->p;
  const double sn = sin(x[2]);
  const double c = cos(x[2]);
  const double mp = p->pole_mass;
  const double len = p->length;
  const double g = p->gravity;
  const double big_m = p->cart_mass + p->pole_mass;
  const double d = big_m + mp * (1.0 - c * c);
  const double d_d3 = 2.0 * mp * sn * c;
  const double n2 = -mp * len * sn * x[3] * x[3] + mp * g * sn * c;
  const double n2_d3 = -mp * len * c * x[3] * x[3] + mp * g * (c * c - sn * sn);
  const double n2_d4 = -2.0 * mp * len * sn * x[3];
  const double n4 = -mp * len * sn * x[3] + mp * g * sn * c + u[0];
  const double n4_d3 = -mp * len * c * x[3] + mp * g * (c * c - sn * sn);
  const double n4_d4 = -mp * len * sn;
  double J[16] = {0}, Ju[4] = {0};
  M_(J, 4, 0, 1) = 1.0;
  M_(J, 4, 1, 2) = (n2_d3 * d - n2 * d_d3) / (d * d * len);
  M_(J, 4, 1, 3) = n2_d4 / (d * len);
  M_(J, 4, 2, 3) = 1.0;
  M_(J, 4, 3, 2) = (n4_d3 * d - n4 * d_d3) / (d * d);
  M_(J, 4, 3, 3) = n4_d4 / d;
  Ju[3] = 1.0 / d;
  double xdot[4];
  cartpole_xdot(p, x, u, xdot);
  for (int i = 0; i < 4; ++i) res[i] = xn[i] - (x[i] + p->dt * xdot[i]);
  for (int j = 0; j < 4; ++j)
    for (int i = 0; i < 4; ++i) {
      double eye = (i == j) ? 1.0 : 0.0;
      M_(jac_x, 4, i, j) = -(eye + p->dt * M_(J, 4, i, j));
    }
  for (int i = 0; i < 4; ++i) jac_u[i] = -(p->dt * Ju[i]);
}

/* ------------------------------------------------------------------ linearize */

/* problem.hpp:157-181 for diagonal input (every shipped family's Hessian is
 * diagonal): the LLT acceptance test passes iff every h_ii - eps > 0; the
 * eigen-clamp of a diagonal matrix is exactly diag(max(h_ii, eps)). */
static int project_pd(double* M, int n, double eps, int* modified) {
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i)
      if (i != j && M[i + j * n] != 0.0) return -1;
  symmetrize(M, n);
  *modified = 0;
  if (n == 1) {
    if (M[0] >= eps) return 0;
    *modified = 1;
    M[0] = eps;
    return 0;
  }
  int pass = 1;
  for (int i = 0; i < n; ++i)
    if (!(M[i + i * n] - eps * 1.0 > 0.0)) pass = 0;
  if (pass) return 0;
  *modified = 1;
  for (int i = 0; i < n; ++i) M[i + i * n] = M[i + i * n] < eps ? eps : M[i + i * n];
  return 0;
}

int port_linearize(port_solver* s, const double* theta, const double* z, double eps_pd, port_status* st) {
  const int nx = s->nx, nu = s->nu, T = s->T;
  double value, grad[64], hess[64 * 64], tmp[64];
  int any = 0;
  ok(st);
  for (int t = 0; t <= T; ++t) {
    const double* x = z + xoff(s, t);
    state_cost(s, theta, x, &value, grad, hess);
    if (!(isfinite(value) && all_finite(grad, nx) && all_finite(hess, nx * nx)))
      return fail(st, PORT_EVALUATION, 0, "state_cost returned non-finite values at stage %d", t);
    int mod = 0;
    if (project_pd(hess, nx, eps_pd, &mod))
      return fail(st, PORT_NUMERICAL, 0, "port: non-diagonal Hessian unsupported");
    any |= mod;
    memcpy(s->Q + (size_t)t * nx * nx, hess, sizeof(double) * (size_t)(nx * nx));
    gemv(hess, nx, nx, x, tmp);
    for (int i = 0; i < nx; ++i) s->q[t * nx + i] = grad[i] - tmp[i];
  }
  for (int t = 0; t < T; ++t) {
    const double* x = z + xoff(s, t);
    const double* u = z + uoff(s, t);
    const double* xn = z + xoff(s, t + 1);
    control_cost(s, theta, u, &value, grad, hess);
    if (!(isfinite(value) && all_finite(grad, nu) && all_finite(hess, nu * nu)))
      return fail(st, PORT_EVALUATION, 0, "control_cost returned non-finite values at stage %d", t);
    int mod = 0;
    if (project_pd(hess, nu, eps_pd, &mod))
      return fail(st, PORT_NUMERICAL, 0, "port: non-diagonal Hessian unsupported");
    any |= mod;
    memcpy(s->R + (size_t)t * nu * nu, hess, sizeof(double) * (size_t)(nu * nu));
    gemv(hess, nu, nu, u, tmp);
    for (int i = 0; i < nu; ++i) s->r[t * nu + i] = grad[i] - tmp[i];

    double res[64], jx[64 * 64], ju[64 * 64];
    dynamics(s, theta, xn, x, u, res, jx, ju);
    double* ap = s->Ap + (size_t)t * nx * nx;
    memset(ap, 0, sizeof(double) * (size_t)(nx * nx));
    for (int i = 0; i < nx; ++i) ap[i + i * nx] = 1.0;
    if (!(all_finite(res, nx) && all_finite(jx, nx * nx) && all_finite(ju, nx * nu)))
      return fail(st, PORT_EVALUATION, 0, "dynamics_residual returned non-finite values at stage %d", t);
    memcpy(s->A + (size_t)t * nx * nx, jx, sizeof(double) * (size_t)(nx * nx));
    memcpy(s->B + (size_t)t * nx * nu, ju, sizeof(double) * (size_t)(nx * nu));
    double p1[64], p2[64], p3[64];
    gemv(ap, nx, nx, xn, p1);
    gemv(jx, nx, nx, x, p2);
    gemv(ju, nx, nu, u, p3);
    for (int i = 0; i < nx; ++i) s->C[t * nx + i] = ((p1[i] + p2[i]) + p3[i]) - res[i];
  }
  const double* x_s = initial_state(s, theta);
  memcpy(s->xs, x_s, sizeof(double) * (size_t)nx);
  if (!all_finite(s->xs, nx))
    return fail(st, PORT_EVALUATION, 0, "initial_state returned non-finite values at stage 0");
  s->pd_projected = any;
  return PORT_OK;
}

void port_flat_b(port_solver* s, double* b) { /* problem.hpp:131-142 */
  for (int t = 0; t < s->T; ++t) {
    memcpy(b + xoff(s, t), s->q + t * s->nx, sizeof(double) * (size_t)s->nx);
    memcpy(b + uoff(s, t), s->r + t * s->nu, sizeof(double) * (size_t)s->nu);
  }
  memcpy(b + xoff(s, s->T), s->q + s->T * s->nx, sizeof(double) * (size_t)s->nx);
}

void port_flat_d(port_solver* s, double* d) { /* problem.hpp:145-150 */
  memcpy(d, s->xs, sizeof(double) * (size_t)s->nx);
  for (int t = 0; t < s->T; ++t) memcpy(d + (t + 1) * s->nx, s->C + t * s->nx, sizeof(double) * (size_t)s->nx);
}

/* ------------------------------------------------------------------ Schur assembly */

int port_assemble(port_solver* s, port_status* st) { /* schur.hpp:114-180 */
  const int nx = s->nx, nu = s->nu, T = s->T;
  const size_t b2 = (size_t)nx * nx;
  ok(st);
  for (int t = 0; t <= T; ++t)
    if (llt(s->Q + t * b2, nx, s->LQ + t * b2))
      return fail(st, PORT_NUMERICAL, 0, "assemble_schur: Cholesky of Q failed at stage %d", t);
  for (int t = 0; t < T; ++t)
    if (llt(s->R + (size_t)t * nu * nu, nu, s->LR + (size_t)t * nu * nu))
      return fail(st, PORT_NUMERICAL, 0, "assemble_schur: Cholesky of R failed at stage %d", t);

  double* eye = s->w + 16 * (size_t)(s->nz + s->nlam);
  double* m1 = eye + b2;
  double* m2 = m1 + b2;
  double* chi = m2 + b2;
  double* tmp = chi + b2;
  double* lchi = tmp + b2;
  double* bt = lchi + b2;  /* nu x nx */
  double* mb = bt + (size_t)nx * nu;
  memset(eye, 0, sizeof(double) * b2);
  for (int i = 0; i < nx; ++i) eye[i + i * nx] = 1.0;

  memcpy(s->Sd, eye, sizeof(double) * b2);
  llt_solve(s->LQ, nx, s->Sd, nx);
  symmetrize(s->Sd, nx);
  for (int t = 0; t < T; ++t) {
    const double* At = s->A + t * b2;
    const double* Bt = s->B + (size_t)t * nx * nu;
    const double* Apt = s->Ap + t * b2;
    /* chi = A Q^-1 A' + B R^-1 B' + A+ Q+^-1 A+' */
    for (int j = 0; j < nx; ++j)
      for (int i = 0; i < nx; ++i) m1[i + j * nx] = At[j + i * nx];
    llt_solve(s->LQ + t * b2, nx, m1, nx);
    gemm(At, 0, m1, 0, nx, nx, nx, chi);
    for (int j = 0; j < nx; ++j)
      for (int i = 0; i < nu; ++i) bt[i + j * nu] = Bt[j + i * nx];
    llt_solve(s->LR + (size_t)t * nu * nu, nu, bt, nx);
    gemm(Bt, 0, bt, 0, nx, nu, nx, tmp);
    for (size_t k = 0; k < b2; ++k) chi[k] = chi[k] + tmp[k];
    for (int j = 0; j < nx; ++j)
      for (int i = 0; i < nx; ++i) m2[i + j * nx] = Apt[j + i * nx];
    llt_solve(s->LQ + (t + 1) * b2, nx, m2, nx);
    gemm(Apt, 0, m2, 0, nx, nx, nx, tmp);
    for (size_t k = 0; k < b2; ++k) chi[k] = chi[k] + tmp[k];
    double* dnext = s->Sd + (t + 1) * b2;
    memcpy(dnext, chi, sizeof(double) * b2);
    symmetrize(dnext, nx);
    /* phi_t = A_t Q_t^-1 A+_{t-1}', A+_{-1} = I */
    if (t == 0) {
      memcpy(mb, eye, sizeof(double) * b2);
    } else {
      const double* prev = s->Ap + (t - 1) * b2;
      for (int j = 0; j < nx; ++j)
        for (int i = 0; i < nx; ++i) mb[i + j * nx] = prev[j + i * nx];
    }
    llt_solve(s->LQ + t * b2, nx, mb, nx);
    gemm(At, 0, mb, 0, nx, nx, nx, s->Ssub + t * b2);
    for (int j = 0; j < nx; ++j)
      for (int i = 0; i < nx; ++i) s->Ssup[t * b2 + i + j * nx] = s->Ssub[t * b2 + j + i * nx];
    if (llt(dnext, nx, lchi))
      return fail(st, PORT_NUMERICAL, 0, "assemble_schur: Cholesky of chi failed at stage %d", t);
    double* pn = s->Pd + (t + 1) * b2;
    memcpy(pn, eye, sizeof(double) * b2);
    llt_solve(lchi, nx, pn, nx);
    symmetrize(pn, nx);
  }
  memcpy(s->Pd, s->Q, sizeof(double) * b2);
  for (int t = 0; t < T; ++t) {
    /* super_t = (-D_t phi_t') D_{t+1} */
    for (size_t k = 0; k < b2; ++k) m1[k] = -s->Pd[t * b2 + k];
    gemm(m1, 0, s->Ssub + t * b2, 1, nx, nx, nx, tmp);
    gemm(tmp, 0, s->Pd + (t + 1) * b2, 0, nx, nx, nx, s->Psup + t * b2);
    for (int j = 0; j < nx; ++j)
      for (int i = 0; i < nx; ++i) s->Psub[t * b2 + i + j * nx] = s->Psup[t * b2 + j + i * nx];
  }
  return PORT_OK;
}

int port_gamma(port_solver* s, const double* b, const double* d, double* out, port_status* st) {
  /* schur.hpp:187-211 */
  const int nx = s->nx, nu = s->nu, T = s->T;
  const size_t b2 = (size_t)nx * nx;
  double sq[64], su[64], p1[64], p2[64], p3[64];
  ok(st);
  memcpy(sq, b + xoff(s, 0), sizeof(double) * (size_t)nx);
  llt_solve(s->LQ, nx, sq, 1);
  for (int i = 0; i < nx; ++i) out[i] = d[i] + sq[i];
  for (int t = 0; t < T; ++t) {
    memcpy(sq, b + xoff(s, t), sizeof(double) * (size_t)nx);
    llt_solve(s->LQ + t * b2, nx, sq, 1);
    gemv(s->A + t * b2, nx, nx, sq, p1);
    memcpy(su, b + uoff(s, t), sizeof(double) * (size_t)nu);
    llt_solve(s->LR + (size_t)t * nu * nu, nu, su, 1);
    gemv(s->B + (size_t)t * nx * nu, nx, nu, su, p2);
    memcpy(sq, b + xoff(s, t + 1), sizeof(double) * (size_t)nx);
    llt_solve(s->LQ + (t + 1) * b2, nx, sq, 1);
    gemv(s->Ap + t * b2, nx, nx, sq, p3);
    for (int i = 0; i < nx; ++i) out[(t + 1) * nx + i] = d[(t + 1) * nx + i] + ((p1[i] + p2[i]) + p3[i]);
  }
  for (int k = 0; k < s->nlam; ++k) out[k] = -out[k];
  return PORT_OK;
}

/* ------------------------------------------------------------------ PCG */

/* schur.hpp:60-72: y_i = D_i v_i (+ L_{i-1} v_{i-1}) (+ U_i v_{i+1}) */
static void btd_matvec(int nx, int nb, const double* D, const double* L, const double* U, const double* v,
                       double* y) {
  const size_t b2 = (size_t)nx * nx;
  double tmp[64];
  for (int i = 0; i < nb; ++i) {
    double* yi = y + (size_t)i * nx;
    gemv(D + i * b2, nx, nx, v + (size_t)i * nx, yi);
    if (i > 0) {
      gemv(L + (i - 1) * b2, nx, nx, v + (size_t)(i - 1) * nx, tmp);
      for (int k = 0; k < nx; ++k) yi[k] = yi[k] + tmp[k];
    }
    if (i + 1 < nb) {
      gemv(U + i * b2, nx, nx, v + (size_t)(i + 1) * nx, tmp);
      for (int k = 0; k < nx; ++k) yi[k] = yi[k] + tmp[k];
    }
  }
}

/* pcg.hpp:37-44 */
static double block_dot(const double* a, const double* b, int nb, int bd) {
  double acc = 0.0;
  for (int i = 0; i < nb; ++i) acc = acc + dotv(a + (size_t)i * bd, b + (size_t)i * bd, bd);
  return acc;
}

int port_pcg_blocks(int nx, int nb, const double* Sd, const double* Ssub, const double* Ssup, const double* Pd,
                    const double* Psub, const double* Psup, const double* gamma, const double* lambda0,
                    double epsilon, int max_iters_cfg, double* lam, int* iters_out, double* final_eta,
                    int* converged, port_status* st) {
  /* pcg.hpp:52-109 */
  ok(st);
  if (!(epsilon > 0.0 && max_iters_cfg >= 0)) return fail(st, PORT_DIMENSION, 0, "pcg: invalid config");
  const int n = nx * nb;
  const int max_iters = max_iters_cfg > 0 ? max_iters_cfg : 2 * n;
  double* r = (double*)malloc(sizeof(double) * (size_t)n * 4);
  double* rt = r + n;
  double* p = rt + n;
  double* y = p + n;
  int iters = 0, code = PORT_OK;
  memcpy(lam, lambda0, sizeof(double) * (size_t)n);
  btd_matvec(nx, nb, Sd, Ssub, Ssup, lam, y);
  for (int k = 0; k < n; ++k) r[k] = gamma[k] - y[k];
  btd_matvec(nx, nb, Pd, Psub, Psup, r, rt);
  memcpy(p, rt, sizeof(double) * (size_t)n);
  double eta = block_dot(r, rt, nb, nx);
  if (eta < 0.0) {
    double scale = normv(r, n) * normv(rt, n);
    if (-eta <= 1e-10 * scale + 1e-300) {
      eta = 0.0;
    } else {
      code = fail(st, PORT_BREAKDOWN, 0, "pcg: preconditioner lost definiteness at iteration %d", 0);
      goto done;
    }
  }
  const double threshold = epsilon * epsilon;
  while (eta > threshold && iters < max_iters) {
    btd_matvec(nx, nb, Sd, Ssub, Ssup, p, y);
    double v = block_dot(p, y, nb, nx);
    if (v <= 0.0) {
      code = fail(st, PORT_BREAKDOWN, iters,
                  "pcg: p'Sp <= 0 (loss of positive definiteness) at iteration %d", iters);
      goto done;
    }
    double alpha = eta / v;
    for (int k = 0; k < n; ++k) lam[k] = lam[k] + alpha * p[k];
    for (int k = 0; k < n; ++k) r[k] = r[k] - alpha * y[k];
    btd_matvec(nx, nb, Pd, Psub, Psup, r, rt);
    double eta_next = block_dot(r, rt, nb, nx);
    if (eta_next < 0.0) {
      double scale = normv(r, n) * normv(rt, n);
      if (-eta_next <= 1e-10 * scale + 1e-300) {
        eta_next = 0.0;
      } else {
        code = fail(st, PORT_BREAKDOWN, iters, "pcg: preconditioner lost definiteness at iteration %d", iters);
        goto done;
      }
    }
    double beta = eta_next / eta;
    for (int k = 0; k < n; ++k) p[k] = rt[k] + beta * p[k];
    eta = eta_next;
    ++iters;
  }
  *final_eta = eta;
  *converged = eta <= threshold;
done:
  *iters_out = iters;
  free(r);
  return code;
}

int port_pcg(port_solver* s, const double* gamma, const double* lambda0, double epsilon, int max_iters,
             double* lambda_out, int* iters, double* final_eta, int* converged, double* eta_hist,
             int eta_hist_cap, port_status* st) {
  (void)eta_hist;
  (void)eta_hist_cap;
  return port_pcg_blocks(s->nx, s->T + 1, s->Sd, s->Ssub, s->Ssup, s->Pd, s->Psub, s->Psup, gamma, lambda0,
                         epsilon, max_iters, lambda_out, iters, final_eta, converged, st);
}

/* ------------------------------------------------------------------ recovery / merit / line search */

int port_recover(port_solver* s, const double* lam, const double* b, double* z, port_status* st) {
  /* sqp.hpp:62-89 */
  const int nx = s->nx, nu = s->nu, T = s->T;
  const size_t b2 = (size_t)nx * nx;
  double rhs[64], tmp[64];
  ok(st);
  for (int t = 0; t <= T; ++t) {
    memcpy(rhs, b + xoff(s, t), sizeof(double) * (size_t)nx);
    if (t == 0) {
      for (int i = 0; i < nx; ++i) rhs[i] = rhs[i] + lam[i];
    } else {
      gemv_t(s->Ap + (t - 1) * b2, nx, nx, lam + t * nx, tmp);
      for (int i = 0; i < nx; ++i) rhs[i] = rhs[i] + tmp[i];
    }
    if (t < T) {
      gemv_t(s->A + t * b2, nx, nx, lam + (t + 1) * nx, tmp);
      for (int i = 0; i < nx; ++i) rhs[i] = rhs[i] + tmp[i];
    }
    llt_solve(s->LQ + t * b2, nx, rhs, 1);
    for (int i = 0; i < nx; ++i) z[xoff(s, t) + i] = -rhs[i];
  }
  for (int t = 0; t < T; ++t) {
    memcpy(rhs, b + uoff(s, t), sizeof(double) * (size_t)nu);
    gemv_t(s->B + (size_t)t * nx * nu, nx, nu, lam + (t + 1) * nx, tmp);
    for (int i = 0; i < nu; ++i) rhs[i] = rhs[i] + tmp[i];
    llt_solve(s->LR + (size_t)t * nu * nu, nu, rhs, 1);
    for (int i = 0; i < nu; ++i) z[uoff(s, t) + i] = -rhs[i];
  }
  return PORT_OK;
}

/* sqp.hpp:98-123 */
static int merit_parts(port_solver* s, const double* theta, const double* z, double* cost, double* viol,
                       port_status* st) {
  const int nx = s->nx, nu = s->nu, T = s->T;
  double c = 0.0, v = 0.0, val;
  double res[64], jx[64 * 64], ju[64 * 64];
  for (int t = 0; t <= T; ++t) {
    state_cost(s, theta, z + xoff(s, t), &val, NULL, NULL);
    if (!isfinite(val)) return fail(st, PORT_EVALUATION, 0, "merit: non-finite state cost at stage %d", t);
    c = c + val;
  }
  for (int t = 0; t < T; ++t) {
    control_cost(s, theta, z + uoff(s, t), &val, NULL, NULL);
    if (!isfinite(val)) return fail(st, PORT_EVALUATION, 0, "merit: non-finite control cost at stage %d", t);
    c = c + val;
    dynamics(s, theta, z + xoff(s, t + 1), z + xoff(s, t), z + uoff(s, t), res, jx, ju);
    v = v + abs_sum(res, nx);
  }
  const double* x_s = initial_state(s, theta);
  double d0[64];
  for (int i = 0; i < nx; ++i) d0[i] = z[i] - x_s[i];
  v = v + abs_sum(d0, nx);
  (void)nu;
  *cost = c;
  *viol = v;
  return PORT_OK;
}

int port_merit(port_solver* s, const double* theta, const double* z, double mu, double* out, port_status* st) {
  double c, v;
  ok(st);
  int e = merit_parts(s, theta, z, &c, &v, st);
  if (e) return e;
  *out = c + mu * v;
  return PORT_OK;
}

static int validate_cfg(const port_sqp_config* cfg, port_status* st) { /* sqp.hpp:23-33 */
  if (cfg->n_alphas < 1) return fail(st, PORT_DIMENSION, 0, "sqp: empty step candidate list");
  for (int i = 0; i < cfg->n_alphas; ++i) {
    int in_range = cfg->alphas[i] > 0.0 && cfg->alphas[i] <= 1.0;
    int decreasing = i == 0 || cfg->alphas[i] < cfg->alphas[i - 1];
    if (!(in_range && decreasing))
      return fail(st, PORT_DIMENSION, 0, "sqp: step candidates must be strictly decreasing in (0,1]");
  }
  if (!(cfg->eta_armijo > 0.0 && cfg->eta_armijo < 1.0)) return fail(st, PORT_DIMENSION, 0, "sqp: eta out of range");
  return PORT_OK;
}

static void interpolate(const double* a, const double* b, double alpha, double* out, int n) {
  for (int k = 0; k < n; ++k) out[k] = a[k] + alpha * (b[k] - a[k]); /* trajectory.hpp:57-62 */
}

int port_line_search(port_solver* s, const double* theta, const double* z_old, const double* z_qp,
                     const port_sqp_config* cfg, double mu_prev, double* z_new, double* alpha_out,
                     int* accepted, double* mu_out, port_status* st) {
  /* sqp.hpp:151-206 */
  const int nx = s->nx, nu = s->nu, T = s->T;
  ok(st);
  int e = validate_cfg(cfg, st);
  if (e) return e;
  double d_cost = 0.0, curvature = 0.0, val, grad[64], dx[64], qdx[64];
  for (int t = 0; t <= T; ++t) {
    for (int i = 0; i < nx; ++i) dx[i] = z_qp[xoff(s, t) + i] - z_old[xoff(s, t) + i];
    state_cost(s, theta, z_old + xoff(s, t), &val, grad, NULL);
    d_cost = d_cost + dotv(grad, dx, nx);
    gemv(s->Q + (size_t)t * nx * nx, nx, nx, dx, qdx);
    curvature = curvature + dotv(dx, qdx, nx);
  }
  for (int t = 0; t < T; ++t) {
    for (int i = 0; i < nu; ++i) dx[i] = z_qp[uoff(s, t) + i] - z_old[uoff(s, t) + i];
    control_cost(s, theta, z_old + uoff(s, t), &val, grad, NULL);
    d_cost = d_cost + dotv(grad, dx, nu);
    gemv(s->R + (size_t)t * nu * nu, nu, nu, dx, qdx);
    curvature = curvature + dotv(dx, qdx, nu);
  }
  double cost, viol;
  e = merit_parts(s, theta, z_old, &cost, &viol, st);
  if (e) return e;
  double mu = mu_prev;
  if (viol >= cfg->mu_floor_denominator) {
    double required = (d_cost + 0.5 * curvature) / ((1.0 - cfg->rho_penalty) * viol);
    if (isfinite(required) && required > mu) mu = required;
  }
  const double phi_old = cost + mu * viol;
  const double descent = d_cost - mu * viol;
  double delta_phi[8];
  double* trial = s->w + 8 * (size_t)(s->nz + s->nlam);
  for (int i = 0; i < cfg->n_alphas; ++i) {
    interpolate(z_old, z_qp, cfg->alphas[i], trial, s->nz);
    double m;
    e = port_merit(s, theta, trial, mu, &m, st);
    if (e) return e;
    delta_phi[i] = m - phi_old - cfg->eta_armijo * cfg->alphas[i] * descent;
  }
  double alpha = cfg->alphas[cfg->n_alphas - 1];
  int acc = 0;
  for (int i = 0; i < cfg->n_alphas; ++i)
    if (delta_phi[i] < 0.0) {
      alpha = cfg->alphas[i];
      acc = 1;
      break;
    }
  interpolate(z_old, z_qp, alpha, z_new, s->nz);
  *alpha_out = alpha;
  *accepted = acc;
  *mu_out = mu;
  return PORT_OK;
}

int port_kkt_inf_norm(port_solver* s, const double* theta, const double* z, const double* lam, double* out,
                      port_status* st) {
  /* problem.hpp:263-300 */
  const int nx = s->nx, nu = s->nu, T = s->T;
  double* gl = s->w + 10 * (size_t)(s->nz + s->nlam);
  double* g = gl + s->nz;
  double val, grad[64], res[64], jx[64 * 64], ju[64 * 64], tmp[64];
  ok(st);
  memset(gl, 0, sizeof(double) * (size_t)(s->nz + s->nlam));
  const double* x_s = initial_state(s, theta);
  for (int i = 0; i < nx; ++i) g[i] = z[i] - x_s[i];
  for (int t = 0; t <= T; ++t) {
    state_cost(s, theta, z + xoff(s, t), &val, grad, NULL);
    memcpy(gl + xoff(s, t), grad, sizeof(double) * (size_t)nx);
  }
  for (int t = 0; t < T; ++t) {
    control_cost(s, theta, z + uoff(s, t), &val, grad, NULL);
    memcpy(gl + uoff(s, t), grad, sizeof(double) * (size_t)nu);
    dynamics(s, theta, z + xoff(s, t + 1), z + xoff(s, t), z + uoff(s, t), res, jx, ju);
    memcpy(g + (t + 1) * nx, res, sizeof(double) * (size_t)nx);
    const double* l1 = lam + (t + 1) * nx;
    gemv_t(jx, nx, nx, l1, tmp);
    for (int i = 0; i < nx; ++i) gl[xoff(s, t) + i] = gl[xoff(s, t) + i] + tmp[i];
    gemv_t(ju, nx, nu, l1, tmp);
    for (int i = 0; i < nu; ++i) gl[uoff(s, t) + i] = gl[uoff(s, t) + i] + tmp[i];
    double eye[64 * 64];
    memset(eye, 0, sizeof(double) * (size_t)(nx * nx));
    for (int i = 0; i < nx; ++i) eye[i + i * nx] = 1.0;
    gemv_t(eye, nx, nx, l1, tmp);
    for (int i = 0; i < nx; ++i) gl[xoff(s, t + 1) + i] = gl[xoff(s, t + 1) + i] + tmp[i];
  }
  for (int i = 0; i < nx; ++i) gl[i] = gl[i] + lam[i];
  double m = fabs(gl[0]);
  for (int k = 1; k < s->nz + s->nlam; ++k)
    if (fabs(gl[k]) > m) m = fabs(gl[k]);
  *out = m;
  return PORT_OK;
}

/* ------------------------------------------------------------------ SQP / backward */

int port_sqp_solve(port_solver* s, const double* theta, const double* z0, const double* lambda0,
                   const port_sqp_config* cfg, double* z_out, double* lambda_out, int* sqp_iters_out,
                   int* converged_out, double* kkt_out, int* pcg_iters, double* step_sizes, port_status* st) {
  /* sqp.hpp:213-261 */
  const int nz = s->nz, nl = s->nlam;
  ok(st);
  int e = validate_cfg(cfg, st);
  if (e) return e;
  if (!(all_finite(z0, nz) && all_finite(lambda0, nl)))
    return fail(st, PORT_DIMENSION, 0, "sqp: initial guess must be finite");
  double* b = s->w;
  double* d = b + nz;
  double* gamma = d + nl;
  double* zqp = gamma + nl;
  double* znew = zqp + nz;
  double* lnew = znew + nz;
  memcpy(s->z, z0, sizeof(double) * (size_t)nz);
  memcpy(s->lam, lambda0, sizeof(double) * (size_t)nl);
  double mu = 1.0;
  int iters = 0, converged = 0;
  for (int iter = 0; iter < cfg->max_sqp_iters; ++iter) {
    if ((e = port_linearize(s, theta, s->z, cfg->eps_pd, st))) return e;
    if ((e = port_assemble(s, st))) return e;
    port_flat_b(s, b);
    port_flat_d(s, d);
    port_gamma(s, b, d, gamma, st);
    int it, conv;
    double feta;
    if ((e = port_pcg(s, gamma, s->lam, cfg->pcg_epsilon, cfg->pcg_max_iters, lnew, &it, &feta, &conv, NULL, 0,
                      st)))
      return e;
    memcpy(s->lam, lnew, sizeof(double) * (size_t)nl);
    if (pcg_iters) pcg_iters[iter] = it;
    port_recover(s, s->lam, b, zqp, st);
    double alpha, mu_new;
    int acc;
    if ((e = port_line_search(s, theta, s->z, zqp, cfg, mu, znew, &alpha, &acc, &mu_new, st))) return e;
    mu = mu_new;
    if (!all_finite(znew, nz))
      return fail(st, PORT_DIVERGENCE, 0, "sqp: non-finite iterate at iteration %d", iter + 1);
    /* trajectory.hpp:64-68: max |dx| then max |du| */
    double step = 0.0, dxm = -1.0, dum = 0.0;
    int have_u = 0;
    for (int t = 0; t <= s->T; ++t)
      for (int i = 0; i < s->nx; ++i) {
        double v = fabs(znew[xoff(s, t) + i] - s->z[xoff(s, t) + i]);
        if (dxm < 0.0 || v > dxm) dxm = v;
      }
    for (int t = 0; t < s->T; ++t)
      for (int i = 0; i < s->nu; ++i) {
        double v = fabs(znew[uoff(s, t) + i] - s->z[uoff(s, t) + i]);
        if (!have_u || v > dum) dum = v;
        have_u = 1;
      }
    step = dxm < dum ? dum : dxm;
    memcpy(s->z, znew, sizeof(double) * (size_t)nz);
    if (step_sizes) step_sizes[iter] = alpha;
    ++iters;
    if (step <= cfg->convergence_tol) {
      converged = 1;
      break;
    }
  }
  if ((e = port_linearize(s, theta, s->z, cfg->eps_pd, st))) return e;
  if ((e = port_assemble(s, st))) return e;
  double kkt;
  if ((e = port_kkt_inf_norm(s, theta, s->z, s->lam, &kkt, st))) return e;
  memcpy(z_out, s->z, sizeof(double) * (size_t)nz);
  memcpy(lambda_out, s->lam, sizeof(double) * (size_t)nl);
  *sqp_iters_out = iters;
  *converged_out = converged;
  *kkt_out = kkt;
  return PORT_OK;
}

/* theta_vjp: affine_quadratic.hpp:82-117 and quadratic_cost.hpp:24-45 */
static void theta_vjp(port_solver* s, const double* theta, const double* z, const double* lam, const double* zt,
                      const double* lt, double* grad) {
  (void)theta;
  const int nx = s->nx, nu = s->nu, T = s->T;
  const double s2 = 2.0 * cost_scale(s);
  memset(grad, 0, sizeof(double) * (size_t)s->ntheta);
  double* gwx = grad;
  double* gwu = grad + nx;
  for (int t = 0; t <= T; ++t)
    for (int i = 0; i < nx; ++i) gwx[i] = gwx[i] - s2 * (z[xoff(s, t) + i] * zt[xoff(s, t) + i]);
  for (int t = 0; t < T; ++t)
    for (int i = 0; i < nu; ++i) gwu[i] = gwu[i] - s2 * (z[uoff(s, t) + i] * zt[uoff(s, t) + i]);
  if (s->p.family == PORT_AFFINE_QUADRATIC) {
    double* ga = grad + nx + nu;
    double* gb = ga + nx * nx;
    double* goff = gb + nx * nu;
    double* gxs = goff + nx;
    for (int t = 0; t < T; ++t) {
      const double* l = lam + (t + 1) * nx;
      const double* m = lt + (t + 1) * nx;
      const double* x = z + xoff(s, t);
      const double* u = z + uoff(s, t);
      const double* zx = zt + xoff(s, t);
      const double* zu = zt + uoff(s, t);
      for (int j = 0; j < nx; ++j)
        for (int i = 0; i < nx; ++i) ga[i + j * nx] = ga[i + j * nx] + l[i] * zx[j];
      for (int j = 0; j < nx; ++j)
        for (int i = 0; i < nx; ++i) ga[i + j * nx] = ga[i + j * nx] + m[i] * x[j];
      for (int j = 0; j < nu; ++j)
        for (int i = 0; i < nx; ++i) gb[i + j * nx] = gb[i + j * nx] + l[i] * zu[j];
      for (int j = 0; j < nu; ++j)
        for (int i = 0; i < nx; ++i) gb[i + j * nx] = gb[i + j * nx] + m[i] * u[j];
      for (int i = 0; i < nx; ++i) goff[i] = goff[i] + m[i];
    }
    for (int i = 0; i < nx; ++i) gxs[i] = gxs[i] + lt[i];
  } else {
    double* gxs = grad + 5;
    for (int i = 0; i < 4; ++i) gxs[i] = gxs[i] + lt[i];
  }
}

int port_backward(port_solver* s, const double* theta, const double* loss_grad_z, const double* lambda_tilde0,
                  double pcg_epsilon, int pcg_max_iters, double* grad_theta, double* lt_out, int* pcg_iters,
                  port_status* st) {
  /* backward.hpp:27-50 */
  const int nz = s->nz, nl = s->nlam;
  double* b = s->w + 2 * (size_t)(nz + nl);
  double* d = b + nz;
  double* gamma = d + nl;
  double* zt = gamma + nl;
  ok(st);
  for (int k = 0; k < nz; ++k) b[k] = -loss_grad_z[k];
  memset(d, 0, sizeof(double) * (size_t)nl);
  port_gamma(s, b, d, gamma, st);
  int conv, e;
  double feta;
  if ((e = port_pcg(s, gamma, lambda_tilde0, pcg_epsilon, pcg_max_iters, lt_out, pcg_iters, &feta, &conv, NULL, 0,
                    st)))
    return e;
  port_recover(s, lt_out, b, zt, st);
  theta_vjp(s, theta, s->z, s->lam, zt, lt_out, grad_theta);
  return PORT_OK;
}

/* ------------------------------------------------------------------ accessors */

void port_get_qp(port_solver* s, double* Q, double* q, double* R, double* r, double* Ap, double* A, double* B,
                 double* C, double* x_s, int* pd) {
  const size_t nx = (size_t)s->nx, nu = (size_t)s->nu, T = (size_t)s->T;
#define CP(dst, src, n) \
  if (dst) memcpy(dst, src, sizeof(double) * (n))
  CP(Q, s->Q, (T + 1) * nx * nx);
  CP(q, s->q, (T + 1) * nx);
  CP(R, s->R, T * nu * nu);
  CP(r, s->r, T * nu);
  CP(Ap, s->Ap, T * nx * nx);
  CP(A, s->A, T * nx * nx);
  CP(B, s->B, T * nx * nu);
  CP(C, s->C, T * nx);
  CP(x_s, s->xs, nx);
  if (pd) *pd = s->pd_projected;
}

void port_get_schur(port_solver* s, double* Sd, double* Ssub, double* Pd, double* Psup) {
  const size_t nx = (size_t)s->nx, T = (size_t)s->T;
  CP(Sd, s->Sd, (T + 1) * nx * nx);
  CP(Ssub, s->Ssub, T * nx * nx);
  CP(Pd, s->Pd, (T + 1) * nx * nx);
  CP(Psup, s->Psup, T * nx * nx);
#undef CP
}

/* ------------------------------------------------------------------ IL epoch */

int port_il_epoch(const port_problem* prob, int batch, const double* thetas, const double* demos,
                  double* lambda_cache, double* lt_cache, const port_sqp_config* cfg, int learn_start,
                  int learn_size, double* loss_sum, double* grad_sum, double* losses, double* grads,
                  int* sqp_iters, long* pcg_iters, port_status* st) {
  /* train.hpp:76-131 */
  port_solver* s = port_create(prob);
  if (!s) return fail(st, PORT_DIMENSION, 0, "port: bad problem");
  const int nz = s->nz, nl = s->nlam, nth = s->ntheta, nx = s->nx, nu = s->nu, T = s->T;
  double* z = (double*)malloc(sizeof(double) * (size_t)(2 * nz + 3 * nl + nth));
  double* lam = z + nz;
  double* lg = lam + nl;
  double* lt = lg + nz;
  double* lt0 = lt + nl;
  double* g = lt0 + nl;
  int first_err = PORT_OK;
  port_status est;
  int* pcg_buf = (int*)malloc(sizeof(int) * (size_t)(cfg->max_sqp_iters + 1));
  for (int j = 0; j < batch; ++j) {
    const double* th = thetas + (size_t)j * nth;
    const double* demo = demos + (size_t)j * nz;
    int it, conv, bit;
    double kkt;
    int e = port_sqp_solve(s, th, demo, lambda_cache + (size_t)j * nl, cfg, z, lam, &it, &conv, &kkt, pcg_buf,
                           NULL, &est);
    if (!e) {
      double l2 = 0.0;
      int first = 1;
      memset(lg, 0, sizeof(double) * (size_t)nz);
      for (int t = 0; t < T; ++t)
        for (int i = 0; i < nu; ++i) {
          double du = z[uoff(s, t) + i] - demo[uoff(s, t) + i];
          l2 = first ? du * du : l2 + du * du;
          first = 0;
          lg[uoff(s, t) + i] = 2.0 / batch * du;
        }
      losses[j] = l2 / batch;
      memcpy(lt0, lt_cache + (size_t)j * nl, sizeof(double) * (size_t)nl);
      e = port_backward(s, th, lg, lt0, cfg->pcg_epsilon, cfg->pcg_max_iters, g, lt, &bit, &est);
      if (!e) {
        memcpy(grads + (size_t)j * learn_size, g + learn_start, sizeof(double) * (size_t)learn_size);
        sqp_iters[j] = it;
        long pc = 0;
        for (int k = 0; k < it; ++k) pc += pcg_buf[k];
        pcg_iters[j] = pc + bit;
        memcpy(lambda_cache + (size_t)j * nl, lam, sizeof(double) * (size_t)nl);
        memcpy(lt_cache + (size_t)j * nl, lt, sizeof(double) * (size_t)nl);
      }
    }
    if (e && first_err == PORT_OK) {
      first_err = e;
      if (st) {
        *st = est;
        char buf[192];
        snprintf(buf, sizeof buf, "demonstration %d: %s", j, est.message);
        memcpy(st->message, buf, sizeof buf);
      }
    }
  }
  (void)nx;
  if (first_err == PORT_OK) {
    double obj = 0.0;
    for (int k = 0; k < learn_size; ++k) grad_sum[k] = 0.0;
    for (int j = 0; j < batch; ++j) {
      obj = obj + losses[j];
      for (int k = 0; k < learn_size; ++k) grad_sum[k] = grad_sum[k] + grads[(size_t)j * learn_size + k];
    }
    *loss_sum = obj;
    ok(st);
  }
  free(pcg_buf);
  free(z);
  port_destroy(s);
  return first_err;
}
