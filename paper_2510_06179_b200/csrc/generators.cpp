// generators.cpp — synthetic inputs of the benchmark shapes, drawn with the
// reference generators' recipe (bench/generators.hpp:52-168) from the same
// libstdc++ engine and distributions, so instance k of seed s is the
// reference's instance k up to the spectral-radius rescale (our Hessenberg-QR
// eigenvalues vs Eigen's EigenSolver agree to rounding).
#include <cmath>
#include <complex>
#include <cstdint>
#include <random>
#include <vector>

#include "docp_cuda.h"

namespace {

/// Eigenvalue moduli of a real n x n (column-major) matrix: Householder
/// Hessenberg reduction + Francis double-shift QR; returns the spectral radius.
double spectral_radius(std::vector<double> a, int n) {
  auto A = [&](int i, int j) -> double& { return a[static_cast<size_t>(i + j * n)]; };
  for (int k = 0; k < n - 2; ++k) {
    double alpha = 0.0;
    for (int i = k + 1; i < n; ++i) alpha += A(i, k) * A(i, k);
    alpha = std::sqrt(alpha);
    if (alpha == 0.0) continue;
    if (A(k + 1, k) > 0) alpha = -alpha;
    std::vector<double> v(static_cast<size_t>(n), 0.0);
    v[k + 1] = A(k + 1, k) - alpha;
    for (int i = k + 2; i < n; ++i) v[i] = A(i, k);
    double vn = 0.0;
    for (int i = k + 1; i < n; ++i) vn += v[i] * v[i];
    if (vn == 0.0) continue;
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      for (int i = k + 1; i < n; ++i) s += v[i] * A(i, j);
      s = 2.0 * s / vn;
      for (int i = k + 1; i < n; ++i) A(i, j) -= s * v[i];
    }
    for (int i = 0; i < n; ++i) {
      double s = 0.0;
      for (int j = k + 1; j < n; ++j) s += A(i, j) * v[j];
      s = 2.0 * s / vn;
      for (int j = k + 1; j < n; ++j) A(i, j) -= s * v[j];
    }
  }
  std::vector<std::complex<double>> ev(static_cast<size_t>(n));
  int nn = n - 1, m = 0, l = 0, its = 0;
  double z = 0, y, x, w, v, u, t = 0.0, s, r = 0, q = 0, p = 0, anorm = 0.0;
  const double eps = std::numeric_limits<double>::epsilon();
  for (int i = 0; i < n; i++)
    for (int j = std::max(i - 1, 0); j < n; j++) anorm += std::abs(A(i, j));
  while (nn >= 0) {
    its = 0;
    do {
      for (l = nn; l > 0; l--) {
        s = std::abs(A(l - 1, l - 1)) + std::abs(A(l, l));
        if (s == 0.0) s = anorm;
        if (std::abs(A(l, l - 1)) <= eps * s) {
          A(l, l - 1) = 0.0;
          break;
        }
      }
      x = A(nn, nn);
      if (l == nn) {
        ev[nn--] = x + t;
      } else {
        y = A(nn - 1, nn - 1);
        w = A(nn, nn - 1) * A(nn - 1, nn);
        if (l == nn - 1) {
          p = 0.5 * (y - x);
          q = p * p + w;
          z = std::sqrt(std::abs(q));
          x += t;
          if (q >= 0.0) {
            z = p + (p >= 0 ? std::abs(z) : -std::abs(z));
            ev[nn - 1] = ev[nn] = x + z;
            if (z != 0.0) ev[nn] = x - w / z;
          } else {
            ev[nn] = {x + p, -z};
            ev[nn - 1] = {x + p, z};
          }
          nn -= 2;
        } else {
          if (its == 60) return -1.0;
          if (its == 10 || its == 20) {
            t += x;
            for (int i = 0; i <= nn; i++) A(i, i) -= x;
            s = std::abs(A(nn, nn - 1)) + std::abs(A(nn - 1, nn - 2));
            y = x = 0.75 * s;
            w = -0.4375 * s * s;
          }
          ++its;
          for (m = nn - 2; m >= l; m--) {
            z = A(m, m);
            r = x - z;
            s = y - z;
            p = (r * s - w) / A(m + 1, m) + A(m, m + 1);
            q = A(m + 1, m + 1) - z - r - s;
            r = A(m + 2, m + 1);
            s = std::abs(p) + std::abs(q) + std::abs(r);
            p /= s;
            q /= s;
            r /= s;
            if (m == l) break;
            u = std::abs(A(m, m - 1)) * (std::abs(q) + std::abs(r));
            v = std::abs(p) * (std::abs(A(m - 1, m - 1)) + std::abs(z) + std::abs(A(m + 1, m + 1)));
            if (u <= eps * v) break;
          }
          for (int i = m; i < nn - 1; i++) {
            A(i + 2, i) = 0.0;
            if (i != m) A(i + 2, i - 1) = 0.0;
          }
          for (int k = m; k < nn; k++) {
            if (k != m) {
              p = A(k, k - 1);
              q = A(k + 1, k - 1);
              r = 0.0;
              if (k + 1 != nn) r = A(k + 2, k - 1);
              if ((x = std::abs(p) + std::abs(q) + std::abs(r)) != 0.0) {
                p /= x;
                q /= x;
                r /= x;
              }
            }
            const double sq = std::sqrt(p * p + q * q + r * r);
            if ((s = (p >= 0 ? sq : -sq)) != 0.0) {
              if (k == m) {
                if (l != m) A(k, k - 1) = -A(k, k - 1);
              } else {
                A(k, k - 1) = -s * x;
              }
              p += s;
              x = p / s;
              y = q / s;
              z = r / s;
              q /= p;
              r /= p;
              for (int j = k; j <= nn; j++) {
                p = A(k, j) + q * A(k + 1, j);
                if (k + 1 != nn) {
                  p += r * A(k + 2, j);
                  A(k + 2, j) -= p * z;
                }
                A(k + 1, j) -= p * y;
                A(k, j) -= p * x;
              }
              const int mmin = nn < k + 3 ? nn : k + 3;
              for (int i = l; i <= mmin; i++) {
                p = x * A(i, k) + y * A(i, k + 1);
                if (k + 1 != nn) {
                  p += z * A(i, k + 2);
                  A(i, k + 2) -= p * r;
                }
                A(i, k + 1) -= p * q;
                A(i, k) -= p;
              }
            }
          }
        }
      }
    } while (l + 1 < nn);
  }
  double rho = 0.0;
  for (const auto& e : ev) rho = std::max(rho, std::abs(e));
  return rho;
}

/// random_linear_instance (generators.hpp:52-79) written in theta layout.
void linear_instance(int nx, int nu, std::mt19937_64& rng, double* th) {
  std::normal_distribution<double> normal(0.0, 1.0);
  double* wx = th;
  double* wu = wx + nx;
  double* a = wu + nu;
  double* b = a + nx * nx;
  double* off = b + nx * nu;
  double* xs = off + nx;
  for (int i = 0; i < nx; ++i) wx[i] = 1.0;
  for (int i = 0; i < nu; ++i) wu[i] = 1.0;
  std::vector<double> delta(static_cast<size_t>(nx * nx));
  for (int j = 0; j < nx; ++j)
    for (int i = 0; i < nx; ++i) delta[i + j * nx] = normal(rng);
  for (int j = 0; j < nx; ++j)
    for (int i = 0; i < nx; ++i) a[i + j * nx] = (i == j ? 1.0 : 0.0) + 0.1 * delta[i + j * nx];
  const double rho = spectral_radius(std::vector<double>(a, a + nx * nx), nx);
  if (rho > 0.99)
    for (int k = 0; k < nx * nx; ++k) a[k] = a[k] * (0.99 / rho);
  for (int j = 0; j < nu; ++j)
    for (int i = 0; i < nx; ++i) b[i + j * nx] = normal(rng);
  for (int i = 0; i < nx; ++i) off[i] = 1e-2 * normal(rng);
  for (int i = 0; i < nx; ++i) xs[i] = 5.0 * normal(rng);
}

}  // namespace

extern "C" {

/// count sequential instances of random_convex_instance (convex != 0,
/// generators.hpp:102-111) or random_linear_instance from mt19937_64(seed),
/// each written as its theta (affine_quadratic.hpp:27-37).
int docp_generate_affine_quadratic(int32_t nx, int32_t nu, uint64_t seed, int32_t count, int32_t convex,
                                   double* thetas) {
  if (nx < 1 || nu < 1 || count < 0 || !thetas) return DOCP_INVALID;
  std::mt19937_64 rng(seed);
  const size_t nth = static_cast<size_t>(nx + nu + nx * nx + nx * nu + 2 * nx);
  for (int k = 0; k < count; ++k) {
    double* th = thetas + nth * static_cast<size_t>(k);
    if (!convex) {
      linear_instance(nx, nu, rng, th);
      continue;
    }
    std::uniform_real_distribution<double> weight(0.5, 2.0);
    std::normal_distribution<double> normal(0.0, 1.0);
    linear_instance(nx, nu, rng, th);
    for (int i = 0; i < nx; ++i) th[i] = weight(rng);
    for (int i = 0; i < nu; ++i) th[nx + i] = weight(rng);
    double* xs = th + nth - nx;
    for (int i = 0; i < nx; ++i) xs[i] = normal(rng);
  }
  return DOCP_OK;
}

/// The drifting instance sequence of pcg_study (study.hpp:74-77, 123-124 and
/// perturb_coefficients, study.hpp:37-48): random_convex_instance from
/// mt19937_64(seed), then after every step each coefficient of A, B, b and
/// x_s (in that order, column-major) is scaled by 1 + U(-magnitude, magnitude)
/// drawn from the same engine. thetas: [steps][n_theta].
int docp_generate_drift_sequence(int32_t nx, int32_t nu, uint64_t seed, int32_t steps, double magnitude,
                                 double* thetas) {
  if (nx < 1 || nu < 1 || steps < 0 || !thetas) return DOCP_INVALID;
  std::mt19937_64 rng(seed);
  const size_t nth = static_cast<size_t>(nx + nu + nx * nx + nx * nu + 2 * nx);
  std::vector<double> cur(nth);
  {
    std::uniform_real_distribution<double> weight(0.5, 2.0);
    std::normal_distribution<double> normal(0.0, 1.0);
    linear_instance(nx, nu, rng, cur.data());
    for (int i = 0; i < nx; ++i) cur[i] = weight(rng);
    for (int i = 0; i < nu; ++i) cur[nx + i] = weight(rng);
    for (int i = 0; i < nx; ++i) cur[nth - nx + i] = normal(rng);
  }
  for (int k = 0; k < steps; ++k) {
    std::copy(cur.begin(), cur.end(), thetas + nth * static_cast<size_t>(k));
    std::uniform_real_distribution<double> u(-magnitude, magnitude);
    for (size_t e = static_cast<size_t>(nx + nu); e < nth; ++e) cur[e] *= 1.0 + u(rng);  // A, B, b, x_s
  }
  return DOCP_OK;
}

/// n draws of uniform_real_distribution(lo, hi) from mt19937_64(seed)
/// (train.hpp:61-64 initial weights; generators.hpp:142-151 initial states).
int docp_generate_uniform(uint64_t seed, int32_t n, double lo, double hi, double* out) {
  if (n < 0 || !out) return DOCP_INVALID;
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u(lo, hi);
  for (int i = 0; i < n; ++i) out[i] = u(rng);
  return DOCP_OK;
}

/// Cart-pole initial states of gen_cartpole (generators.hpp:142-152):
/// U([-.5,.5] x [-.5,.5] x [-pi,pi] x [-1,1]), n x 4.
int docp_generate_cartpole_x0(uint64_t seed, int32_t n, double* x0) {
  if (n < 0 || !x0) return DOCP_INVALID;
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u_half(-0.5, 0.5);
  std::uniform_real_distribution<double> u_pi(-M_PI, M_PI);
  std::uniform_real_distribution<double> u_one(-1.0, 1.0);
  for (int i = 0; i < n; ++i) {
    // Vector x0(4); x0 << u_half(rng), u_half(rng), u_pi(rng), u_one(rng);
    const double a = u_half(rng);
    const double b = u_half(rng);
    const double c = u_pi(rng);
    const double d = u_one(rng);
    x0[4 * i + 0] = a;
    x0[4 * i + 1] = b;
    x0[4 * i + 2] = c;
    x0[4 * i + 3] = d;
  }
  return DOCP_OK;
}

}  // extern "C"
