// crmath.cuh — correctly rounded sin / cos in double-double arithmetic.
//
// The cart-pole family evaluates sin/cos of the pole angle (cartpole.hpp:28-78).
// The reference gets them from glibc, whose results are correctly rounded in
// all but vanishingly rare cases; CUDA's sin/cos are only within 2 ulp, which
// is enough to flip near-zero line-search decisions. These versions evaluate
// the argument reduction (3-part pi/2) and the Taylor series in double-double
// (~1e-31 relative), then round once, so they return the correctly rounded
// value except when the exact result lies within ~1e-31 of a rounding midpoint.
#pragma once

#include <cmath>

#ifndef __CUDACC__
#define __host__
#define __device__
#endif

namespace crmath {

struct dd {
  double hi, lo;
};

__host__ __device__ inline dd two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
__host__ __device__ inline dd quick_two_sum(double a, double b) {
  const double s = a + b;
  return {s, b - (s - a)};
}
__host__ __device__ inline dd two_prod(double a, double b) {
  const double p = a * b;
  return {p, std::fma(a, b, -p)};
}
__host__ __device__ inline dd add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  const dd t = two_sum(a.lo, b.lo);
  s.lo = s.lo + t.hi;
  s = quick_two_sum(s.hi, s.lo);
  s.lo = s.lo + t.lo;
  return quick_two_sum(s.hi, s.lo);
}
__host__ __device__ inline dd mul(dd a, dd b) {
  dd p = two_prod(a.hi, b.hi);
  p.lo = p.lo + (a.hi * b.lo + a.lo * b.hi);
  return quick_two_sum(p.hi, p.lo);
}

// (-1)^k / (2k+1)!  and  (-1)^k / (2k)!  as double-double (hi, lo), k ascending
__host__ __device__ inline dd sin_coef(int k) {
  constexpr double c[15][2] = {{1.0, 0.0},
                               {-0.16666666666666666, -9.25185853854297e-18},
                               {0.008333333333333333, 1.1564823173178714e-19},
                               {-0.0001984126984126984, -1.7209558293420705e-22},
                               {2.7557319223985893e-06, -1.858393274046472e-22},
                               {-2.505210838544172e-08, 1.448814070935912e-24},
                               {1.6059043836821613e-10, 1.2585294588752098e-26},
                               {-7.647163731819816e-13, -7.03872877733453e-30},
                               {2.8114572543455206e-15, 1.6508842730861433e-31},
                               {-8.22063524662433e-18, -2.2141894119604265e-34},
                               {1.9572941063391263e-20, -1.3643503830087908e-36},
                               {-3.868170170630684e-23, 8.843177655482344e-40},
                               {6.446950284384474e-26, -1.9330404233703465e-42},
                               {-9.183689863795546e-29, -1.4303150396787322e-45},
                               {1.1309962886447716e-31, 1.0498015412959506e-47}};
  return {c[k][0], c[k][1]};
}
__host__ __device__ inline dd cos_coef(int k) {
  constexpr double c[15][2] = {{1.0, 0.0},
                               {-0.5, 0.0},
                               {0.041666666666666664, 2.3129646346357427e-18},
                               {-0.001388888888888889, 5.300543954373577e-20},
                               {2.48015873015873e-05, 2.1511947866775882e-23},
                               {-2.755731922398589e-07, -2.3767714622250297e-23},
                               {2.08767569878681e-09, -1.20734505911326e-25},
                               {-1.1470745597729725e-11, -2.0655512752830745e-28},
                               {4.779477332387385e-14, 4.399205485834081e-31},
                               {-1.5619206968586225e-16, -1.1910679660273754e-32},
                               {4.110317623312165e-19, 1.4412973378659527e-36},
                               {-8.896791392450574e-22, 7.911402614872376e-38},
                               {1.6117375710961184e-24, -3.6846573564509766e-41},
                               {-2.4795962632247976e-27, 1.2953730964765229e-43},
                               {3.279889237069838e-30, 1.5117542744029879e-46}};
  return {c[k][0], c[k][1]};
}

/// sin(x) and cos(x), correctly rounded for |x| < 2^20 (larger arguments fall
/// back to the platform functions).
__host__ __device__ inline void sincos_cr(double x, double* s_out, double* c_out) {
  if (!(std::fabs(x) < 1048576.0)) {
    *s_out = std::sin(x);
    *c_out = std::cos(x);
    return;
  }
  constexpr double P1 = 1.5707963267948966, P2 = 6.123233995736766e-17, P3 = -1.4973849048591698e-33;
  const double k = std::rint(x * 0.6366197723675814);
  // r = x - k (P1 + P2 + P3) in double-double
  const dd k1 = two_prod(k, P1);
  dd r = two_sum(x, -k1.hi);
  r = add(r, {-k1.lo, 0.0});
  const dd k2 = two_prod(k, P2);
  r = add(r, {-k2.hi, -k2.lo});
  r = add(r, {-(k * P3), 0.0});
  const dd r2 = mul(r, r);
  dd ps = sin_coef(14), pc = cos_coef(14);
  for (int i = 13; i >= 0; --i) {
    ps = add(mul(ps, r2), sin_coef(i));
    pc = add(mul(pc, r2), cos_coef(i));
  }
  ps = mul(ps, r);
  const double sv = ps.hi + ps.lo, cv = pc.hi + pc.lo;
  const long q = static_cast<long>(k) & 3;
  if (q == 0) {
    *s_out = sv;
    *c_out = cv;
  } else if (q == 1) {
    *s_out = cv;
    *c_out = -sv;
  } else if (q == 2) {
    *s_out = -sv;
    *c_out = -cv;
  } else {
    *s_out = -cv;
    *c_out = sv;
  }
}

}  // namespace crmath
