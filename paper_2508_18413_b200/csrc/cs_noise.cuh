// Distribution transforms of the counter noise (noise.py:140-156) on device.
//
// uniform      ((h >> 11) + 0.5) 2^-53, counter 2k                  (exact)
// normal       sqrt(-2 ln u1) cos(2 pi u2), counters 2k, 2k+1        (~1 ulp)
// chi-squared  2 * gammaincinv(df/2, u), counter 2k: scipy's inverse regularised
//              lower incomplete gamma, restated as Halley iteration on
//              P(a, x) - u with P from its series / continued fraction
//              (|P(a, x) - u| <= 1e-13, the reference pins 1e-12 in
//              test_noise.py:72-80).
#pragma once
#include "cs_rng.cuh"

namespace cs {

// regularised lower incomplete gamma P(a, x), a > 0
CS_D double gamma_p(double a, double x, double lga) {
  if (x <= 0.0) return 0.0;
  const double lpre = a * log(x) - x - lga;
  if (x < a + 1.0) {
    double ap = a, del = 1.0 / a, sum = del;
    for (int n = 0; n < 1000; ++n) {
      ap += 1.0;
      del *= x / ap;
      sum += del;
      if (fabs(del) < fabs(sum) * 1e-17) break;
    }
    return sum * exp(lpre);
  }
  // Lentz continued fraction for Q
  const double tiny = 1e-300;
  double b = x + 1.0 - a, c = 1.0 / tiny, d = 1.0 / b, h = d;
  for (int i = 1; i < 1000; ++i) {
    const double an = -i * (i - a);
    b += 2.0;
    d = an * d + b;
    if (fabs(d) < tiny) d = tiny;
    c = b + an / c;
    if (fabs(c) < tiny) c = tiny;
    d = 1.0 / d;
    const double del = d * c;
    h *= del;
    if (fabs(del - 1.0) < 1e-17) break;
  }
  return 1.0 - exp(lpre) * h;
}

// x with P(a, x) = p (Numerical-Recipes style start, Halley refinement)
CS_D double gamma_p_inv(double a, double p) {
  if (p <= 0.0) return 0.0;
  if (p >= 1.0) return INFINITY;
  const double lga = lgamma(a), a1 = a - 1.0;
  double x, lna1 = 0.0, afac = 0.0;
  if (a > 1.0) {
    lna1 = log(a1);
    afac = exp(a1 * (lna1 - 1.0) - lga);
    const double pp = p < 0.5 ? p : 1.0 - p;
    const double t = sqrt(-2.0 * log(pp));
    double z = (2.30753 + t * 0.27061) / (1.0 + t * (0.99229 + t * 0.04481)) - t;
    if (p < 0.5) z = -z;
    x = fmax(1e-3, a * pow(1.0 - 1.0 / (9.0 * a) - z / (3.0 * sqrt(a)), 3.0));
  } else {
    const double t = 1.0 - a * (0.253 + a * 0.12);
    if (p < t) x = pow(p / t, 1.0 / a);
    else x = 1.0 - log(1.0 - (p - t) / (1.0 - t));
  }
  for (int j = 0; j < 100; ++j) {
    if (x <= 0.0) return 0.0;
    const double err = gamma_p(a, x, lga) - p;
    double dt;
    if (a > 1.0) dt = afac * exp(-(x - a1) + a1 * (log(x) - lna1));
    else dt = exp(-x + a1 * log(x) - lga);
    if (dt == 0.0) break;
    const double u = err / dt;
    const double step = u / (1.0 - 0.5 * fmin(1.0, u * ((a - 1.0) / x - 1.0)));
    x -= step;
    if (x <= 0.0) x = 0.5 * (x + step);
    if (fabs(step) < 1e-15 * x) break;
  }
  return x;
}

CS_D double noise_value(int kind, uint64_t h3, int k, double df) {
  const double u1 = bits_to_unit(hash_c(h3, 2ull * (uint64_t)k));
  switch (kind) {
    case CS_NOISE_UNIFORM: return u1;
    case CS_NOISE_LOG_UNIFORM: return log(u1);
    case CS_NOISE_NORMAL: {
      const double u2 = bits_to_unit(hash_c(h3, 2ull * (uint64_t)k + 1ull));
      return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
    }
    default: return 2.0 * gamma_p_inv(0.5 * df, u1);
  }
}

}  // namespace cs
