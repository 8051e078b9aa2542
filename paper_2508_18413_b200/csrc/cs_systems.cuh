// Transition systems f_t and their solver-form tangents, one thread per step.
//
// Each system exposes
//   prepare(t, s, aux)          forward pass; false if the proposal / trajectory
//                               is non-finite (samplers.py:101-105, 332-336)
//   f(aux, out)                 the hard-gated step (samplers.py:120-122, 344-346)
//   relaxed_f(aux, out)         sigmoid-gated step (124-127, 348-351)
//   jvp_many<NT>(aux, V, out, n, relaxed)   n <= NT tangents J v at the same s
// with the reference's arithmetic order, all in f64 registers.  Noise rows are
// read from the pre-drawn sequence (noise.py:107-113: step t reads row t).
#pragma once
#include "cs_rng.cuh"
#include "cs_targets.cuh"

namespace cs {

// ---------------------------------------------------------------------------
// MALA (samplers.py:71-148)
template <int MD, typename ST, int TK = -1>
struct Mala {
  Target<MD, TK> tg;
  double eps, sq2eps, inv4eps, inv2eps;
  const ST *xi;
  const double *logu;

  struct Aux {
    double S[MD], prop[MD], g0[MD], g1[MD], back[MD];
    double delta, margin;
  };

  CS_D int dim() const { return tg.p.dim; }
  CS_D int mem_index(int k) const { return k < tg.p.dim ? k : -1; }

  CS_D bool prepare(int64_t t, const double (&s)[MD], Aux &a) const {
    const int D = dim();
    bool ok = true;
#pragma unroll
    for (int i = 0; i < MD; ++i) a.S[i] = s[i];
    tg.grad(s, a.g0);
    double xx = 0.0;
#pragma unroll
    for (int i = 0; i < MD; ++i) {
      double z = (i < D) ? ld(xi, t * D + i) : 0.0;
      a.prop[i] = (i < D) ? (s[i] + eps * a.g0[i]) + sq2eps * z : 0.0;
      ok &= (i >= D) || finite(a.prop[i]);
      xx += z * z;
    }
    tg.grad(a.prop, a.g1);
    double rr = 0.0;
#pragma unroll
    for (int i = 0; i < MD; ++i) {
      a.back[i] = (i < D) ? (s[i] - a.prop[i]) - eps * a.g1[i] : 0.0;
      rr += a.back[i] * a.back[i];
    }
    a.delta = ((tg.logp(a.prop) - tg.logp(s)) - rr * inv4eps) + 0.5 * xx;
    a.margin = fmin(0.0, a.delta) - __ldg(logu + t);
    return ok;
  }

  CS_D void f(const Aux &a, double (&o)[MD]) const {
    const bool acc = a.margin > 0.0;
#pragma unroll
    for (int i = 0; i < MD; ++i) o[i] = acc ? a.prop[i] : a.S[i];
  }

  CS_D void relaxed_f(const Aux &a, double (&o)[MD]) const {
    const double w = expit(a.margin);
#pragma unroll
    for (int i = 0; i < MD; ++i) o[i] = w * a.prop[i] + (1.0 - w) * a.S[i];
  }

  template <typename TT = double>
  CS_D void jvp1(const Aux &a, const double (&Vd)[MD], double (&o)[MD], bool relaxed) const {
    TT V[MD], hv[MD], dprop[MD], hd[MD];
#pragma unroll
    for (int i = 0; i < MD; ++i) V[i] = (TT)Vd[i];
    tg.hvpT(a.S, V, hv);
    const TT e = (TT)eps;
#pragma unroll
    for (int i = 0; i < MD; ++i) dprop[i] = V[i] + e * hv[i];
    tg.hvpT(a.prop, dprop, hd);
    TT s1 = 0, s2 = 0, s3 = 0;
#pragma unroll
    for (int i = 0; i < MD; ++i) {
      const TT dback = (V[i] - dprop[i]) - e * hd[i];
      s1 += (TT)a.g1[i] * dprop[i];
      s2 += (TT)a.g0[i] * V[i];
      s3 += (TT)a.back[i] * dback;
    }
    const TT ddelta = (s1 - s2) - s3 * (TT)inv2eps;
    const TT gate = (TT)(relaxed ? expit(a.margin) : (a.margin > 0.0 ? 1.0 : 0.0));
    const TT bend = (TT)sigmoid_prime(a.margin) * (ddelta * (TT)(a.delta < 0.0 ? 1.0 : 0.0));
#pragma unroll
    for (int i = 0; i < MD; ++i)
      o[i] = (double)((gate * dprop[i] + ((TT)1 - gate) * V[i]) + (TT)(a.prop[i] - a.S[i]) * bend);
  }

  template <int NT, typename TT = double>
  CS_D void jvp_many(const Aux &a, const double (&V)[NT][MD], double (&o)[NT][MD], int n,
                     bool relaxed) const {
#pragma unroll
    for (int k = 0; k < NT; ++k)
      if (k < n) jvp1<TT>(a, V[k], o[k], relaxed);
  }
};

// ---------------------------------------------------------------------------
// chain-level HMC (samplers.py:253-387); the L-step leapfrog runs in registers
template <int MD, typename ST, int TK = -1>
struct Hmc {
  Target<MD, TK> tg;
  double eps;
  int L;
  const double *mass;  // nullable
  const ST *mom;
  const double *logu;

  struct Aux {
    double S[MD], vh0[MD], g0[MD], xl[MD], vl[MD], gl[MD];
    double delta, margin;
  };

  CS_D int dim() const { return tg.p.dim; }
  CS_D int mem_index(int k) const { return k < tg.p.dim ? k : -1; }
  CS_D double m(int i) const { return (mass && i < tg.p.dim) ? __ldg(mass + i) : 1.0; }
  CS_D double divm(double x, int i) const { return (mass && i < tg.p.dim) ? x / __ldg(mass + i) : x; }

  CS_D bool prepare(int64_t t, const double (&s)[MD], Aux &a) const {
    const int D = dim();
    double xx = 0.0;
    tg.grad(s, a.g0);
    double x[MD], v[MD], g[MD];
#pragma unroll
    for (int i = 0; i < MD; ++i) {
      double z = (i < D) ? ld(mom, t * D + i) : 0.0;
      xx += z * z;
      a.S[i] = s[i];
      a.vh0[i] = (i < D) ? sqrt(m(i)) * z + (0.5 * eps) * a.g0[i] : 0.0;
      x[i] = s[i];
      v[i] = a.vh0[i];
    }
    const double h0 = 0.5 * xx - tg.logp(s);
    for (int l = 0; l < L; ++l) {
#pragma unroll
      for (int i = 0; i < MD; ++i) x[i] = x[i] + divm(eps * v[i], i);
      tg.grad(x, g);
#pragma unroll
      for (int i = 0; i < MD; ++i) v[i] = v[i] + eps * g[i];
    }
    bool ok = true;
#pragma unroll
    for (int i = 0; i < MD; ++i) ok &= (i >= D) || finite(x[i]);
    tg.grad(x, a.gl);
    double kin = 0.0;
#pragma unroll
    for (int i = 0; i < MD; ++i) {
      a.xl[i] = x[i];
      a.vl[i] = v[i] - (0.5 * eps) * a.gl[i];
      if (i < D) kin += divm(a.vl[i] * a.vl[i], i);
    }
    const double hl = 0.5 * kin - tg.logp(x);
    a.delta = h0 - hl;
    a.margin = fmin(0.0, a.delta) - __ldg(logu + t);
    return ok;
  }

  CS_D void f(const Aux &a, double (&o)[MD]) const {
    const bool acc = a.margin > 0.0;
#pragma unroll
    for (int i = 0; i < MD; ++i) o[i] = acc ? a.xl[i] : a.S[i];
  }

  CS_D void relaxed_f(const Aux &a, double (&o)[MD]) const {
    const double w = expit(a.margin);
#pragma unroll
    for (int i = 0; i < MD; ++i) o[i] = w * a.xl[i] + (1.0 - w) * a.S[i];
  }

  // f_t(s) and ONE tangent J_t V in a single pass of the integrator: prepare()
  // followed by jvp_many<1>() with the same operations in the same order (so
  // the same bits), minus the second primal integration and without the Aux
  // record -- the diag quasi-Newton solve's per-step work (samplers.py:322-381).
  // Returns false when the proposal is non-finite (like prepare()).
  template <typename TT>
  CS_D bool step_tangent(int64_t t, const double (&s)[MD], const double (&V)[MD], double (&fo)[MD],
                         double (&o)[MD]) const {
    const int D = dim();
    double x[MD], v[MD], g[MD];
    TT dx[MD], dv[MD], h[MD], Vk[MD];
    const TT e = (TT)eps, he = (TT)(0.5 * eps);
    tg.grad(s, g);
#pragma unroll
    for (int i = 0; i < MD; ++i) Vk[i] = (TT)V[i];
    tg.hvpT(s, Vk, h);
    double xx = 0.0;
    TT sg = 0;
#pragma unroll
    for (int i = 0; i < MD; ++i) {
      const double z = (i < D) ? ld(mom, t * D + i) : 0.0;
      xx += z * z;
      x[i] = s[i];
      v[i] = (i < D) ? sqrt(m(i)) * z + (0.5 * eps) * g[i] : 0.0;
      dx[i] = Vk[i];
      dv[i] = he * h[i];
      sg += (TT)g[i] * Vk[i];
    }
    const TT dh0 = -sg;
    const double h0 = 0.5 * xx - tg.logp(s);
#pragma unroll 1
    for (int l = 0; l < L; ++l) {
#pragma unroll
      for (int i = 0; i < MD; ++i) x[i] = x[i] + divm(eps * v[i], i);
#pragma unroll
      for (int i = 0; i < MD; ++i) dx[i] = dx[i] + (TT)divm((double)(e * dv[i]), i);
      tg.hvpT(x, dx, h);
#pragma unroll
      for (int i = 0; i < MD; ++i) dv[i] = dv[i] + e * h[i];
      tg.grad(x, g);
#pragma unroll
      for (int i = 0; i < MD; ++i) v[i] = v[i] + eps * g[i];
    }
    // g = grad(x_L) (prepare()'s gl; the loop's last gradient, or grad(s) at L = 0)
    bool ok = true;
#pragma unroll
    for (int i = 0; i < MD; ++i) ok &= (i >= D) || finite(x[i]);
    double kin = 0.0;
#pragma unroll
    for (int i = 0; i < MD; ++i) {
      v[i] = v[i] - (0.5 * eps) * g[i];  // vl
      if (i < D) kin += divm(v[i] * v[i], i);
    }
    const double hl = 0.5 * kin - tg.logp(x);
    const double delta = h0 - hl;
    const double margin = fmin(0.0, delta) - __ldg(logu + t);
    const bool acc = margin > 0.0;
#pragma unroll
    for (int i = 0; i < MD; ++i) fo[i] = acc ? x[i] : s[i];
    const TT gate = (TT)(acc ? 1.0 : 0.0);
    tg.hvpT(x, dx, h);
    TT s1 = 0, s2 = 0;
#pragma unroll
    for (int i = 0; i < MD; ++i) {
      const TT dvl = dv[i] - he * h[i];
      if (i < D) s1 += (TT)divm((double)((TT)v[i] * dvl), i);
      s2 += (TT)g[i] * dx[i];
    }
    const TT ddelta = dh0 - (s1 - s2);
    // sigmoid_prime (an f64 exp + log) only matters where delta < 0
    const TT bend = delta < 0.0 ? (TT)sigmoid_prime(margin) * ddelta : ddelta * (TT)0;
#pragma unroll
    for (int i = 0; i < MD; ++i)
      o[i] = (double)((gate * dx[i] + ((TT)1 - gate) * Vk[i]) + (TT)(x[i] - s[i]) * bend);
    return ok;
  }

  // tangents ride the forward integrator (samplers.py:353-381), all n at once,
  // in tangent precision TT; the positions they are linearised at stay f64
  template <int NT, typename TT = double>
  CS_D void jvp_many(const Aux &a, const double (&V)[NT][MD], double (&o)[NT][MD], int n,
                     bool relaxed) const {
    const int D = dim();
    TT dx[NT][MD], dv[NT][MD], dh0[NT], h[MD];
    double x[MD], v[MD], g[MD];
    const TT e = (TT)eps, he = (TT)(0.5 * eps);
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      if (k >= n) continue;
      TT Vk[MD];
#pragma unroll
      for (int i = 0; i < MD; ++i) Vk[i] = (TT)V[k][i];
      tg.hvpT(a.S, Vk, h);
      TT s = 0;
#pragma unroll
      for (int i = 0; i < MD; ++i) {
        dx[k][i] = Vk[i];
        dv[k][i] = he * h[i];
        s += (TT)a.g0[i] * Vk[i];
      }
      dh0[k] = -s;
    }
#pragma unroll
    for (int i = 0; i < MD; ++i) { x[i] = a.S[i]; v[i] = a.vh0[i]; }
    for (int l = 0; l < L; ++l) {
#pragma unroll
      for (int i = 0; i < MD; ++i) x[i] = x[i] + divm(eps * v[i], i);
#pragma unroll
      for (int k = 0; k < NT; ++k) {
        if (k >= n) continue;
#pragma unroll
        for (int i = 0; i < MD; ++i) dx[k][i] = dx[k][i] + (TT)divm((double)(e * dv[k][i]), i);
        tg.hvpT(x, dx[k], h);
#pragma unroll
        for (int i = 0; i < MD; ++i) dv[k][i] = dv[k][i] + e * h[i];
      }
      tg.grad(x, g);
#pragma unroll
      for (int i = 0; i < MD; ++i) v[i] = v[i] + eps * g[i];
    }
    const TT gate = (TT)(relaxed ? expit(a.margin) : (a.margin > 0.0 ? 1.0 : 0.0));
    const TT sp = (TT)sigmoid_prime(a.margin);
    const TT neg = (TT)(a.delta < 0.0 ? 1.0 : 0.0);
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      if (k >= n) continue;
      tg.hvpT(x, dx[k], h);
      TT s1 = 0, s2 = 0;
#pragma unroll
      for (int i = 0; i < MD; ++i) {
        const TT dvl = dv[k][i] - he * h[i];
        if (i < D) s1 += (TT)divm((double)((TT)a.vl[i] * dvl), i);
        s2 += (TT)a.gl[i] * dx[k][i];
      }
      const TT ddelta = dh0[k] - (s1 - s2);
      const TT bend = sp * (ddelta * neg);
#pragma unroll
      for (int i = 0; i < MD; ++i)
        o[k][i] = (double)((gate * dx[k][i] + ((TT)1 - gate) * (TT)V[k][i]) + (TT)(a.xl[i] - a.S[i]) * bend);
    }
  }
};

// ---------------------------------------------------------------------------
// leapfrog integrator as a system over [x, v] (samplers.py:165-222).  MD is
// the (even) register width; x lives in slots [0, n), v in [H, H + n) with
// H = MD/2, so block elements stay compile-time indexed (see mem_index).
template <int MD, typename ST, int TK = -1>
struct Leapfrog {
  static constexpr int H = MD / 2;
  Target<H, TK> tg;
  double eps;
  const double *mass;
  uint64_t probe_seed;

  struct Aux {
    double S[MD], xn[H], vn[H];
  };

  CS_D int dim() const { return 2 * tg.p.dim; }
  CS_D int mem_index(int k) const {
    const int n = tg.p.dim;
    return k < H ? (k < n ? k : -1) : (k - H < n ? n + k - H : -1);
  }
  CS_D double m(int i) const { return (mass && i < tg.p.dim) ? __ldg(mass + i) : 1.0; }
  CS_D double divm(double x, int i) const { return (mass && i < tg.p.dim) ? x / __ldg(mass + i) : x; }

  CS_D bool prepare(int64_t, const double (&s)[MD], Aux &a) const {
    const int n = tg.p.dim;
    double g[H];
#pragma unroll
    for (int i = 0; i < MD; ++i) a.S[i] = s[i];
#pragma unroll
    for (int i = 0; i < H; ++i) a.xn[i] = (i < n) ? s[i] + divm(eps * s[H + i], i) : 0.0;
    tg.grad(a.xn, g);
#pragma unroll
    for (int i = 0; i < H; ++i) a.vn[i] = (i < n) ? s[H + i] + eps * g[i] : 0.0;
    return true;
  }

  CS_D void f(const Aux &a, double (&o)[MD]) const {
#pragma unroll
    for (int i = 0; i < H; ++i) { o[i] = a.xn[i]; o[H + i] = a.vn[i]; }
  }
  CS_D void relaxed_f(const Aux &a, double (&o)[MD]) const { f(a, o); }

  CS_D void jvp1(const Aux &a, const double (&V)[MD], double (&o)[MD]) const {
    const int n = tg.p.dim;
    double dxn[H], h[H];
#pragma unroll
    for (int i = 0; i < H; ++i) dxn[i] = (i < n) ? V[i] + divm(eps * V[H + i], i) : 0.0;
    tg.hvp(a.xn, dxn, h);
#pragma unroll
    for (int i = 0; i < H; ++i) {
      o[i] = dxn[i];
      o[H + i] = (i < n) ? V[H + i] + eps * h[i] : 0.0;
    }
  }

  template <int NT, typename TT = double>
  CS_D void jvp_many(const Aux &a, const double (&V)[NT][MD], double (&o)[NT][MD], int n,
                     bool) const {
#pragma unroll
    for (int k = 0; k < NT; ++k)
      if (k < n) jvp1(a, V[k], o[k]);
  }

  // block estimate (samplers.py:202-222): a=1, b=eps/m, c=eps dhat, d=1+eps^2 dhat/m
  CS_D void block(const Aux &a, int64_t t, int nsamp, int64_t iteration, double (&ba)[H],
                  double (&bb)[H], double (&bc)[H], double (&bd)[H]) const {
    const int n = tg.p.dim;
    const uint64_t h3 = hash_t(probe_prefix(probe_seed, iteration), (uint64_t)t);
    double dhat[H], z[H], hz[H];
#pragma unroll
    for (int i = 0; i < H; ++i) dhat[i] = 0.0;
    for (int k = 0; k < nsamp; ++k) {
#pragma unroll
      for (int i = 0; i < H; ++i) z[i] = (i < n) ? probe_sign(h3, k, i) : 0.0;
      tg.hvp(a.xn, z, hz);
#pragma unroll
      for (int i = 0; i < H; ++i) dhat[i] += z[i] * hz[i];
    }
#pragma unroll
    for (int i = 0; i < H; ++i) {
      dhat[i] = dhat[i] / (double)nsamp;
      ba[i] = (i < n) ? 1.0 : 0.0;
      bb[i] = (i < n) ? divm(eps, i) : 0.0;
      bc[i] = eps * dhat[i];
      bd[i] = (i < n) ? 1.0 + divm((eps * eps) * dhat[i], i) : 0.0;
    }
  }
};

// ---------------------------------------------------------------------------
// eight-schools systematic Gibbs sweep (samplers.py:464-627); MD = 2S + 2
template <int MD, typename ST>
struct Gibbs {
  static constexpr int S = (MD - 2) / 2;
  static constexpr double kFloor = 1e-8;   // VARIANCE_FLOOR, samplers.py:549
  int D;
  const ST *g_tau, *xi_mu, *xi_theta, *g_sigma;
  const double *prm;  // nu0 tau0_sq mu0 kappa0 alpha0 sigma0_sq S n xbar[S] ss[S]

  struct Aux {
    double mu, th[S], sg[S], raw_ok[S];
    double gt, xm, xt[S], gs[S];
    double tau2n, mun, prec[S], mean[S], thn[S], sgn[S];
  };

  CS_D int dim() const { return D; }
  CS_D int mem_index(int k) const { return k < D ? k : -1; }

  CS_D bool prepare(int64_t t, const double (&s)[MD], Aux &a) const {
    const double nu0 = __ldg(prm + 0), tau0_sq = __ldg(prm + 1), mu0 = __ldg(prm + 2);
    const double kappa0 = __ldg(prm + 3), alpha0 = __ldg(prm + 4), sigma0_sq = __ldg(prm + 5);
    const double n = __ldg(prm + 7);
    a.mu = s[1];
    a.gt = ld(g_tau, t);
    a.xm = ld(xi_mu, t);
    double sth = 0.0, q = 0.0;
#pragma unroll
    for (int i = 0; i < S; ++i) {
      a.th[i] = s[2 + i];
      a.raw_ok[i] = s[2 + S + i] > kFloor ? 1.0 : 0.0;
      a.sg[i] = fmax(s[2 + S + i], kFloor);
      a.xt[i] = ld(xi_theta, t * S + i);
      a.gs[i] = ld(g_sigma, t * S + i);
      double dm = a.th[i] - a.mu;
      q += dm * dm;
      sth += a.th[i];
    }
    const double dmu0 = a.mu - mu0;
    const double q_tau = (nu0 * tau0_sq + kappa0 * (dmu0 * dmu0)) + q;
    a.tau2n = q_tau / a.gt;
    const double kS = kappa0 + (double)S;
    a.mun = (kappa0 * mu0 + sth) / kS + sqrt(a.tau2n / kS) * a.xm;
#pragma unroll
    for (int i = 0; i < S; ++i) {
      const double xbar = __ldg(prm + 8 + i), ss = __ldg(prm + 8 + S + i);
      a.prec[i] = 1.0 / a.tau2n + n / a.sg[i];
      a.mean[i] = (a.mun / a.tau2n + (n * xbar) / a.sg[i]) / a.prec[i];
      a.thn[i] = a.mean[i] + a.xt[i] / sqrt(a.prec[i]);
      const double r = xbar - a.thn[i];
      a.sgn[i] = ((alpha0 * sigma0_sq + ss) + n * (r * r)) / a.gs[i];
    }
    return true;
  }

  CS_D void f(const Aux &a, double (&o)[MD]) const {
    o[0] = a.tau2n;
    o[1] = a.mun;
#pragma unroll
    for (int i = 0; i < S; ++i) { o[2 + i] = a.thn[i]; o[2 + S + i] = a.sgn[i]; }
  }
  CS_D void relaxed_f(const Aux &a, double (&o)[MD]) const { f(a, o); }

  CS_D void jvp1(const Aux &a, const double (&V)[MD], double (&o)[MD]) const {
    const double mu0 = __ldg(prm + 2), kappa0 = __ldg(prm + 3), n = __ldg(prm + 7);
    const double dmu_in = V[1];
    double q = 0.0, sdth = 0.0;
#pragma unroll
    for (int i = 0; i < S; ++i) {
      q += 2.0 * (a.th[i] - a.mu) * (V[2 + i] - dmu_in);
      sdth += V[2 + i];
    }
    const double dq = 2.0 * kappa0 * (a.mu - mu0) * dmu_in + q;
    const double dtau2 = dq / a.gt;
    const double kS = kappa0 + (double)S;
    const double dmu = sdth / kS + a.xm * dtau2 / (2.0 * sqrt(a.tau2n * kS));
    const double t2sq = a.tau2n * a.tau2n;
    o[0] = dtau2;
    o[1] = dmu;
#pragma unroll
    for (int i = 0; i < S; ++i) {
      const double xbar = __ldg(prm + 8 + i);
      const double dsg = a.raw_ok[i] != 0.0 ? V[2 + S + i] : 0.0;
      const double sg2 = a.sg[i] * a.sg[i];
      const double dprec = -dtau2 / t2sq - n * dsg / sg2;
      const double damean = (dmu / a.tau2n - a.mun * dtau2 / t2sq) - n * xbar * dsg / sg2;
      const double dmean = (damean - a.mean[i] * dprec) / a.prec[i];
      const double dth = dmean - 0.5 * a.xt[i] * dprec / pow(a.prec[i], 1.5);
      o[2 + i] = dth;
      o[2 + S + i] = (-2.0 * n * (xbar - a.thn[i]) * dth) / a.gs[i];
    }
  }

  template <int NT, typename TT = double>
  CS_D void jvp_many(const Aux &a, const double (&V)[NT][MD], double (&o)[NT][MD], int n,
                     bool) const {
#pragma unroll
    for (int k = 0; k < NT; ++k)
      if (k < n) jvp1(a, V[k], o[k]);
  }
};

// ---------------------------------------------------------------------------
// build a device system object from the C-ABI descriptor
template <int MD, typename ST, int TK> CS_D Mala<MD, ST, TK> make_mala(const cs_system &s) {
  Mala<MD, ST, TK> m;
  m.tg.p = s.target;
  m.eps = s.eps;
  m.sq2eps = sqrt(2.0 * s.eps);
  m.inv4eps = 1.0 / (4.0 * s.eps);
  m.inv2eps = 1.0 / (2.0 * s.eps);
  m.tg.init();
  m.xi = (const ST *)s.noise_vec;
  m.logu = s.noise_logu;
  return m;
}
template <int MD, typename ST, int TK> CS_D Hmc<MD, ST, TK> make_hmc(const cs_system &s) {
  Hmc<MD, ST, TK> h;
  h.tg.p = s.target;
  h.tg.init();
  h.eps = s.eps;
  h.L = s.L;
  h.mass = s.mass;
  h.mom = (const ST *)s.noise_vec;
  h.logu = s.noise_logu;
  return h;
}
template <int MD, typename ST, int TK> CS_D Leapfrog<MD, ST, TK> make_leapfrog(const cs_system &s) {
  Leapfrog<MD, ST, TK> l;
  l.tg.p = s.target;
  l.tg.init();
  l.eps = s.eps;
  l.mass = s.mass;
  l.probe_seed = s.probe_seed;
  return l;
}
template <int MD, typename ST> CS_D Gibbs<MD, ST> make_gibbs(const cs_system &s) {
  Gibbs<MD, ST> g;
  g.D = s.dim;
  g.g_tau = (const ST *)s.g_tau;
  g.xi_mu = (const ST *)s.xi_mu;
  g.xi_theta = (const ST *)s.xi_theta;
  g.g_sigma = (const ST *)s.g_sigma;
  g.prm = s.gibbs;
  return g;
}

}  // namespace cs
