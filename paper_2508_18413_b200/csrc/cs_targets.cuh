// Register-resident target models for small state dimension (dim <= MD).
//
// Restates chainscan/targets.py per family with the same operation order:
// std-normal (160-166), Gaussian from the Cholesky factor of its precision
// (169-182), Rosenbrock banana (185-212), isotropic mixture (215-251).
// Logistic regression (254-287) is a dense contraction over the data and
// lives in the GEMM path (cs_blr.cu), not here.
#pragma once
#include "cs_common.cuh"

namespace cs {

// TK >= 0 fixes the family at compile time (fused solver kernels); TK = -1
// dispatches on p.kind at run time (batched API kernels).
template <int MD, int TK = -1>
struct Target {
  cs_target p;
  double is1, is2;  // 1/scale1, 1/scale2 (rosenbrock), hoisted out of the hot loops

  CS_D void init() {
    is1 = 1.0 / p.scale1;
    is2 = 1.0 / p.scale2;
  }

  CS_D int dim() const { return p.dim; }
  CS_D int kind() const { return TK >= 0 ? TK : p.kind; }

  CS_D double logp(const double (&x)[MD]) const {
    const int D = p.dim;
    switch (kind()) {
      case CS_TARGET_STD_NORMAL: {
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < MD; ++i) if (i < D) s += x[i] * x[i];
        return -0.5 * s;
      }
      case CS_TARGET_GAUSSIAN: {  // h = (x - mu) @ L ; -0.5 |h|^2
        double r[MD];
#pragma unroll
        for (int i = 0; i < MD; ++i) r[i] = (i < D) ? x[i] - __ldg(p.mu + i) : 0.0;
        double s = 0.0;
        for (int j = 0; j < D; ++j) {
          double h = 0.0;
#pragma unroll
          for (int i = 0; i < MD; ++i) if (i < D) h += r[i] * __ldg(p.chol + i * D + j);
          s += h * h;
        }
        return -0.5 * s;
      }
      case CS_TARGET_ROSENBROCK: {
        double x1 = x[0], x2 = x[MD > 1 ? 1 : 0];
        double r = x2 - p.b * x1 * x1;
        double q = x1 - p.a;
        return -(q * q) * (0.5 * is1) - (r * r) * (0.5 * is2);
      }
      default: {  // mog: log-sum-exp over components (no per-component arrays)
        double top = -INFINITY;
        for (int k = 0; k < p.n_comp; ++k) top = fmax(top, mog_lc(x, k));
        double s = 0.0;
        for (int k = 0; k < p.n_comp; ++k) s += exp(mog_lc(x, k) - top);
        return top + log(s);
      }
    }
  }

  // log component k: log w_k + lognorm_k - |x - m_k|^2 / (2 var_k) (targets.py:220-223)
  CS_D double mog_lc(const double (&x)[MD], int k) const {
    const int D = p.dim;
    double sq = 0.0;
#pragma unroll
    for (int i = 0; i < MD; ++i)
      if (i < D) { double df = x[i] - __ldg(p.means + k * D + i); sq += df * df; }
    return __ldg(p.logw + k) + __ldg(p.lognorm + k) - sq / (2.0 * __ldg(p.variances + k));
  }
  // responsibilities r_k = exp(lc_k - top) / sum (targets.py:230-234): returns top, sum
  CS_D void mog_norm(const double (&x)[MD], double &top, double &sum) const {
    top = -INFINITY;
    for (int k = 0; k < p.n_comp; ++k) top = fmax(top, mog_lc(x, k));
    sum = 0.0;
    for (int k = 0; k < p.n_comp; ++k) sum += exp(mog_lc(x, k) - top);
  }

  CS_D void grad(const double (&x)[MD], double (&g)[MD]) const {
    const int D = p.dim;
    switch (kind()) {
      case CS_TARGET_STD_NORMAL:
#pragma unroll
        for (int i = 0; i < MD; ++i) g[i] = -x[i];
        return;
      case CS_TARGET_GAUSSIAN: {  // -(x - mu) @ P
        double r[MD];
#pragma unroll
        for (int i = 0; i < MD; ++i) r[i] = (i < D) ? x[i] - __ldg(p.mu + i) : 0.0;
#pragma unroll
        for (int j = 0; j < MD; ++j) {
          double s = 0.0;
          if (j < D)
#pragma unroll
            for (int i = 0; i < MD; ++i) if (i < D) s += r[i] * __ldg(p.prec + i * D + j);
          g[j] = -s;
        }
        return;
      }
      case CS_TARGET_ROSENBROCK: {
        double x1 = x[0], x2 = x[MD > 1 ? 1 : 0];
        double r = x2 - p.b * x1 * x1;
        g[0] = -(x1 - p.a) * is1 + 2.0 * p.b * x1 * r * is2;
        if (MD > 1) g[MD > 1 ? 1 : 0] = -r * is2;
#pragma unroll
        for (int i = 2; i < MD; ++i) g[i] = 0.0;
        return;
      }
      default: {  // mog: -sum_k r_k (x - m_k) / var_k
        double top, sum;
        mog_norm(x, top, sum);
#pragma unroll
        for (int i = 0; i < MD; ++i) g[i] = 0.0;
        for (int k = 0; k < p.n_comp; ++k) {
          const double r = exp(mog_lc(x, k) - top) / sum;
          const double var = __ldg(p.variances + k);
#pragma unroll
          for (int i = 0; i < MD; ++i)
            if (i < D) g[i] += r * (x[i] - __ldg(p.means + k * D + i)) / var;
        }
#pragma unroll
        for (int i = 0; i < MD; ++i) g[i] = -g[i];
        return;
      }
    }
  }

  // tangent-precision Hessian-vector product: the curvature is formed from the
  // f64 state, the product runs in TT (float tangents in fp32 storage mode)
  template <typename TT>
  CS_D void hvpT(const double (&x)[MD], const TT (&v)[MD], TT (&o)[MD]) const {
    if constexpr (sizeof(TT) == sizeof(double)) {
      hvp(x, v, o);
    } else {
      const int D = p.dim;
      switch (kind()) {
        case CS_TARGET_STD_NORMAL:
#pragma unroll
          for (int i = 0; i < MD; ++i) o[i] = -v[i];
          return;
        case CS_TARGET_GAUSSIAN:
#pragma unroll
          for (int j = 0; j < MD; ++j) {
            TT s = 0;
            if (j < D)
#pragma unroll
              for (int i = 0; i < MD; ++i) if (i < D) s += v[i] * (TT)__ldg(p.prec + i * D + j);
            o[j] = -s;
          }
          return;
        case CS_TARGET_ROSENBROCK: {
          const double b = p.b;
          const double x1 = x[0], x2 = x[MD > 1 ? 1 : 0];
          const double r = x2 - b * x1 * x1;
          const TT h11 = (TT)(-is1 + (2.0 * b * r - 4.0 * b * b * x1 * x1) * is2);
          const TT h12 = (TT)(2.0 * b * x1 * is2), h22 = (TT)is2;
          const TT v0 = v[0], v1 = v[MD > 1 ? 1 : 0];
          o[0] = h11 * v0 + h12 * v1;
          if (MD > 1) o[MD > 1 ? 1 : 0] = h12 * v0 - v1 * h22;
#pragma unroll
          for (int i = 2; i < MD; ++i) o[i] = 0;
          return;
        }
        default: {
          double vd[MD], od[MD];
#pragma unroll
          for (int i = 0; i < MD; ++i) vd[i] = (double)v[i];
          hvp(x, vd, od);
#pragma unroll
          for (int i = 0; i < MD; ++i) o[i] = (TT)od[i];
          return;
        }
      }
    }
  }

  CS_D void hvp(const double (&x)[MD], const double (&v)[MD], double (&o)[MD]) const {
    const int D = p.dim;
    switch (kind()) {
      case CS_TARGET_STD_NORMAL:
#pragma unroll
        for (int i = 0; i < MD; ++i) o[i] = -v[i];
        return;
      case CS_TARGET_GAUSSIAN:
#pragma unroll
        for (int j = 0; j < MD; ++j) {
          double s = 0.0;
          if (j < D)
#pragma unroll
            for (int i = 0; i < MD; ++i) if (i < D) s += v[i] * __ldg(p.prec + i * D + j);
          o[j] = -s;
        }
        return;
      case CS_TARGET_ROSENBROCK: {
        const double b = p.b;
        double x1 = x[0], x2 = x[MD > 1 ? 1 : 0];
        double r = x2 - b * x1 * x1;
        double h11 = -is1 + (2.0 * b * r - 4.0 * b * b * x1 * x1) * is2;
        double h12 = 2.0 * b * x1 * is2;
        double v0 = v[0], v1 = v[MD > 1 ? 1 : 0];
        o[0] = h11 * v0 + h12 * v1;
        if (MD > 1) o[MD > 1 ? 1 : 0] = h12 * v0 - v1 * is2;
#pragma unroll
        for (int i = 2; i < MD; ++i) o[i] = 0.0;
        return;
      }
      default: {  // mog (targets.py:240-249)
        double top, sum;
        mog_norm(x, top, sum);
        double gbar[MD], term[MD];
#pragma unroll
        for (int i = 0; i < MD; ++i) { gbar[i] = 0.0; term[i] = 0.0; }
        double curv = 0.0;
        for (int k = 0; k < p.n_comp; ++k) {
          const double r = exp(mog_lc(x, k) - top) / sum;
          const double var = __ldg(p.variances + k);
          double gk[MD];
          double gv = 0.0;
#pragma unroll
          for (int i = 0; i < MD; ++i) {
            gk[i] = (i < D) ? -(x[i] - __ldg(p.means + k * D + i)) / var : 0.0;
            gbar[i] += r * gk[i];
            gv += gk[i] * v[i];
          }
#pragma unroll
          for (int i = 0; i < MD; ++i) term[i] += (r * gv) * gk[i];
          curv += r / var;
        }
        double gdot = 0.0;
#pragma unroll
        for (int i = 0; i < MD; ++i) gdot += gbar[i] * v[i];
#pragma unroll
        for (int i = 0; i < MD; ++i) o[i] = (i < D) ? term[i] - curv * v[i] - gbar[i] * gdot : 0.0;
        return;
      }
    }
  }
};

}  // namespace cs
