// MALA element builder for the Bayesian logistic-regression target (BASELINE
// config 3: T = 100K chains steps, D = 100, N = 1000 data rows), diag
// quasi-Newton with K Hutchinson probes.
//
// One Newton update needs, at every step t, grad/logp at the current state S_t
// and at the proposal x~_t, plus hvp(S_t, z_k) and hvp(x~_t, dx~_k) for the
// probe tangents (samplers.py:95-145, targets.py:254-287).  All of them are
// row blocks of four plain GEMMs against the data matrix X:
//   E1 = [S; Z] X^T          logits eta_S and the probes' z X^T
//   G1 = [y - p_S; w_S.(Z X^T)] X       (w = p (1 - p))
//   E2 = [x~; dx~] X^T
//   G2 = [y - p~; w~.(dx~ X^T)] X
// run by cuBLAS (FP64 tensor cores); the sigmoid / weight / row-sum epilogues
// and the per-step MALA gate, tangents, Hutchinson estimate and element
// formation (deer.py:171-183) are our kernels, one warp per step.
#include <cublas_v2.h>

#include <mutex>

#include "cs_apikern.cuh"

namespace cs {

namespace {

constexpr int kBlrMaxD = 128;          // per-lane register slices of 4 columns
constexpr int kBlrCols = kBlrMaxD / 32;

struct BlrCtx {
  std::mutex mu;
  cublasHandle_t h = nullptr;
  double *buf = nullptr;
  size_t cap = 0;
};
BlrCtx g_blr[16];

// A rows [0, T): prev states; rows (k+1)T + r: probe k of step r+1
template <typename ST>
__global__ void k_blr_prologue(cs_system sys, const ST *s0, const ST *guess, int64_t iteration, int K, double *A) {
  const int D = sys.dim;
  const int64_t T = sys.T, total = T * D;
  const uint64_t pre = probe_prefix(sys.seed, iteration);
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / D;
    const int i = (int)(idx - r * D);
    const ST *pr = r == 0 ? s0 : guess + (r - 1) * D;
    A[r * D + i] = (double)pr[i];
    const uint64_t h3 = hash_t(pre, (uint64_t)(r + 1));
    for (int k = 0; k < K; ++k) A[((int64_t)(k + 1) * T + r) * D + i] = probe_sign(h3, k, i);
  }
}

// per step r (one warp, lanes across the N data rows): p = sigmoid(eta),
// E[r] <- y - p, probe rows <- p(1-p) . (z X^T), and the two log-density row
// sums eta.y and sum logaddexp(0, eta).  exp(-eta) serves both the sigmoid and,
// for eta >= 0, logaddexp's exp(-|eta|).
__global__ void __launch_bounds__(256) k_blr_epilogue(double *E, const double *y, int64_t T, int K, int N,
                                                       double *rowsum) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < T; r += nw) {
    double a = 0.0, b = 0.0;
    double *er = E + r * N;
#pragma unroll 4
    for (int n = lane; n < N; n += 32) {
      const double eta = er[n], yn = __ldg(y + n);
      const double em = exp(-eta);
      const double p = 1.0 / (1.0 + em);  // expit / torch.sigmoid
      a += eta * yn;
      b += eta != eta ? eta : fmax(eta, 0.0) + log1p(eta >= 0.0 ? em : exp(eta));  // logaddexp(0, eta)
      er[n] = yn - p;
      const double w = p * (1.0 - p);
      for (int k = 0; k < K; ++k) E[((int64_t)(k + 1) * T + r) * N + n] *= w;
    }
    a = warp_sum(a);
    b = warp_sum(b);
    if (lane == 0) {
      rowsum[2 * r] = a;
      rowsum[2 * r + 1] = b;
    }
  }
}

// gradient at S (kept for the gate derivative), the proposal, and the probe
// tangents dx~_k = z_k + eps hvp(S, z_k), hvp = -(w . zX^T) X - prec z   (warp per step)
template <typename ST>
__global__ void k_blr_propose(cs_system sys, const ST *s0, const ST *guess, const double *A, const double *G, int K,
                              double *A2, double *gS, cs_elem_stats *stats) {
  const int D = sys.dim;
  const int64_t T = sys.T;
  const double prec = sys.target.prior_precision, eps = sys.eps, sq = sqrt(2.0 * eps);
  const ST *xi = (const ST *)sys.noise_vec;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  long long bp = kNoStep;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < T; r += nw) {
    const int64_t t = r + 1;
    const ST *pr = r == 0 ? s0 : guess + (r - 1) * D;
    bool fin = true;
    for (int i = lane; i < D; i += 32) {
      const double s = (double)pr[i];
      const double g = G[r * D + i] - prec * s;  // (y - p) X - prec beta
      gS[r * D + i] = g;
      const double xp = (s + eps * g) + sq * (double)xi[t * D + i];  // samplers.py:206
      fin &= isfinite(xp);
      A2[r * D + i] = xp;
      for (int k = 0; k < K; ++k) {
        const int64_t o = ((int64_t)(k + 1) * T + r) * D + i;
        const double z = A[o];
        const double hv = -G[o] - prec * z;
        A2[o] = z + eps * hv;
      }
    }
    fin = __all_sync(0xffffffffu, fin);
    if (lane == 0 && !fin && t < bp) bp = t;
  }
  if (lane == 0 && bp != kNoStep) atomicMin((long long *)&stats->bad_proposal, bp);
}

// gate, JVPs through the gate, Hutchinson diagonal, element (warp per step)
template <typename ST>
__global__ void k_blr_final(cs_system sys, cs_deer_config cfg, int64_t iteration, const ST *s0, const ST *guess,
                            const double *A, const double *A2, const double *G2, const double *gS,
                            const double *rsS, const double *rsX, ST *jout, ST *uout, cs_elem_stats *stats) {
  const int D = sys.dim;
  const int64_t T = sys.T;
  const int K = cfg.hutchinson_samples;
  const double prec = sys.target.prior_precision, eps = sys.eps;
  const ST *xi = (const ST *)sys.noise_vec;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool do_clip = isfinite(cfg.clip);
  long long bf = kNoStep, bj = kNoStep;
  unsigned pf = 0;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < T; r += nw) {
    const int64_t t = r + 1;
    const ST *pr = r == 0 ? s0 : guess + (r - 1) * D;
    double S[kBlrCols], X[kBlrCols], gp[kBlrCols], rb[kBlrCols], est[kBlrCols];
    double ss = 0.0, sx = 0.0, srb = 0.0, sxi = 0.0;
#pragma unroll
    for (int c = 0; c < kBlrCols; ++c) {
      const int i = lane + 32 * c;
      S[c] = X[c] = gp[c] = rb[c] = est[c] = 0.0;
      if (i < D) {
        S[c] = (double)pr[i];
        X[c] = A2[r * D + i];
        gp[c] = G2[r * D + i] - prec * X[c];
        rb[c] = S[c] - X[c] - eps * gp[c];
        const double z = (double)xi[t * D + i];
        ss += S[c] * S[c];
        sx += X[c] * X[c];
        srb += rb[c] * rb[c];
        sxi += z * z;
      }
    }
    ss = warp_sum(ss);
    sx = warp_sum(sx);
    srb = warp_sum(srb);
    sxi = warp_sum(sxi);
    // logp = eta.y - sum logaddexp(0, eta) - prec/2 |beta|^2   (targets.py:254-270)
    const double lpX = (rsX[2 * r] - rsX[2 * r + 1]) - 0.5 * prec * sx;
    const double lpS = (rsS[2 * r] - rsS[2 * r + 1]) - 0.5 * prec * ss;
    const double delta = lpX - lpS - srb / (4.0 * eps) + 0.5 * sxi;
    const double margin = fmin(0.0, delta) - __ldg(sys.noise_logu + t);
    const double gate = margin > 0.0 ? 1.0 : 0.0;
    const double sp = sigmoid_prime(margin), neg = delta < 0.0 ? 1.0 : 0.0;
    const uint64_t h3 = hash_t(probe_prefix(sys.seed, iteration), (uint64_t)t);
    for (int k = 0; k < K; ++k) {
      const int64_t row = (int64_t)(k + 1) * T + r;
      double z[kBlrCols], dx[kBlrCols];
      double s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
      for (int c = 0; c < kBlrCols; ++c) {
        const int i = lane + 32 * c;
        z[c] = dx[c] = 0.0;
        if (i < D) {
          z[c] = A[row * D + i];
          dx[c] = A2[row * D + i];
          const double hv = -G2[row * D + i] - prec * dx[c];  // hvp(x~, dx~)
          const double dr = (z[c] - dx[c]) - eps * hv;
          s1 += gp[c] * dx[c];
          s2 += gS[r * D + i] * z[c];
          s3 += rb[c] * dr;
        }
      }
      s1 = warp_sum(s1);
      s2 = warp_sum(s2);
      s3 = warp_sum(s3);
      const double ddelta = (s1 - s2) - s3 / (2.0 * eps);
      const double bend = sp * (ddelta * neg);
#pragma unroll
      for (int c = 0; c < kBlrCols; ++c) {
        const double jz = (gate * dx[c] + (1.0 - gate) * z[c]) + (X[c] - S[c]) * bend;
        est[c] += z[c] * jz;
      }
    }
    bool fin = true, jok = true, pfail = false;
    const ST *gr = guess + r * D;
#pragma unroll
    for (int c = 0; c < kBlrCols; ++c) {
      const int i = lane + 32 * c;
      if (i >= D) continue;
      const double f = gate > 0.0 ? X[c] : S[c];
      fin &= isfinite(f);
      pfail |= !(fabs(f - (double)gr[i]) <= cfg.atol + cfg.rtol * fabs(f));
      double v = est[c] / (double)K;
      jok &= isfinite(v);
      if (cfg.preconditioner) v = v * __ldg(cfg.preconditioner + i);
      v = v * cfg.damping;
      if (do_clip) v = clipv(v, cfg.clip);
      jout[r * D + i] = (ST)v;
      uout[r * D + i] = (ST)(f - v * S[c]);
    }
    fin = __all_sync(0xffffffffu, fin);
    jok = __all_sync(0xffffffffu, jok);
    pfail = __any_sync(0xffffffffu, pfail);
    if (lane == 0) {
      if (!fin && t < bf) bf = t;
      if (!jok && t < bj) bj = t;
      pf += pfail ? 1u : 0u;
    }
  }
  if (lane == 0) {
    if (bf != kNoStep) atomicMin((long long *)&stats->bad_step, bf);
    if (bj != kNoStep) atomicMin((long long *)&stats->bad_jacobian, bj);
    if (pf) atomicAdd(&stats->picard_fail, pf);
  }
}

}  // namespace

bool blr_mala_ok(const cs_system &s, int mode) {
  return s.kind == CS_SYS_MALA && s.target.kind == CS_TARGET_BLR && mode == CS_MODE_DIAG && s.dim >= 1 &&
         s.dim <= kBlrMaxD && s.target.dim == s.dim && s.target.X && s.target.y && s.target.n_data > 0 &&
         s.noise_vec && s.noise_logu;
}

template <typename ST>
static cudaError_t blr_run(const cs_system &sys, const cs_deer_config &cfg, int64_t iteration, const ST *s0,
                           const ST *guess, ST *jout, ST *uout, cs_elem_stats *stats, cudaStream_t st) {
  const int D = sys.dim, N = (int)sys.target.n_data;
  const int64_t T = sys.T;
  const int K = cfg.hutchinson_samples < 1 ? 1 : cfg.hutchinson_samples;
  const int64_t M = T * (1 + K);
  int dev = 0;
  cudaGetDevice(&dev);
  BlrCtx &ctx = g_blr[dev & 15];
  std::lock_guard<std::mutex> lock(ctx.mu);
  if (!ctx.h && cublasCreate(&ctx.h) != CUBLAS_STATUS_SUCCESS) return cudaErrorUnknown;
  // A, A2, G (M x D), E (M x N), gS (T x D), row sums 2 x (2T)
  const size_t need = (size_t)3 * M * D + (size_t)M * N + (size_t)T * D + (size_t)4 * T;
  if (ctx.cap < need) {
    if (ctx.buf) cudaFree(ctx.buf);  // synchronises: growth happens once per shape
    ctx.buf = nullptr;
    ctx.cap = 0;
    cudaError_t e = cudaMalloc(&ctx.buf, need * sizeof(double));
    if (e != cudaSuccess) return e;
    ctx.cap = need;
  }
  double *A = ctx.buf, *A2 = A + (size_t)M * D, *G = A2 + (size_t)M * D, *E = G + (size_t)M * D;
  double *gS = E + (size_t)M * N, *rsS = gS + (size_t)T * D, *rsX = rsS + 2 * T;
  const double *X = sys.target.X, *y = sys.target.y;
  const double one = 1.0, zero = 0.0;
  if (cublasSetStream(ctx.h, st) != CUBLAS_STATUS_SUCCESS) return cudaErrorUnknown;
  auto gemm_xt = [&](const double *Ain, double *Cout) {  // row-major C (M x N) = A (M x D) X^T
    return cublasDgemm(ctx.h, CUBLAS_OP_T, CUBLAS_OP_N, N, (int)M, D, &one, X, D, Ain, D, &zero, Cout, N);
  };
  auto gemm_x = [&](const double *Bin, double *Cout) {  // row-major C (M x D) = B (M x N) X
    return cublasDgemm(ctx.h, CUBLAS_OP_N, CUBLAS_OP_N, D, (int)M, N, &one, X, D, Bin, N, &zero, Cout, D);
  };
  const unsigned ge = (unsigned)((T * D + 255) / 256 < 148 * 32 ? (T * D + 255) / 256 : 148 * 32);
  const unsigned gw = (unsigned)((T * 32 + 255) / 256);
  k_blr_prologue<ST><<<ge, 256, 0, st>>>(sys, s0, guess, iteration, K, A);
  if (gemm_xt(A, E) != CUBLAS_STATUS_SUCCESS) return cudaErrorUnknown;
  k_blr_epilogue<<<gw, 256, 0, st>>>(E, y, T, K, N, rsS);
  if (gemm_x(E, G) != CUBLAS_STATUS_SUCCESS) return cudaErrorUnknown;
  k_blr_propose<ST><<<gw, 256, 0, st>>>(sys, s0, guess, A, G, K, A2, gS, stats);
  if (gemm_xt(A2, E) != CUBLAS_STATUS_SUCCESS) return cudaErrorUnknown;
  k_blr_epilogue<<<gw, 256, 0, st>>>(E, y, T, K, N, rsX);
  if (gemm_x(E, G) != CUBLAS_STATUS_SUCCESS) return cudaErrorUnknown;
  k_blr_final<ST><<<gw, 256, 0, st>>>(sys, cfg, iteration, s0, guess, A, A2, G, gS, rsS, rsX, jout, uout, stats);
  return cudaGetLastError();
}

cudaError_t elements_blr(const cs_system &sys, const cs_deer_config &cfg, int dtype, int64_t iteration,
                         const void *s0, const void *guess, void *e0, void *u, cs_elem_stats *stats,
                         cudaStream_t st) {
  if (dtype == CS_F64)
    return blr_run<double>(sys, cfg, iteration, (const double *)s0, (const double *)guess, (double *)e0,
                           (double *)u, stats, st);
  return blr_run<float>(sys, cfg, iteration, (const float *)s0, (const float *)guess, (float *)e0, (float *)u,
                        stats, st);
}

}  // namespace cs
