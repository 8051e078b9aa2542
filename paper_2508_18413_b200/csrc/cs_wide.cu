// Wide leapfrog element builder (block2x2 mode) for a dense Gaussian target:
// the HMC-within-a-proposal system of BASELINE config 4 (D = 1000, L = 100).
//
// Per Newton iteration every step t needs grad(x'_t) = -(x'_t - mu) P and the
// Hutchinson products hvp(x'_t, z_tk) = -z_tk P (samplers.py:188-222), i.e.
// one (T*(1+K)) x n by n x n product -- a plain dense GEMM, done by our DMMA
// GEMM (cs_gemm.cuh) on the FP64 tensor cores.  Two kernels wrap it:
//   k_wide_prologue  x'_t = x + eps v / m  (minus mu) and the +-1 probes,
//                    written as the GEMM's row-major A operand
//   k_wide_epilogue  v'_t, the finite / Picard checks, d_hat, the block
//                    (a, b, c, d) with preconditioner, damping and clip, and
//                    u = f - M prev (deer.py:184-204) -- one CTA per step
// The result feeds cs_scan_block_update exactly like the register builders.

#include <mutex>

#include "cs_apikern.cuh"
#include "cs_gemm.cuh"

namespace cs {

namespace {

struct WideCtx {
  std::mutex mu;
  double *buf = nullptr;  // A (M x n) then C (M x n), f64
  size_t cap = 0;         // doubles
};
WideCtx g_wide[16];

template <typename ST>
__global__ void k_wide_prologue(cs_system sys, const ST *s0, const ST *guess, int64_t iteration, int nsamp,
                                double *A) {
  const int n = sys.dim / 2;
  const int64_t T = sys.T;
  const int64_t total = T * n;
  const double *mu = sys.target.mu;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / n;
    const int i = (int)(idx - r * n);
    const ST *pr = r == 0 ? s0 : guess + (r - 1) * sys.dim;
    const double x = (double)pr[i], v = (double)pr[n + i];
    const double ev = sys.eps * v;
    const double xn = x + (sys.mass ? ev / __ldg(sys.mass + i) : ev);
    A[r * n + i] = xn - (mu ? __ldg(mu + i) : 0.0);
    const uint64_t h3 = hash_t(probe_prefix(sys.probe_seed, iteration), (uint64_t)(r + 1));
    for (int k = 0; k < nsamp; ++k) A[((int64_t)(k + 1) * T + r) * n + i] = probe_sign(h3, k, i);
  }
}

template <typename ST>
__global__ void k_wide_epilogue(cs_system sys, const ST *s0, const ST *guess, const double *A, const double *C,
                                int nsamp, double atol, double rtol, const double *pre, double damping, double clip,
                                ST *ea, ST *eb, ST *ec, ST *ed, ST *u, cs_elem_stats *stats) {
  const int n = sys.dim / 2;
  const int64_t T = sys.T;
  const bool do_clip = isfinite(clip);
  long long bf = kNoStep, bj = kNoStep;
  unsigned pf = 0;
  for (int64_t r = blockIdx.x; r < T; r += gridDim.x) {  // one CTA per step: the n columns across its threads
    const int64_t t = r + 1;
    const ST *pr = r == 0 ? s0 : guess + (r - 1) * sys.dim;
    const ST *gr = guess + r * sys.dim;
    bool fin = true, jok = true, pfail = false;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const double x = (double)pr[i], v = (double)pr[n + i];
      const double ev = sys.eps * v;
      const double xn = x + (sys.mass ? ev / __ldg(sys.mass + i) : ev);  // as in the prologue
      const double g = -C[r * n + i];  // grad = -(x' - mu) P
      const double vn = v + sys.eps * g;
      double dh = 0.0;
      for (int k = 0; k < nsamp; ++k) {
        const int64_t row = (int64_t)(k + 1) * T + r;
        dh += A[row * n + i] * (-C[row * n + i]);  // z * hvp(x', z), hvp = -z P
      }
      dh = dh / (double)nsamp;
      const double m = sys.mass ? __ldg(sys.mass + i) : 1.0;
      double a = 1.0, b = sys.mass ? sys.eps / m : sys.eps, c = sys.eps * dh;
      double d = 1.0 + (sys.mass ? (sys.eps * sys.eps) * dh / m : (sys.eps * sys.eps) * dh);
      fin &= isfinite(xn) && isfinite(vn);
      pfail |= !(fabs(xn - (double)gr[i]) <= atol + rtol * fabs(xn));
      pfail |= !(fabs(vn - (double)gr[n + i]) <= atol + rtol * fabs(vn));
      jok &= isfinite(a) && isfinite(b) && isfinite(c) && isfinite(d);
      if (pre) {
        const double px = __ldg(pre + i), pv = __ldg(pre + n + i);
        b = b * (pv / px);
        c = c * (px / pv);
      }
      a = damping * a; b = damping * b; c = damping * c; d = damping * d;
      if (do_clip) { a = clipv(a, clip); b = clipv(b, clip); c = clipv(c, clip); d = clipv(d, clip); }
      ea[r * n + i] = (ST)a;
      eb[r * n + i] = (ST)b;
      ec[r * n + i] = (ST)c;
      ed[r * n + i] = (ST)d;
      u[r * sys.dim + i] = (ST)(xn - (a * x + b * v));
      u[r * sys.dim + n + i] = (ST)(vn - (c * x + d * v));
    }
    fin = __syncthreads_and(fin);
    jok = __syncthreads_and(jok);
    pfail = __syncthreads_or(pfail);
    if (threadIdx.x == 0) {
      if (!fin && t < bf) bf = t;
      if (!jok && t < bj) bj = t;
      pf += pfail ? 1u : 0u;
    }
  }
  if (threadIdx.x == 0) {
    if (bf != kNoStep) atomicMin((long long *)&stats->bad_step, bf);
    if (bj != kNoStep) atomicMin((long long *)&stats->bad_jacobian, bj);
    if (pf) atomicAdd(&stats->picard_fail, pf);
  }
}

}  // namespace

bool wide_leapfrog_ok(const cs_system &s, int mode) {
  return s.kind == CS_SYS_LEAPFROG && s.target.kind == CS_TARGET_GAUSSIAN && mode == CS_MODE_BLOCK &&
         s.target.prec != nullptr && s.dim % 2 == 0 && s.dim / 2 == s.target.dim;
}

template <typename ST>
static cudaError_t wide_run(const cs_system &sys, const cs_deer_config &cfg, int64_t iteration, const ST *s0,
                            const ST *guess, ST *e0, ST *e1, ST *e2, ST *e3, ST *u, cs_elem_stats *stats,
                            cudaStream_t st) {
  const int n = sys.dim / 2;
  const int64_t T = sys.T;
  const int K = cfg.hutchinson_samples < 1 ? 1 : cfg.hutchinson_samples;
  const int64_t M = T * (1 + K);
  int dev = 0;
  cudaGetDevice(&dev);
  WideCtx &ctx = g_wide[dev & 15];
  std::lock_guard<std::mutex> lock(ctx.mu);
  const size_t need = (size_t)2 * M * n;
  if (ctx.cap < need) {
    if (ctx.buf) cudaFree(ctx.buf);  // cudaFree synchronises: growth happens once per shape
    ctx.buf = nullptr;
    ctx.cap = 0;
    cudaError_t e = cudaMalloc(&ctx.buf, need * sizeof(double));
    if (e != cudaSuccess) return e;
    ctx.cap = need;
  }
  double *A = ctx.buf, *C = ctx.buf + (size_t)M * n;
  const int64_t tot = T * n;
  const unsigned g1 = (unsigned)((tot + 255) / 256 < 148 * 16 ? (tot + 255) / 256 : 148 * 16);
  k_wide_prologue<ST><<<g1 < 1 ? 1 : g1, 256, 0, st>>>(sys, s0, guess, iteration, K, A);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  // C (M x n) = A (M x n) P (n x n), row-major, on the FP64 tensor cores (cs_gemm.cuh)
  e = gemm_rm<double, double, double>(false, (int)M, n, n, A, n, 0, sys.target.prec, n, 0, C, n, 0, 1, st);
  if (e != cudaSuccess) return e;
  const unsigned g2 = (unsigned)(T < 148 * 8 ? T : 148 * 8);
  k_wide_epilogue<ST><<<g2 < 1 ? 1 : g2, 256, 0, st>>>(sys, s0, guess, A, C, K, cfg.atol, cfg.rtol,
                                                        cfg.preconditioner, cfg.damping, cfg.clip, e0, e1, e2, e3, u,
                                                        stats);
  return cudaGetLastError();
}

cudaError_t elements_wide(const cs_system &sys, const cs_deer_config &cfg, int dtype, int64_t iteration,
                          const void *s0, const void *guess, void *e0, void *e1, void *e2, void *e3, void *u,
                          cs_elem_stats *stats, cudaStream_t st) {
  if (dtype == CS_F64)
    return wide_run<double>(sys, cfg, iteration, (const double *)s0, (const double *)guess, (double *)e0,
                            (double *)e1, (double *)e2, (double *)e3, (double *)u, stats, st);
  return wide_run<float>(sys, cfg, iteration, (const float *)s0, (const float *)guess, (float *)e0, (float *)e1,
                         (float *)e2, (float *)e3, (float *)u, stats, st);
}

}  // namespace cs
