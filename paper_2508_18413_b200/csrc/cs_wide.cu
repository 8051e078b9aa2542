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
  ScratchFence fence;
  double *buf = nullptr;  // A (M x n) then C (M x n), f64
  size_t cap = 0;         // doubles
};
WideCtx g_wide[16];

template <typename ST>
__global__ void k_wide_prologue(cs_system sys, const ST *s0, const ST *guess, int64_t iteration, int nsamp,
                                double *A, cs_elem_stats *stats) {
  if (stats && blockIdx.x == 0 && threadIdx.x == 0) {  // this update's stats record (the epilogue adds to it)
    stats->bad_proposal = stats->bad_step = stats->bad_jacobian = kNoStep;
    stats->picard_fail = 0;
    stats->fail_rows = 0;
    stats->dmax = 0.0;
  }
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

// ---------------------------------------------------------------------------
// Batched inner solves for HMC in parallel-leapfrog mode at wide targets
// (samplers.py:301-320 with BASELINE cfg 4's Gaussian, n = 1000, L = 100): B
// proposals' block quasi-Newton solves advance together.  Per Newton pass, for
// every still-active proposal b and step t (rows R = b L + t - 1):
//   k_wb_prologue   x'_t - mu and the +-1 probes of (b, t) as GEMM rows
//   gemm_rm         C = A P for ALL proposals at once (one DMMA GEMM)
//   k_wb_epilogue   f_t = (x', v'), finite / Picard flags per proposal, the
//                   block elements (preconditioner, damping, clip) and u
//   k_wb_decide     run_deer's stops in order (deer.py:263-271), per proposal
//   k_wb_scan       the L-step block recursion from s0_b, one thread per
//                   (proposal, column), in place, with the fail / dmax test
//   k_wb_settle     iterations, guard, no-fail stop (deer.py:272-286)
// and one 4-byte read of the active count.  Each proposal stops exactly where
// its own run_deer would; the caller takes rows in order (errors, fallbacks).
struct WbCtl {
  int status, it, kind, eit;  // status: -1 active, else CS_RUN_*
  long long estep, bad_f, bad_j;
  unsigned pic, fail;
  unsigned long long dmax_bits;
  double d0;
  int update, pad;
};

template <typename ST>
__global__ void k_wb_init(const ST *s0s, int B, int L, int D, ST *G, WbCtl *ctl) {
  const int64_t tot = (int64_t)B * L * D;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = i / ((int64_t)L * D);
    G[i] = s0s[b * D + i % D];  // guess = tile(s0)
  }
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < B; b += gridDim.x * blockDim.x) {
    WbCtl c{};
    c.status = -1;
    c.estep = -1;
    c.eit = -1;
    c.d0 = -1.0;
    ctl[b] = c;
  }
}

__global__ void k_wb_reset(int B, WbCtl *ctl) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < B; b += gridDim.x * blockDim.x) {
    ctl[b].bad_f = ctl[b].bad_j = kNoStep;
    ctl[b].pic = ctl[b].fail = 0u;
    ctl[b].dmax_bits = 0ull;
    ctl[b].update = 0;
  }
}

template <typename ST>
__global__ void k_wb_prologue(cs_system sys, const ST *s0s, const ST *G, const WbCtl *ctl, int B, int L,
                              int64_t iteration, int nsamp, double *A) {
  const int n = sys.dim / 2, D = sys.dim;
  const int64_t rows = (int64_t)B * L, total = rows * n;
  const double *mu = sys.target.mu;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t R = idx / n;
    const int i = (int)(idx - R * n);
    const int b = (int)(R / L), t = (int)(R - (int64_t)b * L) + 1;
    if (ctl[b].status != -1) continue;
    const ST *pr = t == 1 ? s0s + (int64_t)b * D : G + (R - 1) * D;
    const double x = (double)pr[i], v = (double)pr[n + i];
    const double ev = sys.eps * v;
    const double xn = x + (sys.mass ? ev / __ldg(sys.mass + i) : ev);
    A[R * n + i] = xn - (mu ? __ldg(mu + i) : 0.0);
    const uint64_t h3 = hash_t(probe_prefix(sys.probe_seed, iteration), (uint64_t)t);
    for (int k = 0; k < nsamp; ++k) A[((int64_t)(k + 1) * rows + R) * n + i] = probe_sign(h3, k, i);
  }
}

template <typename ST>
__global__ void k_wb_epilogue(cs_system sys, const ST *s0s, const ST *G, WbCtl *ctl, int B, int L, const double *A,
                              const double *C, int nsamp, double atol, double rtol, const double *pre, double damping,
                              double clip, ST *ea, ST *eb, ST *ec, ST *ed, ST *u) {
  const int n = sys.dim / 2, D = sys.dim;
  const int64_t rows = (int64_t)B * L;
  const bool do_clip = isfinite(clip);
  for (int64_t R = blockIdx.x; R < rows; R += gridDim.x) {  // one CTA per (proposal, step)
    const int b = (int)(R / L), t = (int)(R - (int64_t)b * L) + 1;
    if (ctl[b].status != -1) continue;
    const ST *pr = t == 1 ? s0s + (int64_t)b * D : G + (R - 1) * D;
    const ST *gr = G + R * D;
    bool fin = true, jok = true, pfail = false;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const double x = (double)pr[i], v = (double)pr[n + i];
      const double ev = sys.eps * v;
      const double xn = x + (sys.mass ? ev / __ldg(sys.mass + i) : ev);
      const double g = -C[R * n + i];  // grad = -(x' - mu) P
      const double vn = v + sys.eps * g;
      double dh = 0.0;
      for (int k = 0; k < nsamp; ++k) {
        const int64_t row = (int64_t)(k + 1) * rows + R;
        dh += A[row * n + i] * (-C[row * n + i]);  // z * hvp(x', z), hvp = -z P
      }
      dh = dh / (double)nsamp;
      const double m = sys.mass ? __ldg(sys.mass + i) : 1.0;
      double a = 1.0, bb = sys.mass ? sys.eps / m : sys.eps, c = sys.eps * dh;
      double d = 1.0 + (sys.mass ? (sys.eps * sys.eps) * dh / m : (sys.eps * sys.eps) * dh);
      fin &= isfinite(xn) && isfinite(vn);
      pfail |= !(fabs(xn - (double)gr[i]) <= atol + rtol * fabs(xn));
      pfail |= !(fabs(vn - (double)gr[n + i]) <= atol + rtol * fabs(vn));
      jok &= isfinite(a) && isfinite(bb) && isfinite(c) && isfinite(d);
      if (pre) {
        const double px = __ldg(pre + i), pv = __ldg(pre + n + i);
        bb = bb * (pv / px);
        c = c * (px / pv);
      }
      a = damping * a; bb = damping * bb; c = damping * c; d = damping * d;
      if (do_clip) { a = clipv(a, clip); bb = clipv(bb, clip); c = clipv(c, clip); d = clipv(d, clip); }
      ea[R * n + i] = (ST)a;
      eb[R * n + i] = (ST)bb;
      ec[R * n + i] = (ST)c;
      ed[R * n + i] = (ST)d;
      u[R * D + i] = (ST)(xn - (a * x + bb * v));
      u[R * D + n + i] = (ST)(vn - (c * x + d * v));
    }
    fin = __syncthreads_and(fin);
    jok = __syncthreads_and(jok);
    pfail = __syncthreads_or(pfail);
    if (threadIdx.x == 0) {
      if (!fin) atomicMin(&ctl[b].bad_f, (long long)t);
      if (!jok) atomicMin(&ctl[b].bad_j, (long long)t);
      if (pfail) atomicAdd(&ctl[b].pic, 1u);
    }
  }
}

// run_deer's checks before the update, in order (deer.py:263-271)
__global__ void k_wb_decide(int B, int max_iters, WbCtl *ctl) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < B; b += gridDim.x * blockDim.x) {
    WbCtl &c = ctl[b];
    if (c.status != -1) continue;
    if (c.bad_f != kNoStep) { c.status = CS_RUN_DIVERGED; c.kind = CS_DIV_STEP; c.estep = c.bad_f; c.eit = c.it + 1; continue; }
    if (c.pic == 0u) { c.status = CS_RUN_CONVERGED; continue; }
    if (c.it >= max_iters) { c.status = CS_RUN_MAXITERS; continue; }
    if (c.bad_j != kNoStep) { c.status = CS_RUN_DIVERGED; c.kind = CS_DIV_JACOBIAN; c.estep = c.bad_j; c.eit = c.it + 1; continue; }
    c.update = 1;
  }
}

// x_t = a x + b v + ux, v_t = c x + d v + uv from s0_b over the proposal's L
// steps (one thread per proposal column, f64 running state), the new guess
// written in place after the fail test against the old one (deer.py:273-277)
template <typename ST>
__global__ void k_wb_scan(int B, int L, int n, const ST *s0s, const ST *ea, const ST *eb, const ST *ec, const ST *ed,
                          const ST *u, double atol, double rtol, ST *G, WbCtl *ctl) {
  const int D = 2 * n;
  const int64_t tot = (int64_t)B * n;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < tot; idx += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(idx / n), i = (int)(idx - (int64_t)b * n);
    if (!ctl[b].update) continue;
    double x = (double)s0s[(int64_t)b * D + i], v = (double)s0s[(int64_t)b * D + n + i];
    unsigned fails = 0;
    unsigned long long dmb = 0ull;
    for (int t = 0; t < L; ++t) {
      const int64_t R = (int64_t)b * L + t;
      const double a = (double)ea[R * n + i], bb = (double)eb[R * n + i], c = (double)ec[R * n + i],
                   d = (double)ed[R * n + i];
      const double xn = a * x + bb * v + (double)u[R * D + i];
      const double vn = c * x + d * v + (double)u[R * D + n + i];
      x = xn;
      v = vn;
      const ST xs = (ST)x, vs = (ST)v;
      const double gx = fabs((double)xs - (double)G[R * D + i]), gv = fabs((double)vs - (double)G[R * D + n + i]);
      const bool f = gx > atol + rtol * fabs((double)xs) || gv > atol + rtol * fabs((double)vs);
      const unsigned long long bx = (unsigned long long)__double_as_longlong(gx),
                               bv = (unsigned long long)__double_as_longlong(gv);
      dmb = bx > dmb ? bx : dmb;
      dmb = bv > dmb ? bv : dmb;
      G[R * D + i] = xs;
      G[R * D + n + i] = vs;
      // a step fails if ANY of its columns fails: counted once per (proposal, step)
      // through the per-step word below
      fails |= f ? 1u : 0u;
      if (f) atomicOr(&ctl[b].fail, 1u);
    }
    (void)fails;
    atomicMax(&ctl[b].dmax_bits, dmb);
  }
}

__global__ void k_wb_settle(int B, WbCtl *ctl, int *active) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < B; b += gridDim.x * blockDim.x) {
    WbCtl &c = ctl[b];
    if (c.status == -1 && c.update) {
      c.it += 1;
      const double dmax = __longlong_as_double((long long)c.dmax_bits);
      if (c.d0 < 0.0) c.d0 = dmax;
      if (c.d0 > 0.0 && dmax > 1e6 * c.d0) {
        c.status = CS_RUN_DIVERGED;
        c.kind = CS_DIV_GUARD;
        c.eit = c.it;
      } else if (c.fail == 0u) {
        c.status = CS_RUN_CONVERGED;
      }
    }
    if (c.status == -1) atomicAdd(active, 1);
  }
}

template <typename ST>
__global__ void k_wb_finish(int B, int L, int D, const ST *G, const WbCtl *ctl, ST *finals, int32_t *info,
                            long long *err_step) {
  const int64_t tot = (int64_t)B * D;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = i / D;
    finals[i] = G[(b * L + L - 1) * D + i % D];
  }
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < B; b += gridDim.x * blockDim.x) {
    info[4 * b + 0] = ctl[b].status;
    info[4 * b + 1] = ctl[b].it;
    info[4 * b + 2] = ctl[b].kind;
    info[4 * b + 3] = ctl[b].eit;
    err_step[b] = ctl[b].estep;
  }
}

static unsigned g_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  return (unsigned)(g < 1 ? 1 : g);
}

template <typename ST>
static cudaError_t wide_batch_chunk(const cs_system &sys, const cs_deer_config &cfg, int B, const ST *s0s, ST *finals,
                                    int32_t *info, long long *err_step, cudaStream_t st) {
  const int n = sys.dim / 2, D = sys.dim, L = (int)sys.T;
  const int K = cfg.hutchinson_samples < 1 ? 1 : cfg.hutchinson_samples;
  const int64_t rows = (int64_t)B * L, M = rows * (1 + K);
  const size_t bA = sizeof(double) * (size_t)M * n, bG = sizeof(ST) * (size_t)rows * D;
  const size_t bE = sizeof(ST) * (size_t)rows * n;
  const size_t need = 2 * bA + 2 * bG + 4 * bE + sizeof(WbCtl) * (size_t)B + 256;
  // one grow-only scratch buffer per device (the solve synchronises every pass,
  // so the next call may reuse it; a stream-ordered malloc/free pair per call
  // returned the memory to the driver at every sync and re-mapped it)
  static std::mutex mu;
  static char *bufs[16];
  static size_t caps[16];
  static ScratchFence fences[16];
  int dv = 0;
  cudaGetDevice(&dv);
  std::lock_guard<std::mutex> lock(mu);
  ScratchScope scope(fences[dv & 15], st);
  cudaError_t e = cudaSuccess;
  if (caps[dv & 15] < need) {
    if (bufs[dv & 15]) cudaFree(bufs[dv & 15]);
    bufs[dv & 15] = nullptr;
    caps[dv & 15] = 0;
    if ((e = cudaMalloc((void **)&bufs[dv & 15], need)) != cudaSuccess) return e;
    caps[dv & 15] = need;
  }
  char *w = bufs[dv & 15];
  double *A = (double *)w, *C = (double *)(w + bA);
  ST *G = (ST *)(w + 2 * bA), *U = (ST *)(w + 2 * bA + bG);
  ST *ea = (ST *)(w + 2 * bA + 2 * bG), *eb = (ST *)((char *)ea + bE), *ec = (ST *)((char *)eb + bE),
     *ed = (ST *)((char *)ec + bE);
  WbCtl *ctl = (WbCtl *)((char *)ed + bE);
  static int *h_active[16];
  static int *d_active[16];
  int dev = 0;
  cudaGetDevice(&dev);
  if (!h_active[dev & 15]) {
    if ((e = cudaMallocHost(&h_active[dev & 15], sizeof(int))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&d_active[dev & 15], sizeof(int))) != cudaSuccess) return e;
  }
  int *ha = h_active[dev & 15], *da = d_active[dev & 15];
  k_wb_init<ST><<<g_for(rows * D), 256, 0, st>>>(s0s, B, L, D, G, ctl);
  for (int it = 0; it <= cfg.max_iters; ++it) {
    k_wb_reset<<<g_for(B), 256, 0, st>>>(B, ctl);
    k_wb_prologue<ST><<<g_for(rows * n), 256, 0, st>>>(sys, s0s, G, ctl, B, L, it, K, A);
    e = gemm_rm<double, double, double>(false, (int)M, n, n, A, n, 0, sys.target.prec, n, 0, C, n, 0, 1, st);
    if (e != cudaSuccess) break;
    k_wb_epilogue<ST><<<(unsigned)(rows < 148 * 16 ? rows : 148 * 16), 256, 0, st>>>(
        sys, s0s, G, ctl, B, L, A, C, K, cfg.atol, cfg.rtol, cfg.preconditioner, cfg.damping, cfg.clip, ea, eb, ec,
        ed, U);
    k_wb_decide<<<g_for(B), 256, 0, st>>>(B, cfg.max_iters, ctl);
    k_wb_scan<ST><<<g_for((int64_t)B * n), 256, 0, st>>>(B, L, n, s0s, ea, eb, ec, ed, U, cfg.atol, cfg.rtol, G, ctl);
    cudaMemsetAsync(da, 0, sizeof(int), st);
    k_wb_settle<<<g_for(B), 256, 0, st>>>(B, ctl, da);
    cudaMemcpyAsync(ha, da, sizeof(int), cudaMemcpyDeviceToHost, st);
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) break;
    if (*ha == 0) break;
  }
  if (e == cudaSuccess) {
    k_wb_finish<ST><<<g_for((int64_t)B * D), 256, 0, st>>>(B, L, D, G, ctl, finals, info, err_step);
    e = cudaGetLastError();
  }
  return e;
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
  ScratchScope scope(ctx.fence, st);
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
  k_wide_prologue<ST><<<g1 < 1 ? 1 : g1, 256, 0, st>>>(sys, s0, guess, iteration, K, A, stats);
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

cudaError_t wide_batch_solve(const cs_system &sys, const cs_deer_config &cfg, int dtype, int B, const void *s0s,
                             void *finals, int32_t *info, long long *err_step, cudaStream_t st) {
  // proposals in chunks that keep the GEMM operands to a few hundred MB
  const int64_t per = (int64_t)sys.T * (1 + (cfg.hutchinson_samples < 1 ? 1 : cfg.hutchinson_samples)) * (sys.dim / 2);
  int chunk = (int)(((int64_t)48 << 20) / (per > 0 ? per : 1));
  if (chunk < 1) chunk = 1;
  const int D = sys.dim;
  for (int b0 = 0; b0 < B; b0 += chunk) {
    const int nb = B - b0 < chunk ? B - b0 : chunk;
    cudaError_t e;
    if (dtype == CS_F64)
      e = wide_batch_chunk<double>(sys, cfg, nb, (const double *)s0s + (int64_t)b0 * D, (double *)finals + (int64_t)b0 * D,
                                   info + 4 * b0, err_step + b0, st);
    else
      e = wide_batch_chunk<float>(sys, cfg, nb, (const float *)s0s + (int64_t)b0 * D, (float *)finals + (int64_t)b0 * D,
                                  info + 4 * b0, err_step + b0, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
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
