// MALA element builder for the Bayesian logistic-regression target (BASELINE
// config 3: T = 100K chains steps, D = 100, N = 1000 data rows), diag
// quasi-Newton with K Hutchinson probes.
//
// One Newton update needs, at every step t, grad/logp at the current state S_t
// and at the proposal x~_t, plus hvp(S_t, z_k) and hvp(x~_t, dx~_k) for the
// probe tangents (samplers.py:95-145, targets.py:254-287).  All of them are
// row blocks of four plain GEMMs against the data matrix X (the fused builder
// in cs_blr_fused.cu does all of this in one kernel for <= 7 probes; this
// pipeline serves more probes):
//   E1 = [S; Z] X^T          logits eta_S and the probes' z X^T
//   G1 = [y - p_S; w_S.(Z X^T)] X       (w = p (1 - p))
//   E2 = [x~; dx~] X^T
//   G2 = [y - p~; w~.(dx~ X^T)] X
// run by our DMMA GEMM (cs_gemm.cuh, FP64 tensor cores); the sigmoid / weight / row-sum epilogues
// and the per-step MALA gate, tangents, Hutchinson estimate and element
// formation (deer.py:171-183) are our kernels, one warp per step.
#include <cstdlib>
#include <mutex>

#include "cs_apikern.cuh"
#include "cs_dispatch.h"
#include "cs_gemm.cuh"
#include "cs_umma.cuh"

namespace cs {

namespace {

constexpr int kBlrMaxD = 128;          // per-lane register slices of 4 columns
constexpr int kBlrCols = kBlrMaxD / 32;

struct BlrCtx {
  std::mutex mu;
  ScratchFence fence;
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

// float offset of element (row, k) in the tiled operand layout: tile (row / 128,
// k / 32) is 128 rows x 128 B, 16-byte chunk c of row rr stored at c ^ (rr & 7)
CS_D int64_t swz_index(int64_t row, int k, int nkb) {
  const int rr = (int)(row & 127), c = (k & 31) >> 2;
  return (((row >> 7) * nkb + (k >> 5)) * 128 + rr) * 32 + ((c ^ (rr & 7)) << 2) + (k & 3);
}

// first packed index of triangle row i (pairs (i, j >= i), row-major)
CS_D int pair_row_start(int i, int D) { return i * D - i * (i - 1) / 2; }

// zero the K padding (data rows N .. 32 nkb) of the tiled weight operand
__global__ void k_wt_pad(float *wsw, int64_t T, int N, int nkb) {
  const int pad = 32 * nkb - N;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < T * pad; i += (int64_t)gridDim.x * blockDim.x)
    wsw[swz_index(i / pad, N + (int)(i % pad), nkb)] = 0.0f;
}

// per step r (one warp, lanes across the N data rows): p = sigmoid(eta),
// E[r] <- y - p, probe rows <- p(1-p) . (z X^T), and the two log-density row
// sums eta.y and sum logaddexp(0, eta).  exp(-eta) serves both the sigmoid and,
// for eta >= 0, logaddexp's exp(-|eta|).
// wsw (optional): the weights again as f32 in the tiled tcgen05 operand layout
// of the pair-Gram GEMM (k_pair_gram): 128-step x 32-row tiles, K-major,
// SWIZZLE_128B, zero past N (nkb = padded data rows / 32)
__global__ void __launch_bounds__(256) k_blr_epilogue(double *E, const double *y, int64_t T, int K, int N,
                                                       double *rowsum, double *wout = nullptr,
                                                       float *wsw = nullptr, int nkb = 0) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < T; r += nw) {
    double a = 0.0, b = 0.0;
    double *er = E + r * N;
#pragma unroll 4
    for (int n = lane; n < N; n += 32) {
      const double eta = er[n], yn = __ldg(y + n);
      double p, lae;
      sigmoid_logaddexp(eta, p, lae);  // expit, logaddexp(0, eta)
      a += eta * yn;
      b += lae;
      er[n] = yn - p;
      const double w = p * (1.0 - p);
      if (wout) wout[r * N + n] = w;
      if (wsw) wsw[swz_index(r, n, nkb)] = (float)w;
      for (int k = 0; k < K; ++k) E[((int64_t)(k + 1) * T + r) * N + n] *= w;
    }
    if (wsw)
      for (int n = N + lane; n < 32 * nkb; n += 32) wsw[swz_index(r, n, nkb)] = 0.0f;
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

// ---------------------------------------------------------------------------
// Dense (full-Jacobian) Newton for BLR MALA (BASELINE cfg 3 "full").  The
// reference assembles J column by column from D jvps (core.py:125-134); the
// jvp is linear in V, so J has the closed form
//   A = I + eps H(S),  r = S - x~ - eps g(x~)
//   w = A g(x~) - g(S) + (H(S) r + A H(x~) r) / 2
//   J = gate A + (1 - gate) I + c (x~ - S) w^T,  c = sigma'(margin) 1(delta < 0)
// with H(x) = -X^T diag(p(1-p)) X - prec I.  H(x~) r is one GEMM pair against
// X; H(S) is formed explicitly per step (it is J's main term) by k_bd_final,
// which then forms the vectors, the gate and the element (preconditioner,
// damping, clip, u = f - J prev; deer.py:161-170) in the same CTA.

// g~ = G - prec x~ and r = S - x~ - eps g~ (T x D)
template <typename ST>
__global__ void k_bd_resid(cs_system sys, const ST *s0, const ST *guess, const double *A2, const double *G,
                           double *GX, double *R) {
  const int D = sys.dim;
  const int64_t total = sys.T * D;
  const double prec = sys.target.prior_precision, eps = sys.eps;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / D;
    const int i = (int)(idx - r * D);
    const double s = (double)(r == 0 ? s0[i] : guess[(r - 1) * D + i]);
    const double xt = A2[idx], gt = G[idx] - prec * xt;
    GX[idx] = gt;
    R[idx] = (s - xt) - eps * gt;
  }
}

constexpr int kBdThr = 256;

// one CTA per step r: H_raw = X^T diag(w_S) X (register-tiled, X streamed
// through shared memory in 16-row slices, the next slice prefetched into
// registers), then the closed-form J and the dense element
CS_D unsigned tf32_of(float x) {
  unsigned r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
CS_D void mma_tf32(float (&c)[4], unsigned a0, unsigned a1, unsigned a2, unsigned a3, unsigned b0, unsigned b1) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
               "{%0,%1,%2,%3};"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
               : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
CS_D void cp_async16_zfill(void *dst, const void *src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}

// X as f32 rows padded to 128 columns (the tensor-core Hessian's operand)
__global__ void k_bd_xf(const double *X, int N, int D, float *Xf) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N * 128; i += gridDim.x * blockDim.x) {
    const int n = i >> 7, d = i & 127;
    Xf[i] = d < D ? (float)X[(int64_t)n * D + d] : 0.0f;
  }
}

constexpr int kTcKB = 32, kTcLD = 136;  // n rows per staged block; padded row stride (conflict-free fragments)

// TCM: 0 = FP32/FP64 pipes, 1 = mma.sync TF32, 2 = tcgen05 (UMMA, TMEM accumulator),
// 3 = H_raw read from the pair-Gram GEMM's output (Xf = Hp, ldx = its row stride;
// the next step's packed triangle is copied in by cp.async behind this step)
template <typename ST, int DP, int TCM>
__global__ void __launch_bounds__(kBdThr)
k_bd_final(cs_system sys, cs_deer_config cfg, const ST *s0, const ST *guess, const double *A2, const double *GX,
           const double *gS, const double *R, const double *HR, const double *WS, const double *rsS,
           const double *rsX, const float *Xf, int ldx, ST *Jout, ST *uout, cs_elem_stats *stats) {
  using CT = ST;
  constexpr bool TC = TCM == 1;
  constexpr int NA = DP / 16, SL = 16, PER = SL * DP / kBdThr;
  constexpr int XS = TCM == 1 ? 2 * kTcKB * kTcLD + 2 * kTcKB : 2 * SL * DP;  // staging elements
  const int D = sys.dim, N = (int)sys.target.n_data;
  const double prec = sys.target.prior_precision, eps = sys.eps;
  const double *X = sys.target.X;
  const ST *xi = (const ST *)sys.noise_vec;
  extern __shared__ __align__(16) unsigned char bsm[];
  // TCM 2: the UMMA operand stages (1024-aligned) alias the Hessian tile
  CT *Hs = TCM == 2 ? smem_align<CT, 1024>(bsm) : (CT *)bsm;  // DP x DP
  // Hessian tile row stride: DP + 1 makes row and column walks bank-conflict
  // free; TCM 3 takes DP + 4 so the element rows are read as 16-byte vectors
  constexpr int HLD = TCM == 3 ? DP + 4 : DP + 1;
  constexpr int HS = TCM == 2 && 2 * kUmmaStages * kUmmaTile > DP * HLD ? 2 * kUmmaStages * kUmmaTile : DP * HLD;
  CT *Xs = Hs + HS;  // SIMT: 2 x SL x DP; mma.sync: 2 x kTcKB x kTcLD + 2 x kTcKB weights; tcgen05: ldx weights
  double *vS = TCM >= 2 ? smem_align<double, 16>(Xs + ldx)
                        : (double *)(Xs + XS + ((XS & 1) ? 1 : 0));
  double *vX = vS + DP, *vG = vX + DP, *vR = vG + DP, *vW = vR + DP, *vH = vW + DP, *vP = vH + DP;
  __shared__ double red[4][kBdThr / 32];
  __shared__ __align__(16) CT s_vwf[128], s_pcol[128];  // w_j in the storage type, p_j (the element rows)
  // matvec partials [4][2][128]: for TCM 2 in the stage region past the Hessian tile
  __shared__ double mpart_s[TCM == 2 ? 1 : 4 * 2 * 128];
  double(*mpart)[2][128] = (double(*)[2][128])(TCM == 2 ? (double *)(Hs + ((DP * HLD + 1) & ~1)) : mpart_s);
  __shared__ int flags[3];
  __shared__ __align__(8) uint64_t s_ubar[2 * kUmmaStages + 1];
  __shared__ uint32_t s_tmem;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4, lane = tid & 31, wid = tid >> 5;
  const bool do_clip = isfinite(cfg.clip);
  UmmaPipe pipe;
  if constexpr (TCM == 2) {
    static_assert(TCM != 2 || (DP == 128 && sizeof(ST) == 4), "tcgen05 Hessian: f32, 128 padded columns");
    pipe.full = s_ubar;
    pipe.empty = s_ubar + kUmmaStages;
    pipe.done = s_ubar + 2 * kUmmaStages;
    umma_pipe_init(pipe);
    pipe.tmem = tmem_alloc128(&s_tmem);  // its barrier also publishes the mbarrier inits
  }
  // TCM 2: the next step's weight row is loaded into registers behind this
  // step's Hessian, so the weights never cost an exposed round trip
  constexpr int WP = 8;  // weights per thread held in registers (N <= 2048; beyond: direct loads)
  float wpre[WP];
  auto wload = [&](int64_t rr) {
#pragma unroll
    for (int p = 0; p < WP; ++p) {
      const int n = tid + p * kBdThr;
      wpre[p] = (rr < sys.T && n < N) ? (float)__ldg(WS + rr * N + n) : 0.0f;
    }
  };
  if constexpr (TCM == 2) wload(blockIdx.x);
  static_assert(TCM != 3 || sizeof(ST) == 4, "pair-Gram Hessian: f32");
  const int hp_chunks = (D * (D + 1) / 2 + 3) / 4;
  auto hp_fetch = [&](int64_t rr) {  // step rr's packed triangle -> the staging row Xs
    if (rr < sys.T)
      for (int q = tid; q < hp_chunks; q += kBdThr) cp_async16(Xs + 4 * q, Xf + rr * ldx + 4 * q);
  };
  if constexpr (TCM == 3) hp_fetch(blockIdx.x);
  for (int64_t r = blockIdx.x; r < sys.T; r += gridDim.x) {
    const int64_t t = r + 1;
    const double *w = WS + r * N;
    // this step's vectors are requested now and used after the Hessian
    const ST *pr = r == 0 ? s0 : guess + (r - 1) * D;
    double pS = 0.0, pX = 0.0, pR = 0.0, pZ = 0.0, pG = 0.0, pH = 0.0, pgS = 0.0, pgu = 0.0;
    if (tid < D) {
      pS = (double)pr[tid];
      pX = A2[r * D + tid];
      pR = R[r * D + tid];
      pZ = (double)xi[t * D + tid];
      pG = GX[r * D + tid];
      pH = HR[r * D + tid];
      pgS = gS[r * D + tid];
      pgu = (double)guess[r * D + tid];
    }
    if constexpr (TCM == 2) {
      float *wbuf = (float *)Xs;
#pragma unroll
      for (int p = 0; p < WP; ++p) {
        const int n = tid + p * kBdThr;
        if (n < ldx) wbuf[n] = wpre[p];
      }
      for (int n = tid + WP * kBdThr; n < ldx; n += kBdThr) wbuf[n] = n < N ? (float)__ldg(w + n) : 0.0f;
      __syncthreads();
      gram_tcgen05<kBdThr>(pipe, Xf, ldx, N, wbuf, (float *)Hs, (float *)Hs, HLD);
      wload(r + gridDim.x);
    } else if constexpr (TCM == 3) {
      cp_async_wait_all();
      __syncthreads();
      // unpack: warp per triangle row, both halves of the symmetric tile
      for (int i = wid; i < D; i += kBdThr / 32) {
        const float *src = (const float *)Xs + pair_row_start(i, D) - i;
        for (int j = i + lane; j < D; j += 32) {
          const float v = src[j];
          Hs[i * HLD + j] = v;
          Hs[j * HLD + i] = v;
        }
      }
    } else if constexpr (TC) {
      // H_raw on the tensor cores (mma.sync m16n8k8 TF32, f32 accumulate):
      // warp wid owns output rows 16 wid .. 16 wid + 15, all 16 column blocks
      // of 8; A[d][n] = w_n X[n][d], B[n][e] = X[n][e], K = the N data rows
      // in blocks of 32 staged by cp.async (double-buffered)
      static_assert(!TC || (DP == 128 && sizeof(ST) == 4), "tensor-core Hessian: f32, 128 padded columns");
      float *xs = (float *)Xs, *wsl = xs + 2 * kTcKB * kTcLD;
      // warp wid owns output rows 16 wid .. 16 wid + 15, all 16 column blocks
      // (multiplying only the upper-triangle blocks measured slower: the
      // per-block operand selection costs more than the saved MMAs)
      const int g = lane >> 2, tq = lane & 3;
      float acc[16][4];
#pragma unroll
      for (int cb = 0; cb < 16; ++cb) acc[cb][0] = acc[cb][1] = acc[cb][2] = acc[cb][3] = 0.0f;
      const int nkb = (N + kTcKB - 1) / kTcKB;
      auto stage = [&](int kb, int buf) {
#pragma unroll
        for (int p = 0; p < kTcKB * 32 / kBdThr; ++p) {
          const int idx = tid + p * kBdThr, row = idx >> 5, c16 = idx & 31, n = kb * kTcKB + row;
          cp_async16_zfill(xs + buf * kTcKB * kTcLD + row * kTcLD + c16 * 4, Xf + (int64_t)(n < N ? n : 0) * 128 + c16 * 4,
                           n < N);
        }
        if (tid < kTcKB) {
          const int n = kb * kTcKB + tid;
          wsl[buf * kTcKB + tid] = n < N ? (float)__ldg(w + n) : 0.0f;
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
      };
      stage(0, 0);
      for (int kb = 0; kb < nkb; ++kb) {
        if (kb + 1 < nkb) {
          stage(kb + 1, (kb + 1) & 1);
          asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
          asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        const float *xb = xs + (kb & 1) * kTcKB * kTcLD, *wb = wsl + (kb & 1) * kTcKB;
#pragma unroll
        for (int ks = 0; ks < kTcKB / 8; ++ks) {
          const int n0 = ks * 8;
          const float w0 = wb[n0 + tq], w1 = wb[n0 + tq + 4];
          const float *r0 = xb + (n0 + tq) * kTcLD, *r1 = xb + (n0 + tq + 4) * kTcLD;
          const int d0 = 16 * wid + g;
          const unsigned a0 = tf32_of(w0 * r0[d0]), a1 = tf32_of(w0 * r0[d0 + 8]);
          const unsigned a2 = tf32_of(w1 * r1[d0]), a3 = tf32_of(w1 * r1[d0 + 8]);
#pragma unroll
          for (int cb = 0; cb < 16; ++cb)
            mma_tf32(acc[cb], a0, a1, a2, a3, tf32_of(r0[8 * cb + g]), tf32_of(r1[8 * cb + g]));
        }
        __syncthreads();  // the buffer is restaged two blocks on
      }
#pragma unroll
      for (int cb = 0; cb < 16; ++cb) {
        const int row = 16 * wid + g, col = 8 * cb + 2 * tq;
#pragma unroll
        for (int e = 0; e < 4; ++e) {  // upper triangle, mirrored: Hs is exactly symmetric
          const int ri = row + (e >> 1) * 8, ci = col + (e & 1);
          if (ci >= ri) {
            Hs[ri * HLD + ci] = acc[cb][e];
            Hs[ci * HLD + ri] = acc[cb][e];
          }
        }
      }
    } else {
    CT pf[PER];
    auto fetch = [&](int n0) {
#pragma unroll
      for (int p = 0; p < PER; ++p) {
        const int idx = tid + p * kBdThr, nn = idx / DP, d = idx - nn * DP, n = n0 + nn;
        pf[p] = (n < N && d < D) ? (CT)(__ldg(X + (int64_t)n * D + d) * __ldg(w + n)) : CT(0);
      }
    };
    auto stash = [&](int buf) {
#pragma unroll
      for (int p = 0; p < PER; ++p) Xs[buf * SL * DP + tid + p * kBdThr] = pf[p];
    };
    // the unweighted operand X[n][e] is read straight from the L2-resident X
    CT acc[NA][NA];
#pragma unroll
    for (int x = 0; x < NA; ++x)
#pragma unroll
      for (int y = 0; y < NA; ++y) acc[x][y] = CT(0);
    const int nsl = (N + SL - 1) / SL;
    fetch(0);
    stash(0);
    __syncthreads();
    for (int sl = 0; sl < nsl; ++sl) {
      if (sl + 1 < nsl) fetch((sl + 1) * SL);
      const CT *Xc = Xs + (sl & 1) * SL * DP;
#pragma unroll 4
      for (int nn = 0; nn < SL; ++nn) {
        const int n = sl * SL + nn;
        CT a[NA], b[NA];
#pragma unroll
        for (int x = 0; x < NA; ++x) a[x] = Xc[nn * DP + ty + 16 * x];  // w_n X[n][i]
        const double *xr = X + (int64_t)(n < N ? n : 0) * D;
#pragma unroll
        for (int y = 0; y < NA; ++y) {
          const int e = tx + 16 * y;
          b[y] = (n < N && e < D) ? (CT)__ldg(xr + e) : CT(0);
        }
#pragma unroll
        for (int x = 0; x < NA; ++x)
#pragma unroll
          for (int y = 0; y < NA; ++y) acc[x][y] = fma(a[x], b[y], acc[x][y]);
      }
      if (sl + 1 < nsl) stash((sl + 1) & 1);
      __syncthreads();
    }
#pragma unroll
    for (int x = 0; x < NA; ++x)
#pragma unroll
      for (int y = 0; y < NA; ++y) {  // upper triangle, mirrored: Hs is exactly symmetric
        const int ri = ty + 16 * x, ci = tx + 16 * y;
        if (ci >= ri) {
          Hs[ri * HLD + ci] = acc[x][y];
          Hs[ci * HLD + ri] = acc[x][y];
        }
      }
    }
    // vectors
    double ss = 0.0, sx = 0.0, sr = 0.0, sxi = 0.0, hxr = 0.0;
    if (tid < D) {
      const double S = pS, xt = pX, rr = pR, z = pZ;
      vS[tid] = S;
      vX[tid] = xt;
      vG[tid] = pG;
      vR[tid] = rr;
      hxr = -pH - prec * rr;  // H(x~) r
      vH[tid] = hxr;
      vP[tid] = cfg.preconditioner ? S * __ldg(cfg.preconditioner + tid) : S;  // p . S
      ss = S * S;
      sx = xt * xt;
      sr = rr * rr;
      sxi = z * z;
    }
    ss = warp_sum(ss);
    sx = warp_sum(sx);
    sr = warp_sum(sr);
    sxi = warp_sum(sxi);
    if (lane == 0) {
      red[0][wid] = ss;
      red[1][wid] = sx;
      red[2][wid] = sr;
      red[3][wid] = sxi;
    }
    if (tid < 3) flags[tid] = 0;
    __syncthreads();  // Hs, vectors, partial sums
    if constexpr (TCM == 3) hp_fetch(r + gridDim.x);  // the staging row is free again
    ss = sx = sr = sxi = 0.0;
#pragma unroll
    for (int k = 0; k < kBdThr / 32; ++k) {
      ss += red[0][k];
      sx += red[1][k];
      sr += red[2][k];
      sxi += red[3][k];
    }
    const double lpX = (rsX[2 * r] - rsX[2 * r + 1]) - 0.5 * prec * sx;
    const double lpS = (rsS[2 * r] - rsS[2 * r + 1]) - 0.5 * prec * ss;
    const double delta = lpX - lpS - sr / (4.0 * eps) + 0.5 * sxi;  // samplers.py:111-116
    const double margin = fmin(0.0, delta) - __ldg(sys.noise_logu + t);
    const double gate = margin > 0.0 ? 1.0 : 0.0;
    const double cb = sigmoid_prime(margin) * (delta < 0.0 ? 1.0 : 0.0);
    // w_i = A g~ - g(S) + (H(S) r + A H(x~) r)/2, H(S) v = -(H_raw v) - prec v; also
    // H(S) (p.S) for the closed-form u.  Two threads per row (column halves).
    {
      const int i = tid & 127, hf = tid >> 7;
      if (i < D) {
        const int jm = (D + 1) / 2, j0 = hf ? jm : 0, j1 = hf ? D : jm;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        for (int j = j0; j < j1; ++j) {
          const double h = (double)Hs[j * HLD + i];  // = H[i][j] (symmetric), bank-conflict free
          a0 = fma(h, vG[j], a0);
          a1 = fma(h, vR[j], a1);
          a2 = fma(h, vH[j], a2);
          a3 = fma(h, vP[j], a3);
        }
        mpart[0][hf][i] = a0;
        mpart[1][hf][i] = a1;
        mpart[2][hf][i] = a2;
        mpart[3][hf][i] = a3;
      }
    }
    __syncthreads();
    double wps = 0.0;
    if (tid < D) {
      const double hg = -(mpart[0][0][tid] + mpart[0][1][tid]) - prec * vG[tid];
      const double hr = -(mpart[1][0][tid] + mpart[1][1][tid]) - prec * vR[tid];
      const double hh = -(mpart[2][0][tid] + mpart[2][1][tid]) - prec * vH[tid];
      const double wv = (vG[tid] + eps * hg) - pgS + 0.5 * (hr + (hxr + eps * hh));
      vW[tid] = wv;
      wps = wv * vP[tid];
      s_vwf[tid] = (CT)wv;
      s_pcol[tid] = cfg.preconditioner ? (CT)__ldg(cfg.preconditioner + tid) : CT(1);
    }
    wps = warp_sum(wps);
    if (lane == 0) red[0][wid] = wps;
    __syncthreads();
    // element: J_ij = gate (d_ij + eps H_ij) + (1 - gate) d_ij + cb (x~_i - S_i) w_j, then the
    // preconditioner ratio p_j / p_i, damping and clip (deer.py:161-170)
    auto Jij = [&](int i, int j, double hraw) {  // hraw = H_raw[i][j]
      const double hij = -hraw - (i == j ? prec : 0.0);
      const double dij = i == j ? 1.0 : 0.0;
      double v = gate * (dij + eps * hij) + (1.0 - gate) * dij + cb * (vX[i] - vS[i]) * vW[j];
      if (cfg.preconditioner) v = v * (__ldg(cfg.preconditioner + j) / __ldg(cfg.preconditioner + i));
      v = v * cfg.damping;
      if (do_clip) v = clipv(v, cfg.clip);
      return v;
    };
    ST *Jr = Jout + r * (int64_t)D * D;
    bool jok = true;
    {
      // warp per row, lanes across the row (coalesced stores, no index division);
      // the entries are formed in the storage precision, the f64 parts hoisted
      const CT g1 = (CT)gate, g0 = (CT)(1.0 - gate), ce = (CT)(gate * eps), lam = (CT)cfg.damping;
      const CT cl = (CT)cfg.clip;
      const CT pdiag = (CT)prec;
      const bool pre = cfg.preconditioner != nullptr;
      auto elem = [&](int i, int j, CT h, CT ci, CT pinv) {
        const CT hij = -h - (i == j ? pdiag : CT(0));
        CT v = ce * hij + ci * s_vwf[j] + (i == j ? g1 + g0 : CT(0));
        if (pre) v = v * (s_pcol[j] * pinv);
        v = v * lam;
        if (do_clip) v = v < -cl ? -cl : (v > cl ? cl : v);
        jok &= isfinite(v);
        return v;
      };
      auto rows_scalar = [&]() {
        for (int i = wid; i < D; i += kBdThr / 32) {
          const CT ci = (CT)(cb * (vX[i] - vS[i]));
          const CT pinv = pre ? (CT)(1.0 / __ldg(cfg.preconditioner + i)) : CT(1);
          const CT *hrow = Hs + i * HLD;
          ST *jrow = Jr + (int64_t)i * D;
          for (int j = lane; j < D; j += 32) jrow[j] = (ST)elem(i, j, hrow[j], ci, pinv);
        }
      };
      if constexpr (TCM == 3) {
        if ((D & 3) == 0) {
          // four columns per lane: 16-byte Hessian reads and J stores
          for (int i = wid; i < D; i += kBdThr / 32) {
            const CT ci = (CT)(cb * (vX[i] - vS[i]));
            const CT pinv = pre ? (CT)(1.0 / __ldg(cfg.preconditioner + i)) : CT(1);
            const CT *hrow = Hs + i * HLD;
            ST *jrow = Jr + (int64_t)i * D;
            for (int j = 4 * lane; j < D; j += 128) {
              const float4 h = *(const float4 *)(hrow + j);
              float4 o;
              o.x = elem(i, j, h.x, ci, pinv);
              o.y = elem(i, j + 1, h.y, ci, pinv);
              o.z = elem(i, j + 2, h.z, ci, pinv);
              o.w = elem(i, j + 3, h.w, ci, pinv);
              *(float4 *)(jrow + j) = o;
            }
          }
        } else {
          rows_scalar();
        }
      } else {
        rows_scalar();
      }
    }
    if (!jok) flags[1] = 1;
    if (tid < D) {
      const double f = gate > 0.0 ? vX[tid] : vS[tid];
      double jp = 0.0;
      if (do_clip) {  // clipped entries: the elementwise row sum
        for (int j = 0; j < D; ++j) jp = fma(Jij(tid, j, (double)Hs[j * HLD + tid]), vS[j], jp);
      } else {
        // (J prev)_i = (damping / p_i) [gate (pS_i + eps (H pS)_i) + (1 - gate) pS_i + cb dx_i (w . pS)]
        double wp = 0.0;
#pragma unroll
        for (int k = 0; k < kBdThr / 32; ++k) wp += red[0][k];
        const double ps = vP[tid];
        const double hp = -(mpart[3][0][tid] + mpart[3][1][tid]) - prec * ps;
        const double pi = cfg.preconditioner ? __ldg(cfg.preconditioner + tid) : 1.0;
        jp = (cfg.damping / pi) *
             (gate * (ps + eps * hp) + (1.0 - gate) * ps + cb * (vX[tid] - vS[tid]) * wp);
      }
      uout[r * D + tid] = (ST)(f - jp);
      if (!isfinite(f)) flags[0] = 1;
      if (!(fabs(f - pgu) <= cfg.atol + cfg.rtol * fabs(f))) flags[2] = 1;
    }
    __syncthreads();
    if (tid == 0) {
      if (flags[0]) atomicMin((long long *)&stats->bad_step, (long long)t);
      if (flags[1]) atomicMin((long long *)&stats->bad_jacobian, (long long)t);
      if (flags[2]) atomicAdd(&stats->picard_fail, 1u);
    }
    __syncthreads();
  }
  if constexpr (TCM == 2) tmem_free128(pipe.tmem);
}

// X^T as f32 [128][ldx] (rows >= D and columns >= N zero): the UMMA operand source
__global__ void k_bd_xt(const double *X, int N, int D, int ldx, float *XT) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 128 * ldx; i += gridDim.x * blockDim.x) {
    const int d = i / ldx, n = i - d * ldx;
    XT[i] = (d < D && n < N) ? (float)X[(int64_t)n * D + d] : 0.0f;
  }
}

// ---- H_t for every step as ONE GEMM over data-row pairs ---------------------
// H_raw,t[i][j] = sum_n w_t[n] X[n][i] X[n][j] = (W Q^T)[t][p(i, j)] with
// Q[p(i, j)][n] = X[n][i] X[n][j] over the upper-triangle pairs p (row-major,
// p(i, j) = i D - i (i - 1) / 2 + j - i).  The per-step weights become the A
// operand and the data products a fixed B operand, so the tensor cores stream
// TMA-loaded tiles instead of re-forming w . X^T per step (k_bd_final TCM 2).

// Q in the tiled operand layout (see swz_index), pairs >= P and data rows >= N zero
__global__ void k_pair_operand(const double *X, int N, int D, int nkb, int P, int64_t total, float *Qt) {
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    const int e = (int)(o & 3), sc = (int)((o >> 2) & 7), rr = (int)((o >> 5) & 127);
    const int64_t tile = o >> 12;
    const int kb = (int)(tile % nkb), nt = (int)(tile / nkb);
    const int p = nt * 128 + rr, n = kb * 32 + ((sc ^ (rr & 7)) << 2) + e;
    float v = 0.0f;
    if (p < P && n < N) {
      const double b = 2.0 * D + 1.0;
      int i = (int)floor((b - sqrt(b * b - 8.0 * p)) * 0.5);
      i = i < 0 ? 0 : (i >= D ? D - 1 : i);
      while (i + 1 < D && pair_row_start(i + 1, D) <= p) ++i;
      while (i > 0 && pair_row_start(i, D) > p) --i;
      const int j = i + p - pair_row_start(i, D);
      v = (float)(X[(int64_t)n * D + i] * X[(int64_t)n * D + j]);
    }
    Qt[o] = v;
  }
}

// Hp (f32, row stride ldp) = W Q^T: one 128-step x 128-pair tile per CTA, K =
// the data rows in blocks of 32.  Warp 0 lane 0 moves the pre-tiled operand
// blocks with 1-D bulk copies (TMA engine), warp 1 lane 0 issues kind::tf32
// MMAs into a TMEM accumulator; all four warps then drain TMEM through shared
// memory and write the tile rows back with bulk stores.  Two CTAs per SM: one's
// epilogue overlaps the other's MMAs.
constexpr int kPgStages = 3;
constexpr int kPgLd = 132;  // staged output row stride (floats): conflict-free v4 stores, 16-byte rows
static_assert(128 * kPgLd <= kPgStages * 2 * kUmmaTile, "output staging fits the operand stages");

__global__ void __launch_bounds__(128) k_pair_gram(const float *__restrict__ Wt, const float *__restrict__ Qt, int nkb,
                                                  float *Hp, int64_t ldp) {
  extern __shared__ __align__(16) unsigned char psm[];
  float *tiles = smem_align<float, 1024>(psm);
  __shared__ __align__(8) uint64_t full[kPgStages], empty[kPgStages], done;
  __shared__ uint32_t s_tmem;
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  const int nt = blockIdx.x;
  const int64_t mt = blockIdx.y;
  if (tid == 0) {
    for (int s = 0; s < kPgStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&done, 1);
    fence_mbar_init();
  }
  const uint32_t tmem = tmem_alloc128(&s_tmem);  // its barrier also publishes the mbarrier inits
  const float *Ab = Wt + mt * nkb * kUmmaTile, *Bb = Qt + (int64_t)nt * nkb * kUmmaTile;
  if (wid == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % kPgStages;
        if (kb >= kPgStages) mbar_wait(&empty[s], ((kb / kPgStages) - 1) & 1);
        float *A = tiles + s * 2 * kUmmaTile;
        mbar_expect_tx(&full[s], 2 * kUmmaTile * sizeof(float));
        bulk_g2s(A, Ab + (int64_t)kb * kUmmaTile, kUmmaTile * sizeof(float), &full[s]);
        bulk_g2s(A + kUmmaTile, Bb + (int64_t)kb * kUmmaTile, kUmmaTile * sizeof(float), &full[s]);
      }
    }
    __syncwarp();
  } else if (wid == 1) {
    if (lane == 0) {
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % kPgStages;
        mbar_wait(&full[s], (kb / kPgStages) & 1);
        tc_fence_after();
        const float *A = tiles + s * 2 * kUmmaTile;
        const uint64_t da = umma_desc_sw128(A), db = umma_desc_sw128(A + kUmmaTile);
#pragma unroll
        for (int k = 0; k < kUmmaKB / 8; ++k)
          umma_tf32(tmem, da + 2 * k, db + 2 * k, kIdescTf32_128x128, (kb | k) != 0);
        umma_commit(&empty[s]);
      }
      umma_commit(&done);
    }
    __syncwarp();
  }
  mbar_wait(&done, 0);
  tc_fence_after();
  // TMEM lanes 32 w .. 32 w + 31 = this warp's tile rows -> staged rows -> bulk stores
  const int row = 32 * wid + lane;
  float *srow = tiles + row * kPgLd;
#pragma unroll
  for (int cc = 0; cc < 128; cc += 16) {
    float v[16];
    tmem_ld16(tmem + ((uint32_t)(32 * wid) << 16) + (uint32_t)cc, v);
#pragma unroll
    for (int q = 0; q < 4; ++q) *(float4 *)(srow + cc + 4 * q) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  }
  fence_proxy_async_smem();
  bulk_s2g(Hp + (mt * 128 + row) * ldp + (int64_t)nt * 128, srow, 128 * sizeof(float));
  bulk_commit();
  bulk_wait_read();
  tmem_free128(tmem);
}

}  // namespace

// test hook: H_t = X^T diag(W_t) X through the tcgen05 path, one CTA per t
__global__ void __launch_bounds__(kBdThr) k_gram_debug(const float *XT, int ldx, int N, const double *W, int64_t T,
                                                       float *Hout) {
  extern __shared__ __align__(16) unsigned char gsm[];
  float *tiles = smem_align<float, 1024>(gsm);
  constexpr int kHs = 2 * kUmmaStages * kUmmaTile > 128 * 129 ? 2 * kUmmaStages * kUmmaTile : 128 * 129;
  float *wbuf = tiles + kHs;  // after the operand stages / the (aliased) Hessian tile
  __shared__ __align__(8) uint64_t bars[2 * kUmmaStages + 1];
  __shared__ uint32_t s_tmem;
  UmmaPipe pipe;
  pipe.full = bars;
  pipe.empty = bars + kUmmaStages;
  pipe.done = bars + 2 * kUmmaStages;
  umma_pipe_init(pipe);
  pipe.tmem = tmem_alloc128(&s_tmem);
  for (int64_t r = blockIdx.x; r < T; r += gridDim.x) {
    for (int n = threadIdx.x; n < ldx; n += blockDim.x) wbuf[n] = n < N ? (float)W[r * N + n] : 0.0f;
    __syncthreads();
    gram_tcgen05<kBdThr>(pipe, XT, ldx, N, wbuf, tiles, tiles, 129);
    for (int i = threadIdx.x; i < 128 * 128; i += blockDim.x) Hout[r * 128 * 128 + i] = tiles[(i >> 7) * 129 + (i & 127)];
    __syncthreads();
  }
  tmem_free128(pipe.tmem);
}

bool blr_mala_ok(const cs_system &s, int mode) {
  return s.kind == CS_SYS_MALA && s.target.kind == CS_TARGET_BLR && (mode == CS_MODE_DIAG || mode == CS_MODE_DENSE) &&
         s.dim >= 1 &&
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
  ScratchScope scope(ctx.fence, st);
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
  // the two data products on the FP64 tensor cores (cs_gemm.cuh), row-major
  auto gemm_xt = [&](const double *Ain, double *Cout) {  // C (M x N) = A (M x D) X^T
    return gemm_rm<double, double, double>(true, (int)M, N, D, Ain, D, 0, X, D, 0, Cout, N, 0, 1, st);
  };
  auto gemm_x = [&](const double *Bin, double *Cout) {  // C (M x D) = B (M x N) X
    return gemm_rm<double, double, double>(false, (int)M, D, N, Bin, N, 0, X, D, 0, Cout, D, 0, 1, st);
  };
  const unsigned ge = (unsigned)((T * D + 255) / 256 < 148 * 32 ? (T * D + 255) / 256 : 148 * 32);
  const unsigned gw = (unsigned)((T * 32 + 255) / 256);
  k_blr_prologue<ST><<<ge, 256, 0, st>>>(sys, s0, guess, iteration, K, A);
  if (cudaError_t ge = gemm_xt(A, E)) return ge;
  k_blr_epilogue<<<gw, 256, 0, st>>>(E, y, T, K, N, rsS);
  if (cudaError_t ge = gemm_x(E, G)) return ge;
  k_blr_propose<ST><<<gw, 256, 0, st>>>(sys, s0, guess, A, G, K, A2, gS, stats);
  if (cudaError_t ge = gemm_xt(A2, E)) return ge;
  k_blr_epilogue<<<gw, 256, 0, st>>>(E, y, T, K, N, rsX);
  if (cudaError_t ge = gemm_x(E, G)) return ge;
  k_blr_final<ST><<<gw, 256, 0, st>>>(sys, cfg, iteration, s0, guess, A, A2, G, gS, rsS, rsX, jout, uout, stats);
  return cudaGetLastError();
}

// f32 Hessian (CS_BLR_DENSE_TC): 3 pair-Gram GEMM on tcgen05 (default), 2 per-step
// tcgen05 Gram, 1 mma.sync, 0 FP32 pipes
static int bd_tensor_cores() {
  static const int v = [] {
    const char *e = getenv("CS_BLR_DENSE_TC");
    return e ? atoi(e) : 3;
  }();
  return v;
}

template <typename ST, int DP, int TCM = 0>
static cudaError_t bd_final_launch(const cs_system &sys, const cs_deer_config &cfg, const ST *s0, const ST *guess,
                                   const double *A2, const double *GX, const double *gS, const double *R,
                                   const double *HR, const double *WS, const double *rsS, const double *rsX,
                                   const float *Xf, ST *J, ST *u, cs_elem_stats *stats, cudaStream_t st,
                                   int ldx = 0) {
  const size_t xs = TCM == 1 ? 2 * kTcKB * kTcLD + 2 * kTcKB : TCM >= 2 ? (size_t)ldx + 4 : 2 * 16 * DP;
  const size_t hld = TCM == 3 ? DP + 4 : DP + 1;
  const size_t hs = TCM == 2 && 2 * kUmmaStages * kUmmaTile > DP * hld ? 2 * kUmmaStages * kUmmaTile : DP * hld;
  const size_t smem = sizeof(ST) * (hs + xs) + 8 + 7 * DP * sizeof(double) + (TCM == 2 ? 1024 : 0);
  auto k = k_bd_final<ST, DP, TCM>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t grid = sys.T < 148 * 16 ? sys.T : 148 * 16;
  k<<<(unsigned)grid, kBdThr, smem, st>>>(sys, cfg, s0, guess, A2, GX, gS, R, HR, WS, rsS, rsX, Xf, ldx, J, u,
                                          stats);
  return cudaGetLastError();
}

template <typename ST>
static cudaError_t blr_dense_run(const cs_system &sys, const cs_deer_config &cfg, int64_t iteration, const ST *s0,
                                 const ST *guess, ST *J, ST *uout, cs_elem_stats *stats, cudaStream_t st) {
  const int D = sys.dim, N = (int)sys.target.n_data;
  const int64_t T = sys.T;
  int dev = 0;
  cudaGetDevice(&dev);
  BlrCtx &ctx = g_blr[dev & 15];
  std::lock_guard<std::mutex> lock(ctx.mu);
  ScratchScope scope(ctx.fence, st);
  // A, A2, G, gS, GX, R, HR (T x D); E, WS, WX (T x N); row sums 2 x (2T)
  // + Xf: X as f32 (N x 128, or its transpose 128 x ldx for tcgen05)
  // pair-Gram path: W tiles (Tpad x 32 nkb), Q tiles (ldp x 32 nkb), Hp (Tpad x ldp), f32
  const bool pg = sizeof(ST) == 4 && bd_tensor_cores() == 3;
  const int nkb = (N + 31) / 32, npairs = D * (D + 1) / 2;
  const int64_t Tpad = (T + 127) / 128 * 128, ldp = (int64_t)(npairs + 127) / 128 * 128;
  const size_t pg_floats = pg ? (size_t)(Tpad * 32 * nkb + ldp * 32 * nkb + Tpad * ldp) : 0;
  // + the fused GEMM epilogue's row partials (T x npart x 2)
  const int npart = (N + 63) / 64 * 2;
  const size_t need = (size_t)7 * T * D + (size_t)3 * T * N + (size_t)4 * T + (size_t)64 * (N + 32) +
                      (pg_floats + 1) / 2 + 64 + (size_t)2 * T * npart + 64;
  if (ctx.cap < need) {
    if (ctx.buf) cudaFree(ctx.buf);
    ctx.buf = nullptr;
    ctx.cap = 0;
    cudaError_t e = cudaMalloc(&ctx.buf, need * sizeof(double));
    if (e != cudaSuccess) return e;
    ctx.cap = need;
  }
  double *A = ctx.buf, *A2 = A + (size_t)T * D, *G = A2 + (size_t)T * D, *gS = G + (size_t)T * D;
  double *GX = gS + (size_t)T * D, *R = GX + (size_t)T * D, *HR = R + (size_t)T * D;
  double *E = HR + (size_t)T * D, *WS = E + (size_t)T * N, *WX = WS + (size_t)T * N;
  double *rsS = WX + (size_t)T * N, *rsX = rsS + 2 * T;
  float *Xf = (float *)(rsX + 2 * T);
  float *Wt = (float *)(((uintptr_t)(rsX + 2 * T + 64 * (N + 32)) + 255) & ~(uintptr_t)255);
  float *Qt = Wt + Tpad * 32 * nkb, *Hp = Qt + ldp * 32 * nkb;
  double *part = (double *)(((uintptr_t)(pg ? Hp + Tpad * ldp : Wt) + 255) & ~(uintptr_t)255);
  const double *X = sys.target.X, *y = sys.target.y;
  auto gemm_xt = [&](const double *Ain, double *Cout) {  // C (T x N) = A (T x D) X^T
    return gemm_rm<double, double, double>(true, (int)T, N, D, Ain, D, 0, X, D, 0, Cout, N, 0, 1, st);
  };
  // the same product with the logistic epilogue fused into its tile stores
  auto gemm_xt_logit = [&](const double *Ain, double *wout, float *wsw, double *rowsum) {
    return gemm_xt_logistic((int)T, N, D, Ain, D, X, D, E, N, y, wout, wsw, nkb, part, rowsum, st);
  };
  auto gemm_x = [&](const double *Bin, double *Cout) {  // C (T x D) = B (T x N) X
    return gemm_rm<double, double, double>(false, (int)T, D, N, Bin, N, 0, X, D, 0, Cout, D, 0, 1, st);
  };
  const unsigned ge = (unsigned)((T * D + 255) / 256 < 148 * 32 ? (T * D + 255) / 256 : 148 * 32);
  const unsigned gw = (unsigned)((T * 32 + 255) / 256);
  k_blr_prologue<ST><<<ge, 256, 0, st>>>(sys, s0, guess, iteration, 0, A);
  if (pg) {  // the weights go straight into the GEMM's operand tiles; H_raw for every step in one GEMM
    if (cudaError_t ge = gemm_xt_logit(A, nullptr, Wt, rsS)) return ge;
    if (N < 32 * nkb) k_wt_pad<<<(unsigned)((T * 32 + 255) / 256), 256, 0, st>>>(Wt, T, N, nkb);
    const int64_t qn = ldp * 32 * nkb;
    k_pair_operand<<<(unsigned)((qn + 255) / 256 < 148 * 64 ? (qn + 255) / 256 : 148 * 64), 256, 0, st>>>(
        X, N, D, nkb, npairs, qn, Qt);
    const size_t smem = 1024 + (size_t)kPgStages * 2 * kUmmaTile * sizeof(float);
    static bool attr = false;
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute(k_pair_gram, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      attr = true;
    }
    k_pair_gram<<<dim3((unsigned)(ldp / 128), (unsigned)(Tpad / 128)), 128, smem, st>>>(Wt, Qt, nkb, Hp, ldp);
  } else {
    if (cudaError_t ge = gemm_xt_logit(A, WS, nullptr, rsS)) return ge;
  }
  if (cudaError_t ge = gemm_x(E, G)) return ge;
  k_blr_propose<ST><<<gw, 256, 0, st>>>(sys, s0, guess, A, G, 0, A2, gS, stats);
  if (cudaError_t ge = gemm_xt_logit(A2, WX, nullptr, rsX)) return ge;
  if (cudaError_t ge = gemm_x(E, G)) return ge;
  k_bd_resid<ST><<<ge, 256, 0, st>>>(sys, s0, guess, A2, G, GX, R);
  // H(x~) r: (r X^T) . w~ straight out of the GEMM, then against X
  if (cudaError_t ge = gemm_xt_scaled((int)T, N, D, R, D, X, D, E, N, WX, st)) return ge;
  if (cudaError_t ge = gemm_x(E, HR)) return ge;
  if constexpr (sizeof(ST) == 4) {
    if (pg) {
      if (D <= 112)
        return bd_final_launch<ST, 112, 3>(sys, cfg, s0, guess, A2, GX, gS, R, HR, WS, rsS, rsX, Hp, J, uout, stats,
                                           st, (int)ldp);
      return bd_final_launch<ST, 128, 3>(sys, cfg, s0, guess, A2, GX, gS, R, HR, WS, rsS, rsX, Hp, J, uout, stats,
                                         st, (int)ldp);
    }
    if (bd_tensor_cores() == 2) {  // f32 storage: H(S) on the 5th-gen tensor cores (tcgen05, TMEM accumulator)
      const int ldx = (N + 31) / 32 * 32;
      k_bd_xt<<<(128 * ldx + 255) / 256, 256, 0, st>>>(X, N, D, ldx, Xf);
      return bd_final_launch<ST, 128, 2>(sys, cfg, s0, guess, A2, GX, gS, R, HR, WS, rsS, rsX, Xf, J, uout,
                                         stats, st, ldx);
    }
    if (bd_tensor_cores() == 1) {  // mma.sync TF32
      k_bd_xf<<<(N * 128 + 255) / 256, 256, 0, st>>>(X, N, D, Xf);
      return bd_final_launch<ST, 128, 1>(sys, cfg, s0, guess, A2, GX, gS, R, HR, WS, rsS, rsX, Xf, J, uout,
                                         stats, st);
    }
  }
  const int dp = D <= 16 ? 16 : D <= 32 ? 32 : D <= 64 ? 64 : D <= 112 ? 112 : 128;
  switch (dp) {
    case 16: return bd_final_launch<ST, 16>(sys, cfg, s0, guess, A2, GX, gS, R, HR, WS, rsS, rsX, Xf, J, uout, stats, st);
    case 32: return bd_final_launch<ST, 32>(sys, cfg, s0, guess, A2, GX, gS, R, HR, WS, rsS, rsX, Xf, J, uout, stats, st);
    case 64: return bd_final_launch<ST, 64>(sys, cfg, s0, guess, A2, GX, gS, R, HR, WS, rsS, rsX, Xf, J, uout, stats, st);
    case 112: return bd_final_launch<ST, 112>(sys, cfg, s0, guess, A2, GX, gS, R, HR, WS, rsS, rsX, Xf, J, uout, stats, st);
    default: return bd_final_launch<ST, 128>(sys, cfg, s0, guess, A2, GX, gS, R, HR, WS, rsS, rsX, Xf, J, uout, stats, st);
  }
}

cudaError_t debug_gram(const double *X, int N, int D, const double *W, int64_t T, float *H, cudaStream_t st) {
  const int ldx = (N + 31) / 32 * 32;
  float *XT = nullptr;
  cudaError_t e = scratch_alloc((void **)&XT, sizeof(float) * 128 * ldx, st);
  if (e != cudaSuccess) return e;
  k_bd_xt<<<(128 * ldx + 255) / 256, 256, 0, st>>>(X, N, D, ldx, XT);
  const size_t hs = 2 * kUmmaStages * kUmmaTile > 128 * 129 ? 2 * kUmmaStages * kUmmaTile : 128 * 129;
  const size_t smem = 1024 + sizeof(float) * (hs + ldx + 4);
  cudaFuncSetAttribute(k_gram_debug, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_gram_debug<<<(unsigned)(T < 148 ? T : 148), kBdThr, smem, st>>>(XT, ldx, N, W, T, H);
  e = cudaGetLastError();
  cudaFreeAsync(XT, st);
  return e;
}

namespace {
__global__ void k_w_tiles(const double *W, int64_t T, int N, int nkb, float *Wt) {  // W (T x N) -> operand tiles
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < T * 32 * nkb; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / (32 * nkb);
    const int n = (int)(i - r * 32 * nkb);
    Wt[swz_index(r, n, nkb)] = n < N ? (float)W[r * N + n] : 0.0f;
  }
}
__global__ void k_pair_unpack(const float *Hp, int64_t ldp, int64_t T, int D, float *H) {  // -> T x 128 x 128
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < T * 128 * 128; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i >> 14;
    const int a = (int)((i >> 7) & 127), b = (int)(i & 127);
    const int lo = a < b ? a : b, hi = a < b ? b : a;
    H[i] = (a < D && b < D) ? Hp[t * ldp + pair_row_start(lo, D) + hi - lo] : 0.0f;
  }
}
}  // namespace

// ---- target model functions on the device (targets.py:160-287 ModelFns) -------
// The GEMM-shaped targets -- logistic regression and dense Gaussians of any
// width -- evaluated for a batch of n states with our DMMA GEMM and small row
// kernels: log density (n), gradient (n x D), Hessian-vector product (n x D).
namespace {
// rows of E (n x N): logp partials eta.y - sum logaddexp(0, eta) - prec/2 |x|^2 (warp per row)
__global__ void k_tgt_blr_logp(const double *E, const double *y, const double *x, int64_t n, int N, int D,
                               double prec, double *out) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += nw) {
    double a = 0.0, b = 0.0, q = 0.0;
    for (int k = lane; k < N; k += 32) {
      const double eta = E[r * N + k];
      a += eta * __ldg(y + k);
      b += logaddexp0(eta);
    }
    for (int d = lane; d < D; d += 32) q += x[r * D + d] * x[r * D + d];
    a = warp_sum(a);
    b = warp_sum(b);
    q = warp_sum(q);
    if (lane == 0) out[r] = (a - b) - 0.5 * prec * q;
  }
}
// E <- y - sigmoid(E)  (what 1), or T <- sigmoid'(E) . T (what 2)
__global__ void k_tgt_blr_map(double *E, const double *y, double *T, int64_t total, int N, int what) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const double eta = E[i];
    const double p = expit(eta);
    if (what == 1) E[i] = __ldg(y + i % N) - p;
    else T[i] *= p * (1.0 - p);
  }
}
// out = sgn * G - c * z (the prior / precision terms), elementwise
__global__ void k_tgt_axpy(double *out, const double *G, const double *z, int64_t total, double sgn, double c) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = sgn * G[i] - (z ? c * z[i] : 0.0);
}
__global__ void k_tgt_diff(const double *x, const double *mu, int64_t n, int D, double *out) {  // x - mu
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n * D; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = x[i] - __ldg(mu + i % D);
}
__global__ void k_tgt_halfsq(const double *H, int64_t n, int D, double *out) {  // -|h|^2 / 2 per row
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += nw) {
    double q = 0.0;
    for (int d = lane; d < D; d += 32) q += H[r * D + d] * H[r * D + d];
    q = warp_sum(q);
    if (lane == 0) out[r] = -0.5 * q;
  }
}
unsigned egrid(int64_t total) { return (unsigned)((total + 255) / 256 < 148 * 16 ? (total + 255) / 256 : 148 * 16); }
}  // namespace

cudaError_t target_eval_gemm(const cs_target &tg, int what, int64_t n, const double *x, const double *v,
                             double *out, cudaStream_t st) {
  const int D = tg.dim;
  if (n <= 0) return cudaSuccess;
  const unsigned gw = (unsigned)((n * 32 + 255) / 256 < 148 * 16 ? (n * 32 + 255) / 256 : 148 * 16);
  if (tg.kind == CS_TARGET_BLR) {
    const int N = (int)tg.n_data;
    double *E = nullptr, *Tm = nullptr;
    const size_t eb = sizeof(double) * (size_t)n * N;
    cudaError_t e = scratch_alloc((void **)&E, what == 2 ? 2 * eb : eb, st);
    if (e != cudaSuccess) return e;
    Tm = what == 2 ? E + (size_t)n * N : nullptr;
    // eta = x X^T
    e = gemm_rm<double, double, double>(true, (int)n, N, D, x, D, 0, tg.X, D, 0, E, N, 0, 1, st);
    if (e == cudaSuccess) {
      if (what == 0) {
        k_tgt_blr_logp<<<gw, 256, 0, st>>>(E, tg.y, x, n, N, D, tg.prior_precision, out);
      } else if (what == 1) {  // (y - p) X - prec x
        k_tgt_blr_map<<<egrid(n * N), 256, 0, st>>>(E, tg.y, nullptr, n * N, N, 1);
        e = gemm_rm<double, double, double>(false, (int)n, D, N, E, N, 0, tg.X, D, 0, out, D, 0, 1, st);
        if (e == cudaSuccess) k_tgt_axpy<<<egrid(n * D), 256, 0, st>>>(out, out, x, n * D, 1.0, tg.prior_precision);
      } else {  // -((p (1 - p)) . (v X^T)) X - prec v
        e = gemm_rm<double, double, double>(true, (int)n, N, D, v, D, 0, tg.X, D, 0, Tm, N, 0, 1, st);
        if (e == cudaSuccess) {
          k_tgt_blr_map<<<egrid(n * N), 256, 0, st>>>(E, nullptr, Tm, n * N, N, 2);
          e = gemm_rm<double, double, double>(false, (int)n, D, N, Tm, N, 0, tg.X, D, 0, out, D, 0, 1, st);
          if (e == cudaSuccess)
            k_tgt_axpy<<<egrid(n * D), 256, 0, st>>>(out, out, v, n * D, -1.0, tg.prior_precision);
        }
      }
    }
    cudaFreeAsync(E, st);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
  }
  if (tg.kind == CS_TARGET_GAUSSIAN) {
    double *W = nullptr;
    cudaError_t e = scratch_alloc((void **)&W, sizeof(double) * (size_t)n * D * 2, st);
    if (e != cudaSuccess) return e;
    double *Z = W, *H = W + (size_t)n * D;
    if (what == 2) {  // -(v P)
      e = gemm_rm<double, double, double>(false, (int)n, D, D, v, D, 0, tg.prec, D, 0, H, D, 0, 1, st);
      if (e == cudaSuccess) k_tgt_axpy<<<egrid(n * D), 256, 0, st>>>(out, H, nullptr, n * D, -1.0, 0.0);
    } else {
      k_tgt_diff<<<egrid(n * D), 256, 0, st>>>(x, tg.mu, n, D, Z);
      if (what == 1) {  // -((x - mu) P)
        e = gemm_rm<double, double, double>(false, (int)n, D, D, Z, D, 0, tg.prec, D, 0, H, D, 0, 1, st);
        if (e == cudaSuccess) k_tgt_axpy<<<egrid(n * D), 256, 0, st>>>(out, H, nullptr, n * D, -1.0, 0.0);
      } else {  // -|(x - mu) L|^2 / 2
        e = gemm_rm<double, double, double>(false, (int)n, D, D, Z, D, 0, tg.chol, D, 0, H, D, 0, 1, st);
        if (e == cudaSuccess) k_tgt_halfsq<<<gw, 256, 0, st>>>(H, n, D, out);
      }
    }
    cudaFreeAsync(W, st);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
  }
  return cudaErrorNotSupported;
}

cudaError_t debug_pair_gram(const double *X, int N, int D, const double *W, int64_t T, float *H, cudaStream_t st) {
  const int nkb = (N + 31) / 32, npairs = D * (D + 1) / 2;
  const int64_t Tpad = (T + 127) / 128 * 128, ldp = (int64_t)(npairs + 127) / 128 * 128;
  if (T == 0) return cudaSuccess;
  float *buf = nullptr;
  const size_t nf = (size_t)(Tpad * 32 * nkb + ldp * 32 * nkb + Tpad * ldp);
  cudaError_t e = scratch_alloc((void **)&buf, sizeof(float) * nf, st);
  if (e != cudaSuccess) return e;
  cudaMemsetAsync(buf, 0, sizeof(float) * Tpad * 32 * nkb, st);
  float *Wt = buf, *Qt = Wt + Tpad * 32 * nkb, *Hp = Qt + ldp * 32 * nkb;
  k_w_tiles<<<148 * 8, 256, 0, st>>>(W, T, N, nkb, Wt);
  k_pair_operand<<<148 * 8, 256, 0, st>>>(X, N, D, nkb, npairs, ldp * 32 * nkb, Qt);
  const size_t smem = 1024 + (size_t)kPgStages * 2 * kUmmaTile * sizeof(float);
  cudaFuncSetAttribute(k_pair_gram, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_pair_gram<<<dim3((unsigned)(ldp / 128), (unsigned)(Tpad / 128)), 128, smem, st>>>(Wt, Qt, nkb, Hp, ldp);
  k_pair_unpack<<<148 * 8, 256, 0, st>>>(Hp, ldp, T, D, H);
  e = cudaGetLastError();
  cudaFreeAsync(buf, st);
  return e;
}

cudaError_t elements_blr(const cs_system &sys, const cs_deer_config &cfg, int dtype, int64_t iteration,
                         const void *s0, const void *guess, void *e0, void *u, cs_elem_stats *stats,
                         cudaStream_t st) {
  if (cfg.mode == CS_MODE_DENSE) {
    if (dtype == CS_F64)
      return blr_dense_run<double>(sys, cfg, iteration, (const double *)s0, (const double *)guess, (double *)e0,
                                   (double *)u, stats, st);
    return blr_dense_run<float>(sys, cfg, iteration, (const float *)s0, (const float *)guess, (float *)e0,
                                (float *)u, stats, st);
  }
  // diag: the fused DMMA builder (cs_blr_fused.cu); more than 7 probes per step
  // take the GEMM pipeline below
  if (blr_fused_ok(sys, cfg))
    return elements_blr_fused(sys, cfg, dtype, iteration, 0, sys.T, s0, guess, e0, u, stats, st);
  if (dtype == CS_F64)
    return blr_run<double>(sys, cfg, iteration, (const double *)s0, (const double *)guess, (double *)e0,
                           (double *)u, stats, st);
  return blr_run<float>(sys, cfg, iteration, (const float *)s0, (const float *)guess, (float *)e0, (float *)u,
                        stats, st);
}

}  // namespace cs
