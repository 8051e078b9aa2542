// Fused MALA element builder for the Bayesian logistic-regression target, diag
// quasi-Newton (BASELINE config 3: T = 100K steps, D = 100, N = 1000 rows).
//
// ONE kernel per Newton update builds f_t and the Hutchinson diagonal of every
// step (samplers.py:95-145, targets.py:254-287, deer.py:171-183).  A CTA owns
// TS consecutive steps; its Q tile holds their states S and their K probe rows
// z_k (TS * (1 + K) <= 64 rows, D <= 104 columns, f64).  Two passes:
//
//   pass 1  Q = [S; z]        for each 64-row tile of X (staged by cp.async,
//                             double-buffered):
//                               E = Q X_tile^T                 (DMMA, f64)
//                               P = [y - sigma(E_S); w . E_z]  (in smem, w = p(1-p))
//                               G += P X_tile                  (DMMA, f64)
//                             with the log-density row sums eta.y and
//                             sum logaddexp(0, eta) kept per step;
//           propose           g(S) = G_S - prec S,  x~ = S + eps g + sqrt(2 eps) xi,
//                             dx~_k = z_k + eps hvp(S, z_k) -> Q = [x~; dx~]
//   pass 2  the same tiles at x~ -> g(x~), hvp(x~, dx~), logp(x~)
//   final   gate, the tangents through it, est = mean_k z_k . J z_k, the element
//           (preconditioner, damping, clip), u = f - d prev, finite / Picard flags.
//
// The T x N logit matrices never leave the SM (the previous realisation wrote
// and re-read them through HBM around four cuBLAS DGEMMs); X (N x D, 800 KB)
// stays L2-resident.  The f64 products run on the FP64 tensor cores as
// mma.sync m8n8k4 (DMMA): the contractions are the reference's f64 matmuls, in a
// fixed order, so a solve is reproducible bit for bit.
//
// The kernel also takes a step range (t0, n) with the state before it (the halo
// row), so a T-sharded solve builds its shard's elements.
#include "cs_apikern.cuh"

namespace cs {

namespace {

constexpr int kFR = 64;    // rows of the Q tile: TS steps x (1 + K) row groups
constexpr int kFN = 32;    // data rows per staged X tile
constexpr int kFDP = 104;  // D padded to the DMMA grid (13 n8 tiles; D <= 104)
constexpr int kFLD = 108;  // smem stride of Q / X rows: conflict-free DMMA fragments
constexpr int kFPL = 36;   // smem stride of P rows
constexpr int kFGrp = 256; // threads per role group
constexpr int kFThr = 2 * kFGrp;
constexpr int kFXBuf = 2;  // X tiles per group (double buffer)
constexpr int kFMaxK = 7;
constexpr int kFNT = kFDP / 8;  // 13 column tiles

// per-step scalars kept in shared memory
struct StepScal {
  double aS[kFR], bS[kFR], aX[kFR], bX[kFR];  // eta.y and sum logaddexp, at S and at x~
  double ssS[kFR], sxi[kFR], sxX[kFR];
  double s2[kFMaxK][kFR];  // g(S) . z_k
  double gate[kFR], sp[kFR], neg[kFR];
  int flags[kFR];  // bit 0: non-finite proposal, 1: non-finite f, 2: Picard fail, 3: non-finite Jacobian
};

constexpr size_t kFQ = (size_t)kFR * kFLD, kFX = (size_t)kFN * kFLD, kFP = (size_t)kFR * kFPL;
constexpr size_t kFSmem = sizeof(double) * (kFQ + 2 * kFXBuf * kFX + 2 * kFP) + sizeof(StepScal);

CS_D void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

CS_D void cp_async8(void *dst, const void *src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(valid ? 8 : 0)
               : "memory");
}
CS_D void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> CS_D void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// named barrier of one warp group (ids 1, 2)
CS_D void bar_group(int g) { asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "n"(kFGrp) : "memory"); }

// X rows [n0, n0 + kFN) into a staging tile (zero beyond N and D), one group
CS_D void stage_x(double *Xs, const double *X, int n0, int N, int D, int gtid) {
  for (int i = gtid; i < kFN * kFDP; i += kFGrp) {
    const int r = i / kFDP, d = i - r * kFDP;
    const int n = n0 + r;
    const bool ok = n < N && d < D;
    cp_async8(Xs + r * kFLD + d, X + (ok ? (size_t)n * D + d : 0), ok);
  }
  cp_async_commit();
}

// One pass over the data.  Two warp groups of 8 take alternate X tiles
// (ping-pong): each stages its tiles (cp.async, double-buffered), forms
//   E = Q X_tile^T (DMMA), P = [y - sigmoid(E_S); w . E_z] in its own smem
//   tile, G_grp += P X_tile (DMMA; warp w owns rows 8w..8w+7, 13 column tiles)
// so one group's transcendental epilogue runs while the other's products keep
// the FP64 tensor pipe busy.  The two partial sums are added in a fixed order
// (even tiles + odd tiles) into group 0's registers, which return G; the
// log-density row sums of the state rows land in a_out / b_out.
CS_D void blr_pass(const double *Qs, double *Xs, double *Ps, const double *X, const double *y, int N, int D,
                   int TS, int K, double (&acc)[kFNT][2], double *a_out, double *b_out) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grp = warp >> 3, gw = warp & 7, gtid = tid & (kFGrp - 1);
  const int ntiles = (N + kFN - 1) / kFN;
  double *Xg = Xs + (size_t)grp * kFXBuf * kFX;
  double *Pg = Ps + (size_t)grp * kFP;
  const int wr = gw >> 1, wc = gw & 1;  // GEMM 1 warp grid: 4 x 2 of 16 x 16
  double ra[4], rb[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) ra[q] = rb[q] = 0.0;
#pragma unroll
  for (int jt = 0; jt < kFNT; ++jt) acc[jt][0] = acc[jt][1] = 0.0;
  if (grp < ntiles) stage_x(Xg, X, grp * kFN, N, D, gtid);
  for (int j = grp, it = 0; j < ntiles; j += 2, ++it) {
    const double *Xc = Xg + (size_t)(it & 1) * kFX;
    cp_async_wait<0>();
    bar_group(grp);  // X(j) visible to the group; the other buffer's last reader (tile j-2) is done
    if (j + 2 < ntiles) stage_x(Xg + (size_t)((it + 1) & 1) * kFX, X, (j + 2) * kFN, N, D, gtid);
    {
      double c1[2][2][2];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) c1[mi][ni][0] = c1[mi][ni][1] = 0.0;
      const double *qa = Qs + (size_t)(wr * 16 + (lane >> 2)) * kFLD + (lane & 3);
      const double *xb = Xc + (size_t)(wc * 16 + (lane >> 2)) * kFLD + (lane & 3);
#pragma unroll 2
      for (int d0 = 0; d0 < kFDP; d0 += 4) {
        double a[2], b[2];
#pragma unroll
        for (int mi = 0; mi < 2; ++mi) a[mi] = qa[mi * 8 * kFLD + d0];
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) b[ni] = xb[ni * 8 * kFLD + d0];
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int ni = 0; ni < 2; ++ni) dmma(c1[mi][ni], a[mi], b[ni]);
      }
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) {
          double *p = Pg + (size_t)(wr * 16 + mi * 8 + (lane >> 2)) * kFPL + wc * 16 + ni * 8 + 2 * (lane & 3);
          p[0] = c1[mi][ni][0];
          p[1] = c1[mi][ni][1];
        }
    }
    bar_group(grp);
    // p = sigmoid(eta), P_S = y - p, P_z *= w = p (1 - p); row sums.  Thread:
    // column lane of the tile, steps gw, gw + 8, gw + 16, gw + 24
    {
      const int n = j * kFN + lane;
      const bool ok = n < N;
      const double yn = ok ? __ldg(y + n) : 0.0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int s = gw + 8 * q;
        if (s >= TS) break;
        double *ps = Pg + (size_t)s * kFPL + lane;
        if (!ok) {
          *ps = 0.0;
          for (int k = 0; k < K; ++k) ps[(size_t)(k + 1) * TS * kFPL] = 0.0;
          continue;
        }
        const double eta = *ps;
        double p, lae;
        sigmoid_logaddexp(eta, p, lae);  // expit, logaddexp(0, eta)
        ra[q] += eta * yn;
        rb[q] += lae;
        *ps = yn - p;
        const double w = p * (1.0 - p);
        for (int k = 0; k < K; ++k) ps[(size_t)(k + 1) * TS * kFPL] *= w;
      }
    }
    bar_group(grp);
    {
      const double *pa = Pg + (size_t)(gw * 8 + (lane >> 2)) * kFPL + (lane & 3);
      const double *xb = Xc + (size_t)(lane & 3) * kFLD + (lane >> 2);
#pragma unroll 2
      for (int k0 = 0; k0 < kFN; k0 += 4) {
        const double a = pa[k0];
#pragma unroll
        for (int jt = 0; jt < kFNT; ++jt) dmma(acc[jt], a, xb[(size_t)k0 * kFLD + jt * 8]);
      }
    }
  }
  // combine: group 1's partial products and row sums go through smem (the X
  // tiles are free), group 0 adds them in a fixed order
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    ra[q] = warp_sum(ra[q]);
    rb[q] = warp_sum(rb[q]);
  }
  __syncthreads();
  double *xch = Xs;  // kFR x kFDP partial G + 2 x 32 row sums
  double *rsx = Xs + (size_t)kFR * kFDP;
  if (grp == 1) {
#pragma unroll
    for (int jt = 0; jt < kFNT; ++jt) {
      double *p = xch + (size_t)(gw * 8 + (lane >> 2)) * kFDP + jt * 8 + 2 * (lane & 3);
      p[0] = acc[jt][0];
      p[1] = acc[jt][1];
    }
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        rsx[2 * (gw + 8 * q)] = ra[q];
        rsx[2 * (gw + 8 * q) + 1] = rb[q];
      }
  }
  __syncthreads();
  if (grp == 0) {
#pragma unroll
    for (int jt = 0; jt < kFNT; ++jt) {
      const double *p = xch + (size_t)(gw * 8 + (lane >> 2)) * kFDP + jt * 8 + 2 * (lane & 3);
      acc[jt][0] += p[0];
      acc[jt][1] += p[1];
    }
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int s = gw + 8 * q;
        if (s < TS) {
          a_out[s] = ra[q] + rsx[2 * s];
          b_out[s] = rb[q] + rsx[2 * s + 1];
        }
      }
  }
  __syncthreads();
}

template <typename ST>
__global__ void __launch_bounds__(kFThr, 1)
k_blr_fused(cs_system sys, cs_deer_config cfg, int64_t iteration, int64_t t0, int64_t n, const ST *s0,
            const ST *guess, ST *jout, ST *uout, cs_elem_stats *stats) {
  extern __shared__ __align__(16) double fsm[];
  double *Qs = fsm;                  // kFR x kFLD
  double *Xs = Qs + kFQ;             // 2 groups x kFXBuf x kFN x kFLD
  double *Ps = Xs + 2 * kFXBuf * kFX;  // 2 groups x kFR x kFPL
  StepScal &sc = *(StepScal *)(Ps + 2 * kFP);
  const int D = sys.dim, N = (int)sys.target.n_data;
  const int K = cfg.hutchinson_samples;
  const int TS = kFR / (1 + K);
  const double prec = sys.target.prior_precision, eps = sys.eps, sq = sqrt(2.0 * eps);
  const double *X = sys.target.X, *y = sys.target.y;
  const ST *xi = (const ST *)sys.noise_vec;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t pre = probe_prefix(sys.seed, iteration);
  long long bp = kNoStep, bf = kNoStep, bj = kNoStep;
  unsigned pf = 0;
  const bool do_clip = isfinite(cfg.clip);

  for (int64_t r0 = (int64_t)blockIdx.x * TS; r0 < n; r0 += (int64_t)gridDim.x * TS) {
    const int ts = (int)(n - r0 < TS ? n - r0 : TS);  // steps of this tile
    // ---- Q = [S; z_1 .. z_K] (rows beyond the tile's steps and columns beyond D: 0)
    for (int i = tid; i < kFR * kFDP; i += kFThr) {
      const int row = i / kFDP, d = i - row * kFDP;
      const int g = row / TS, s = row - g * TS;
      double v = 0.0;
      if (g <= K && s < ts && d < D) {
        const int64_t r = r0 + s;
        if (g == 0) v = (double)(r == 0 ? s0[d] : guess[(r - 1) * D + d]);
        else v = probe_sign(hash_t(pre, (uint64_t)(t0 + r + 1)), g - 1, d);
      }
      Qs[(size_t)row * kFLD + d] = v;
    }
    if (tid < kFR) sc.flags[tid] = 0;
    __syncthreads();

    double acc[kFNT][2];
    blr_pass(Qs, Xs, Ps, X, y, N, D, TS, K, acc, sc.aS, sc.bS);

    // ---- propose: warp w holds rows 8w + lane/4, columns 8j + 2(lane%4) + e
    {
      const int row = warp * 8 + (lane >> 2);
      const int g = row / TS, s = row - g * TS;
      const bool live = g <= K && s < ts;
      double *gS = Ps;  // g(S) rows (TS x kFLD) for the probe rows' s2 = g(S).z
      double ss = 0.0, sx = 0.0, sxx = 0.0;
      bool fin = true;
      if (live && g == 0) {
        const int64_t t = t0 + r0 + s + 1;
#pragma unroll
        for (int j = 0; j < kFNT; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int d = j * 8 + 2 * (lane & 3) + e;
            if (d >= D) continue;
            double *q = Qs + (size_t)row * kFLD + d;
            const double S = *q;
            const double gr = acc[j][e] - prec * S;  // (y - p) X - prec beta
            gS[(size_t)s * kFLD + d] = gr;
            const double z = (double)xi[t * D + d];
            const double xp = (S + eps * gr) + sq * z;  // samplers.py:206
            fin &= isfinite(xp);
            ss += S * S;
            sx += z * z;
            sxx += xp * xp;
            *q = xp;
          }
      }
      ss += __shfl_xor_sync(0xffffffffu, ss, 1);
      ss += __shfl_xor_sync(0xffffffffu, ss, 2);
      sx += __shfl_xor_sync(0xffffffffu, sx, 1);
      sx += __shfl_xor_sync(0xffffffffu, sx, 2);
      sxx += __shfl_xor_sync(0xffffffffu, sxx, 1);
      sxx += __shfl_xor_sync(0xffffffffu, sxx, 2);
      {
        const int f1 = __shfl_xor_sync(0xffffffffu, (int)fin, 1);
        const int f2 = __shfl_xor_sync(0xffffffffu, (int)fin, 2);
        fin = fin && f1 && f2;
      }
      if (live && g == 0 && (lane & 3) == 0) {
        sc.ssS[s] = ss;
        sc.sxi[s] = sx;
        sc.sxX[s] = sxx;
        if (!fin) sc.flags[s] |= 1;
      }
      __syncthreads();  // g(S) rows complete
      double s2 = 0.0;
      if (live && g > 0) {
#pragma unroll
        for (int j = 0; j < kFNT; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int d = j * 8 + 2 * (lane & 3) + e;
            if (d >= D) continue;
            double *q = Qs + (size_t)row * kFLD + d;
            const double z = *q;
            s2 += gS[(size_t)s * kFLD + d] * z;
            const double hv = -acc[j][e] - prec * z;  // hvp(S, z) = -(w . zX^T) X - prec z
            *q = z + eps * hv;                        // dx~ = z + eps hvp
          }
      }
      s2 += __shfl_xor_sync(0xffffffffu, s2, 1);
      s2 += __shfl_xor_sync(0xffffffffu, s2, 2);
      if (live && g > 0 && (lane & 3) == 0) sc.s2[g - 1][s] = s2;
      __syncthreads();
    }

    blr_pass(Qs, Xs, Ps, X, y, N, D, TS, K, acc, sc.aX, sc.bX);

    // ---- final: state rows first (g(x~), r, |r|^2, gate), then the probe rows
    double *GXs = Xs;                          // g(x~) rows   TS x kFLD
    double *RBs = Xs + (size_t)TS * kFLD;      // r rows       TS x kFLD
    double *ESTs = RBs + (size_t)TS * kFLD;    // z . J z      K x TS x kFDP (fits: (2 + K) TS <= 3 x 64)
    {
      const int row = warp * 8 + (lane >> 2);
      const int g = row / TS, s = row - g * TS;
      const bool live = g <= K && s < ts;
      double srb = 0.0;
      if (live && g == 0) {
        const int64_t r = r0 + s;
        const ST *pr = r == 0 ? s0 : guess + (r - 1) * D;
#pragma unroll
        for (int j = 0; j < kFNT; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int d = j * 8 + 2 * (lane & 3) + e;
            if (d >= D) continue;
            const double xp = Qs[(size_t)row * kFLD + d];
            const double gp = acc[j][e] - prec * xp;
            const double rbv = ((double)pr[d] - xp) - eps * gp;
            GXs[(size_t)s * kFLD + d] = gp;
            RBs[(size_t)s * kFLD + d] = rbv;
            srb += rbv * rbv;
          }
      }
      srb += __shfl_xor_sync(0xffffffffu, srb, 1);
      srb += __shfl_xor_sync(0xffffffffu, srb, 2);
      if (live && g == 0 && (lane & 3) == 0) {
        const int64_t t = t0 + r0 + s + 1;
        // logp = eta.y - sum logaddexp(0, eta) - prec/2 |beta|^2   (targets.py:254-270)
        const double lpX = (sc.aX[s] - sc.bX[s]) - 0.5 * prec * sc.sxX[s];
        const double lpS = (sc.aS[s] - sc.bS[s]) - 0.5 * prec * sc.ssS[s];
        const double delta = lpX - lpS - srb / (4.0 * eps) + 0.5 * sc.sxi[s];
        const double margin = fmin(0.0, delta) - __ldg(sys.noise_logu + t);
        sc.gate[s] = margin > 0.0 ? 1.0 : 0.0;
        sc.sp[s] = sigmoid_prime(margin);
        sc.neg[s] = delta < 0.0 ? 1.0 : 0.0;
      }
      __syncthreads();
      double s1 = 0.0, s3 = 0.0;
      if (live && g > 0) {
#pragma unroll
        for (int j = 0; j < kFNT; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int d = j * 8 + 2 * (lane & 3) + e;
            if (d >= D) continue;
            const double dx = Qs[(size_t)row * kFLD + d];
            const double z = probe_sign(hash_t(pre, (uint64_t)(t0 + r0 + s + 1)), g - 1, d);
            const double hv = -acc[j][e] - prec * dx;  // hvp(x~, dx~)
            const double dr = (z - dx) - eps * hv;
            s1 += GXs[(size_t)s * kFLD + d] * dx;
            s3 += RBs[(size_t)s * kFLD + d] * dr;
          }
      }
      s1 += __shfl_xor_sync(0xffffffffu, s1, 1);
      s1 += __shfl_xor_sync(0xffffffffu, s1, 2);
      s3 += __shfl_xor_sync(0xffffffffu, s3, 1);
      s3 += __shfl_xor_sync(0xffffffffu, s3, 2);
      if (live && g > 0) {
        const int64_t r = r0 + s;
        const ST *pr = r == 0 ? s0 : guess + (r - 1) * D;
        const double ddelta = (s1 - sc.s2[g - 1][s]) - s3 / (2.0 * eps);
        const double bend = sc.sp[s] * (ddelta * sc.neg[s]);
        const double gate = sc.gate[s];
        const uint64_t h3 = hash_t(pre, (uint64_t)(t0 + r + 1));
#pragma unroll
        for (int j = 0; j < kFNT; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int d = j * 8 + 2 * (lane & 3) + e;
            if (d >= D) continue;
            const double dx = Qs[(size_t)row * kFLD + d];
            const double z = probe_sign(h3, g - 1, d);
            const double xp = Qs[(size_t)s * kFLD + d];
            const double jz = (gate * dx + (1.0 - gate) * z) + (xp - (double)pr[d]) * bend;
            ESTs[((size_t)(g - 1) * TS + s) * kFDP + d] = z * jz;
          }
      }
      __syncthreads();
    }
    // ---- elements: est = mean_k z_k J z_k (probes in order), precond, damping, clip
    for (int i = tid; i < ts * D; i += kFThr) {
      const int s = i / D, d = i - s * D;
      const int64_t r = r0 + s;
      const int64_t t = t0 + r + 1;
      const ST *pr = r == 0 ? s0 : guess + (r - 1) * D;
      const double S = (double)pr[d];
      const double f = sc.gate[s] > 0.0 ? Qs[(size_t)s * kFLD + d] : S;
      double est = 0.0;
      for (int k = 0; k < K; ++k) est += ESTs[((size_t)k * TS + s) * kFDP + d];
      double v = est / (double)K;
      int fl = 0;
      if (!isfinite(f)) fl |= 2;
      if (!(fabs(f - (double)guess[r * D + d]) <= cfg.atol + cfg.rtol * fabs(f))) fl |= 4;
      if (!isfinite(v)) fl |= 8;
      if (cfg.preconditioner) v = v * __ldg(cfg.preconditioner + d);
      v = v * cfg.damping;
      if (do_clip) v = clipv(v, cfg.clip);
      jout[r * D + d] = (ST)v;
      uout[r * D + d] = (ST)(f - v * S);
      if (fl) atomicOr(&sc.flags[s], fl);
      (void)t;
    }
    __syncthreads();
    if (tid < ts) {
      const int fl = sc.flags[tid];
      const long long t = (long long)(t0 + r0 + tid + 1);
      if (fl & 1) bp = min(bp, t);
      if (fl & 2) bf = min(bf, t);
      if (fl & 8) bj = min(bj, t);
      if (fl & 4) ++pf;
    }
    __syncthreads();
  }
  if (warp < (kFR + 31) / 32) {  // the threads that saw per-step flags
    bp = warp_min_nn64(bp);
    bf = warp_min_nn64(bf);
    bj = warp_min_nn64(bj);
    pf = warp_sum_u32(pf);
    if (lane == 0) {
      if (bp != kNoStep) atomicMin((long long *)&stats->bad_proposal, bp);
      if (bf != kNoStep) atomicMin((long long *)&stats->bad_step, bf);
      if (bj != kNoStep) atomicMin((long long *)&stats->bad_jacobian, bj);
      if (pf) atomicAdd(&stats->picard_fail, pf);
    }
  }
}

// ---------------------------------------------------------------------------
// sequential_evaluate (core.py:163-184) for BLR MALA: one CTA walks the chain
// in order, f64.  The state's logits, gradient and log density are carried from
// step to step (the next state is either the proposal or the state itself), so
// each step evaluates the target once, at the proposal: eta = X x~ (a warp per
// data row, lanes across D), p = sigmoid(eta), g = (y - p) X - prec x~ (a thread
// per column over a slice of the rows, slices summed in order), the MALA gate
// (samplers.py:95-122).  X (800 KB at cfg 3) is read from L2 every step.
constexpr int kSeqThr = 1024;
constexpr int kSeqMaxN = 4096;

CS_D double seq_eval(const double *X, const double *y, int N, int D, double prec, const double *xs, double *eta,
                     double *P, double *part, double *g, double *red) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = kSeqThr / 32;
  // eta_n = X[n] . x  and the log-density terms eta.y, logaddexp(0, eta)
  double a = 0.0, b = 0.0;
  for (int n = warp; n < N; n += nw) {
    double e = 0.0;
    for (int d = lane; d < D; d += 32) e += __ldg(X + (size_t)n * D + d) * xs[d];
    e = warp_sum(e);
    if (lane == 0) {
      const double em = exp(-e), p = 1.0 / (1.0 + em), yn = __ldg(y + n);
      eta[n] = e;
      P[n] = yn - p;
      a += e * yn;
      b += e != e ? e : fmax(e, 0.0) + log1p(e >= 0.0 ? em : exp(e));
    }
  }
  if (lane == 0) {
    red[2 * warp] = a;
    red[2 * warp + 1] = b;
  }
  __syncthreads();
  // g_d = sum_n P_n X[n][d] - prec x_d: column d, rows split into kSeqThr / 128 slices
  const int ns = kSeqThr / 128, d = tid & 127, sl = tid >> 7;
  if (d < D) {
    double acc = 0.0;
    const int n0 = sl * ((N + ns - 1) / ns), n1 = min(N, n0 + (N + ns - 1) / ns);
#pragma unroll 4
    for (int n = n0; n < n1; ++n) acc += P[n] * __ldg(X + (size_t)n * D + d);
    part[sl * 128 + d] = acc;
  }
  __syncthreads();
  double lp = 0.0;
  if (tid < D) {
    double acc = 0.0;
    for (int q = 0; q < ns; ++q) acc += part[q * 128 + tid];
    g[tid] = acc - prec * xs[tid];
  }
  if (tid == 0) {
    double aa = 0.0, bb = 0.0, ss = 0.0;
    for (int w = 0; w < nw; ++w) {
      aa += red[2 * w];
      bb += red[2 * w + 1];
    }
    for (int k = 0; k < D; ++k) ss += xs[k] * xs[k];
    red[2 * nw] = (aa - bb) - 0.5 * prec * ss;  // logp = eta.y - sum logaddexp - prec/2 |x|^2
  }
  __syncthreads();
  lp = red[2 * nw];
  return lp;
}

template <typename ST>
__global__ void __launch_bounds__(kSeqThr, 1)
k_blr_sequential(cs_system sys, const ST *s0, int64_t T, ST *out, long long *bad) {
  __shared__ double xs[128], xp[128], gS[128], gX[128], part[kSeqThr], red[2 * (kSeqThr / 32) + 2];
  __shared__ int s_bad;
  extern __shared__ double seq_dyn[];  // eta[N], P[N]
  const int D = sys.dim, N = (int)sys.target.n_data;
  const double prec = sys.target.prior_precision, eps = sys.eps, sq = sqrt(2.0 * eps);
  const double *X = sys.target.X, *y = sys.target.y;
  const ST *xi = (const ST *)sys.noise_vec;
  double *eta = seq_dyn, *P = seq_dyn + N;
  const int tid = threadIdx.x;
  if (tid < D) xs[tid] = (double)s0[tid];
  if (tid == 0) s_bad = 0;
  __syncthreads();
  double lpS = seq_eval(X, y, N, D, prec, xs, eta, P, part, gS, red);
  for (int64_t t = 1; t <= T; ++t) {
    // proposal x~ = S + eps g(S) + sqrt(2 eps) xi_t  (samplers.py:206)
    if (tid < D) {
      const double xv = (xs[tid] + eps * gS[tid]) + sq * (double)xi[t * D + tid];
      xp[tid] = xv;
      if (!isfinite(xv)) s_bad = 1;
    }
    __syncthreads();
    if (s_bad) {
      if (tid == 0) *bad = t;
      return;
    }
    const double lpX = seq_eval(X, y, N, D, prec, xp, eta, P, part, gX, red);
    // gate: delta = logp(x~) - logp(S) - |r|^2/(4 eps) + |xi|^2/2, r = S - x~ - eps g(x~)
    if (tid == 0) {
      double srb = 0.0, sxi = 0.0;
      for (int k = 0; k < D; ++k) {
        const double r = (xs[k] - xp[k]) - eps * gX[k];
        const double z = (double)xi[t * D + k];
        srb += r * r;
        sxi += z * z;
      }
      const double delta = lpX - lpS - srb / (4.0 * eps) + 0.5 * sxi;
      const double margin = fmin(0.0, delta) - __ldg(sys.noise_logu + t);
      red[2 * (kSeqThr / 32) + 1] = margin > 0.0 ? 1.0 : 0.0;
    }
    __syncthreads();
    const bool acc = red[2 * (kSeqThr / 32) + 1] > 0.0;
    if (acc) {
      if (tid < D) {
        xs[tid] = xp[tid];
        gS[tid] = gX[tid];
      }
      lpS = lpX;
    }
    __syncthreads();
    if (tid < D) out[(t - 1) * D + tid] = (ST)xs[tid];  // the walk itself stays f64 (as k_sys_seq)
    __syncthreads();
  }
}

}  // namespace

bool blr_fused_ok(const cs_system &s, const cs_deer_config &cfg) {
  return cfg.mode == CS_MODE_DIAG && s.dim <= kFDP && cfg.hutchinson_samples >= 1 &&
         cfg.hutchinson_samples <= kFMaxK;
}

cudaError_t elements_blr_fused(const cs_system &sys, const cs_deer_config &cfg, int dtype, int64_t iteration,
                               int64_t t0, int64_t n, const void *s0, const void *guess, void *j, void *u,
                               cs_elem_stats *stats, cudaStream_t st) {
  if (n < 1) return cudaSuccess;
  const int TS = kFR / (1 + cfg.hutchinson_samples);
  const int64_t tiles = (n + TS - 1) / TS;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = (unsigned)(tiles < (int64_t)sms * 64 ? tiles : (int64_t)sms * 64);
  if (dtype == CS_F64) {
    auto k = k_blr_fused<double>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFSmem);
    if (e != cudaSuccess) return e;
    k<<<grid, kFThr, kFSmem, st>>>(sys, cfg, iteration, t0, n, (const double *)s0, (const double *)guess,
                                   (double *)j, (double *)u, stats);
  } else {
    auto k = k_blr_fused<float>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFSmem);
    if (e != cudaSuccess) return e;
    k<<<grid, kFThr, kFSmem, st>>>(sys, cfg, iteration, t0, n, (const float *)s0, (const float *)guess,
                                   (float *)j, (float *)u, stats);
  }
  return cudaGetLastError();
}

}  // namespace cs

namespace cs {

cudaError_t blr_sequential(const cs_system &sys, int dtype, const void *s0, int64_t T, void *out, long long *bad,
                           cudaStream_t st) {
  const int N = (int)sys.target.n_data;
  if (sys.dim > 128 || N > kSeqMaxN) return cudaErrorNotSupported;
  const size_t smem = sizeof(double) * 2 * (size_t)N;
  if (dtype == CS_F64) {
    cudaFuncSetAttribute(k_blr_sequential<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_blr_sequential<double><<<1, kSeqThr, smem, st>>>(sys, (const double *)s0, T, (double *)out, bad);
  } else {
    cudaFuncSetAttribute(k_blr_sequential<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_blr_sequential<float><<<1, kSeqThr, smem, st>>>(sys, (const float *)s0, T, (float *)out, bad);
  }
  return cudaGetLastError();
}

}  // namespace cs
