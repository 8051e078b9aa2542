// Row-major strided-batched GEMM on the FP64 tensor cores (DMMA, mma.sync
// m8n8k4 f64), the library's one dense-product building block:
//
//   C[b] (M x N, ldc) = A[b] (M x K, lda) . op(B[b])
//   op(B) = B (K x N, ldb)            BT = false
//         = B^T with B given N x K    BT = true   (e.g. X^T of a data matrix X)
//
// Inputs are f32 or f64 and are widened to f64 on their way into shared
// memory; accumulation is f64, the result is rounded once to C's type.  Tiles:
// BM x 64 outputs per CTA -- BM = 128: 8 warps of 32 x 32 (4 x 4 DMMA tiles);
// BM = 64 / 32: 16 / 8 warps of 16 x 16 for smaller problems; K in steps of 16, the next step's operands
// loaded into registers while the current one is multiplied (double-buffered
// shared memory).  Strides of the staged tiles are chosen so every DMMA
// fragment load is bank-conflict free.  The summation order is fixed (k
// ascending per output), so results are reproducible bit for bit.
//
// Used by the wide leapfrog builder (A . P, cfg 4), the dense logistic-
// regression builder ([S; z] X^T and P X, cfg 3 "full") and the dense affine
// aggregates / D > 128 dense scans (products of augmented maps).
#pragma once
#include <cstdlib>
#include <type_traits>

#include "cs_common.cuh"

namespace cs {

// Optional fused epilogue on the C tile (mode 0: plain store):
//   1 logistic: eta = the product; C <- y[col] - sigmoid(eta); weights
//     p (1 - p) to `wout` (f64, C's layout) and / or `wsw` (f32 tcgen05 operand
//     tiles, see swz_index in cs_blr.cu); per-row partial sums
//     (eta . y, sum logaddexp(0, eta)) over this warp's 32 columns to
//     part[row][npart] -- folded in a fixed order afterwards (deterministic)
//   2 scale: C <- product . S[row][col]
struct GemmEpi {
  int mode = 0;
  const double *y = nullptr;
  double *part = nullptr;
  int npart = 0;
  double *wout = nullptr;
  float *wsw = nullptr;
  int nkb = 0;
  const double *S = nullptr;
};

namespace gemm_detail {

constexpr int kBN = 64;
constexpr int kLDB = kBN + 4;  // 68 doubles: B fragments conflict free

CS_D void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <typename T>
CS_D double ldg_d(const T *p) {
  return (double)__ldg(p);
}

// BM = 32 / 64: 16 x 16 warp tiles (BM/16 x 4 warps); BM = 128: 32 x 32 warp
// tiles (4 x 2 warps), twice the DMMAs per fragment load for large products
template <int BM> struct GemmWarps {
  static constexpr int WT = BM == 128 ? 32 : 16;  // warp tile edge
  static constexpr int WN = kBN / WT;             // warps across N
  static constexpr int NT = (BM / WT) * WN * 32;  // threads
  static constexpr int MI = WT / 8;               // DMMA tiles per warp edge
  static constexpr int BK = BM == 128 ? 8 : 16;   // K per staged step (48 KB of static smem)
  static constexpr int LDA = BK + 4;              // 12 / 20 doubles: A fragments conflict free
};

template <int BM, bool BT, typename TA, typename TB, typename TC, int EPI = 0>
__global__ void __launch_bounds__(GemmWarps<BM>::NT)
k_gemm(int M, int N, int K, const TA *__restrict__ A, int64_t lda, int64_t sA, const TB *__restrict__ B,
       int64_t ldb, int64_t sB, TC *__restrict__ C, int64_t ldc, int64_t sC, GemmEpi ep = GemmEpi()) {
  using GW = GemmWarps<BM>;
  constexpr int kBK = GW::BK, kLDA = GW::LDA;
  constexpr int NT = GW::NT;                     // threads
  constexpr int MI = GW::MI;
  constexpr int EA = BM * kBK / NT;              // A elements per thread per K step
  constexpr int EB = kBK * kBN / NT;             // B elements per thread per K step
  __shared__ __align__(16) double As[2][BM * kLDA];
  __shared__ __align__(16) double Bs[2][kBK * kLDB];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / GW::WN, wn = warp % GW::WN;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * kBN;
  A += (int64_t)blockIdx.z * sA;
  B += (int64_t)blockIdx.z * sB;
  C += (int64_t)blockIdx.z * sC;
  double ra[EA], rb[EB];
  auto load = [&](int k0) {
#pragma unroll
    for (int e = 0; e < EA; ++e) {
      const int i = tid + e * NT, r = i / kBK, k = i % kBK;
      const int gm = m0 + r, gk = k0 + k;
      ra[e] = (gm < M && gk < K) ? ldg_d(A + (int64_t)gm * lda + gk) : 0.0;
    }
#pragma unroll
    for (int e = 0; e < EB; ++e) {
      const int i = tid + e * NT;
      if constexpr (BT) {  // B^T given N x K: walk k fastest (coalesced)
        const int n = i / kBK, k = i % kBK;
        const int gn = n0 + n, gk = k0 + k;
        rb[e] = (gn < N && gk < K) ? ldg_d(B + (int64_t)gn * ldb + gk) : 0.0;
      } else {
        const int k = i / kBN, n = i % kBN;
        const int gn = n0 + n, gk = k0 + k;
        rb[e] = (gn < N && gk < K) ? ldg_d(B + (int64_t)gk * ldb + gn) : 0.0;
      }
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int e = 0; e < EA; ++e) {
      const int i = tid + e * NT;
      As[buf][(i / kBK) * kLDA + i % kBK] = ra[e];
    }
#pragma unroll
    for (int e = 0; e < EB; ++e) {
      const int i = tid + e * NT;
      if constexpr (BT) Bs[buf][(i % kBK) * kLDB + i / kBK] = rb[e];
      else Bs[buf][(i / kBN) * kLDB + i % kBN] = rb[e];
    }
  };
  double c[MI][MI][2];
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < MI; ++ni) c[mi][ni][0] = c[mi][ni][1] = 0.0;
  const int nk = (K + kBK - 1) / kBK;
  load(0);
  store(0);
  __syncthreads();
  for (int s = 0; s < nk; ++s) {
    const int buf = s & 1;
    if (s + 1 < nk) load((s + 1) * kBK);  // in flight while this step multiplies
    const double *as = As[buf] + (wm * GW::WT + (lane >> 2)) * kLDA + (lane & 3);
    const double *bs = Bs[buf] + (lane & 3) * kLDB + wn * GW::WT + (lane >> 2);
#pragma unroll
    for (int k0 = 0; k0 < kBK; k0 += 4) {
      double av[MI], bv[MI];
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        av[i] = as[i * 8 * kLDA + k0];
        bv[i] = bs[k0 * kLDB + i * 8];
      }
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < MI; ++ni) dmma884(c[mi][ni], av[mi], bv[ni]);
    }
    if (s + 1 < nk) {
      store(buf ^ 1);  // the other buffer's last readers finished before the previous barrier
      __syncthreads();
    }
  }
  if constexpr (EPI == 0) {
#pragma unroll
    for (int mi = 0; mi < MI; ++mi)
#pragma unroll
      for (int ni = 0; ni < MI; ++ni) {
        const int gm = m0 + wm * GW::WT + mi * 8 + (lane >> 2);
        const int gn = n0 + wn * GW::WT + ni * 8 + 2 * (lane & 3);
        if (gm >= M) continue;
        if (gn < N) C[(int64_t)gm * ldc + gn] = (TC)c[mi][ni][0];
        if (gn + 1 < N) C[(int64_t)gm * ldc + gn + 1] = (TC)c[mi][ni][1];
      }
  } else {
#pragma unroll
    for (int mi = 0; mi < MI; ++mi) {
      const int gm = m0 + wm * GW::WT + mi * 8 + (lane >> 2);
      double pa = 0.0, pb = 0.0;
#pragma unroll
      for (int ni = 0; ni < MI; ++ni)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int gn = n0 + wn * GW::WT + ni * 8 + 2 * (lane & 3) + h;
          if (gm >= M || gn >= N) continue;
          const int64_t o = (int64_t)gm * ldc + gn;
          const double v = c[mi][ni][h];
          if constexpr (EPI == 1) {
            const double yn = __ldg(ep.y + gn);
            double p, lae;
            sigmoid_logaddexp(v, p, lae);  // expit, logaddexp(0, eta)
            pa += v * yn;
            pb += lae;
            C[o] = (TC)(yn - p);
            const double w = p * (1.0 - p);
            if (ep.wout) ep.wout[o] = w;
            if (ep.wsw) {
              const int rr = gm & 127, cc = (gn & 31) >> 2;
              ep.wsw[((((int64_t)gm >> 7) * ep.nkb + (gn >> 5)) * 128 + rr) * 32 + ((cc ^ (rr & 7)) << 2) + (gn & 3)] =
                  (float)w;
            }
          } else {
            C[o] = (TC)(v * ep.S[o]);
          }
        }
      if constexpr (EPI == 1) {
        // the 4 lanes of a row (lane & 3), then one partial per (row, warp column)
        pa += __shfl_xor_sync(0xffffffffu, pa, 1);
        pb += __shfl_xor_sync(0xffffffffu, pb, 1);
        pa += __shfl_xor_sync(0xffffffffu, pa, 2);
        pb += __shfl_xor_sync(0xffffffffu, pb, 2);
        if ((lane & 3) == 0 && gm < M) {
          double *q = ep.part + ((int64_t)gm * ep.npart + (int64_t)blockIdx.x * GW::WN + wn) * 2;
          q[0] = pa;
          q[1] = pb;
        }
      }
    }
  }
}

// f64, non-transposed operands: the same tiles fed by a 3-stage cp.async ring
// (global -> shared without a register round trip, two K-steps in flight)
constexpr int kCpStages = 3;
CS_D void cp_async8_zfill(void *dst, const void *src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src),
               "r"(valid ? 8 : 0)
               : "memory");
}
template <int BM, typename TC, int CBK = GemmWarps<BM>::BK>
__global__ void __launch_bounds__(GemmWarps<BM>::NT)
k_gemm_cp(int M, int N, int K, const double *__restrict__ A, int64_t lda, int64_t sA, const double *__restrict__ B,
          int64_t ldb, int64_t sB, TC *__restrict__ C, int64_t ldc, int64_t sC) {
  using GW = GemmWarps<BM>;
  constexpr int kBK = CBK, kLDA = CBK + 4, NT = GW::NT, MI = GW::MI;
  constexpr int EA = BM * kBK / NT, EB = kBK * kBN / NT;
  constexpr int SA = BM * kLDA, SB = kBK * kLDB;
  extern __shared__ __align__(16) double cp_sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / GW::WN, wn = warp % GW::WN;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * kBN;
  A += (int64_t)blockIdx.z * sA;
  B += (int64_t)blockIdx.z * sB;
  C += (int64_t)blockIdx.z * sC;
  const int nk = (K + kBK - 1) / kBK;
  auto issue = [&](int st) {
    if (st < nk) {
      double *As = cp_sm + (st % kCpStages) * (SA + SB), *Bs = As + SA;
      const int k0 = st * kBK;
#pragma unroll
      for (int e = 0; e < EA; ++e) {
        const int i = tid + e * NT, r = i / kBK, k = i % kBK;
        const int gm = m0 + r, gk = k0 + k;
        const bool ok = gm < M && gk < K;
        cp_async8_zfill(As + r * kLDA + k, ok ? A + (int64_t)gm * lda + gk : A, ok);
      }
#pragma unroll
      for (int e = 0; e < EB; ++e) {
        const int i = tid + e * NT, k = i / kBN, n = i % kBN;
        const int gn = n0 + n, gk = k0 + k;
        const bool ok = gn < N && gk < K;
        cp_async8_zfill(Bs + k * kLDB + n, ok ? B + (int64_t)gk * ldb + gn : B, ok);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double c[MI][MI][2];
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < MI; ++ni) c[mi][ni][0] = c[mi][ni][1] = 0.0;
#pragma unroll
  for (int st = 0; st < kCpStages - 1; ++st) issue(st);
  for (int s = 0; s < nk; ++s) {
    asm volatile("cp.async.wait_group %0;" ::"n"(kCpStages - 2) : "memory");
    __syncthreads();  // stage s landed everywhere; stage s-1's readers are done
    issue(s + kCpStages - 1);
    const double *As = cp_sm + (s % kCpStages) * (SA + SB), *Bs = As + SA;
    const double *as = As + (wm * GW::WT + (lane >> 2)) * kLDA + (lane & 3);
    const double *bs = Bs + (lane & 3) * kLDB + wn * GW::WT + (lane >> 2);
#pragma unroll
    for (int k0 = 0; k0 < kBK; k0 += 4) {
      double av[MI], bv[MI];
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        av[i] = as[i * 8 * kLDA + k0];
        bv[i] = bs[k0 * kLDB + i * 8];
      }
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < MI; ++ni) dmma884(c[mi][ni], av[mi], bv[ni]);
    }
  }
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < MI; ++ni) {
      const int gm = m0 + wm * GW::WT + mi * 8 + (lane >> 2);
      const int gn = n0 + wn * GW::WT + ni * 8 + 2 * (lane & 3);
      if (gm >= M) continue;
      if (gn < N) C[(int64_t)gm * ldc + gn] = (TC)c[mi][ni][0];
      if (gn + 1 < N) C[(int64_t)gm * ldc + gn + 1] = (TC)c[mi][ni][1];
    }
}

// fixed-order fold of the logistic epilogue's row partials (warp per row)
static __global__ void k_gemm_rowfold(const double *part, int64_t M, int npart, double *rowsum) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < M; r += nw) {
    double a = 0.0, b = 0.0;
    for (int j = lane; j < npart; j += 32) {  // lane-sequential, then a fixed butterfly
      a += part[(r * npart + j) * 2];
      b += part[(r * npart + j) * 2 + 1];
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, off);
      b += __shfl_xor_sync(0xffffffffu, b, off);
    }
    if (lane == 0) {
      rowsum[2 * r] = a;
      rowsum[2 * r + 1] = b;
    }
  }
}

}  // namespace gemm_detail

// C = eta = A X^T (M x N, f64) with the logistic epilogue fused (GemmEpi mode 1):
// C <- y - sigmoid(eta), weights to wout / wsw, row sums (eta . y, sum
// logaddexp(0, eta)) to rowsum[2 M].  part: scratch of M * ceil(N / 32) * 2
// doubles.  One batch, 128-row tiles.
inline cudaError_t gemm_xt_logistic(int M, int N, int K, const double *A, int64_t lda, const double *X, int64_t ldx,
                                    double *C, int64_t ldc, const double *y, double *wout, float *wsw, int nkb,
                                    double *part, double *rowsum, cudaStream_t st) {
  using namespace gemm_detail;
  if (M <= 0 || N <= 0) return cudaSuccess;
  GemmEpi ep;
  ep.mode = 1;
  ep.y = y;
  ep.wout = wout;
  ep.wsw = wsw;
  ep.nkb = nkb;
  ep.part = part;
  ep.npart = (int)((N + kBN - 1) / kBN) * GemmWarps<128>::WN;
  const dim3 grid((unsigned)((N + kBN - 1) / kBN), (M + 127) / 128, 1);
  k_gemm<128, true, double, double, double, 1><<<grid, GemmWarps<128>::NT, 0, st>>>(M, N, K, A, lda, 0, X, ldx, 0, C,
                                                                                    ldc, 0, ep);
  const int64_t wr = (int64_t)M * 32;
  k_gemm_rowfold<<<(unsigned)((wr + 255) / 256 < 148 * 16 ? (wr + 255) / 256 : 148 * 16), 256, 0, st>>>(
      part, M, ep.npart, rowsum);
  return cudaGetLastError();
}

// C = (A X^T) . S elementwise (GemmEpi mode 2), 128-row tiles, one batch
inline cudaError_t gemm_xt_scaled(int M, int N, int K, const double *A, int64_t lda, const double *X, int64_t ldx,
                                  double *C, int64_t ldc, const double *S, cudaStream_t st) {
  using namespace gemm_detail;
  if (M <= 0 || N <= 0) return cudaSuccess;
  GemmEpi ep;
  ep.mode = 2;
  ep.S = S;
  const dim3 grid((unsigned)((N + kBN - 1) / kBN), (M + 127) / 128, 1);
  k_gemm<128, true, double, double, double, 2><<<grid, GemmWarps<128>::NT, 0, st>>>(M, N, K, A, lda, 0, X, ldx, 0, C,
                                                                                    ldc, 0, ep);
  return cudaGetLastError();
}

// C = A . op(B) for `batch` independent problems (see the header comment).
// Small problems (fewer than ~2 waves of 64 x 64 tiles) take 32 x 64 tiles.
template <typename TA, typename TB, typename TC>
cudaError_t gemm_rm(bool bt, int M, int N, int K, const TA *A, int64_t lda, int64_t sA, const TB *B, int64_t ldb,
                    int64_t sB, TC *C, int64_t ldc, int64_t sC, int batch, cudaStream_t st) {
  using namespace gemm_detail;
  if (M <= 0 || N <= 0 || batch <= 0) return cudaSuccess;
  const int64_t nt = (N + kBN - 1) / kBN;
  const int64_t tiles128 = (int64_t)((M + 127) / 128) * nt * batch, tiles64 = (int64_t)((M + 63) / 64) * nt * batch;
  // the largest tile that still gives every SM a couple of CTAs
  const int BM = tiles128 >= 4 * 148 ? 128 : tiles64 >= 2 * 148 ? 64 : 32;
  const dim3 grid((unsigned)nt, (M + BM - 1) / BM, batch);
  if constexpr (std::is_same<TA, double>::value && std::is_same<TB, double>::value) {
    static const bool use_cp = [] {
      const char *e = getenv("CS_GEMM_CP");
      return e ? atoi(e) != 0 : true;
    }();
    if (!bt && use_cp) {  // f64 operands as stored: the cp.async ring
      auto cp = [&](auto bm) -> cudaError_t {
        constexpr int kBM = decltype(bm)::value, kBK = 16;
        using GW = GemmWarps<kBM>;
        constexpr size_t smem = sizeof(double) * kCpStages * ((size_t)kBM * (kBK + 4) + (size_t)kBK * kLDB);
        static const cudaError_t attr =  // once per tile shape (each kBM is its own lambda body)
            cudaFuncSetAttribute(k_gemm_cp<kBM, TC, kBK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (attr != cudaSuccess) return attr;
        k_gemm_cp<kBM, TC, kBK><<<grid, GW::NT, smem, st>>>(M, N, K, A, lda, sA, B, ldb, sB, C, ldc, sC);
        return cudaGetLastError();
      };
      if (BM == 128) return cp(std::integral_constant<int, 128>());
      if (BM == 64) return cp(std::integral_constant<int, 64>());
      return cp(std::integral_constant<int, 32>());
    }
  }
  auto go = [&](auto kern, int threads) {
    kern<<<grid, threads, 0, st>>>(M, N, K, A, lda, sA, B, ldb, sB, C, ldc, sC, GemmEpi());
  };
  if (BM == 128) {
    if (bt) go(k_gemm<128, true, TA, TB, TC>, GemmWarps<128>::NT);
    else go(k_gemm<128, false, TA, TB, TC>, GemmWarps<128>::NT);
  } else if (BM == 64) {
    if (bt) go(k_gemm<64, true, TA, TB, TC>, GemmWarps<64>::NT);
    else go(k_gemm<64, false, TA, TB, TC>, GemmWarps<64>::NT);
  } else {
    if (bt) go(k_gemm<32, true, TA, TB, TC>, GemmWarps<32>::NT);
    else go(k_gemm<32, false, TA, TB, TC>, GemmWarps<32>::NT);
  }
  return cudaGetLastError();
}

}  // namespace cs
