// Dense affine scan for wide states, 8 < D <= 128 (pscan.py:196-213 and
// _scan_kernels.py:47-99; SURVEY.md 8a row A12 at BASELINE cfg 3, D = 100).
//
// The recurrence s_t = J_t s_{t-1} + u_t with full D x D Jacobians is split in
// chunks of c steps and solved in three launches:
//   k_dense_reduce  one CTA per chunk composes (M, w) = (J_last...J_first,
//                   the chunk's affine part) -- the 2 T D^3 flop of the scan,
//                   a register-tiled product chain with J streamed through
//                   shared memory in 16-column slices
//   k_dense_carry   one CTA walks the chunk aggregates in order (f64) and
//                   writes every chunk's entry state (D^2 per chunk)
//   k_dense_replay  one CTA per chunk replays s_t = J_t s_{t-1} + u_t from
//                   its entry, warp-per-row dot products with f64 sums; the
//                   J_t reads (4 D^2 bytes per step) make it HBM-bound
// Aggregates and carries are f64 whatever the storage type.
#include <cstdlib>

#include "cs_common.cuh"
#include "cs_scan.cuh"
#include "cs_umma.cuh"

namespace cs {

constexpr int kDwSlice = 16;     // columns of J_t per shared-memory slice
constexpr int kDwReduceThr = 256;
constexpr int kDwThr = 512;      // carry / replay

template <typename ST, int DP>
__global__ void __launch_bounds__(kDwReduceThr)
k_dense_reduce(const ST *__restrict__ J, const ST *__restrict__ u, int64_t T, int D, int c, double *aggM,
               double *aggw) {
  constexpr int NA = DP / 16;
  constexpr int NS = DP / kDwSlice;                          // slices per step
  constexpr int PER = DP * kDwSlice / kDwReduceThr;          // slice elements per thread (DP*16/256)
  extern __shared__ __align__(16) unsigned char dsm[];
  ST *Ms = (ST *)dsm;              // DP x DP running product (zero padded)
  ST *Js = Ms + DP * DP;           // 2 x (DP x kDwSlice) slices of J_t, double-buffered
  ST *wv = Js + 2 * DP * kDwSlice; // DP running affine part
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t q = blockIdx.x, t0 = q * (int64_t)c;
  const int64_t t1 = t0 + c < T ? t0 + c : T;
  const int64_t DD = (int64_t)D * D;
  {
    const ST *J0 = J + t0 * DD;
    for (int idx = tid; idx < DP * DP; idx += kDwReduceThr) {
      const int i = idx / DP, k = idx - i * DP;
      Ms[idx] = (i < D && k < D) ? J0[i * D + k] : ST(0);
    }
    for (int i = tid; i < DP; i += kDwReduceThr) wv[i] = i < D ? u[t0 * D + i] : ST(0);
  }
  // slice n of the chunk's stream (step t0+1+n/NS, columns (n%NS)*16..): each
  // thread owns PER fixed (row, column) positions of it; the next slice is
  // loaded into registers while the current one is multiplied
  ST pf[PER];
  auto fetch = [&](int64_t n) {
    const int64_t t = t0 + 1 + n / NS;
    const int k0 = (int)(n % NS) * kDwSlice;
    const ST *Jt = J + t * DD;
#pragma unroll
    for (int p = 0; p < PER; ++p) {
      const int idx = tid + p * kDwReduceThr;
      const int i = idx / kDwSlice, k = k0 + (idx - i * kDwSlice);
      pf[p] = (t < t1 && i < D && k < D) ? __ldg(Jt + i * D + k) : ST(0);
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int p = 0; p < PER; ++p) Js[buf * DP * kDwSlice + tid + p * kDwReduceThr] = pf[p];
  };
  const int64_t nslices = (t1 - t0 - 1) * NS;
  if (nslices > 0) {
    fetch(0);
    stash(0);
  }
  __syncthreads();
  int64_t n = 0;
  for (int64_t t = t0 + 1; t < t1; ++t) {
    ST acc[NA][NA];
#pragma unroll
    for (int x = 0; x < NA; ++x)
#pragma unroll
      for (int y = 0; y < NA; ++y) acc[x][y] = ST(0);
    double wacc = 0.0;  // thread i < D: row i of J_t w
#pragma unroll 1
    for (int sl = 0; sl < NS; ++sl, ++n) {
      const int k0 = sl * kDwSlice;
      if (n + 1 < nslices) fetch(n + 1);
      const ST *Jc = Js + (n & 1) * DP * kDwSlice;
#pragma unroll
      for (int kk = 0; kk < kDwSlice; ++kk) {
        ST a[NA], b[NA];
#pragma unroll
        for (int x = 0; x < NA; ++x) a[x] = Jc[(ty + 16 * x) * kDwSlice + kk];
#pragma unroll
        for (int y = 0; y < NA; ++y) b[y] = Ms[(k0 + kk) * DP + tx + 16 * y];
#pragma unroll
        for (int x = 0; x < NA; ++x)
#pragma unroll
          for (int y = 0; y < NA; ++y) acc[x][y] = fma(a[x], b[y], acc[x][y]);
      }
      if (tid < DP)
#pragma unroll
        for (int kk = 0; kk < kDwSlice; ++kk) wacc += (double)Jc[tid * kDwSlice + kk] * (double)wv[k0 + kk];
      if (n + 1 < nslices) stash((int)((n + 1) & 1));  // the other buffer: last read a slice ago
      if (sl + 1 < NS) __syncthreads();
    }
    __syncthreads();  // every product read of Ms done
#pragma unroll
    for (int x = 0; x < NA; ++x)
#pragma unroll
      for (int y = 0; y < NA; ++y) Ms[(ty + 16 * x) * DP + tx + 16 * y] = acc[x][y];
    if (tid < DP) wv[tid] = tid < D ? (ST)(wacc + (double)u[t * D + tid]) : ST(0);
    __syncthreads();
  }
  double *M = aggM + q * DD;
  for (int idx = tid; idx < D * D; idx += kDwReduceThr) {
    const int i = idx / D, k = idx - i * D;
    M[idx] = (double)Ms[i * DP + k];
  }
  for (int i = tid; i < D; i += kDwReduceThr) aggw[q * D + i] = (double)wv[i];
}

// entries[q] = state entering chunk q; e_{q+1} = M_q e_q + w_q.  Warp w owns
// rows w, w + 16, ...; lanes stride the columns (coalesced row reads), and
// the next chunk's matrix is loaded into registers while this one is applied.
// CTA g walks chunks [g per, g per + per) from its entry: gent[g] when given,
// else s0 (one CTA over everything).
template <typename ST, int DP>
__global__ void __launch_bounds__(kDwThr)
k_dense_carry(const double *aggM, const double *aggw, const ST *s0, const double *gent, int64_t nch_all, int D,
              int64_t per, double *entries) {
  constexpr int NW = kDwThr / 32, RPW = DP / NW, KL = (DP + 31) / 32;
  __shared__ double e[2][128];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t DD = (int64_t)D * D;
  const int64_t q0 = (int64_t)blockIdx.x * per;
  const int64_t nch = q0 + per < nch_all ? per : nch_all - q0;
  aggM += q0 * DD;
  aggw += q0 * D;
  entries += q0 * D;
  if (tid < D) e[0][tid] = gent ? gent[(int64_t)blockIdx.x * D + tid] : (double)s0[tid];
  double m[RPW][KL];
  auto load = [&](int64_t q) {
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      const int i = w + NW * r;
#pragma unroll
      for (int k = 0; k < KL; ++k) {
        const int col = lane + 32 * k;
        m[r][k] = (i < D && col < D) ? __ldcg(aggM + q * DD + (int64_t)i * D + col) : 0.0;
      }
    }
  };
  if (nch > 0) load(0);
  __syncthreads();
  for (int64_t q = 0; q < nch; ++q) {
    const double *cur = e[q & 1];
    double acc[RPW];
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      acc[r] = 0.0;
#pragma unroll
      for (int k = 0; k < KL; ++k) {
        const int col = lane + 32 * k;
        acc[r] = fma(m[r][k], col < D ? cur[col] : 0.0, acc[r]);
      }
    }
    if (q + 1 < nch) load(q + 1);
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], off);
      const int i = w + NW * r;
      if (lane == 0 && i < D) {
        entries[q * D + i] = cur[i];
        e[(q + 1) & 1][i] = acc[r] + __ldcg(aggw + q * D + i);
      }
    }
    __syncthreads();
  }
}

// replay chunk q from its entry: warp w owns rows w, w + 16, ...; lanes
// stride the columns, f64 sums, one barrier per step; J_{t+1} is loaded into
// a second register set while step t is applied
template <typename ST, int DP>
__global__ void __launch_bounds__(kDwThr)
k_dense_replay(const ST *__restrict__ J, const ST *__restrict__ u, const double *entries, int64_t T, int D, int c,
               ST *out) {
  constexpr int NW = kDwThr / 32, RPW = DP / NW, KL = (DP + 31) / 32;
  __shared__ double s[2][128];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t q = blockIdx.x, t0 = q * (int64_t)c;
  const int64_t t1 = t0 + c < T ? t0 + c : T;
  const int64_t DD = (int64_t)D * D;
  if (tid < D) s[0][tid] = entries[q * D + tid];
  ST ja[RPW][KL];
  ST jb[sizeof(ST) == 4 ? RPW : 1][sizeof(ST) == 4 ? KL : 1];  // f64: one set (registers)
  auto load = [&](int64_t t, ST (&jv)[RPW][KL]) {
    const ST *Jt = J + t * DD;
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      const int i = w + NW * r;
#pragma unroll
      for (int m = 0; m < KL; ++m) {
        const int k = lane + 32 * m;
        jv[r][m] = (t < t1 && i < D && k < D) ? __ldcs(Jt + (int64_t)i * D + k) : ST(0);
      }
    }
  };
  auto step = [&](int64_t t, const ST (&jv)[RPW][KL], int par) {
    const double *cur = s[par];
    double acc[RPW];
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      acc[r] = 0.0;
#pragma unroll
      for (int m = 0; m < KL; ++m) {
        const int k = lane + 32 * m;
        acc[r] = fma((double)jv[r][m], k < D ? cur[k] : 0.0, acc[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], off);
      const int i = w + NW * r;
      if (lane == 0 && i < D) {
        const ST v = (ST)(acc[r] + (double)u[t * D + i]);
        s[par ^ 1][i] = (double)v;
        out[t * D + i] = v;
      }
    }
    __syncthreads();
  };
  __syncthreads();
  int par = 0;
  if constexpr (sizeof(ST) == 8) {
    for (int64_t t = t0; t < t1; ++t) {
      load(t, ja);
      step(t, ja, par);
      par ^= 1;
    }
    return;
  } else {
  load(t0, ja);
  for (int64_t t = t0; t < t1; t += 2) {
    load(t + 1, jb);
    step(t, ja, par);
    par ^= 1;
    if (t + 1 >= t1) break;
    load(t + 2, ja);
    step(t + 1, jb, par);
    par ^= 1;
  }
  }
}

// f32 replay with the step maps streamed through shared memory: J_t and u_t of
// the next kRpStages steps are in flight as 1-D bulk copies (TMA engine) while
// step t is applied, so a chunk's walk runs at its HBM rate instead of one
// exposed load latency per step (D % 4 == 0: every map is whole 16-byte lines)
constexpr int kRpStages = 2;

template <int DP>
__global__ void __launch_bounds__(kDwThr, 1)
k_dense_replay_tma(const float *__restrict__ J, const float *__restrict__ u, const double *entries, int64_t T, int D,
                   int c, float *out) {
  constexpr int NW = kDwThr / 32, RPW = DP / NW, KL = (DP + 31) / 32;
  extern __shared__ __align__(16) unsigned char rsm[];
  __shared__ double s[2][128];
  __shared__ __align__(8) uint64_t bar[kRpStages];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t q = blockIdx.x, t0 = q * (int64_t)c;
  const int64_t t1 = t0 + c < T ? t0 + c : T;
  const int64_t DD = (int64_t)D * D;
  const int slot = (int)(((size_t)DD + D + 3) / 4 * 4);  // floats per stage (16-byte multiple)
  float *ring = (float *)rsm;
  if (tid == 0) {
    for (int k = 0; k < kRpStages; ++k) mbar_init(&bar[k], 1);
    fence_mbar_init();
  }
  if (tid < D) s[0][tid] = entries[q * D + tid];
  __syncthreads();
  auto issue = [&](int64_t t) {  // thread 0: step t's J_t and u_t into its stage
    const int k = (int)((t - t0) % kRpStages);
    float *dst = ring + (size_t)k * slot;
    mbar_expect_tx(&bar[k], (unsigned)((DD + D) * sizeof(float)));
    bulk_g2s(dst, J + t * DD, (unsigned)(DD * sizeof(float)), &bar[k]);
    bulk_g2s(dst + DD, u + t * D, (unsigned)(D * sizeof(float)), &bar[k]);
  };
  if (tid == 0)
    for (int64_t t = t0; t < t1 && t < t0 + kRpStages; ++t) issue(t);
  int par = 0;
  for (int64_t t = t0; t < t1; ++t) {
    const int k = (int)((t - t0) % kRpStages);
    mbar_wait(&bar[k], (unsigned)(((t - t0) / kRpStages) & 1));
    const float *Js = ring + (size_t)k * slot, *us = Js + DD;
    const double *cur = s[par];
    double acc[RPW];
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      const int i = w + NW * r;
      acc[r] = 0.0;
#pragma unroll
      for (int m = 0; m < KL; ++m) {
        const int kk = lane + 32 * m;
        if (i < D && kk < D) acc[r] = fma((double)Js[i * D + kk], cur[kk], acc[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], off);
      const int i = w + NW * r;
      if (lane == 0 && i < D) {
        const float v = (float)(acc[r] + (double)us[i]);
        s[par ^ 1][i] = (double)v;
        out[t * D + i] = v;
      }
    }
    __syncthreads();  // every read of stage k and of s[par] is done
    if (tid == 0 && t + kRpStages < t1) issue(t + kRpStages);
    par ^= 1;
  }
}

static bool dense_replay_tma() {  // CS_DENSE_REPLAY_TMA=0 keeps the register-prefetch replay
  static const bool v = [] {
    const char *e = getenv("CS_DENSE_REPLAY_TMA");
    return e ? atoi(e) != 0 : true;
  }();
  return v;
}

// ---------------------------------------------------------------------------
int dense_wide_chunk(int64_t T) {
  const char *e = getenv("CS_DENSE_CHUNK");
  if (e && atoi(e) > 0) return atoi(e);
  // enough chunks to fill the machine with replay CTAs, few enough that the
  // serial carry stays short: the power of two nearest T / 768 (128 steps per
  // chunk at T = 1e5), so the tree composition covers whole chunks
  const double want = (double)T / 768.0;
  int c = 8;
  while (c < 512 && (double)c * 1.4142135623730951 < want) c *= 2;
  return c;
}

static bool dense_tc() {  // CS_DENSE_TC=0 keeps the f32 composition on the FP32 pipes
  static const bool v = [] {
    const char *e = getenv("CS_DENSE_TC");
    return e ? atoi(e) != 0 : true;
  }();
  return v;
}

static int dense_dp(int D) { return D <= 16 ? 16 : D <= 32 ? 32 : D <= 64 ? 64 : D <= 112 ? 112 : 128; }

template <typename ST, int DP>
static cudaError_t launch_reduce(const ScanArgs<ST> &a, int c, int64_t nch, double *aggM, double *aggw,
                                 cudaStream_t st) {
  const size_t smem = sizeof(ST) * ((size_t)DP * DP + 2 * (size_t)DP * kDwSlice + DP);
  auto k = k_dense_reduce<ST, DP>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k<<<(unsigned)nch, kDwReduceThr, smem, st>>>(a.e0, a.u, a.T, a.D, c, aggM, aggw);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Tensor-core composition (f32 storage, D < 128, D % 4 == 0): the chunk's
// product chain M <- J_t M on the 5th-gen tensor cores.  The chain needs f32
// accuracy (the carry applies M to the entry state), so every operand is
// split x = hi + lo in TF32 and each product is hi.hi + hi.lo + lo.hi (3xTF32,
// error ~2^-21 per product against f32's 2^-24).  The affine part rides along
// as column D of the B operand, M_aug = [M | w]: J_t M_aug = [J_t M | J_t w],
// and u_t is added to that column in the epilogue.  Per step: J_t streams in
// four 32-column K-blocks (staging warps 1..7, two blocks ahead in registers),
// warp 0 lane 0 issues 4 x 3 kind::tf32 MMAs per block into a 128 x 128 f32
// TMEM accumulator, then all warps read it back (tcgen05.ld) and write the new
// M_aug^T, split, as the next step's B operand (K-major, SWIZZLE_128B).
constexpr int kDrtThr = 256;

CS_D void tf32_split(float x, float &hi, float &lo) {
  unsigned h;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
  hi = __uint_as_float(h);
  unsigned l;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(x - hi));
  lo = __uint_as_float(l);
}
// x = hi + lo with hi = x rounded to TF32 (nearest, ties away -- cvt.rna for
// finite x) by integer arithmetic; lo is left in f32 (the tensor core reads its
// top 19 bits)
CS_D void tf32_split_fast(float x, float &hi, float &lo) {
  hi = __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
  lo = x - hi;
}
// float offset of element (row, k) in a K-major SW128 operand of 128 rows whose
// K extent is split into 32-column atoms of 128 x 32 floats
CS_D int sw128_off(int row, int k) {
  return (k >> 5) * kUmmaTile + row * 32 + ((((k & 31) >> 2) ^ (row & 7)) << 2) + (k & 3);
}

__global__ void __launch_bounds__(kDrtThr, 1)
k_dense_reduce_tc(const float *__restrict__ J, const float *__restrict__ u, int64_t T, int D, int c, double *aggM,
                  double *aggw) {
  extern __shared__ __align__(16) unsigned char dsm[];
  float *Bh = smem_align<float, 1024>(dsm);  // 4 atoms: M_aug^T hi
  float *Bl = Bh + 4 * kUmmaTile;                                      // lo
  float *As = Bl + 4 * kUmmaTile;                                      // 2 stages x (hi, lo) of J_t K-blocks
  __shared__ __align__(8) uint64_t bars[2 * kUmmaStages + 1];
  __shared__ uint32_t s_tmem;
  UmmaPipe pipe;
  pipe.full = bars;
  pipe.empty = bars + kUmmaStages;
  pipe.done = bars + 2 * kUmmaStages;
  umma_pipe_init(pipe);  // full barriers count blockDim.x - 32: the staging warps
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t q = blockIdx.x, t0 = q * (int64_t)c;
  const int64_t t1 = t0 + c < T ? t0 + c : T;
  const int64_t DD = (int64_t)D * D;
  // initial B = M_aug^T with M_aug = [J_t0 | u_t0]
  {
    const float *J0 = J + t0 * DD;
    for (int idx = tid; idx < 128 * 128; idx += kDrtThr) {
      const int k = idx >> 7, j = idx & 127;  // coalesced over j (row k of M_aug)
      float v = 0.0f;
      if (k < D) v = j < D ? J0[k * D + j] : (j == D ? u[t0 * D + k] : 0.0f);
      float hi, lo;
      tf32_split(v, hi, lo);
      Bh[sw128_off(j, k)] = hi;
      Bl[sw128_off(j, k)] = lo;
    }
  }
  pipe.tmem = tmem_alloc128(&s_tmem);  // its barrier also publishes the B writes and barrier inits
  if (t1 - t0 == 1) {
    for (int idx = tid; idx < D * D; idx += kDrtThr) aggM[q * DD + idx] = (double)J[t0 * DD + idx];
    for (int i = tid; i < D; i += kDrtThr) aggw[q * D + i] = (double)u[t0 * D + i];
    tmem_free128(pipe.tmem);
    return;
  }
  fence_proxy_async_smem();
  __syncthreads();
  const int nblk = (int)(t1 - t0 - 1) * 4;  // K-blocks of the chunk's stream: step t0 + 1 + b / 4, columns 32 (b % 4)
  constexpr int NS = kDrtThr - 32, PER = (128 * 8 + NS - 1) / NS;
  const int st = tid - 32;
  float4 xr[2][PER];
  auto load = [&](int b, float4 (&dst)[PER]) {
    const int64_t t = t0 + 1 + b / 4;
    const float *Jt = J + t * DD;
    const int kb = b & 3;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int qq = st + i * NS, r = qq >> 3, ch = qq & 7, k0 = 32 * kb + 4 * ch;
      dst[i] = (b < nblk && qq < 1024 && r < D && k0 < D) ? __ldg((const float4 *)(Jt + r * D + k0))
                                                          : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  if (wid > 0) {
    load(0, xr[0]);
    load(1, xr[1]);
  }
  int b = 0;
  const int erow = 32 * (wid & 3) + lane;  // this thread's accumulator row in the epilogue
  for (int64_t t = t0 + 1; t < t1; ++t) {
    const float ut = erow < D ? __ldg(u + t * D + erow) : 0.0f;  // issued now, used after the MMAs
    if (wid == 0) {
      if (lane == 0) {
        for (int kb = 0; kb < 4; ++kb) {
          const uint32_t g = pipe.kb + kb;
          const int s = (int)(g % kUmmaStages);
          mbar_wait(&pipe.full[s], (g / kUmmaStages) & 1);
          tc_fence_after();
          const float *Ah = As + s * 2 * kUmmaTile, *Al = Ah + kUmmaTile;
          const uint64_t dah = umma_desc_sw128(Ah), dal = umma_desc_sw128(Al);
          const uint64_t dbh = umma_desc_sw128(Bh + kb * kUmmaTile), dbl = umma_desc_sw128(Bl + kb * kUmmaTile);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            umma_tf32(pipe.tmem, dah + 2 * k, dbh + 2 * k, kIdescTf32_128x128, (kb | k) != 0);
            umma_tf32(pipe.tmem, dah + 2 * k, dbl + 2 * k, kIdescTf32_128x128, 1);
            umma_tf32(pipe.tmem, dal + 2 * k, dbh + 2 * k, kIdescTf32_128x128, 1);
          }
          umma_commit(&pipe.empty[s]);
        }
        umma_commit(pipe.done);
      }
      __syncwarp();
    } else {
      for (int kb = 0; kb < 4; ++kb, ++b) {
        const uint32_t g = pipe.kb + kb;
        const int s = (int)(g % kUmmaStages);
        const uint32_t use = g / kUmmaStages;
        if (use > 0) mbar_wait(&pipe.empty[s], (use - 1) & 1);
        float *Ah = As + s * 2 * kUmmaTile, *Al = Ah + kUmmaTile;
#pragma unroll
        for (int i = 0; i < PER; ++i) {
          const int qq = st + i * NS, r = qq >> 3, ch = qq & 7;
          if (qq < 1024) {
            const float4 x = xr[b & 1][i];
            float4 h, l;
            tf32_split(x.x, h.x, l.x);
            tf32_split(x.y, h.y, l.y);
            tf32_split(x.z, h.z, l.z);
            tf32_split(x.w, h.w, l.w);
            const int off = r * 32 + ((ch ^ (r & 7)) << 2);
            *(float4 *)(Ah + off) = h;
            *(float4 *)(Al + off) = l;
          }
        }
        if (b + 2 < nblk) load(b + 2, xr[b & 1]);
        fence_proxy_async_smem();
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&pipe.full[s])) : "memory");
      }
    }
    pipe.kb += 4;
    // epilogue: the new M_aug = J_t M_aug (+ u_t in column D) back into B, or the aggregate
    mbar_wait(pipe.done, pipe.steps & 1);
    ++pipe.steps;
    tc_fence_after();
    const bool last = t + 1 == t1;
    const int row = erow, c0 = 64 * (wid >> 2);
#pragma unroll
    for (int cc = 0; cc < 64; cc += 16) {
      float v[16];
      tmem_ld16(pipe.tmem + ((uint32_t)(32 * (wid & 3)) << 16) + (uint32_t)(c0 + cc), v);
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int j = c0 + cc + e;
        float val = v[e];
        if (j == D) val += ut;
        if (last) {
          if (row < D) {
            if (j < D) aggM[q * DD + (int64_t)row * D + j] = (double)val;
            else if (j == D) aggw[q * D + row] = (double)val;
          }
        } else {
          float hi, lo;
          tf32_split(val, hi, lo);
          Bh[sw128_off(j, row)] = hi;
          Bl[sw128_off(j, row)] = lo;
        }
      }
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
  }
  tmem_free128(pipe.tmem);
}

// ---------------------------------------------------------------------------
// Tree-ordered composition (f32 storage, D < 128, D % 4 == 0): chunk aggregates
// over chunks of c = 2^L steps as L levels of INDEPENDENT pair products,
//   (M, w)_p <- (M_{2p+1} M_{2p}, M_{2p+1} w_{2p} + w_{2p+1})
// (an odd tail is carried through as I . (M, w)), so every level is one
// throughput-bound batched product instead of a dependent chain per chunk.
// Persistent CTAs walk the level's products; per product, K (= D padded to
// 128) streams in four 32-row blocks through a 3-stage ring:
//   warps 5..11   stage A = M_{2p+1} (K-major SW128) and B = [M_{2p} | w_{2p}]
//                 (MN-major, SWIZZLE_128B_BASE32B: rows k, the 128 columns j
//                 contiguous -- the maps' own row-major order, so no
//                 transposition), both split
//                 hi + lo in TF32
//   warp 4        issues 4 x 3 kind::tf32 MMAs per block (hi.hi + hi.lo +
//                 lo.hi) into one of two TMEM accumulators
//   warps 0..3    drain the other accumulator (tcgen05.ld, row per lane), add
//                 w_{2p+1}, store the product (f32, or f64 at the last level)
// so staging, MMAs and the epilogue of consecutive products overlap.
constexpr int kDtThr = 384;
constexpr int kDtStages = 3;
constexpr int kDtStaging = kDtThr - 160;  // warps 5..11
// MN-major tf32 operand descriptor (the only MN-major layout tf32 takes:
// SWIZZLE_128B_BASE32B, layout type 1): rows (K) of 128 B = 32 columns, the
// four 32-byte granules of row k stored at granule ^ (k & 3); 4-row atoms
// `sbo` bytes apart, 32-column groups `lbo` bytes apart
CS_D uint64_t umma_desc_sw128_mn(const void *smem_tile, uint32_t lbo, uint32_t sbo = 512) {
  const uint64_t a = (uint64_t)smem_u32(smem_tile);
  return ((a & 0x3FFFFull) >> 4) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) | (1ull << 46) |
         (1ull << 61);
}
// D f32, A/B tf32, A K-major, B MN-major (bit 16), N = 128, M = 128
constexpr uint32_t kIdescTf32_128x128_BMN = kIdescTf32_128x128 | (1u << 16);

__global__ void __launch_bounds__(kDtThr, 1)
k_dense_tree_tc(const float *__restrict__ Min, const float *__restrict__ win, int64_t K, int D, float *Mout,
                float *wout, double *Mout64, double *wout64) {
  extern __shared__ __align__(16) unsigned char dsm[];
  // stage s: A hi, A lo (128 rows x 32 k), B hi, B lo (4 column groups x 32 k-rows x 32)
  float *stg = smem_align<float, 1024>(dsm);
  __shared__ __align__(8) uint64_t full[kDtStages], empty[kDtStages], accf[2], acce[2];
  __shared__ uint32_t s_tmem;
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  const int64_t nprod = (K + 1) / 2;
  const int64_t DD = (int64_t)D * D;
  if (tid == 0) {
    for (int s = 0; s < kDtStages; ++s) {
      mbar_init(&full[s], kDtStaging);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accf[b], 1);
      mbar_init(&acce[b], 128);
    }
    fence_mbar_init();
  }
  if (wid == 0) {  // two 128-column accumulators
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&s_tmem))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  if (wid >= 5) {
    // ---- staging: 2 x 1024 16-byte chunks per block (A: row i, k chunk; B: k-row, j chunk).
    // Block g's in-range chunks are copied raw by cp.async straight to their
    // swizzled places in the hi tiles, two blocks ahead; when they land, the
    // thread that copied a chunk rewrites it as (rna hi, lo) -- no cross-thread
    // hand-off, no register staging.  Chunks out of range (zero), the identity
    // of an odd tail and the affine column are formed at conversion.
    constexpr int PER = (2048 + kDtStaging - 1) / kDtStaging;
    const int st = tid - 160;
    float *wS = (float *)(stg + kDtStages * 4 * kUmmaTile);  // [stage][32]: w_{2p} rows of the block
    const int64_t nloc = nprod > blockIdx.x ? (nprod - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int64_t nblk = 4 * nloc;
    // per slot e (chunk q = st + 224 e, fixed for the whole kernel): its place in
    // the stage (floats past A hi), its offset in the source map at kb = 0, the
    // row / column it covers (validity per kb), A or B
    int dsto[PER], soff[PER], rc[PER];
#pragma unroll
    for (int e = 0; e < PER; ++e) {
      const int q = st + e * kDtStaging;
      if (q < 1024) {
        const int r = q >> 3, c = q & 7;
        dsto[e] = r * 32 + ((c ^ (r & 7)) << 2);
        soff[e] = r * D + 4 * c;
        rc[e] = (r << 8) | (4 * c);  // i, k0
      } else {
        const int qb = q < 2048 ? q - 1024 : 0, r = qb >> 5, j4 = qb & 31, grp = j4 >> 3, c = j4 & 7;
        dsto[e] = 2 * kUmmaTile + grp * 1024 + r * 32 + ((((c >> 1) ^ (r & 3)) << 3) | ((c & 1) << 2));
        soff[e] = r * D + 4 * j4;
        rc[e] = (r << 8) | (4 * j4);  // k0, j
      }
    }
    const int stepB = 32 * D;
    auto issue = [&](int64_t g) {
      const int s = (int)(g % kDtStages);
      const int64_t p = blockIdx.x + (g >> 2) * gridDim.x;
      const int kb = (int)(g & 3);
      float *Ah = stg + s * 4 * kUmmaTile;
      const bool tail = 2 * p + 1 >= K;
      const float *M1 = Min + (2 * p + 1) * DD + 32 * kb, *M0 = Min + 2 * p * DD + (int64_t)stepB * kb;
#pragma unroll
      for (int e = 0; e < PER; ++e) {
        const int q = st + e * kDtStaging;
        const int a = rc[e] >> 8, b = rc[e] & 255;
        if (q < 1024) {
          if (!tail && a < D && b + 32 * kb < D) cp_async16(Ah + dsto[e], M1 + soff[e]);
        } else if (q < 2048 && a + 32 * kb < D) {
          if (b < D) cp_async16(Ah + dsto[e], M0 + soff[e]);
          else if (b == D)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(wS + s * 32 + a)),
                         "l"(win + 2 * p * D + 32 * kb + a)
                         : "memory");
        }
      }
    };
    auto convert = [&](int64_t g) {
      const int s = (int)(g % kDtStages);
      const int64_t p = blockIdx.x + (g >> 2) * gridDim.x;
      const int kb = (int)(g & 3);
      float *Ah = stg + s * 4 * kUmmaTile;
      const bool tail = 2 * p + 1 >= K;
#pragma unroll
      for (int e = 0; e < PER; ++e) {
        const int q = st + e * kDtStaging;
        if (q < 2048) {
          const int a = rc[e] >> 8, b = rc[e] & 255;
          float *dh = Ah + dsto[e], *dl = dh + kUmmaTile;  // lo tiles sit one tile past their hi tiles
          float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
          if (q < 1024) {
            const int k = b + 32 * kb;
            if (a < D && k < D) {
              if (!tail) x = *(const float4 *)dh;
              else x = make_float4(a == k, a == k + 1, a == k + 2, a == k + 3);
            }
          } else if (a + 32 * kb < D) {
            if (b < D) x = *(const float4 *)dh;
            else if (b == D) x.x = wS[s * 32 + a];
          }
          float4 h, l;
          tf32_split_fast(x.x, h.x, l.x);
          tf32_split_fast(x.y, h.y, l.y);
          tf32_split_fast(x.z, h.z, l.z);
          tf32_split_fast(x.w, h.w, l.w);
          *(float4 *)dh = h;
          *(float4 *)dl = l;
        }
      }
    };
    // block g: converted (and handed to the MMA) two iterations after its copies
    // were issued, before this iteration's wait for a free stage
    for (int64_t g = 0; g < nblk + 2; ++g) {
      if (g >= 2) {
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        convert(g - 2);
        fence_proxy_async_smem();
        mbar_arrive(&full[(g - 2) % kDtStages]);
      }
      if (g < nblk) {
        const uint32_t use = (uint32_t)(g / kDtStages);
        if (use > 0) mbar_wait(&empty[g % kDtStages], (use - 1) & 1);
        issue(g);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
  } else if (wid == 4) {
    // ---- MMA issue
    if (lane == 0) {
      uint32_t g = 0, n = 0;
      for (int64_t p = blockIdx.x; p < nprod; p += gridDim.x, ++n) {
        const uint32_t b = n & 1;
        if (n >= 2) mbar_wait(&acce[b], ((n >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t acc = tmem + 128 * b;
        for (int kb = 0; kb < 4; ++kb, ++g) {
          const int s = (int)(g % kDtStages);
          mbar_wait(&full[s], (g / kDtStages) & 1);
          tc_fence_after();
          const float *Ah = stg + s * 4 * kUmmaTile, *Al = Ah + kUmmaTile, *Bh = Al + kUmmaTile, *Bl = Bh + kUmmaTile;
          const uint64_t dah = umma_desc_sw128(Ah), dal = umma_desc_sw128(Al);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {  // 8 k-rows per MMA: A start + 32 B, B start + 8 rows (1 KB)
            const uint64_t dbh = umma_desc_sw128_mn(Bh + kk * 256, 4096), dbl = umma_desc_sw128_mn(Bl + kk * 256, 4096);
            constexpr uint32_t idesc = kIdescTf32_128x128_BMN;
            umma_tf32(acc, dah + 2 * kk, dbh, idesc, (kb | kk) != 0);
            umma_tf32(acc, dah + 2 * kk, dbl, idesc, 1);
            umma_tf32(acc, dal + 2 * kk, dbh, idesc, 1);
          }
          umma_commit(&empty[s]);
        }
        umma_commit(&accf[b]);
      }
    }
    __syncwarp();
  } else {
    // ---- epilogue: warp w drains TMEM lanes 32 w .. (row i = 32 w + lane)
    const int i = 32 * wid + lane;
    uint32_t n = 0;
    for (int64_t p = blockIdx.x; p < nprod; p += gridDim.x, ++n) {
      const uint32_t b = n & 1;
      const bool tail = 2 * p + 1 >= K;
      const float w1 = (!tail && i < D) ? __ldcs(win + (2 * p + 1) * D + i) : 0.0f;
      mbar_wait(&accf[b], (n >> 1) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int cc = 0; cc < 128; cc += 16) {
        float v[16];
        tmem_ld16(tmem + 128 * b + ((uint32_t)(32 * wid) << 16) + (uint32_t)cc, v);
        if (i >= D || cc > D) continue;
        if (Mout64) {
          double *row = Mout64 + p * DD + (int64_t)i * D;
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const int j = cc + e;
            if (j < D) row[j] = (double)v[e];
            else if (j == D) wout64[p * D + i] = (double)v[e] + (double)w1;
          }
        } else {
          float *row = Mout + p * DD + (int64_t)i * D;
#pragma unroll
          for (int e = 0; e < 16; e += 4) {
            const int j = cc + e;
            if (j + 4 <= D) *(float4 *)(row + j) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
            else if (j == D) wout[p * D + i] = v[e] + w1;
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&acce[b]);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (wid == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
}

static bool dense_tree() {  // CS_DENSE_TREE=0 keeps the per-chunk product chain (k_dense_reduce_tc)
  static const bool v = [] {
    const char *e = getenv("CS_DENSE_TREE");
    return e ? atoi(e) != 0 : true;
  }();
  return v;
}

static bool tree_ok(int D, int esize) { return esize == 4 && D % 4 == 0 && D < 128 && dense_tree(); }

// f32 scratch of the tree levels: ceil(T/2) + ceil(T/4) maps (ping-pong)
static size_t tree_scratch_floats(int64_t T, int D) {
  return (size_t)(((T + 1) / 2) + ((T + 3) / 4)) * ((size_t)D * D + D) + 64;
}

// chunk aggregates over chunks of c = 2^L steps (c from dense_wide_chunk)
static cudaError_t launch_tree(const float *J, const float *u, int64_t T, int D, int c, double *aggM, double *aggw,
                               float *scratch, cudaStream_t st) {
  int L = 0;
  while ((1 << L) < c) ++L;
  const size_t smem = 1024 + sizeof(float) * ((size_t)kDtStages * 4 * kUmmaTile + kDtStages * 32);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_dense_tree_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int64_t DD = (int64_t)D * D;
  float *bufA = scratch, *bufB = scratch + ((T + 1) / 2) * (DD + D);
  const float *inM = J, *inw = u;
  int64_t K = T;
  for (int l = 1; l <= L; ++l) {
    const int64_t np = (K + 1) / 2;
    float *o = (l & 1) ? bufA : bufB;
    float *oM = o, *ow = o + np * DD;
    const bool last = l == L;
    const unsigned grid = (unsigned)(np < sms ? np : sms);
    k_dense_tree_tc<<<grid, kDtThr, smem, st>>>(inM, inw, K, D, last ? nullptr : oM, last ? nullptr : ow,
                                                last ? aggM : nullptr, last ? aggw : nullptr);
    inM = oM;
    inw = ow;
    K = np;
  }
  return cudaGetLastError();
}

// Chunk entries: one serial walk over the chunk aggregates when they are few;
// otherwise two levels -- groups of kDwGroup chunk aggregates are composed in
// parallel (the reduce kernel again, on f64 aggregates), one CTA walks the
// group aggregates, and every group then walks its own chunks from its entry.
constexpr int kDwGroup = 16;

template <typename ST, int DP>
static cudaError_t launch_tail(const ScanArgs<ST> &a, int c, int64_t nch, const double *aggM, const double *aggw,
                               double *entries, double *gM, cudaStream_t st) {
  const int D = a.D;
  if (nch <= 4 * kDwGroup) {
    k_dense_carry<ST, DP><<<1, kDwThr, 0, st>>>(aggM, aggw, a.s0, nullptr, nch, D, nch, entries);
  } else {
    const int64_t ng = (nch + kDwGroup - 1) / kDwGroup;
    double *gw = gM + ng * (int64_t)D * D, *gent = gw + ng * (int64_t)D;
    ScanArgs<double> g{aggM, nullptr, nullptr, nullptr, aggw, nullptr, nullptr, nch, D};
    cudaError_t e = launch_reduce<double, DP>(g, kDwGroup, ng, gM, gw, st);
    if (e != cudaSuccess) return e;
    k_dense_carry<ST, DP><<<1, kDwThr, 0, st>>>(gM, gw, a.s0, nullptr, ng, D, ng, gent);
    k_dense_carry<ST, DP><<<(unsigned)ng, kDwThr, 0, st>>>(aggM, aggw, a.s0, gent, nch, D, kDwGroup, entries);
  }
  if constexpr (sizeof(ST) == 4) {
    if (dense_replay_tma() && D % 4 == 0 && ((((uintptr_t)a.e0) | ((uintptr_t)a.u)) & 15) == 0) {
      const size_t slot = ((size_t)D * D + D + 3) / 4 * 4;
      const size_t smem = sizeof(float) * slot * kRpStages;
      cudaError_t e = cudaFuncSetAttribute(k_dense_replay_tma<DP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem);
      if (e != cudaSuccess) return e;
      k_dense_replay_tma<DP><<<(unsigned)nch, kDwThr, smem, st>>>((const float *)a.e0, (const float *)a.u, entries,
                                                                  a.T, D, c, (float *)a.out);
      return cudaGetLastError();
    }
  }
  k_dense_replay<ST, DP><<<(unsigned)nch, kDwThr, 0, st>>>(a.e0, a.u, entries, a.T, D, c, a.out);
  return cudaGetLastError();
}

template <typename ST>
cudaError_t launch_dense_wide_t(ScanArgs<ST> a, void *ws, cudaStream_t st, double *agg_out) {
  const int64_t T = a.T;
  const int D = a.D;
  if (T == 0) return cudaSuccess;
  const int c = dense_wide_chunk(T);
  const int64_t nch = (T + c - 1) / c;
  double *aggM = (double *)ws;
  double *aggw = aggM + nch * (int64_t)D * D;
  double *entries = aggw + nch * (int64_t)D;
  double *gM = entries + nch * (int64_t)D;  // group level: ng x (D*D + 2D)
  cudaError_t e;
  const int64_t ngt = (nch + kDwGroup - 1) / kDwGroup;
  double *tree_end = (double *)(((uintptr_t)(gM + ngt * ((int64_t)D * D + 2 * D)) + 255) & ~(uintptr_t)255);
  if (tree_ok(D, (int)sizeof(ST)) && (c & (c - 1)) == 0) {
    // scratch past the aggregate-fold tree (see dense_wide_ws_bytes)
    const int64_t nf = nch <= 64 ? nch : ngt;
    float *scratch = (float *)(((uintptr_t)tree_end + dense_tree_bytes(nf, D) + 255) & ~(uintptr_t)255);
    e = launch_tree((const float *)a.e0, (const float *)a.u, T, D, c, aggM, aggw, scratch, st);
  } else if (sizeof(ST) == 4 && dense_tc() && D % 4 == 0 && D < 128) {
    const size_t smem = 1024 + sizeof(float) * (8 + 2 * kUmmaStages) * kUmmaTile;  // B hi/lo + A stages
    e = cudaFuncSetAttribute(k_dense_reduce_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_dense_reduce_tc<<<(unsigned)nch, kDrtThr, smem, st>>>((const float *)a.e0, (const float *)a.u, T, D, c, aggM,
                                                            aggw);
    e = cudaGetLastError();
  } else
  switch (dense_dp(D)) {
    case 16: e = launch_reduce<ST, 16>(a, c, nch, aggM, aggw, st); break;
    case 32: e = launch_reduce<ST, 32>(a, c, nch, aggM, aggw, st); break;
    case 64: e = launch_reduce<ST, 64>(a, c, nch, aggM, aggw, st); break;
    case 112: e = launch_reduce<ST, 112>(a, c, nch, aggM, aggw, st); break;
    default: e = launch_reduce<ST, 128>(a, c, nch, aggM, aggw, st); break;
  }
  if (e != cudaSuccess) return e;
  if (agg_out) {  // whole-sequence map: fold chunk (or group) aggregates as a tree of DGEMMs
    double *tree = (double *)(((uintptr_t)(gM + ((nch + kDwGroup - 1) / kDwGroup) * ((int64_t)D * D + 2 * D)) + 255) &
                              ~(uintptr_t)255);
    if (nch <= 64) return dense_fold_aggregates(aggM, aggw, nch, D, tree, agg_out, st);
    const int64_t ng = (nch + kDwGroup - 1) / kDwGroup;
    double *gw = gM + ng * (int64_t)D * D;
    ScanArgs<double> g{aggM, nullptr, nullptr, nullptr, aggw, nullptr, nullptr, nch, D};
    switch (dense_dp(D)) {
      case 16: e = launch_reduce<double, 16>(g, kDwGroup, ng, gM, gw, st); break;
      case 32: e = launch_reduce<double, 32>(g, kDwGroup, ng, gM, gw, st); break;
      case 64: e = launch_reduce<double, 64>(g, kDwGroup, ng, gM, gw, st); break;
      case 112: e = launch_reduce<double, 112>(g, kDwGroup, ng, gM, gw, st); break;
      default: e = launch_reduce<double, 128>(g, kDwGroup, ng, gM, gw, st); break;
    }
    if (e != cudaSuccess) return e;
    return dense_fold_aggregates(gM, gw, ng, D, tree, agg_out, st);
  }
  switch (dense_dp(D)) {
    case 16: e = launch_tail<ST, 16>(a, c, nch, aggM, aggw, entries, gM, st); break;
    case 32: e = launch_tail<ST, 32>(a, c, nch, aggM, aggw, entries, gM, st); break;
    case 64: e = launch_tail<ST, 64>(a, c, nch, aggM, aggw, entries, gM, st); break;
    case 112: e = launch_tail<ST, 112>(a, c, nch, aggM, aggw, entries, gM, st); break;
    default: e = launch_tail<ST, 128>(a, c, nch, aggM, aggw, entries, gM, st); break;
  }
  return e;
}

size_t dense_wide_ws_bytes(int64_t T, int D, int esize) {
  const int c = dense_wide_chunk(T);
  const int64_t nch = (T + c - 1) / c;
  const int64_t ng = (nch + 15) / 16;
  // + the tree scratch of the whole-sequence aggregate (cs_scan_aggregate):
  // the chunk aggregates when there are few, else the group aggregates;
  // + the f32 levels of the tree-ordered chunk composition
  const int64_t nf = nch <= 64 ? nch : ng;
  return (size_t)(nch + ng) * ((size_t)D * D + 2 * D) * sizeof(double) + 256 + dense_tree_bytes(nf, D) + 256 +
         (tree_ok(D, esize) ? tree_scratch_floats(T, D) * sizeof(float) + 256 : 0);
}

template cudaError_t launch_dense_wide_t<float>(ScanArgs<float>, void *, cudaStream_t, double *);
template cudaError_t launch_dense_wide_t<double>(ScanArgs<double>, void *, cudaStream_t, double *);

}  // namespace cs
