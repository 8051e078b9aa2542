// Dense affine scans for any width D > 128, and the whole-sequence dense
// aggregate (the T-sharded driver's shard carry) for D > 8 (pscan.py:196-213,
// _scan_kernels.py:47-99; deer.py:161-170 builds these elements for any D).
//
// D > 128 is past the register/shared-memory tiling of cs_dense.cu, so the
// chunk compositions -- the scan's 2 T D^3 flop -- are batched DMMA GEMMs
// (cs_gemm.cuh):
//   per step k of a chunk, every chunk at once:  [M|w]_q <- J_{t0_q+k} [M|w]_q
//     (one strided-batched GEMM over the chunks, row-major D x (D+1) operands,
//      the affine column riding along) + u_{t0_q+k} added to the last column
//   k_xl_carry   one CTA walks the chunk maps in order (f64) -> chunk entries
//   k_xl_replay  one CTA per chunk replays s_t = J_t s_{t-1} + u_t from its
//                entry; warp-per-row dot products, f64 sums, the state rounded
//                to the storage type each step (as k_dense_replay)
// The composition inside a chunk runs in the storage type, everything that
// crosses chunks in f64 -- the same split as the narrower scans.
//
// Aggregates: chunk maps (this file's or cs_dense.cu's) are lifted to
// augmented (D+1) x (D+1) f64 matrices [[M, w], [0, 1]], where composing two
// affine maps is a plain product, and folded as a balanced tree of batched
// DMMA GEMMs (log2(n) launches).
#include "cs_common.cuh"
#include "cs_gemm.cuh"
#include "cs_scan.cuh"

namespace cs {

namespace {

constexpr int kXlThr = 512;

inline size_t al(size_t b) { return (b + 255) & ~(size_t)255; }

}  // namespace

// chunk length for D > 128: at most ~148 chunks (one reduce chain per SM's
// worth of batch), at least 8 steps per chunk
int dense_xl_chunk(int64_t T) {
  int64_t c = (T + 147) / 148;
  if (c < 8) c = 8;
  return (int)c;
}

// f64 tree buffers for n maps of width D: n + ceil(n/2) augmented matrices
static size_t tree_bytes(int64_t n, int D) {
  const size_t S = (size_t)(D + 1) * (D + 1);
  return al((size_t)(n + (n + 1) / 2) * S * sizeof(double));
}

size_t dense_xl_ws_bytes(int64_t T, int D, int elem_bytes) {
  const int c = dense_xl_chunk(T);
  const int64_t nch = T > 0 ? (T + c - 1) / c : 1;
  const size_t mb = al((size_t)nch * D * (D + 1) * elem_bytes);
  return 2 * mb + al((size_t)nch * D * sizeof(double)) + tree_bytes(nch, D) + 256;
}

// [M|w]_q = [J_{t0} | u_{t0}]
template <typename ST>
__global__ void k_xl_init(const ST *__restrict__ J, const ST *__restrict__ u, int D, int c, ST *M) {
  const int64_t q = blockIdx.y, t0 = q * (int64_t)c;
  const int64_t W = D + 1, n = (int64_t)D * W;
  ST *Mq = M + q * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / W, k = idx - i * W;
    Mq[idx] = k < D ? J[t0 * D * D + i * D + k] : u[t0 * D + i];
  }
}

// last column of [M|w]_q += u_{t0_q + k}
template <typename ST>
__global__ void k_xl_addu(const ST *__restrict__ u, int D, int c, int k, int64_t nq, ST *M) {
  const int64_t W = D + 1;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < nq * D; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = idx / D, i = idx - q * D;
    M[q * D * W + i * W + D] += u[(q * c + k) * D + i];
  }
}

// entries[q] = state entering chunk q; e_{q+1} = M_q e_q + w_q (f64)
template <typename ST>
__global__ void __launch_bounds__(kXlThr) k_xl_carry(const ST *__restrict__ M, const ST *s0, int64_t nch, int D,
                                                      double *entries) {
  extern __shared__ double xs[];  // 2 x D
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, NW = kXlThr / 32;
  const int64_t W = D + 1;
  for (int i = threadIdx.x; i < D; i += kXlThr) xs[i] = (double)s0[i];
  __syncthreads();
  for (int64_t q = 0; q < nch; ++q) {
    const double *cur = xs + (q & 1) * D;
    double *nxt = xs + ((q + 1) & 1) * D;
    const ST *Mq = M + q * D * W;
    for (int i = threadIdx.x; i < D; i += kXlThr) entries[q * D + i] = cur[i];
    for (int i = w; i < D; i += NW) {
      double acc = 0.0;
      for (int k = lane; k < D; k += 32) acc = fma((double)Mq[i * W + k], cur[k], acc);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
      if (lane == 0) nxt[i] = acc + (double)Mq[i * W + D];
    }
    __syncthreads();
  }
}

template <typename ST>
__global__ void __launch_bounds__(kXlThr) k_xl_replay(const ST *__restrict__ J, const ST *__restrict__ u,
                                                       const double *entries, int64_t T, int D, int c, ST *out) {
  extern __shared__ double xs[];  // 2 x D
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, NW = kXlThr / 32;
  const int64_t q = blockIdx.x, t0 = q * (int64_t)c;
  const int64_t t1 = t0 + c < T ? t0 + c : T;
  const int64_t DD = (int64_t)D * D;
  for (int i = threadIdx.x; i < D; i += kXlThr) xs[i] = entries[q * D + i];
  __syncthreads();
  int par = 0;
  for (int64_t t = t0; t < t1; ++t, par ^= 1) {
    const double *cur = xs + par * D;
    double *nxt = xs + (par ^ 1) * D;
    const ST *Jt = J + t * DD;
    for (int i = w; i < D; i += NW) {
      double acc = 0.0;
      for (int k = lane; k < D; k += 32) acc = fma((double)__ldcs(Jt + (int64_t)i * D + k), cur[k], acc);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
      if (lane == 0) {
        const ST v = (ST)(acc + (double)u[t * D + i]);
        nxt[i] = (double)v;
        out[t * D + i] = v;
      }
    }
    __syncthreads();
  }
}

// augmented f64 lift: aug[q] = [[M_q, w_q], [0, 1]] from row-major [M|w] (ST)
template <typename ST>
__global__ void k_aug_from_mw(const ST *__restrict__ M, int64_t n, int D, double *aug) {
  const int64_t W = D + 1, S = W * W;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n * S; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = idx / S, r = idx - q * S, i = r / W, k = r - i * W;
    aug[idx] = i < D ? (double)M[q * D * W + i * W + k] : (k == D ? 1.0 : 0.0);
  }
}

// the same from separate f64 (M, w) arrays (cs_dense.cu's chunk aggregates)
__global__ void k_aug_from_split(const double *__restrict__ aggM, const double *__restrict__ aggw, int64_t n, int D,
                                 double *aug) {
  const int64_t W = D + 1, S = W * W;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n * S; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = idx / S, r = idx - q * S, i = r / W, k = r - i * W;
    aug[idx] = i < D ? (k < D ? aggM[q * D * D + i * D + k] : aggw[q * D + i]) : (k == D ? 1.0 : 0.0);
  }
}

// flat [M (row-major D x D) | w (D)] from the augmented total
__global__ void k_aug_to_flat(const double *__restrict__ aug, int D, double *out) {
  const int64_t W = D + 1;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)D * D + D; idx += (int64_t)gridDim.x * blockDim.x) {
    if (idx < (int64_t)D * D) {
      const int64_t i = idx / D, k = idx - i * D;
      out[idx] = aug[i * W + k];
    } else {
      const int64_t i = idx - (int64_t)D * D;
      out[idx] = aug[i * W + D];
    }
  }
}

static unsigned grid1(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  return (unsigned)(g < 1 ? 1 : g);
}

// fold n augmented maps (earliest first) into the flat aggregate; buf holds
// n + ceil(n/2) augmented matrices, the first n filled
static cudaError_t tree_fold(double *buf, int64_t n, int D, double *out, cudaStream_t st) {
  const int W = D + 1;
  const long long S = (long long)W * W;
  double *a = buf, *b = buf + n * S;
  while (n > 1) {
    const int64_t pairs = n / 2;
    // pair i: C = A_{2i+1} A_{2i} (the later map applied last), batched DMMA GEMM
    cudaError_t e = gemm_rm<double, double, double>(false, W, W, W, a + S, W, 2 * S, a, W, 2 * S, b, W, S,
                                                    (int)pairs, st);
    if (e != cudaSuccess) return e;
    if (n & 1) {
      e = cudaMemcpyAsync(b + pairs * S, a + (n - 1) * S, S * sizeof(double), cudaMemcpyDeviceToDevice, st);
      if (e != cudaSuccess) return e;
    }
    n = (n + 1) / 2;
    double *tmp = a;
    a = b;
    b = tmp;
  }
  k_aug_to_flat<<<grid1((int64_t)D * D + D), 256, 0, st>>>(a, D, out);
  return cudaGetLastError();
}

// chunk maps [M|w]_q of the storage type for D > 128, into Ma; returns the
// buffer holding the final maps
template <typename ST>
static cudaError_t xl_reduce(const ScanArgs<ST> &a, int c, int64_t nch, ST *Ma, ST *Mb, ST **fin, cudaStream_t st) {
  const int D = a.D;
  const int64_t W = D + 1, n = (int64_t)D * W;
  k_xl_init<ST><<<dim3((unsigned)((n + 255) / 256 < 64 ? (n + 255) / 256 : 64), (unsigned)nch), 256, 0, st>>>(
      a.e0, a.u, D, c, Ma);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int64_t last_len = a.T - (nch - 1) * (int64_t)c;
  ST *cur = Ma, *nxt = Mb;
  for (int k = 1; k < c; ++k) {
    const int64_t nq = k < last_len ? nch : nch - 1;  // only the last chunk can be short
    if (nq <= 0) break;
    // [M|w]' = J_t [M|w] for every chunk at once (row-major, batched DMMA GEMM;
    // storage-type operands widened to f64, the product rounded back)
    e = gemm_rm<ST, ST, ST>(false, D, (int)W, D, a.e0 + (int64_t)k * D * D, D, (int64_t)c * D * D, cur, W, n, nxt,
                            W, n, (int)nq, st);
    if (e != cudaSuccess) return e;
    k_xl_addu<ST><<<grid1(nq * D), 256, 0, st>>>(a.u, D, c, k, nq, nxt);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if (nq < nch) {  // the short last chunk keeps its finished map
      e = cudaMemcpyAsync(nxt + (nch - 1) * n, cur + (nch - 1) * n, n * sizeof(ST), cudaMemcpyDeviceToDevice, st);
      if (e != cudaSuccess) return e;
    }
    ST *tmp = cur;
    cur = nxt;
    nxt = tmp;
  }
  *fin = cur;
  return cudaSuccess;
}

template <typename ST>
cudaError_t launch_dense_xl_t(ScanArgs<ST> a, void *ws, double *agg_out, cudaStream_t st) {
  const int64_t T = a.T;
  const int D = a.D;
  if (T == 0) return cudaSuccess;
  const int c = dense_xl_chunk(T);
  const int64_t nch = (T + c - 1) / c;
  const size_t mb = al((size_t)nch * D * (D + 1) * sizeof(ST));
  ST *Ma = (ST *)ws, *Mb = (ST *)((char *)ws + mb);
  double *entries = (double *)((char *)ws + 2 * mb);
  double *tree = (double *)((char *)entries + al((size_t)nch * D * sizeof(double)));
  ST *fin = nullptr;
  cudaError_t e = xl_reduce<ST>(a, c, nch, Ma, Mb, &fin, st);
  if (e != cudaSuccess) return e;
  if (agg_out) {
    k_aug_from_mw<ST><<<grid1(nch * (int64_t)(D + 1) * (D + 1)), 256, 0, st>>>(fin, nch, D, tree);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    return tree_fold(tree, nch, D, agg_out, st);
  }
  const size_t smem = 2 * (size_t)D * sizeof(double);
  if (smem > 48 * 1024) {
    e = cudaFuncSetAttribute(k_xl_carry<ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_xl_replay<ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k_xl_carry<ST><<<1, kXlThr, smem, st>>>(fin, a.s0, nch, D, entries);
  k_xl_replay<ST><<<(unsigned)nch, kXlThr, smem, st>>>(a.e0, a.u, entries, T, D, c, a.out);
  return cudaGetLastError();
}

// fold cs_dense.cu's f64 chunk aggregates (n maps) into the flat aggregate;
// tree: n + ceil(n/2) augmented matrices of scratch
cudaError_t dense_fold_aggregates(const double *aggM, const double *aggw, int64_t n, int D, double *tree,
                                  double *out, cudaStream_t st) {
  k_aug_from_split<<<grid1(n * (int64_t)(D + 1) * (D + 1)), 256, 0, st>>>(aggM, aggw, n, D, tree);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return tree_fold(tree, n, D, out, st);
}

size_t dense_tree_bytes(int64_t n, int D) { return tree_bytes(n, D); }

template cudaError_t launch_dense_xl_t<float>(ScanArgs<float>, void *, double *, cudaStream_t);
template cudaError_t launch_dense_xl_t<double>(ScanArgs<double>, void *, double *, cudaStream_t);

}  // namespace cs
