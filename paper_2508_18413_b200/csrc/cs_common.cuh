// Shared device/host helpers for the chainscan_b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>

#include "../../include/chainscan_b200.h"

#define CS_HD __host__ __device__ __forceinline__
#define CS_D __device__ __forceinline__

namespace cs {

constexpr int64_t kNoStep = INT64_MAX;   // "no offending step" sentinel for atomicMin

// Stream-ordered hand-off of a scratch buffer shared by all streams of a
// device (the host mutex only orders the enqueueing): a user's stream first
// waits for the previous user's queued work on the buffer, and on scope exit
// records its own, so a call on another stream cannot overwrite it mid-flight.
struct ScratchFence {
  cudaEvent_t ev = nullptr;
  void acquire(cudaStream_t st) {
    if (ev) cudaStreamWaitEvent(st, ev, 0);
  }
  void release(cudaStream_t st) {
    if (!ev && cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) {
      ev = nullptr;
      cudaDeviceSynchronize();  // no event: fall back to draining the device
      return;
    }
    cudaEventRecord(ev, st);
  }
};
// Stream-ordered scratch (cudaMallocAsync) from the device's default pool, which
// keeps freed blocks instead of returning them at every synchronisation (the
// default release threshold of 0 re-maps memory on each call: milliseconds).
inline cudaError_t scratch_alloc(void **p, size_t bytes, cudaStream_t st) {
  static bool done[16] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!done[dev & 15]) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    done[dev & 15] = true;
  }
  return cudaMallocAsync(p, bytes, st);
}

struct ScratchScope {  // acquire now, release when the enqueueing function returns
  ScratchFence &f;
  cudaStream_t st;
  ScratchScope(ScratchFence &fence, cudaStream_t s) : f(fence), st(s) { f.acquire(st); }
  ~ScratchScope() { f.release(st); }
};

// ---- storage <-> f64 ------------------------------------------------------
template <typename ST> CS_D double ld(const ST *p, int64_t i) { return (double)__ldg(p + i); }
template <typename ST> CS_D void st(ST *p, int64_t i, double v) { p[i] = (ST)v; }
// coherent (non-.nc) load for buffers written earlier in the same launch
template <typename ST> CS_D double ldv(const ST *p, int64_t i) {
  return (double)*((const volatile ST *)(p + i));
}

// ---- numerics mirroring numpy / scipy --------------------------------------
CS_D double logaddexp0(double x) {  // np.logaddexp(0, x)
  if (x != x) return x;
  return fmax(x, 0.0) + log1p(exp(-fabs(x)));
}
CS_D double log_sigmoid(double z) { return -logaddexp0(-z); }            // samplers.py:53-54
// sigma'(z) = sigma(z) sigma(-z) = e^-|z| / (1 + e^-|z|)^2: the saturation-safe value of
// samplers.py:57-59 with one exp instead of three transcendental calls
CS_D double sigmoid_prime(double z) {
  const double e = exp(-fabs(z));
  const double q = 1.0 + e;
  return e / (q * q);
}
CS_D double expit(double x) { return 1.0 / (1.0 + exp(-x)); }
// sigmoid(x) and logaddexp(0, x) from ONE exponential, t = e^{-|x|}:
// p = 1 / (1 + t) for x >= 0 and t / (1 + t) below (expit to within an ulp),
// logaddexp(0, x) = max(x, 0) + log1p(t), numpy's own form (same bits)
CS_D void sigmoid_logaddexp(double x, double &p, double &lae) {
  if (x != x) {
    p = x;
    lae = x;
    return;
  }
  const double t = exp(-fabs(x));
  const double r = 1.0 / (1.0 + t);
  p = x >= 0.0 ? r : t * r;
  lae = fmax(x, 0.0) + log1p(t);
}             // scipy.special.expit
CS_D double clipv(double x, double c) { return fmin(fmax(x, -c), c); }    // np.clip

// ---- atomics ------------------------------------------------------------------
// max of non-negative doubles via their bit patterns (NaN with clear sign bit
// sorts above +inf, so a NaN gap propagates like numpy's max).
CS_D void atomic_max_nonneg(unsigned long long *addr, double v) {
  atomicMax(addr, (unsigned long long)__double_as_longlong(v));
}
CS_D void atomic_min_i64(long long *addr, long long v) { atomicMin(addr, v); }

// ---- warp reductions -------------------------------------------------------------
CS_D double warp_sum(double v) {  // butterfly: every lane ends with the full sum
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}
CS_D double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
CS_D unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  return v;
}
CS_D long long warp_min_i64(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w < v ? w : v;
  }
  return v;
}
CS_D int warp_sum_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// single-instruction warp reductions (redux.sync) for the solver's flags:
// sums of u32 counts, and min / max of NON-NEGATIVE 64-bit words (step indices
// with the INT64_MAX sentinel; f64 bit patterns of |x|) as hi-word then lo-word
CS_D unsigned warp_sum_u32(unsigned v) { return __reduce_add_sync(0xffffffffu, v); }
CS_D long long warp_min_nn64(long long v) {
  const unsigned hi = (unsigned)((unsigned long long)v >> 32), lo = (unsigned)v;
  const unsigned mh = __reduce_min_sync(0xffffffffu, hi);
  const unsigned ml = __reduce_min_sync(0xffffffffu, hi == mh ? lo : 0xffffffffu);
  return (long long)(((unsigned long long)mh << 32) | ml);
}
CS_D unsigned long long warp_max_nn64(unsigned long long v) {
  const unsigned hi = (unsigned)(v >> 32), lo = (unsigned)v;
  const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
  const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
  return ((unsigned long long)mh << 32) | ml;
}

CS_D bool finite(double x) { return isfinite(x); }

}  // namespace cs
