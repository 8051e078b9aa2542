// extern "C" boundary of libchainscan_b200.so (include/chainscan_b200.h).
//
// Host-side validation mirrors the reference's error behaviour; every compute
// call launches hand-written sm_100a kernels on the caller's stream.
#include <cstdio>
#include <cstring>
#include <atomic>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "cs_dispatch.h"
#include "cs_gen_tables.h"
#include "cs_noise.cuh"
#include "cs_scan.cuh"

using namespace cs;

namespace {
thread_local std::string g_err;

int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char *where) {
  return fail(CS_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
inline cudaStream_t S(void *p) { return (cudaStream_t)p; }
inline unsigned grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  if (g > 148LL * 64) g = 148LL * 64;
  return (unsigned)(g < 1 ? 1 : g);
}
inline int esize(int dtype) { return dtype == CS_F64 ? 8 : 4; }
inline bool dtype_ok(int dtype) { return dtype == CS_F32 || dtype == CS_F64; }
inline size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

int sm_count() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 148;
}
}  // namespace

// ---------------------------------------------------------------------------
// kernels
namespace cs {

template <typename OT>
__global__ void k_noise_fill(int kind, uint64_t seed, uint64_t slot, int64_t t0, int64_t nt,
                             int count, double df, OT *out) {
  const uint64_t h2 = hash_prefix(seed, slot);
  const int64_t n = nt * count;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / count;
    const int k = (int)(idx - i * count);
    const uint64_t h3 = hash_t(h2, (uint64_t)(t0 + i));
    out[idx] = (OT)noise_value(kind, h3, k, df);
  }
}

template <typename OT>
__global__ void k_rademacher(uint64_t seed, int64_t iteration, const int64_t *ts, int64_t t0,
                             int64_t n, int sample, int dim, OT *out) {
  const uint64_t h2 = probe_prefix(seed, iteration);
  const int64_t tot = n * dim;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < tot;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / dim;
    const int d = (int)(idx - i * dim);
    const int64_t t = ts ? ts[i] : t0 + i;
    out[idx] = (OT)probe_sign(hash_t(h2, (uint64_t)t), sample, d);
  }
}

template <typename ST>
__global__ void k_first_nonfinite(const ST *x, int64_t n, int64_t width, long long *out) {
  long long best = kNoStep;
  const int64_t tot = n * width;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < tot;
       idx += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite((double)x[idx])) {
      const long long r = idx / width;
      best = r < best ? r : best;
    }
  best = warp_min_i64(best);
  if ((threadIdx.x & 31) == 0 && best != kNoStep) atomicMin(out, best);
}

template <typename ST>
__global__ void k_converged(const ST *prev, const ST *next, int64_t n, double atol, double rtol,
                            unsigned *notok, unsigned long long *dmax) {
  unsigned bad = 0;
  unsigned long long dm = 0ull;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double nx = (double)next[i];
    const double gap = fabs(nx - (double)prev[i]);
    bad += (gap <= atol + rtol * fabs(nx)) ? 0u : 1u;
    const unsigned long long gb = (unsigned long long)__double_as_longlong(gap);
    dm = gb > dm ? gb : dm;
  }
  bad = (unsigned)warp_sum_i((int)bad);
  dm = warp_max_u64(dm);
  if ((threadIdx.x & 31) == 0) {
    if (bad) atomicAdd(notok, bad);
    atomicMax(dmax, dm);
  }
}

template <typename ST>
__global__ void k_bookkeeping(const ST *guess, const ST *next, int64_t T, int D, double atol,
                              double rtol, int iteration, int32_t *last_fail, unsigned *nfail,
                              unsigned long long *dmax) {
  unsigned cnt = 0;
  unsigned long long dm = 0ull;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < T;
       r += (int64_t)gridDim.x * blockDim.x) {
    bool f = false;
    for (int d = 0; d < D; ++d) {
      const double nx = (double)next[r * D + d];
      const double gap = fabs(nx - (double)guess[r * D + d]);
      f |= gap > atol + rtol * fabs(nx);
      const unsigned long long gb = (unsigned long long)__double_as_longlong(gap);
      dm = gb > dm ? gb : dm;
    }
    if (f) { last_fail[r] = iteration; ++cnt; }
  }
  cnt = (unsigned)warp_sum_i((int)cnt);
  dm = warp_max_u64(dm);
  if ((threadIdx.x & 31) == 0) {
    if (cnt) atomicAdd(nfail, cnt);
    atomicMax(dmax, dm);
  }
}

// wide rows (D >= 32): one warp per row, lanes across the state
template <typename ST>
__global__ void k_bookkeeping_wide(const ST *guess, const ST *next, int64_t T, int D, double atol,
                                   double rtol, int iteration, int32_t *last_fail, unsigned *nfail,
                                   unsigned long long *dmax) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned cnt = 0;
  unsigned long long dm = 0ull;
  for (int64_t r = w0; r < T; r += nw) {
    int f = 0;
    for (int d = lane; d < D; d += 32) {
      const double nx = (double)next[r * D + d];
      const double gap = fabs(nx - (double)guess[r * D + d]);
      f |= gap > atol + rtol * fabs(nx);
      const unsigned long long gb = (unsigned long long)__double_as_longlong(gap);
      dm = gb > dm ? gb : dm;
    }
    if (__any_sync(0xffffffffu, f)) {
      if (lane == 0) { last_fail[r] = iteration; ++cnt; }
    }
  }
  cnt = (unsigned)warp_sum_i((int)cnt);
  dm = warp_max_u64(dm);
  if (lane == 0) {
    if (cnt) atomicAdd(nfail, cnt);
    atomicMax(dmax, dm);
  }
}

template <typename ST>
CS_D double prev_at(const ST *s0, const ST *guess, int64_t r, int D, int d) {
  return r == 0 ? (double)s0[d] : (double)guess[(r - 1) * D + d];
}

// deer.py:171-183
template <typename ST>
__global__ void k_form_diag(const ST *est, const ST *f, const ST *s0, const ST *guess, int64_t T,
                            int D, const double *pre, double lam, double clip, ST *j, ST *u) {
  const int64_t n = T * D;
  const bool do_clip = isfinite(clip);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / D;
    const int d = (int)(i - r * D);
    double v = (double)est[i];
    if (pre) v = v * pre[d];
    v = v * lam;
    if (do_clip) v = clipv(v, clip);
    j[i] = (ST)v;
    u[i] = (ST)((double)f[i] - v * prev_at(s0, guess, r, D, d));
  }
}

// deer.py:161-170; one thread per row
template <typename ST>
__global__ void k_form_dense(const ST *Jin, const ST *f, const ST *s0, const ST *guess, int64_t T,
                             int D, const double *pre, double lam, double clip, ST *J, ST *u) {
  const bool do_clip = isfinite(clip);
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < T;
       r += (int64_t)gridDim.x * blockDim.x) {
    for (int a = 0; a < D; ++a) {
      double acc = 0.0;
      for (int c = 0; c < D; ++c) {
        const int64_t q = (r * D + a) * D + c;
        double v = (double)Jin[q];
        if (pre) v = v * (pre[c] / pre[a]);
        v = v * lam;
        if (do_clip) v = clipv(v, clip);
        J[q] = (ST)v;
        acc += v * prev_at(s0, guess, r, D, c);
      }
      u[r * D + a] = (ST)((double)f[r * D + a] - acc);
    }
  }
}

// deer.py:184-204; D = position dim (state 2D)
template <typename ST>
__global__ void k_form_block(const ST *ai, const ST *bi, const ST *ci, const ST *di, const ST *f,
                             const ST *s0, const ST *guess, int64_t T, int D, const double *pre,
                             double lam, double clip, ST *ao, ST *bo, ST *co, ST *dout, ST *u) {
  const int64_t n = T * D;
  const bool do_clip = isfinite(clip);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / D;
    const int k = (int)(i - r * D);
    double a = (double)ai[i], b = (double)bi[i], c = (double)ci[i], d = (double)di[i];
    if (pre) {
      const double px = pre[k], pv = pre[D + k];
      b = b * (pv / px);
      c = c * (px / pv);
    }
    a = lam * a; b = lam * b; c = lam * c; d = lam * d;
    if (do_clip) { a = clipv(a, clip); b = clipv(b, clip); c = clipv(c, clip); d = clipv(d, clip); }
    ao[i] = (ST)a; bo[i] = (ST)b; co[i] = (ST)c; dout[i] = (ST)d;
    const double x = prev_at(s0, guess, r, 2 * D, k), v = prev_at(s0, guess, r, 2 * D, D + k);
    u[r * 2 * D + k] = (ST)((double)f[r * 2 * D + k] - (a * x + b * v));
    u[r * 2 * D + D + k] = (ST)((double)f[r * 2 * D + D + k] - (c * x + d * v));
  }
}

template <typename ST>
__global__ void k_hutch(ST *est, const ST *z, const ST *jz, int64_t n, int first, double div) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v = (first ? 0.0 : (double)est[i]) + (double)z[i] * (double)jz[i];
    if (div > 0.0) v = v / div;
    est[i] = (ST)v;
  }
}

__global__ void k_set_i64(long long *p, long long v) { *p = v; }

__global__ void k_init_stats(cs_elem_stats *s) {
  s->bad_proposal = s->bad_step = s->bad_jacobian = kNoStep;
  s->picard_fail = 0;
  s->fail_rows = 0;
  s->dmax = 0.0;
}

// first row whose last-fail stamp is `it` (the window advance of deer.py:318)
__global__ void k_first_stamp(const int32_t *lf, int64_t n, int32_t it, long long *out) {
  long long best = kNoStep;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    if (lf[r] == it) {
      best = r;
      break;
    }
  best = warp_min_nn64(best);
  if ((threadIdx.x & 31) == 0 && best != kNoStep) atomicMin(out, best);
}

// Per (device, stream) solver state that outlives a call: the grid control
// block and halo stamps (zeroed once here, left zeroed by every solve), the
// host-mapped outcome record and a pair of timing events.
struct SolveState {
  int dev;
  cudaStream_t st;
  std::thread::id host;  // per host thread too: two threads sharing a stream get separate outcome records
  SolveCtl *ctl;
  int *ready;
  SolveOut *out;  // host-mapped (UVA: the same pointer on the device)
  cudaEvent_t ev0, ev1;
  unsigned seq;   // solves launched on this state
};

}  // namespace cs

// ---------------------------------------------------------------------------
extern "C" {

const char *cs_last_error(void) { return g_err.c_str(); }

static unsigned long long *h_probe = nullptr;
static int h_probe_n = 0;
int cs_debug_gram(const double *X, int32_t N, int32_t D, const double *W, int64_t T, float *H_out, void *stream) {
  if (!X || !W || !H_out || N < 1 || D < 1 || D > 128 || T < 0) return fail(CS_ERR_CONFIG, "bad gram arguments");
  const cudaError_t e = debug_gram(X, N, D, W, T, H_out, S(stream));
  return e == cudaSuccess ? CS_OK : cuda_fail(e, "cs_debug_gram");
}
int cs_debug_pair_gram(const double *X, int32_t N, int32_t D, const double *W, int64_t T, float *H_out,
                       void *stream) {
  if (!X || !W || !H_out || N < 1 || D < 1 || D > 128 || T < 0) return fail(CS_ERR_CONFIG, "bad gram arguments");
  const cudaError_t e = debug_pair_gram(X, N, D, W, T, H_out, S(stream));
  return e == cudaSuccess ? CS_OK : cuda_fail(e, "cs_debug_pair_gram");
}

int cs_debug_probe(unsigned long long *dev_buf, int n) {
  h_probe = dev_buf;
  h_probe_n = dev_buf ? n : 0;
  return CS_OK;
}
int cs_version(void) { return 1; }

int cs_target_eval(const cs_target *target, int what, int64_t n, const double *x, const double *v, double *out,
                   void *stream) {
  if (!target || !x || !out || n < 0 || what < 0 || what > 2 || (what == 2 && !v))
    return fail(CS_ERR_CONFIG, "bad target_eval arguments");
  if (target->dim < 1) return fail(CS_ERR_CONFIG, "bad target dimension");
  if (target->kind == CS_TARGET_BLR && (!target->X || !target->y || target->n_data < 1))
    return fail(CS_ERR_CONFIG, "logistic-regression target without data");
  if (target->kind == CS_TARGET_GAUSSIAN && (!target->mu || !target->chol || !target->prec))
    return fail(CS_ERR_CONFIG, "gaussian target without mean / factors");
  const cudaError_t e = target_eval_gemm(*target, what, n, x, v, out, S(stream));
  if (e == cudaErrorNotSupported) return fail(CS_ERR_CONFIG, "target_eval: logistic regression and gaussian only");
  return e == cudaSuccess ? CS_OK : cuda_fail(e, "cs_target_eval");
}

int cs_stream_sync(void *stream) {
  const cudaError_t e = cudaStreamSynchronize(S(stream));
  return e == cudaSuccess ? CS_OK : cuda_fail(e, "cs_stream_sync");
}

int cs_device_sm_count(int *out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  e = cudaDeviceGetAttribute(out, cudaDevAttrMultiProcessorCount, dev);
  return e == cudaSuccess ? CS_OK : cuda_fail(e, "cudaDeviceGetAttribute");
}

int cs_noise_fill(int kind, uint64_t seed, uint64_t slot_id, int64_t t0, int64_t nt, int32_t count,
                  double df, int dtype, void *out, void *stream) {
  if (kind < 0 || kind > CS_NOISE_LOG_UNIFORM) return fail(CS_ERR_CONFIG, "unknown noise kind");
  if (!dtype_ok(dtype)) return fail(CS_ERR_CONFIG, "bad dtype");
  if (count < 1 || nt < 0) return fail(CS_ERR_CONFIG, "slot count must be >= 1");
  if (kind == CS_NOISE_CHI2 && !(df > 0)) return fail(CS_ERR_CONFIG, "chi-squared slot needs df > 0");
  const int64_t n = nt * count;
  if (n == 0) return CS_OK;
  if (dtype == CS_F64)
    k_noise_fill<double><<<grid_for(n, 256), 256, 0, S(stream)>>>(kind, seed, slot_id, t0, nt, count, df, (double *)out);
  else
    k_noise_fill<float><<<grid_for(n, 256), 256, 0, S(stream)>>>(kind, seed, slot_id, t0, nt, count, df, (float *)out);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? CS_OK : cuda_fail(e, "cs_noise_fill");
}

int cs_rademacher_fill(uint64_t seed, int64_t iteration, const int64_t *ts, int64_t t0, int64_t n,
                       int32_t sample, int32_t dim, int dtype, void *out, void *stream) {
  if (!dtype_ok(dtype) || dim < 1 || n < 0) return fail(CS_ERR_STRUCTURAL, "bad probe shape");
  if (n == 0) return CS_OK;
  if (dtype == CS_F64)
    k_rademacher<double><<<grid_for(n * dim, 256), 256, 0, S(stream)>>>(seed, iteration, ts, t0, n, sample, dim, (double *)out);
  else
    k_rademacher<float><<<grid_for(n * dim, 256), 256, 0, S(stream)>>>(seed, iteration, ts, t0, n, sample, dim, (float *)out);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? CS_OK : cuda_fail(e, "cs_rademacher_fill");
}

// ---- scans -----------------------------------------------------------------
size_t cs_scan_workspace_bytes(int mode, int dtype, int64_t T, int32_t D) {
  const int var = mode == CS_MODE_DIAG ? SCAN_DIAG : mode == CS_MODE_BLOCK ? SCAN_BLOCK : SCAN_DENSE;
  if (var == SCAN_DENSE && D > 128) return dense_xl_ws_bytes(T, D, dtype == CS_F64 ? 8 : 4);
  if (var == SCAN_DENSE && D > 8) return dense_wide_ws_bytes(T, D, dtype == CS_F64 ? 8 : 4);
  return scan_ws_bytes(var, dtype, T, D);
}

// wide dense scans (D > 8) and their whole-sequence aggregate (agg_out != null):
// cs_dense.cu up to D = 128, cs_dense_xl.cu beyond
static int dense_wide_call(int dtype, const void *J, const void *u, const void *s0, void *out, int64_t T, int D,
                           void *ws, size_t ws_bytes, double *agg_out, void *stream) {
  const size_t need = D > 128 ? dense_xl_ws_bytes(T, D, dtype == CS_F64 ? 8 : 4) : dense_wide_ws_bytes(T, D, dtype == CS_F64 ? 8 : 4);
  if (ws_bytes < need) return fail(CS_ERR_CONFIG, "scan workspace too small");
  cudaError_t e;
  if (dtype == CS_F64) {
    ScanArgs<double> a{(const double *)J, nullptr, nullptr, nullptr, (const double *)u, (const double *)s0,
                       (double *)out, T, D};
    e = D > 128 ? launch_dense_xl_t<double>(a, ws, agg_out, S(stream))
                : launch_dense_wide_t<double>(a, ws, S(stream), agg_out);
  } else {
    ScanArgs<float> a{(const float *)J, nullptr, nullptr, nullptr, (const float *)u, (const float *)s0,
                      (float *)out, T, D};
    e = D > 128 ? launch_dense_xl_t<float>(a, ws, agg_out, S(stream))
                : launch_dense_wide_t<float>(a, ws, S(stream), agg_out);
  }
  return e == cudaSuccess ? CS_OK : cuda_fail(e, agg_out ? "dense aggregate launch" : "dense scan launch");
}

static int do_scan(int var, int dtype, const void *e0, const void *e1, const void *e2, const void *e3,
                   const void *u, const void *s0, void *out, int64_t T, int D, void *ws, size_t ws_bytes,
                   void *stream) {
  if (!dtype_ok(dtype)) return fail(CS_ERR_CONFIG, "bad dtype");
  if (T < 0 || D < 1) return fail(CS_ERR_STRUCTURAL, "bad scan shape");
  if (var != SCAN_DENSE && D > 4096) return fail(CS_ERR_CONFIG, "scan D too large");
  if (var == SCAN_DENSE && D > 8) return dense_wide_call(dtype, e0, u, s0, out, T, D, ws, ws_bytes, nullptr, stream);
  const ScanPlan p = scan_plan(var, dtype, T, D);
  if (ws_bytes < p.ws_bytes) return fail(CS_ERR_CONFIG, "scan workspace too small");
  if (T == 0) return CS_OK;
  // plain diag scans take the single-pass kernel when the workspace covers its
  // tile records and the element / output arrays are 16-byte aligned (bulk copies)
  const bool a16 = ((((uintptr_t)e0) | ((uintptr_t)u) | ((uintptr_t)out)) & 15) == 0;
  const bool one_pass = a16 && scan_1p_eligible(var, T, D) && ws_bytes >= scan_plan_1p(var, dtype, T, D).ws_bytes;
  // (any alignment: the local scan falls back to plain loads for unaligned arrays)
  const bool local = scan_local_eligible(var, T, D) &&
                     ws_bytes >= (var == SCAN_BLOCK ? scan_local_blk_ws_bytes(dtype, T, D)
                                                    : scan_local_ws_bytes(dtype, T, D));
  // reduce-then-replay for plain diag scans up to CS_SCAN_RR_PLAIN_MAX_T
  static const int64_t rr_max = [] {
    const char *e = getenv("CS_SCAN_RR_PLAIN_MAX_T");
    return e ? (int64_t)atoll(e) : ((int64_t)1 << 20);  // D = 18: 2^17 0.053 -> 0.046 ms, 2^18 0.069 -> 0.051, 2^19 0.085 -> 0.070; even at 2^20; local ahead above (tools/sweep_rr_plain.sh)
  }();
  // (D > 64: every T from 2^16 -- the column scan's tile chain is latency-bound there)
  const bool rr = (T < rr_max || D > 64) && scan_rr_eligible(var, T, D) && ws_bytes >= scan_rr_ws_bytes(dtype, T, D);
  cudaError_t e;
  if (rr) {
    if (dtype == CS_F64) {
      ScanArgs<double> a{(const double *)e0, nullptr, nullptr, nullptr, (const double *)u, (const double *)s0,
                         (double *)out, T, D};
      e = launch_scan_rr_t<double, false>(a, ws, S(stream));
    } else {
      ScanArgs<float> a{(const float *)e0, nullptr, nullptr, nullptr, (const float *)u, (const float *)s0,
                        (float *)out, T, D};
      e = launch_scan_rr_t<float, false>(a, ws, S(stream));
    }
    return e == cudaSuccess ? CS_OK : cuda_fail(e, "scan launch");
  }
  if (dtype == CS_F64) {
    ScanArgs<double> a{(const double *)e0, (const double *)e1, (const double *)e2, (const double *)e3,
                       (const double *)u, (const double *)s0, (double *)out, T, D};
    a.probe = h_probe;
    a.probe_n = h_probe_n;
    e = local      ? (var == SCAN_BLOCK ? launch_scan_local_blk_t<double>(a, ws, S(stream))
                                        : launch_scan_local_t<double, false>(a, ws, S(stream)))
        : one_pass ? launch_scan_1p_t<double>(scan_plan_1p(var, dtype, T, D), a, ws, S(stream))
                   : launch_scan_t<double>(p, a, ws, S(stream));
  } else {
    ScanArgs<float> a{(const float *)e0, (const float *)e1, (const float *)e2, (const float *)e3,
                      (const float *)u, (const float *)s0, (float *)out, T, D};
    a.probe = h_probe;
    a.probe_n = h_probe_n;
    e = local      ? (var == SCAN_BLOCK ? launch_scan_local_blk_t<float>(a, ws, S(stream))
                                        : launch_scan_local_t<float, false>(a, ws, S(stream)))
        : one_pass ? launch_scan_1p_t<float>(scan_plan_1p(var, dtype, T, D), a, ws, S(stream))
                   : launch_scan_t<float>(p, a, ws, S(stream));
  }
  return e == cudaSuccess ? CS_OK : cuda_fail(e, "scan launch");
}

int cs_scan_diag(int dtype, const void *j, const void *u, const void *s0, void *out, int64_t T,
                 int32_t D, void *ws, size_t ws_bytes, void *stream) {
  return do_scan(SCAN_DIAG, dtype, j, nullptr, nullptr, nullptr, u, s0, out, T, D, ws, ws_bytes, stream);
}
int cs_scan_block(int dtype, const void *a, const void *b, const void *c, const void *d, const void *u,
                  const void *s0, void *out, int64_t T, int32_t D, void *ws, size_t ws_bytes, void *stream) {
  return do_scan(SCAN_BLOCK, dtype, a, b, c, d, u, s0, out, T, D, ws, ws_bytes, stream);
}
int cs_scan_dense(int dtype, const void *J, const void *u, const void *s0, void *out, int64_t T,
                  int32_t D, void *ws, size_t ws_bytes, void *stream) {
  return do_scan(SCAN_DENSE, dtype, J, nullptr, nullptr, nullptr, u, s0, out, T, D, ws, ws_bytes, stream);
}

int cs_scan_aggregate(int mode, int dtype, const void *e0, const void *e1, const void *e2, const void *e3,
                      const void *u, int64_t T, int32_t D, double *agg_out, void *ws, size_t ws_bytes,
                      void *stream) {
  if (!dtype_ok(dtype)) return fail(CS_ERR_CONFIG, "bad dtype");
  if (T < 1 || D < 1) return fail(CS_ERR_STRUCTURAL, "bad aggregate shape");
  const int var = mode == CS_MODE_DIAG ? SCAN_DIAG : mode == CS_MODE_BLOCK ? SCAN_BLOCK : SCAN_DENSE;
  if (var == SCAN_DENSE && D > 8)
    return dense_wide_call(dtype, e0, u, nullptr, nullptr, T, D, ws, ws_bytes, agg_out, stream);
  const ScanPlan p = scan_plan(var, dtype, T, D);
  if (ws_bytes < p.ws_bytes) return fail(CS_ERR_CONFIG, "scan workspace too small");
  cudaError_t e;
  if (dtype == CS_F64) {
    ScanArgs<double> a{(const double *)e0, (const double *)e1, (const double *)e2, (const double *)e3,
                       (const double *)u, nullptr, nullptr, T, D};
    e = launch_aggregate_t<double>(p, a, ws, agg_out, S(stream));
  } else {
    ScanArgs<float> a{(const float *)e0, (const float *)e1, (const float *)e2, (const float *)e3,
                      (const float *)u, nullptr, nullptr, T, D};
    e = launch_aggregate_t<float>(p, a, ws, agg_out, S(stream));
  }
  return e == cudaSuccess ? CS_OK : cuda_fail(e, "aggregate launch");
}

// ---- building blocks -------------------------------------------------------------
int cs_first_stamped_row(const int32_t *last_fail, int64_t n, int32_t iteration, int64_t *d_first, void *stream) {
  if (!last_fail || !d_first || n < 0) return fail(CS_ERR_CONFIG, "bad arguments");
  k_set_i64<<<1, 1, 0, S(stream)>>>((long long *)d_first, kNoStep);
  if (n > 0) k_first_stamp<<<grid_for(n, 256), 256, 0, S(stream)>>>(last_fail, n, iteration, (long long *)d_first);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? CS_OK : cuda_fail(e, "cs_first_stamped_row");
}

int cs_first_nonfinite_row(int dtype, const void *x, int64_t n, int64_t width, int64_t *d_first,
                           void *stream) {
  if (!dtype_ok(dtype)) return fail(CS_ERR_CONFIG, "bad dtype");
  k_set_i64<<<1, 1, 0, S(stream)>>>((long long *)d_first, kNoStep);
  if (n * width > 0) {
    if (dtype == CS_F64)
      k_first_nonfinite<double><<<grid_for(n * width, 256), 256, 0, S(stream)>>>((const double *)x, n, width, (long long *)d_first);
    else
      k_first_nonfinite<float><<<grid_for(n * width, 256), 256, 0, S(stream)>>>((const float *)x, n, width, (long long *)d_first);
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? CS_OK : cuda_fail(e, "cs_first_nonfinite_row");
}

int cs_converged(int dtype, const void *prev, const void *next, int64_t n, double atol, double rtol,
                 uint32_t *d_notok, double *d_dmax, void *stream) {
  if (!dtype_ok(dtype)) return fail(CS_ERR_CONFIG, "bad dtype");
  cudaMemsetAsync(d_notok, 0, sizeof(uint32_t), S(stream));
  cudaMemsetAsync(d_dmax, 0, sizeof(double), S(stream));
  if (n > 0) {
    if (dtype == CS_F64)
      k_converged<double><<<grid_for(n, 256), 256, 0, S(stream)>>>((const double *)prev, (const double *)next, n, atol, rtol, d_notok, (unsigned long long *)d_dmax);
    else
      k_converged<float><<<grid_for(n, 256), 256, 0, S(stream)>>>((const float *)prev, (const float *)next, n, atol, rtol, d_notok, (unsigned long long *)d_dmax);
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? CS_OK : cuda_fail(e, "cs_converged");
}

int cs_update_bookkeeping(int dtype, const void *guess, const void *next, int64_t T, int32_t D,
                          double atol, double rtol, int32_t iteration, int32_t *last_fail,
                          uint32_t *d_fail_rows, double *d_dmax, void *stream) {
  if (!dtype_ok(dtype)) return fail(CS_ERR_CONFIG, "bad dtype");
  cudaMemsetAsync(d_fail_rows, 0, sizeof(uint32_t), S(stream));
  cudaMemsetAsync(d_dmax, 0, sizeof(double), S(stream));
  if (T > 0 && D >= 32) {
    const int64_t threads = T * 32;
    if (dtype == CS_F64)
      k_bookkeeping_wide<double><<<grid_for(threads, 256), 256, 0, S(stream)>>>((const double *)guess, (const double *)next, T, D, atol, rtol, iteration, last_fail, d_fail_rows, (unsigned long long *)d_dmax);
    else
      k_bookkeeping_wide<float><<<grid_for(threads, 256), 256, 0, S(stream)>>>((const float *)guess, (const float *)next, T, D, atol, rtol, iteration, last_fail, d_fail_rows, (unsigned long long *)d_dmax);
  } else if (T > 0) {
    if (dtype == CS_F64)
      k_bookkeeping<double><<<grid_for(T, 256), 256, 0, S(stream)>>>((const double *)guess, (const double *)next, T, D, atol, rtol, iteration, last_fail, d_fail_rows, (unsigned long long *)d_dmax);
    else
      k_bookkeeping<float><<<grid_for(T, 256), 256, 0, S(stream)>>>((const float *)guess, (const float *)next, T, D, atol, rtol, iteration, last_fail, d_fail_rows, (unsigned long long *)d_dmax);
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? CS_OK : cuda_fail(e, "cs_update_bookkeeping");
}

int cs_form_diag(int dtype, const void *est, const void *f, const void *s0, const void *guess, int64_t T,
                 int32_t D, const double *pre, double damping, double clip, void *j, void *u, void *stream) {
  if (!dtype_ok(dtype)) return fail(CS_ERR_CONFIG, "bad dtype");
  if (T * D == 0) return CS_OK;
  if (dtype == CS_F64)
    k_form_diag<double><<<grid_for(T * D, 256), 256, 0, S(stream)>>>((const double *)est, (const double *)f, (const double *)s0, (const double *)guess, T, D, pre, damping, clip, (double *)j, (double *)u);
  else
    k_form_diag<float><<<grid_for(T * D, 256), 256, 0, S(stream)>>>((const float *)est, (const float *)f, (const float *)s0, (const float *)guess, T, D, pre, damping, clip, (float *)j, (float *)u);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? CS_OK : cuda_fail(e, "cs_form_diag");
}

int cs_form_dense(int dtype, const void *J_in, const void *f, const void *s0, const void *guess, int64_t T,
                  int32_t D, const double *pre, double damping, double clip, void *J, void *u, void *stream) {
  if (!dtype_ok(dtype)) return fail(CS_ERR_CONFIG, "bad dtype");
  if (T == 0) return CS_OK;
  if (dtype == CS_F64)
    k_form_dense<double><<<grid_for(T, 128), 128, 0, S(stream)>>>((const double *)J_in, (const double *)f, (const double *)s0, (const double *)guess, T, D, pre, damping, clip, (double *)J, (double *)u);
  else
    k_form_dense<float><<<grid_for(T, 128), 128, 0, S(stream)>>>((const float *)J_in, (const float *)f, (const float *)s0, (const float *)guess, T, D, pre, damping, clip, (float *)J, (float *)u);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? CS_OK : cuda_fail(e, "cs_form_dense");
}

int cs_form_block(int dtype, const void *a_in, const void *b_in, const void *c_in, const void *d_in,
                  const void *f, const void *s0, const void *guess, int64_t T, int32_t D, const double *pre,
                  double damping, double clip, void *a, void *b, void *c, void *d, void *u, void *stream) {
  if (!dtype_ok(dtype)) return fail(CS_ERR_CONFIG, "bad dtype");
  if (T * D == 0) return CS_OK;
  if (dtype == CS_F64)
    k_form_block<double><<<grid_for(T * D, 256), 256, 0, S(stream)>>>(
        (const double *)a_in, (const double *)b_in, (const double *)c_in, (const double *)d_in, (const double *)f,
        (const double *)s0, (const double *)guess, T, D, pre, damping, clip, (double *)a, (double *)b, (double *)c,
        (double *)d, (double *)u);
  else
    k_form_block<float><<<grid_for(T * D, 256), 256, 0, S(stream)>>>(
        (const float *)a_in, (const float *)b_in, (const float *)c_in, (const float *)d_in, (const float *)f,
        (const float *)s0, (const float *)guess, T, D, pre, damping, clip, (float *)a, (float *)b, (float *)c,
        (float *)d, (float *)u);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? CS_OK : cuda_fail(e, "cs_form_block");
}

int cs_hutchinson_accumulate(int dtype, void *est, const void *z, const void *jz, int64_t n, int32_t first,
                             double final_div, void *stream) {
  if (!dtype_ok(dtype)) return fail(CS_ERR_CONFIG, "bad dtype");
  if (n == 0) return CS_OK;
  if (dtype == CS_F64)
    k_hutch<double><<<grid_for(n, 256), 256, 0, S(stream)>>>((double *)est, (const double *)z, (const double *)jz, n, first, final_div);
  else
    k_hutch<float><<<grid_for(n, 256), 256, 0, S(stream)>>>((float *)est, (const float *)z, (const float *)jz, n, first, final_div);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? CS_OK : cuda_fail(e, "cs_hutchinson_accumulate");
}

// ---- transition systems -------------------------------------------------------------
// a change of basis is fused into the MALA and HMC register kernels only
static bool basis_ok(const cs_system *sys) {
  return !sys->basis || sys->kind == CS_SYS_MALA || sys->kind == CS_SYS_HMC;
}

static int check_sys(const cs_system *sys, int dtype, int *md_out) {
  if (!sys) return fail(CS_ERR_CONFIG, "null system");
  if (!dtype_ok(dtype)) return fail(CS_ERR_CONFIG, "bad dtype");
  if (!basis_ok(sys)) return fail(CS_ERR_CONFIG, "a change of basis is fused into the MALA and HMC kernels only");
  int md = 0;
  if (sys->kind == CS_SYS_GIBBS) {
    md = sys->dim == 18 ? 18 : 0;
    if (!md) return fail(CS_ERR_CONFIG, "device GibbsKernel is built for the eight-schools layout (dim 18)");
  } else {
    if (sys->target.kind == CS_TARGET_BLR)
      return fail(CS_ERR_CONFIG, "logistic-regression targets run on the GEMM path (cs_blr), not the register path");
    md = api_md(sys->kind, sys->target.kind, sys->dim);
    if (!md) return fail(CS_ERR_CONFIG, "state dimension too large for the register-resident system kernels");
  }
  *md_out = md;
  return CS_OK;
}

int cs_system_supported(const cs_system *sys, int dtype) {
  if (!sys || !dtype_ok(dtype) || !basis_ok(sys)) return 0;
  if (sys->kind == CS_SYS_GIBBS) return sys->dim == 18 ? 1 : 0;
  if (sys->target.kind == CS_TARGET_BLR) return 0;
  return api_md(sys->kind, sys->target.kind, sys->dim) ? 1 : 0;
}

static int syscall(const cs_system *sys, int dtype, SysCall c, void *stream, const char *what) {
  int md = 0;
  int rc = check_sys(sys, dtype, &md);
  if (rc != CS_OK) return rc;
  if (c.op == 2 && sys->kind != CS_SYS_LEAPFROG)
    return fail(CS_ERR_CONFIG, "system does not provide a block2x2 Jacobian estimate");
  if (c.bad) k_set_i64<<<1, 1, 0, S(stream)>>>(c.bad, kNoStep);
  cudaError_t e = syscall_dispatch(*sys, dtype, md, c, S(stream));
  if (e == cudaErrorNotSupported) return fail(CS_ERR_CONFIG, "no kernel instantiated for this system/target/width");
  return e == cudaSuccess ? CS_OK : cuda_fail(e, what);
}

int cs_system_step(const cs_system *sys, int dtype, const int64_t *ts, int64_t t0, int64_t n, const void *Sx,
                   void *out, int64_t *bad_step, void *stream) {
  SysCall c{0, ts, t0, n, Sx, nullptr, out, nullptr, nullptr, nullptr, (long long *)bad_step, 0, 0, 0};
  return syscall(sys, dtype, c, stream, "cs_system_step");
}
int cs_system_relaxed_step(const cs_system *sys, int dtype, const int64_t *ts, int64_t t0, int64_t n,
                           const void *Sx, void *out, void *stream) {
  SysCall c{0, ts, t0, n, Sx, nullptr, out, nullptr, nullptr, nullptr, nullptr, 1, 0, 0};
  return syscall(sys, dtype, c, stream, "cs_system_relaxed_step");
}
int cs_system_jvp(const cs_system *sys, int dtype, const int64_t *ts, int64_t t0, int64_t n, const void *Sx,
                  const void *V, void *out, int32_t relaxed, void *stream) {
  SysCall c{1, ts, t0, n, Sx, V, out, nullptr, nullptr, nullptr, nullptr, relaxed, 0, 0};
  return syscall(sys, dtype, c, stream, "cs_system_jvp");
}
int cs_system_block_jacobian(const cs_system *sys, int dtype, const int64_t *ts, int64_t t0, int64_t n,
                             const void *Sx, int32_t n_samples, int64_t iteration, void *a, void *b, void *c,
                             void *d, void *stream) {
  if (n_samples < 1) return fail(CS_ERR_CONFIG, "hutchinson_samples must be >= 1");
  SysCall cc{2, ts, t0, n, Sx, nullptr, a, b, c, d, nullptr, 0, n_samples, iteration};
  return syscall(sys, dtype, cc, stream, "cs_system_block_jacobian");
}
int cs_system_sequential(const cs_system *sys, int dtype, const void *s0, int64_t T, void *out, int64_t *bad_step,
                         void *stream) {
  if (sys && dtype_ok(dtype) && !sys->basis && blr_mala_ok(*sys, CS_MODE_DIAG)) {
    // logistic-regression MALA: one CTA walks the chain with the target's data
    // products in the CTA (not the register path)
    k_set_i64<<<1, 1, 0, S(stream)>>>((long long *)bad_step, kNoStep);
    if (T < 1) return CS_OK;
    const cudaError_t e = blr_sequential(*sys, dtype, s0, T, out, (long long *)bad_step, S(stream));
    if (e == cudaErrorNotSupported) return fail(CS_ERR_CONFIG, "sequential walk: D <= 128 and N <= 4096 data rows");
    return e == cudaSuccess ? CS_OK : cuda_fail(e, "cs_system_sequential (logistic regression)");
  }
  SysCall c{3, nullptr, 1, T, s0, nullptr, out, nullptr, nullptr, nullptr, (long long *)bad_step, 0, 0, 0};
  return syscall(sys, dtype, c, stream, "cs_system_sequential");
}

// ---- fused element builder + update scans (the streamed solver path) ---------------
int cs_system_elements_supported(const cs_system *sys, int32_t mode, int dtype) {
  if (!sys || !dtype_ok(dtype)) return 0;
  if (sys->basis && (!basis_ok(sys) || mode == CS_MODE_BLOCK || sys->target.kind == CS_TARGET_BLR)) return 0;
  if (mode == CS_MODE_BLOCK && sys->kind != CS_SYS_LEAPFROG) return 0;
  int md = 0;
  if (sys->kind == CS_SYS_GIBBS) md = (sys->dim == 18 && mode == CS_MODE_DIAG) ? 18 : 0;
  else if (sys->target.kind != CS_TARGET_BLR) md = elem_md(sys->kind, sys->target.kind, sys->dim);
  return md > 0 || wide_leapfrog_ok(*sys, mode) || blr_mala_ok(*sys, mode) ? 1 : 0;
}

int cs_system_elements_range_supported(const cs_system *sys, const cs_deer_config *cfg, int dtype) {
  if (!sys || !cfg || !dtype_ok(dtype)) return 0;
  if (!cs_system_elements_supported(sys, cfg->mode, dtype)) return 0;
  if (sys->target.kind == CS_TARGET_BLR && sys->kind == CS_SYS_MALA)
    return blr_mala_ok(*sys, cfg->mode) && (cfg->mode == CS_MODE_DENSE || blr_fused_ok(*sys, *cfg)) ? 1 : 0;
  return !wide_leapfrog_ok(*sys, cfg->mode) || elem_md(sys->kind, sys->target.kind, sys->dim) > 0 ? 1 : 0;
}

static int elem_width(const cs_system *sys) {
  if (sys->kind == CS_SYS_GIBBS) return sys->dim == 18 ? 18 : 0;
  if (sys->target.kind == CS_TARGET_BLR) return 0;
  return elem_md(sys->kind, sys->target.kind, sys->dim);
}

int cs_system_elements(const cs_system *sys, const cs_deer_config *cfg, int dtype, int64_t iteration,
                       const void *s0, const void *guess, void *e0, void *e1, void *e2, void *e3, void *u,
                       cs_elem_stats *d_stats, void *stream) {
  if (!sys || !cfg || !d_stats) return fail(CS_ERR_CONFIG, "null argument");
  if (!dtype_ok(dtype)) return fail(CS_ERR_CONFIG, "bad dtype");
  if (sys->basis && !cs_system_elements_supported(sys, cfg->mode, dtype))
    return fail(CS_ERR_CONFIG, "a change of basis is fused into the MALA / HMC diag and dense builders only");
  const int md = elem_width(sys);
  const bool wide = !md && wide_leapfrog_ok(*sys, cfg->mode);
  const bool blr = !md && !wide && blr_mala_ok(*sys, cfg->mode);
  if (!md && !wide && !blr) return fail(CS_ERR_CONFIG, "no fused element builder for this system");
  if (cfg->mode == CS_MODE_BLOCK && sys->kind != CS_SYS_LEAPFROG)
    return fail(CS_ERR_CONFIG, "system does not provide a block2x2 Jacobian estimate");
  cudaStream_t st = S(stream);
  if (!wide || sys->T < 1) k_init_stats<<<1, 1, 0, st>>>(d_stats);  // (the wide prologue resets it itself)
  if (sys->T < 1) return CS_OK;
  cudaError_t e;
  if (wide) {
    e = elements_wide(*sys, *cfg, dtype, iteration, s0, guess, e0, e1, e2, e3, u, d_stats, st);
    return e == cudaSuccess ? CS_OK : cuda_fail(e, "cs_system_elements (wide leapfrog, cuBLAS)");
  }
  if (blr) {
    e = elements_blr(*sys, *cfg, dtype, iteration, s0, guess, e0, u, d_stats, st);
    return e == cudaSuccess ? CS_OK : cuda_fail(e, "cs_system_elements (logistic-regression MALA)");
  }
  if (dtype == CS_F64) {
    SolveArgs<double> A{};
    A.sys = *sys; A.mode = cfg->mode; A.max_iters = cfg->max_iters; A.nsamp = cfg->hutchinson_samples;
    A.atol = cfg->atol; A.rtol = cfg->rtol; A.damping = cfg->damping; A.clip = cfg->clip;
    A.pre = cfg->preconditioner; A.s0 = (const double *)s0; A.T = sys->T; A.D = sys->dim;
    e = elements_dispatch(*sys, dtype, md, cfg->mode, &A, (int)iteration, guess, e0, e1, e2, e3, u, d_stats, st);
  } else {
    SolveArgs<float> A{};
    A.sys = *sys; A.mode = cfg->mode; A.max_iters = cfg->max_iters; A.nsamp = cfg->hutchinson_samples;
    A.atol = cfg->atol; A.rtol = cfg->rtol; A.damping = cfg->damping; A.clip = cfg->clip;
    A.pre = cfg->preconditioner; A.s0 = (const float *)s0; A.T = sys->T; A.D = sys->dim;
    e = elements_dispatch(*sys, dtype, md, cfg->mode, &A, (int)iteration, guess, e0, e1, e2, e3, u, d_stats, st);
  }
  if (e == cudaErrorNotSupported) return fail(CS_ERR_CONFIG, "element builder not instantiated for this system/mode");
  return e == cudaSuccess ? CS_OK : cuda_fail(e, "cs_system_elements");
}

int cs_system_elements_range(const cs_system *sys, const cs_deer_config *cfg, int dtype, int64_t iteration,
                             int64_t t0, int64_t n, const void *s0, const void *guess, void *e0, void *e1, void *e2,
                             void *e3, void *u, cs_elem_stats *d_stats, void *stream) {
  if (!sys || !cfg || !d_stats) return fail(CS_ERR_CONFIG, "null argument");
  if (t0 < 0 || n < 0 || t0 + n > sys->T) return fail(CS_ERR_STRUCTURAL, "step range outside [1, T]");
  if (t0 == 0 && n == sys->T)
    return cs_system_elements(sys, cfg, dtype, iteration, s0, guess, e0, e1, e2, e3, u, d_stats, stream);
  if (sys->basis && !cs_system_elements_supported(sys, cfg->mode, dtype))
    return fail(CS_ERR_CONFIG, "a change of basis is fused into the MALA / HMC diag and dense builders only");
  if (!dtype_ok(dtype)) return fail(CS_ERR_CONFIG, "bad dtype");
  const int md = elem_width(sys);
  const bool blr = !md && blr_mala_ok(*sys, cfg->mode);
  if (!md && !blr)
    return fail(CS_ERR_CONFIG, "step ranges need a register-kernel system or the logistic-regression builders "
                               "(the wide leapfrog builder takes whole chains)");
  if (cfg->mode == CS_MODE_BLOCK && sys->kind != CS_SYS_LEAPFROG)
    return fail(CS_ERR_CONFIG, "system does not provide a block2x2 Jacobian estimate");
  cudaStream_t st = S(stream);
  k_init_stats<<<1, 1, 0, st>>>(d_stats);
  if (n < 1) return CS_OK;
  cudaError_t e;
  if (blr) {
    if (blr_fused_ok(*sys, *cfg)) {
      e = elements_blr_fused(*sys, *cfg, dtype, iteration, t0, n, s0, guess, e0, u, d_stats, st);
    } else {
      // the dense (and many-probe) pipelines index noise by local row: hand them
      // the shard as a chain of n steps whose noise tables start at step t0 + 1
      // (their probes, the many-probe diag case, hash the local step: refused)
      if (cfg->mode != CS_MODE_DENSE)
        return fail(CS_ERR_CONFIG, "step ranges of the logistic-regression diag builder need <= 7 probes");
      cs_system loc = *sys;
      loc.T = n;
      loc.noise_vec = (const char *)sys->noise_vec + (size_t)t0 * sys->dim * esize(dtype);
      loc.noise_logu = sys->noise_logu + t0;
      e = elements_blr(loc, *cfg, dtype, iteration, s0, guess, e0, u, d_stats, st);
    }
    return e == cudaSuccess ? CS_OK : cuda_fail(e, "cs_system_elements_range (logistic-regression MALA)");
  }
  if (dtype == CS_F64) {
    SolveArgs<double> A{};
    A.sys = *sys; A.mode = cfg->mode; A.max_iters = cfg->max_iters; A.nsamp = cfg->hutchinson_samples;
    A.atol = cfg->atol; A.rtol = cfg->rtol; A.damping = cfg->damping; A.clip = cfg->clip;
    A.pre = cfg->preconditioner; A.s0 = (const double *)s0; A.T = n; A.D = sys->dim; A.t0 = t0;
    e = elements_dispatch(*sys, dtype, md, cfg->mode, &A, (int)iteration, guess, e0, e1, e2, e3, u, d_stats, st);
  } else {
    SolveArgs<float> A{};
    A.sys = *sys; A.mode = cfg->mode; A.max_iters = cfg->max_iters; A.nsamp = cfg->hutchinson_samples;
    A.atol = cfg->atol; A.rtol = cfg->rtol; A.damping = cfg->damping; A.clip = cfg->clip;
    A.pre = cfg->preconditioner; A.s0 = (const float *)s0; A.T = n; A.D = sys->dim; A.t0 = t0;
    e = elements_dispatch(*sys, dtype, md, cfg->mode, &A, (int)iteration, guess, e0, e1, e2, e3, u, d_stats, st);
  }
  if (e == cudaErrorNotSupported) return fail(CS_ERR_CONFIG, "element builder not instantiated for this system/mode");
  return e == cudaSuccess ? CS_OK : cuda_fail(e, "cs_system_elements_range");
}

static int do_scan_update(int var, int dtype, const void *e0, const void *e1, const void *e2, const void *e3,
                          const void *u, const void *s0, void *out, int64_t T, int D, void *ws, size_t ws_bytes,
                          const void *guess, double atol, double rtol, int it, int32_t *last_fail,
                          cs_elem_stats *stats, void *stream) {
  if (!dtype_ok(dtype)) return fail(CS_ERR_CONFIG, "bad dtype");
  if (T < 0 || D < 1 || D > 4096) return fail(CS_ERR_STRUCTURAL, "bad scan shape");
  const ScanPlan p = scan_plan(var, dtype, T, D, true);
  if (ws_bytes < p.ws_bytes) return fail(CS_ERR_CONFIG, "scan workspace too small");
  if (T == 0) return CS_OK;
  {  // out and guess must not overlap (guess is read through the read-only path)
    const size_t nb = (size_t)T * (size_t)D * (var == SCAN_BLOCK ? 2 : 1) * (size_t)esize(dtype);
    const uintptr_t o0 = (uintptr_t)out, g0 = (uintptr_t)guess;
    if (guess && o0 < g0 + nb && g0 < o0 + nb) return fail(CS_ERR_CONFIG, "scan update: out overlaps guess");
  }
  // very long diag scans: the local scan + fix-up with the bookkeeping on each tile's
  // final states.  Newton iterates' maps often contract slowly, so the fix-up covers
  // much of each range and the two-pass scan stays ahead at moderate T (cfg 5, T = 1M:
  // 79.0 -> 83.9 ms per solve with the local scan)
  const bool local = T >= ((int64_t)1 << 22) && var == SCAN_DIAG && scan_local_eligible(var, T, D) &&
                     ws_bytes >= scan_local_ws_bytes(dtype, T, D);
  // reduce-then-replay (default everywhere from 2^16): the local scan's per-tile
  // bookkeeping is latency-bound on its guess loads -- T = 2^22 / 2^24, D = 18:
  // 0.89 / 3.40 ms local vs 0.35 / 1.30 ms (tools/update_scan_time.py)
  static const int rr_mode = [] {  // 0 off, 1 below the local scan's range, 2 everywhere
    const char *e = getenv("CS_SCAN_RR");
    return e ? atoi(e) : 2;
  }();
  const bool rr = (rr_mode == 2 || (rr_mode == 1 && !local)) && scan_rr_eligible(var, T, D) &&
                  ws_bytes >= scan_rr_ws_bytes(dtype, T, D);
  cudaError_t e;
  if (dtype == CS_F64) {
    ScanArgs<double> a{(const double *)e0, (const double *)e1, (const double *)e2, (const double *)e3,
                       (const double *)u, (const double *)s0, (double *)out, T, D, (const double *)guess,
                       atol, rtol, it, last_fail, stats};
    e = rr      ? launch_scan_rr_t<double, true>(a, ws, S(stream))
        : local ? launch_scan_local_t<double, true>(a, ws, S(stream))
              : launch_scan_t<double>(p, a, ws, S(stream), true);
  } else {
    ScanArgs<float> a{(const float *)e0, (const float *)e1, (const float *)e2, (const float *)e3,
                      (const float *)u, (const float *)s0, (float *)out, T, D, (const float *)guess,
                      atol, rtol, it, last_fail, stats};
    e = rr      ? launch_scan_rr_t<float, true>(a, ws, S(stream))
        : local ? launch_scan_local_t<float, true>(a, ws, S(stream))
              : launch_scan_t<float>(p, a, ws, S(stream), true);
  }
  return e == cudaSuccess ? CS_OK : cuda_fail(e, "scan update launch");
}

int cs_scan_diag_update(int dtype, const void *j, const void *u, const void *s0, void *out, int64_t T, int32_t D,
                        void *ws, size_t ws_bytes, const void *guess, double atol, double rtol, int32_t iteration,
                        int32_t *last_fail, cs_elem_stats *d_stats, void *stream) {
  return do_scan_update(SCAN_DIAG, dtype, j, nullptr, nullptr, nullptr, u, s0, out, T, D, ws, ws_bytes, guess, atol,
                        rtol, iteration, last_fail, d_stats, stream);
}
int cs_scan_block_update(int dtype, const void *a, const void *b, const void *c, const void *d, const void *u,
                         const void *s0, void *out, int64_t T, int32_t D, void *ws, size_t ws_bytes,
                         const void *guess, double atol, double rtol, int32_t iteration, int32_t *last_fail,
                         cs_elem_stats *d_stats, void *stream) {
  return do_scan_update(SCAN_BLOCK, dtype, a, b, c, d, u, s0, out, T, D, ws, ws_bytes, guess, atol, rtol,
                        iteration, last_fail, d_stats, stream);
}

// ---- whole-chain solve ------------------------------------------------------------
static int solver_width(const cs_system *sys) {
  if (sys->kind == CS_SYS_GIBBS) return sys->dim == 18 ? 18 : 0;
  if (sys->target.kind == CS_TARGET_BLR) return 0;
  return solve_md(sys->kind, sys->target.kind, sys->dim);
}

int cs_deer_supported(const cs_system *sys, int mode, int dtype) {
  if (!sys || !dtype_ok(dtype) || sys->basis) return 0;  // bases run on the streamed engine
  const int md = solver_width(sys);
  if (!md) return 0;
  if (mode == CS_MODE_BLOCK && sys->kind != CS_SYS_LEAPFROG) return 0;
  return 1;
}

int cs_leapfrog_batch_supported(const cs_system *sys, int32_t mode, int dtype) {
  return sys && dtype_ok(dtype) && (leapfrog_batch_ok(*sys, mode) || wide_leapfrog_ok(*sys, mode)) ? 1 : 0;
}

int cs_leapfrog_batch_solve(const cs_system *sys, const cs_deer_config *cfg, int dtype, int32_t B, const void *s0s,
                            void *finals, int32_t *info, int64_t *err_step, void *stream) {
  if (!sys || !cfg || !info || !err_step) return fail(CS_ERR_CONFIG, "null argument");
  if (!dtype_ok(dtype)) return fail(CS_ERR_CONFIG, "bad dtype");
  const bool narrow = leapfrog_batch_ok(*sys, cfg->mode);
  if (!narrow && !wide_leapfrog_ok(*sys, cfg->mode))
    return fail(CS_ERR_CONFIG, "batched leapfrog solve: unsupported system/mode");
  if (cfg->max_iters < 1 || cfg->hutchinson_samples < 1 || !(cfg->atol > 0) || !(cfg->rtol >= 0) ||
      !(cfg->damping > 0 && cfg->damping <= 1) || !(cfg->clip > 0))
    return fail(CS_ERR_CONFIG, "bad solver configuration");
  if (B < 0) return fail(CS_ERR_STRUCTURAL, "negative batch");
  if (B == 0) return CS_OK;
  // register-width trajectories: one CTA per proposal; dense Gaussian targets
  // of any width (cfg 4): all proposals' passes share one DMMA GEMM per iteration
  const cudaError_t e =
      narrow ? leapfrog_batch_solve(*sys, *cfg, dtype, B, s0s, finals, info, (long long *)err_step, S(stream))
             : wide_batch_solve(*sys, *cfg, dtype, B, s0s, finals, info, (long long *)err_step, S(stream));
  return e == cudaSuccess ? CS_OK : cuda_fail(e, "batched leapfrog solve");
}

size_t cs_deer_workspace_bytes(const cs_system *sys, int dtype, int32_t max_iters) {
  (void)max_iters;
  if (!sys) return 0;
  const int md = solver_width(sys);
  const int W = md * md + md;
  const size_t T = (size_t)sys->T, D = (size_t)sys->dim;
  return al(T * D * esize(dtype)) + al(sizeof(SolveCtl)) + al(sizeof(double) * 2 * kAggReplicas * 8 * (size_t)sm_count() * (W > 0 ? W : 1)) +
         al(sizeof(int) * 8 * (size_t)sm_count());
}

int cs_deer_solve(const cs_system *sys, const cs_deer_config *cfg, int dtype, const void *s0, void *trace,
                  int32_t *per_step_converged_at, double *delta_history, void *ws, size_t ws_bytes,
                  cs_deer_result *res, void *stream) {
  if (!sys || !cfg || !res) return fail(CS_ERR_CONFIG, "null argument");
  if (!dtype_ok(dtype)) return fail(CS_ERR_CONFIG, "bad dtype");
  if (cfg->mode < 0 || cfg->mode > 2) return fail(CS_ERR_CONFIG, "unknown mode");
  if (!(cfg->atol > 0) || !(cfg->rtol >= 0)) return fail(CS_ERR_CONFIG, "need atol > 0 and rtol >= 0");
  if (cfg->max_iters < 1) return fail(CS_ERR_CONFIG, "max_iters must be >= 1");
  if (cfg->hutchinson_samples < 1) return fail(CS_ERR_CONFIG, "hutchinson_samples must be >= 1");
  if (!(cfg->damping > 0 && cfg->damping <= 1)) return fail(CS_ERR_CONFIG, "damping must lie in (0, 1]");
  if (!(cfg->clip > 0)) return fail(CS_ERR_CONFIG, "clip must be positive");
  if (!cs_deer_supported(sys, cfg->mode, dtype))
    return fail(CS_ERR_CONFIG, "system/mode not handled by the fused solver (use the host-driven path)");
  if (sys->T < 1) return fail(CS_ERR_CONFIG, "T must be >= 1");
  const size_t need = cs_deer_workspace_bytes(sys, dtype, cfg->max_iters);
  if (ws_bytes < need) return fail(CS_ERR_CONFIG, "solver workspace too small");
  const int md = solver_width(sys);
  const int64_t T = sys->T;
  const int D = sys->dim;
  cudaStream_t st = S(stream);
  const int sms = sm_count();
  SolveState *ss = nullptr;
  {
    static std::mutex mu;
    static std::vector<SolveState *> states;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    const std::thread::id me = std::this_thread::get_id();
    for (SolveState *x : states)
      if (x->dev == dev && x->st == st && x->host == me) ss = x;
    if (!ss) {
      SolveState n{};
      n.dev = dev;
      n.st = st;
      n.host = me;
      cudaError_t e = cudaMalloc(&n.ctl, sizeof(SolveCtl) + sizeof(int) * kReadyStride * 8 * (size_t)sms);
      if (e == cudaSuccess) e = cudaHostAlloc(&n.out, sizeof(SolveOut), cudaHostAllocMapped);
      if (e == cudaSuccess) memset((void *)n.out, 0, sizeof(SolveOut));  // seq 0: no solve signalled yet
      if (e == cudaSuccess) e = cudaEventCreate(&n.ev0);
      if (e == cudaSuccess) e = cudaEventCreate(&n.ev1);
      if (e != cudaSuccess) return cuda_fail(e, "solver state");
      n.ready = (int *)(n.ctl + 1);
      std::vector<SolveCtl> z(1);
      memset(z.data(), 0, sizeof(SolveCtl));
      for (int q = 0; q < 4; ++q)
        for (int g = 0; g < kMaxSlotGroups; ++g)
          z[0].slot[q][g].bad_prop = z[0].slot[q][g].bad_f = z[0].slot[q][g].bad_jac = kNoStep;
      e = cudaMemcpy(n.ctl, z.data(), sizeof(SolveCtl), cudaMemcpyHostToDevice);
      if (e == cudaSuccess) e = cudaMemset(n.ready, 0, sizeof(int) * kReadyStride * 8 * (size_t)sms);
      if (e != cudaSuccess) return cuda_fail(e, "solver state init");
      ss = new SolveState(n);
      states.push_back(ss);
    }
  }
  unsigned char *w = (unsigned char *)ws;
  void *G1 = w;
  w += al((size_t)T * D * esize(dtype));
  w += al(sizeof(SolveCtl));
  double *agg = (double *)w;
  SolvePick pick{};
  cudaError_t e;
  const unsigned seq = ++ss->seq;
  if (dtype == CS_F64) {
    SolveArgs<double> A{};
    A.sys = *sys; A.mode = cfg->mode; A.max_iters = cfg->max_iters; A.nsamp = cfg->hutchinson_samples;
    A.atol = cfg->atol; A.rtol = cfg->rtol; A.damping = cfg->damping; A.clip = cfg->clip;
    A.pre = cfg->preconditioner; A.s0 = (const double *)s0; A.G0 = (double *)trace; A.G1 = (double *)G1;
    A.last_fail = per_step_converged_at; A.hist = delta_history; A.ctl = ss->ctl; A.out = ss->out; A.agg = agg;
    A.seq = seq;
    A.ready = ss->ready; A.probe = h_probe; A.probe_n = h_probe_n; A.T = T; A.D = D;
    e = solve_dispatch(*sys, dtype, md, cfg->mode, &A, sms, st, &pick);
  } else {
    SolveArgs<float> A{};
    A.sys = *sys; A.mode = cfg->mode; A.max_iters = cfg->max_iters; A.nsamp = cfg->hutchinson_samples;
    A.atol = cfg->atol; A.rtol = cfg->rtol; A.damping = cfg->damping; A.clip = cfg->clip;
    A.pre = cfg->preconditioner; A.s0 = (const float *)s0; A.G0 = (float *)trace; A.G1 = (float *)G1;
    A.last_fail = per_step_converged_at; A.hist = delta_history; A.ctl = ss->ctl; A.out = ss->out; A.agg = agg;
    A.seq = seq;
    A.ready = ss->ready; A.probe = h_probe; A.probe_n = h_probe_n; A.T = T; A.D = D;
    e = solve_dispatch(*sys, dtype, md, cfg->mode, &A, sms, st, &pick);
  }
  if (e == cudaErrorNotSupported) return fail(CS_ERR_CONFIG, "fused solver not instantiated for this system");
  if (e != cudaSuccess) return cuda_fail(e, "cooperative solve launch");
  cudaEventRecord(ss->ev1, st);
  // the kernel writes its outcome straight into host-mapped memory and signals
  // it with the sequence number: spin on that word (it lands before the grid's
  // last CTAs retire; everything after is stream-ordered), polling the event
  // now and then so a failed launch cannot hang the host
  const volatile unsigned *sig = (const volatile unsigned *)&ss->out->seq;
  for (unsigned n = 1; *sig != seq; ++n) {
    if ((n & 1023u) == 0u) {
      e = cudaEventQuery(ss->ev1);
      if (e == cudaErrorNotReady) continue;
      if (e != cudaSuccess) return cuda_fail(e, "solve");
      if (*sig != seq) return fail(CS_ERR_CUDA, "solve finished without its outcome record");
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  SolveOut h;
  memcpy(&h, (const void *)ss->out, sizeof h);
  const float ms = (float)((double)(h.t_end - h.t_start) * 1e-6);
  res->iterations = h.iterations;
  res->status = h.status;
  res->err_kind = h.err_kind;
  res->err_step = h.err_step;
  res->err_iteration = h.err_iter;
  res->launches = 1;
  res->guard_dmax = h.guard_dmax;
  res->guard_d0 = h.guard_d0;
  res->stop_reason = h.stop;
  res->grid_blocks = pick.nblocks;
  res->steps_per_thread = pick.seg;
  res->kept_in_registers = pick.keep;
  res->fused_tangent = pick.fused_tangent;
  res->device_ms = ms;
  if (h.status == CS_RUN_DIVERGED) {
    char buf[256];
    snprintf(buf, sizeof buf, "chain diverged (kind %d) at step %lld, iteration %d", h.err_kind,
             (long long)h.err_step, h.err_iter);
    return fail(CS_ERR_DIVERGED, buf);
  }
  return CS_OK;
}

}  // extern "C"
