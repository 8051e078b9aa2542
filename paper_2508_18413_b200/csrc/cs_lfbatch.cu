// Every proposal's inner leapfrog solve of an HMC chain in parallel-leapfrog
// mode, batched on the device (samplers.py:301-320 HmcKernel._integrate_parallel;
// SURVEY.md 8f item 2).  The reference runs one run_deer per chain row, one
// after another; here one CTA owns one proposal -- thread t owns leapfrog step
// t of the L-step trajectory -- and runs the whole Newton loop of deer.py:
// 259-286 for it (forward pass, finite check, Picard pre-check, max_iters,
// block2x2 element with the Hutchinson probes of samplers.py:202-222, CTA scan,
// update bookkeeping, divergence guard), so B proposals cost one launch.  Each
// chain stops on its own, exactly as its own run_deer would; rows that fail to
// converge are reported for the caller's sequential fallback.
#include "cs_apikern.cuh"

namespace cs {

namespace {

constexpr int kLfbThreads = kSolveThreads;  // trajectory steps per CTA (L <= 256)

template <int MD, typename ST, int TK>
__global__ void __launch_bounds__(kLfbThreads)
k_leapfrog_batch(SolveArgs<ST> A, int B, const ST *s0s, ST *finals, int32_t *info, long long *err_step) {
  using Sys = Leapfrog<MD, ST, TK>;
  using E = Elem<CS_MODE_BLOCK, MD>;
  const Sys sys = make_leapfrog<MD, ST, TK>(A.sys);
  __shared__ double rows[kLfbThreads * MD];
  __shared__ E s_warp[kLfbThreads / 32 + 1];
  __shared__ long long s_bad[2];
  __shared__ unsigned s_fail[2];
  __shared__ unsigned long long s_dm;
  const int L = (int)A.T, D = A.D, tid = threadIdx.x;
  const bool act = tid < L;
  const int64_t t = tid + 1;
  for (int b = blockIdx.x; b < B; b += gridDim.x) {
    double s0r[MD], g[MD];
    load_row<Sys, MD, ST>(sys, s0s + (int64_t)b * D, s0r);
#pragma unroll
    for (int i = 0; i < MD; ++i) g[i] = s0r[i];  // guess = tile(s0)
    int it = 0, status = CS_RUN_MAXITERS, kind = CS_DIV_NONE, eit = -1;
    long long estep = -1;
    double d0 = -1.0;
    for (;;) {
      // prev = [s0; guess[:-1]]: each thread publishes its row, reads its predecessor's
#pragma unroll
      for (int i = 0; i < MD; ++i) rows[tid * MD + i] = g[i];
      if (tid == 0) {
        s_bad[0] = s_bad[1] = kNoStep;
        s_fail[0] = s_fail[1] = 0u;
        s_dm = 0ull;
      }
      __syncthreads();
      double prev[MD];
#pragma unroll
      for (int i = 0; i < MD; ++i) prev[i] = tid == 0 ? s0r[i] : rows[(tid - 1) * MD + i];
      typename Sys::Aux aux;
      double f[MD];
      bool pfail = false;
      E e;
      e.ident();
      bool jok = true;
      if (act) {
        sys.prepare(t, prev, aux);
        sys.f(aux, f);
        bool fin = true;
#pragma unroll
        for (int i = 0; i < MD; ++i) {
          if (sys.mem_index(i) < 0) continue;
          fin &= finite(f[i]);
          pfail |= !(fabs(f[i] - g[i]) <= A.atol + A.rtol * fabs(f[i]));
        }
        if (!fin) atomicMin(&s_bad[0], (long long)t);
        if (pfail) atomicAdd(&s_fail[0], 1u);
        if (it < A.max_iters) {
          build_elem<Sys, CS_MODE_BLOCK, MD, ST>(sys, aux, prev, f, t, it, A, e, jok);
          if (!jok) atomicMin(&s_bad[1], (long long)t);
        }
      }
      __syncthreads();
      // deer.py:264-270, in order
      if (s_bad[0] != kNoStep) { status = CS_RUN_DIVERGED; kind = CS_DIV_STEP; estep = s_bad[0]; eit = it + 1; break; }
      if (s_fail[0] == 0u) { status = CS_RUN_CONVERGED; break; }
      if (it >= A.max_iters) { status = CS_RUN_MAXITERS; break; }
      if (s_bad[1] != kNoStep) { status = CS_RUN_DIVERGED; kind = CS_DIV_JACOBIAN; estep = s_bad[1]; eit = it + 1; break; }
      // the affine solve over the trajectory: CTA scan of the step elements
      E excl, total;
      block_scan(e, excl, total, s_warp);
      double x[MD];
#pragma unroll
      for (int i = 0; i < MD; ++i) x[i] = s0r[i];
      excl.apply(x);
      e.apply(x);
      ++it;
      bool fail = false;
      unsigned long long dmb = 0ull;
      if (act) {
#pragma unroll
        for (int i = 0; i < MD; ++i) {
          if (sys.mem_index(i) < 0) continue;
          const double xs = (double)(ST)x[i];  // the stored iterate
          const double gap = fabs(xs - g[i]);
          fail |= gap > A.atol + A.rtol * fabs(xs);
          const unsigned long long gb = (unsigned long long)__double_as_longlong(gap);
          dmb = gb > dmb ? gb : dmb;
          g[i] = xs;
        }
      }
      dmb = warp_max_u64(dmb);
      if ((tid & 31) == 0) atomicMax(&s_dm, dmb);
      if (fail) atomicAdd(&s_fail[1], 1u);
      __syncthreads();
      const double dmax = __longlong_as_double((long long)s_dm);
      if (d0 < 0.0) d0 = dmax;
      if (d0 > 0.0 && dmax > 1e6 * d0) { status = CS_RUN_DIVERGED; kind = CS_DIV_GUARD; eit = it; break; }
      if (s_fail[1] == 0u) { status = CS_RUN_CONVERGED; break; }
      __syncthreads();  // s_fail / s_dm are reset at the top of the next pass
    }
    if (tid == L - 1) {
#pragma unroll
      for (int i = 0; i < MD; ++i) {
        const int m = sys.mem_index(i);
        if (m >= 0) finals[(int64_t)b * D + m] = (ST)g[i];
      }
    }
    if (tid == 0) {
      info[4 * b + 0] = status;
      info[4 * b + 1] = it;
      info[4 * b + 2] = kind;
      info[4 * b + 3] = eit;
      err_step[b] = estep;
    }
    __syncthreads();
  }
}

template <int MD, typename ST, int TK>
cudaError_t launch_lfb(const SolveArgs<ST> &A, int B, const void *s0s, void *finals, int32_t *info,
                       long long *err_step, cudaStream_t st) {
  const int grid = B < 148 * 8 ? B : 148 * 8;
  k_leapfrog_batch<MD, ST, TK><<<grid, kLfbThreads, 0, st>>>(A, B, (const ST *)s0s, (ST *)finals, info, err_step);
  return cudaGetLastError();
}

template <typename ST>
cudaError_t lfb_dispatch(int tk, const SolveArgs<ST> &A, int B, const void *s0s, void *finals, int32_t *info,
                         long long *err_step, cudaStream_t st) {
  switch (tk) {
    case CS_TARGET_STD_NORMAL: return launch_lfb<4, ST, 0>(A, B, s0s, finals, info, err_step, st);
    case CS_TARGET_GAUSSIAN: return launch_lfb<4, ST, 1>(A, B, s0s, finals, info, err_step, st);
    case CS_TARGET_ROSENBROCK: return launch_lfb<4, ST, 2>(A, B, s0s, finals, info, err_step, st);
    case CS_TARGET_MOG: return launch_lfb<4, ST, 3>(A, B, s0s, finals, info, err_step, st);
  }
  return cudaErrorNotSupported;
}

}  // namespace

bool leapfrog_batch_ok(const cs_system &s, int mode) {
  return s.kind == CS_SYS_LEAPFROG && mode == CS_MODE_BLOCK && s.T >= 1 && s.T <= kLfbThreads &&
         s.target.kind >= CS_TARGET_STD_NORMAL && s.target.kind <= CS_TARGET_MOG && s.dim >= 2 && s.dim <= 4 &&
         s.dim % 2 == 0;
}

cudaError_t leapfrog_batch_solve(const cs_system &sys, const cs_deer_config &cfg, int dtype, int B, const void *s0s,
                                 void *finals, int32_t *info, long long *err_step, cudaStream_t st) {
  if (dtype == CS_F64) {
    SolveArgs<double> A{};
    A.sys = sys; A.mode = CS_MODE_BLOCK; A.max_iters = cfg.max_iters; A.nsamp = cfg.hutchinson_samples;
    A.atol = cfg.atol; A.rtol = cfg.rtol; A.damping = cfg.damping; A.clip = cfg.clip; A.pre = cfg.preconditioner;
    A.T = sys.T; A.D = sys.dim; A.seg = 1; A.nblocks = 1;
    return lfb_dispatch<double>(sys.target.kind, A, B, s0s, finals, info, err_step, st);
  }
  SolveArgs<float> A{};
  A.sys = sys; A.mode = CS_MODE_BLOCK; A.max_iters = cfg.max_iters; A.nsamp = cfg.hutchinson_samples;
  A.atol = cfg.atol; A.rtol = cfg.rtol; A.damping = cfg.damping; A.clip = cfg.clip; A.pre = cfg.preconditioner;
  A.T = sys.T; A.D = sys.dim; A.seg = 1; A.nblocks = 1;
  return lfb_dispatch<float>(sys.target.kind, A, B, s0s, finals, info, err_step, st);
}

}  // namespace cs
