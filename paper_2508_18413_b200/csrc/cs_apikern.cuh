// Batched TransitionSystem entry points (core.py:104-152) as one-thread-per-row
// kernels over the fused system objects, plus the sequential chain walk
// (core.py:163-184) and the persistent-solver launcher.
#pragma once
#include "cs_solver.cuh"

namespace cs {

constexpr int kRowThreads = 128;

template <class Sys, int MD, typename ST>
CS_D void load_row_ro(const Sys &sys, const ST *row, double (&x)[MD]) {
#pragma unroll
  for (int k = 0; k < MD; ++k) {
    const int m = sys.mem_index(k);
    x[k] = m >= 0 ? (double)row[m] : 0.0;
  }
}
template <class Sys, int MD, typename ST>
CS_D void store_row(const Sys &sys, ST *row, const double (&x)[MD]) {
#pragma unroll
  for (int k = 0; k < MD; ++k) {
    const int m = sys.mem_index(k);
    if (m >= 0) row[m] = (ST)x[k];
  }
}

template <class Sys, int MD, typename ST>
__global__ void __launch_bounds__(kRowThreads)
k_sys_step(cs_system s, const int64_t *ts, int64_t t0, int64_t n, const ST *S, ST *out,
           long long *bad, int relaxed) {
  const int64_t i = (int64_t)blockIdx.x * kRowThreads + threadIdx.x;
  if (i >= n) return;
  const Sys sys = SysFactory<Sys>::make(s);
  const int D = s.dim;
  const int64_t t = ts ? ts[i] : t0 + i;
  double x[MD], f[MD];
  load_row_ro<Sys, MD, ST>(sys, S + i * D, x);
  if (s.basis) {  // z -> Q' f(Q z)
    double z[MD];
#pragma unroll
    for (int k = 0; k < MD; ++k) z[k] = x[k];
    basis_in<Sys, MD>(sys, s.basis, D, z, x);
  }
  typename Sys::Aux aux;
  const bool ok = sys.prepare(t, x, aux);
  if (!ok && bad) atomicMin(bad, (long long)t);
  if (relaxed) sys.relaxed_f(aux, f);
  else sys.f(aux, f);
  if (s.basis) {
    double fx[MD];
#pragma unroll
    for (int k = 0; k < MD; ++k) fx[k] = f[k];
    basis_out<Sys, MD>(sys, s.basis, D, fx, f);
  }
  store_row<Sys, MD, ST>(sys, out + i * D, f);
}

template <class Sys, int MD, typename ST>
__global__ void __launch_bounds__(kRowThreads)
k_sys_jvp(cs_system s, const int64_t *ts, int64_t t0, int64_t n, const ST *S, const ST *V,
          ST *out, int relaxed) {
  const int64_t i = (int64_t)blockIdx.x * kRowThreads + threadIdx.x;
  if (i >= n) return;
  const Sys sys = SysFactory<Sys>::make(s);
  const int D = s.dim;
  const int64_t t = ts ? ts[i] : t0 + i;
  double x[MD], v[1][MD], o[1][MD];
  load_row_ro<Sys, MD, ST>(sys, S + i * D, x);
  load_row_ro<Sys, MD, ST>(sys, V + i * D, v[0]);
  if (s.basis) {
    double z[MD];
#pragma unroll
    for (int k = 0; k < MD; ++k) z[k] = x[k];
    basis_in<Sys, MD>(sys, s.basis, D, z, x);
  }
  typename Sys::Aux aux;
  sys.prepare(t, x, aux);
  jvp_basis<1, double>(sys, s.basis, D, aux, v, o, 1, relaxed != 0);
  store_row<Sys, MD, ST>(sys, out + i * D, o[0]);
}

template <class Sys, int MD, typename ST>
__global__ void __launch_bounds__(kRowThreads)
k_sys_block(cs_system s, const int64_t *ts, int64_t t0, int64_t n, const ST *S, int nsamp,
            int64_t iteration, ST *a, ST *b, ST *c, ST *d) {
  if constexpr (HasBlock<Sys>::value) {
    const int64_t i = (int64_t)blockIdx.x * kRowThreads + threadIdx.x;
    if (i >= n) return;
    const Sys sys = SysFactory<Sys>::make(s);
    constexpr int H = MD / 2;
    const int h = s.dim / 2;
    const int64_t t = ts ? ts[i] : t0 + i;
    double x[MD];
    load_row_ro<Sys, MD, ST>(sys, S + i * s.dim, x);
    typename Sys::Aux aux;
    sys.prepare(t, x, aux);
    double ba[H], bb[H], bc[H], bd[H];
    sys.block(aux, t, nsamp, iteration, ba, bb, bc, bd);
#pragma unroll
    for (int k = 0; k < H; ++k)
      if (k < h) {
        a[i * h + k] = (ST)ba[k];
        b[i * h + k] = (ST)bb[k];
        c[i * h + k] = (ST)bc[k];
        d[i * h + k] = (ST)bd[k];
      }
  }
}

// sequential_evaluate: one thread walks the chain; stops at the first
// non-finite proposal/state (core.py:178-182, samplers.py:101-105).
template <class Sys, int MD, typename ST>
__global__ void k_sys_seq(cs_system s, const ST *s0, int64_t T, ST *out, long long *bad) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  const Sys sys = SysFactory<Sys>::make(s);
  const int D = s.dim;
  double x[MD];
  load_row_ro<Sys, MD, ST>(sys, s0, x);
  for (int64_t t = 1; t <= T; ++t) {
    typename Sys::Aux aux;
    bool ok;
    if (s.basis) {  // the chain in z coordinates: z_t = Q' f(Q z_{t-1})
      double xs[MD], fx[MD];
      basis_in<Sys, MD>(sys, s.basis, D, x, xs);
      ok = sys.prepare(t, xs, aux);
      sys.f(aux, fx);
      basis_out<Sys, MD>(sys, s.basis, D, fx, x);
    } else {
      ok = sys.prepare(t, x, aux);
      sys.f(aux, x);
    }
#pragma unroll
    for (int k = 0; k < MD; ++k)
      if (sys.mem_index(k) >= 0) ok &= finite(x[k]);
    if (!ok) { *bad = t; return; }
    store_row<Sys, MD, ST>(sys, out + (t - 1) * D, x);
  }
}

// One fused pass over all steps: f_t, finite checks, Picard residual, the
// Jacobian estimate and the element (cs_system_elements).
template <class Sys, int MODE, int MD, typename ST>
__global__ void __launch_bounds__(kRowThreads)
k_sys_elements(SolveArgs<ST> A, int iteration, const ST *guess, ST *e0, ST *e1, ST *e2, ST *e3, ST *u,
               cs_elem_stats *stats) {
  using E = Elem<MODE, MD>;
  __shared__ long long smin[3];
  __shared__ unsigned scnt;
  if (threadIdx.x == 0) {
    smin[0] = smin[1] = smin[2] = kNoStep;
    scnt = 0;
  }
  __syncthreads();
  const Sys sys = SysFactory<Sys>::make(A.sys);
  const int D = A.D;
  const int64_t r = (int64_t)blockIdx.x * kRowThreads + threadIdx.x;
  long long bp = kNoStep, bf = kNoStep, bj = kNoStep;
  unsigned pf = 0;
  if (r < A.T) {
    const int64_t t = A.t0 + r + 1;
    double prev[MD], gr[MD];
    load_row_ro<Sys, MD, ST>(sys, r == 0 ? A.s0 : guess + (r - 1) * D, prev);
    load_row_ro<Sys, MD, ST>(sys, guess + r * D, gr);
    typename Sys::Aux aux;
    double f[MD];
    if (A.sys.basis) {  // z coordinates: prepare at Q z, f -> Q' f (build_elem conjugates the tangents)
      double xs[MD], fx[MD];
      basis_in<Sys, MD>(sys, A.sys.basis, D, prev, xs);
      if (!sys.prepare(t, xs, aux)) bp = t;
      sys.f(aux, fx);
      basis_out<Sys, MD>(sys, A.sys.basis, D, fx, f);
    } else {
      if (!sys.prepare(t, prev, aux)) bp = t;
      sys.f(aux, f);
    }
    bool fin = true, pfail = false;
#pragma unroll
    for (int i = 0; i < MD; ++i) {
      if (sys.mem_index(i) < 0) continue;
      fin &= finite(f[i]);
      pfail |= !(fabs(f[i] - gr[i]) <= A.atol + A.rtol * fabs(f[i]));
    }
    if (!fin) bf = t;
    pf = pfail ? 1u : 0u;
    E e;
    bool jok;
    build_elem<Sys, MODE, MD, ST>(sys, aux, prev, f, t, iteration, A, e, jok);
    if (!jok) bj = t;
    if constexpr (MODE == CS_MODE_DIAG) {
#pragma unroll
      for (int k = 0; k < MD; ++k) {
        const int m = sys.mem_index(k);
        if (m >= 0) { e0[r * D + m] = (ST)e.j(k); u[r * D + m] = (ST)e.u(k); }
      }
    } else if constexpr (MODE == CS_MODE_DENSE) {
#pragma unroll
      for (int a = 0; a < MD; ++a) {
        const int ma = sys.mem_index(a);
        if (ma < 0) continue;
        u[r * D + ma] = (ST)e.u(a);
#pragma unroll
        for (int c = 0; c < MD; ++c) {
          const int mc = sys.mem_index(c);
          if (mc >= 0) e0[(r * D + ma) * D + mc] = (ST)e.M(a, c);
        }
      }
    } else {
      constexpr int H = MD / 2;
      const int n = D / 2;
#pragma unroll
      for (int i = 0; i < H; ++i)
        if (i < n) {
          e0[r * n + i] = (ST)e.ba(i);
          e1[r * n + i] = (ST)e.bb(i);
          e2[r * n + i] = (ST)e.bc(i);
          e3[r * n + i] = (ST)e.bd(i);
          u[r * D + i] = (ST)e.u(i);
          u[r * D + n + i] = (ST)e.u(H + i);
        }
    }
  }
  bp = warp_min_i64(bp);
  bf = warp_min_i64(bf);
  bj = warp_min_i64(bj);
  pf = (unsigned)warp_sum_i((int)pf);
  if ((threadIdx.x & 31) == 0) {
    if (bp != kNoStep) atomicMin(&smin[0], bp);
    if (bf != kNoStep) atomicMin(&smin[1], bf);
    if (bj != kNoStep) atomicMin(&smin[2], bj);
    if (pf) atomicAdd(&scnt, pf);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (smin[0] != kNoStep) atomicMin((long long *)&stats->bad_proposal, smin[0]);
    if (smin[1] != kNoStep) atomicMin((long long *)&stats->bad_step, smin[1]);
    if (smin[2] != kNoStep) atomicMin((long long *)&stats->bad_jacobian, smin[2]);
    if (scnt) atomicAdd(&stats->picard_fail, scnt);
  }
}

template <class Sys, int MODE, int MD, typename ST>
cudaError_t launch_elements(SolveArgs<ST> A, int iteration, const void *guess, void *e0, void *e1, void *e2,
                            void *e3, void *u, cs_elem_stats *stats, cudaStream_t st) {
  const unsigned grid = (unsigned)((A.T + kRowThreads - 1) / kRowThreads);
  k_sys_elements<Sys, MODE, MD, ST><<<grid, kRowThreads, 0, st>>>(A, iteration, (const ST *)guess, (ST *)e0,
                                                                    (ST *)e1, (ST *)e2, (ST *)e3, (ST *)u, stats);
  return cudaGetLastError();
}

struct SysCall {
  int op;  // 0 step, 1 jvp, 2 block, 3 sequential
  const int64_t *ts;
  int64_t t0, n;
  const void *S, *V;
  void *out, *out_b, *out_c, *out_d;
  long long *bad;
  int relaxed, nsamp;
  int64_t iteration;
};

template <class Sys, int MD, typename ST>
cudaError_t run_syscall(const cs_system &s, const SysCall &c, cudaStream_t st) {
  const unsigned grid = (unsigned)((c.n + kRowThreads - 1) / kRowThreads);
  if (c.op != 3 && c.n == 0) return cudaSuccess;
  switch (c.op) {
    case 0:
      k_sys_step<Sys, MD, ST><<<grid, kRowThreads, 0, st>>>(s, c.ts, c.t0, c.n, (const ST *)c.S,
                                                          (ST *)c.out, c.bad, c.relaxed);
      break;
    case 1:
      k_sys_jvp<Sys, MD, ST><<<grid, kRowThreads, 0, st>>>(s, c.ts, c.t0, c.n, (const ST *)c.S,
                                                         (const ST *)c.V, (ST *)c.out, c.relaxed);
      break;
    case 2:
      k_sys_block<Sys, MD, ST><<<grid, kRowThreads, 0, st>>>(s, c.ts, c.t0, c.n, (const ST *)c.S,
                                                           c.nsamp, c.iteration, (ST *)c.out,
                                                           (ST *)c.out_b, (ST *)c.out_c, (ST *)c.out_d);
      break;
    default:
      k_sys_seq<Sys, MD, ST><<<1, 1, 0, st>>>(s, (const ST *)c.S, c.n, (ST *)c.out, c.bad);
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// persistent solver launch: pick register-kept vs recompute variant and the
// co-resident grid from the occupancy calculator.
struct SolvePick {
  int nblocks, seg, keep, fused_tangent;
};

template <class Sys, int MODE, int MD, typename ST, bool FT>
cudaError_t launch_solve_ft(SolveArgs<ST> A, int sms, cudaStream_t st, SolvePick *pick) {
  // register-kept elements only pay off (and only fit) for narrow states
  constexpr bool kKeepOK = MD <= 4;
  auto kk = deer_persistent<Sys, MODE, MD, ST, kKeepOK, FT>;
  auto kr = deer_persistent<Sys, MODE, MD, ST, false, FT>;
  const size_t keep_smem = sizeof(double) * kSegKeep * Elem<MODE, MD>::W * kSolveThreads;
  // occupancy is a property of the instantiation: query once per device
  static int s_bk[16], s_br[16];
  static bool s_done[16];
  int dev = 0;
  cudaGetDevice(&dev);
  dev &= 15;
  cudaError_t e;
  if (!s_done[dev]) {
    int bk = 0, br = 0;
    if constexpr (kKeepOK) {
      e = cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)keep_smem);
      if (e != cudaSuccess) return e;
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bk, kk, kSolveThreads, keep_smem);
      if (e != cudaSuccess) return e;
    }
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&br, kr, kSolveThreads, 0);
    if (e != cudaSuccess) return e;
    s_bk[dev] = bk;
    s_br[dev] = br;
    s_done[dev] = true;
  }
  int bk = s_bk[dev], br = s_br[dev];
  if (bk > 8) bk = 8;
  if (br > 8) br = 8;
  const int64_t T = A.T;
  int64_t cap = (int64_t)bk * sms;
  int64_t seg = cap > 0 ? (T + cap * kSolveThreads - 1) / (cap * kSolveThreads) : kSegKeep + 1;
  bool keep = cap > 0 && seg <= kSegKeep;
  if (!keep) {
    cap = (int64_t)br * sms;
    if (cap <= 0) return cudaErrorInvalidConfiguration;
    seg = (T + cap * kSolveThreads - 1) / (cap * kSolveThreads);
  }
  if (seg < 1) seg = 1;
  // every co-resident CTA gets an equal contiguous share (at most seg steps per
  // thread); once the grid spans every SM, round it up to a whole number of
  // CTAs per SM so no SM carries an extra CTA's steps (T = 100K at 3 CTAs/SM:
  // 444 CTAs x 225 steps instead of 391 x 256, where 95 SMs ran 3 CTAs and 53
  // ran 2 and the grid waited on the busy ones)
  int64_t nb = (T + kSolveThreads - 1) / kSolveThreads;
  if (nb >= sms) nb = (nb + sms - 1) / sms * sms;
  if (nb > cap) nb = cap;
  A.seg = (int)seg;
  A.nblocks = (int)(nb < 1 ? 1 : nb);
  pick->nblocks = A.nblocks;
  pick->seg = A.seg;
  pick->keep = keep;
  pick->fused_tangent = FT;
  void *args[] = {&A};
  void *fn = (void *)kr;
  size_t smem = 0;
  if constexpr (kKeepOK) {
    if (keep) {
      fn = (void *)kk;
      smem = keep_smem;
    }
  }
  return cudaLaunchCooperativeKernel(fn, dim3(A.nblocks), dim3(kSolveThreads), args, smem, st);
}

template <class Sys, int MODE, int MD, typename ST>
cudaError_t launch_solve(SolveArgs<ST> A, int sms, cudaStream_t st, SolvePick *pick) {
  if constexpr (MODE == CS_MODE_DIAG && HasStepTangent<Sys>::value) {
    if (A.nsamp == 1) return launch_solve_ft<Sys, MODE, MD, ST, true>(A, sms, st, pick);
  }
  return launch_solve_ft<Sys, MODE, MD, ST, false>(A, sms, st, pick);
}

}  // namespace cs
