// Device-resident Newton driver: run_deer (deer.py:230-328) as ONE cooperative
// persistent kernel.
//
// Grid = co-resident CTAs (cooperative launch); CTA b owns a contiguous range of
// steps, thread i of it a contiguous segment of `seg` steps.  Per iteration:
//
//  phase A  for each owned step t: prev = guess[t-1] (s0 at t=1), f_t(prev) via
//           the fused system (noise row t), finite checks, Picard residual
//           |f - guess| <= atol + rtol|f| (deer.py:263-268), Jacobian estimate
//           (Hutchinson probes hashed on device / D tangent columns / leapfrog
//           block) -> element (J, u = f - J prev) with preconditioner, damping,
//           clip in the reference's order (deer.py:161-204); fold the segment
//           into one element (kept in registers when seg <= kSegKeep).
//           Block scan (warp shuffles + smem) -> CTA aggregate -> global.
//  sync     grid barrier; every CTA reads the same reduced flags and takes the
//           same branch: proposal/step errors, Picard stop, max_iters stop,
//           Jacobian errors (deer.py:264-271 order).
//  phase B  carry-in = ordered fold of preceding CTA aggregates applied to s0;
//           replay the segment, write guess', per-row fail test and
//           last_fail[t] = iteration (deer.py:273-277), dmax.
//  sync     history, divergence guard (deer.py:221-227, 281-283), stop if no
//           row failed (deer.py:284-286).
//
// No host round trip inside the solve: the only host sync is after the launch.
#pragma once
#include "cs_elem.cuh"
#include "cs_lookback.cuh"
#include "cs_systems.cuh"

namespace cs {

constexpr int kSolveThreads = 256;
constexpr int kSegKeep = 4;
constexpr int kTanMax = 4;

// Per-iteration reduction slot.  One per group of kSlotGroup consecutive CTAs,
// each on its own 128-byte line: the CTAs of a group combine their flags with
// atomics (16-way, groups in parallel on different L2 slices) instead of the
// whole grid serialising on one line, and after the barrier every CTA folds
// the few group slots.
struct __align__(128) SolveSlot {
  long long bad_prop, bad_f, bad_jac;
  unsigned picard_fail, any_fail;
  unsigned long long dmax_bits;
};
static_assert(offsetof(SolveSlot, bad_jac) == 16 && offsetof(SolveSlot, picard_fail) == 24 &&
                  offsetof(SolveSlot, any_fail) == 28 && offsetof(SolveSlot, dmax_bits) == 32,
              "the solver reads slots as three 16-byte words");
constexpr int kSlotGroup = 16;
constexpr int kMaxSlotGroups = 80;  // 8 CTAs/SM x 148 SMs / 16, rounded up
constexpr int kReadyStride = 32;    // halo stamps one 128-byte line apart

// Grid control block.  It lives in library-owned device memory (one per
// device and stream, zeroed once) and the kernel leaves it zeroed on exit: the
// last CTA out resets the slots, the barrier counter and the halo stamps, so a
// solve is ONE launch (no init kernel).
struct SolveCtl {
  SolveSlot slot[4][kMaxSlotGroups];
  unsigned arrive, gen, exit_count, pad0;
};

// Outcome of a solve, written by CTA 0 into host-mapped memory at exit.
struct SolveOut {
  int iterations, status, err_kind, final_buf, stop;
  int err_iter;
  long long err_step;
  double guard_dmax, guard_d0;
  unsigned long long t_start, t_end;  // %globaltimer (ns) at CTA 0's entry and at the outcome write
  unsigned seq;                       // written last: the host's completion signal for solve `seq`
};

template <typename ST>
struct SolveArgs {
  cs_system sys;
  int mode, max_iters, nsamp;
  double atol, rtol, damping, clip;
  const double *pre;
  const ST *s0;
  ST *G0, *G1;
  int32_t *last_fail;
  double *hist;
  SolveCtl *ctl;
  SolveOut *out;  // host-mapped
  unsigned seq;   // this solve's sequence number (SolveOut::seq on completion)
  double *agg;  // [2][nblocks][W]
  int *ready;   // [nblocks] iterate stamp: rows of guess_it written by CTA b
  unsigned long long *probe;  // cs_debug_probe buffer or null
  int probe_n;
  int64_t T;
  int D, seg, nblocks;
  int64_t t0;  // element builders: rows are steps t0+1 .. t0+T (a T shard); 0 elsewhere
};

// ---------------------------------------------------------------------------
template <class Sys> struct SysFactory;
template <int MD, typename ST, int TK> struct SysFactory<Mala<MD, ST, TK>> {
  static CS_D Mala<MD, ST, TK> make(const cs_system &s) { return make_mala<MD, ST, TK>(s); }
};
template <int MD, typename ST, int TK> struct SysFactory<Hmc<MD, ST, TK>> {
  static CS_D Hmc<MD, ST, TK> make(const cs_system &s) { return make_hmc<MD, ST, TK>(s); }
};
template <int MD, typename ST, int TK> struct SysFactory<Leapfrog<MD, ST, TK>> {
  static CS_D Leapfrog<MD, ST, TK> make(const cs_system &s) { return make_leapfrog<MD, ST, TK>(s); }
};
template <int MD, typename ST> struct SysFactory<Gibbs<MD, ST>> {
  static CS_D Gibbs<MD, ST> make(const cs_system &s) { return make_gibbs<MD, ST>(s); }
};

template <class Sys> struct HasBlock { static constexpr bool value = false; };
template <int MD, typename ST, int TK> struct HasBlock<Leapfrog<MD, ST, TK>> { static constexpr bool value = true; };

template <class Sys, int MD, typename ST>
CS_D void load_row(const Sys &sys, const ST *row, double (&x)[MD]) {
#pragma unroll
  for (int k = 0; k < MD; ++k) {
    const int m = sys.mem_index(k);
    x[k] = m >= 0 ? (double)__ldcg(row + m) : 0.0;
  }
}

// Orthogonal change of basis (targets.py:473-517): a system in z = Q' s
// coordinates steps z -> Q' f(Q z).  Q is dim x dim row-major f64; registers
// past dim (mem_index < 0) stay zero.  x = Q z, and z = Q' x.
template <class Sys, int MD>
CS_D void basis_in(const Sys &sys, const double *Q, int D, const double (&z)[MD], double (&x)[MD]) {
#pragma unroll
  for (int i = 0; i < MD; ++i) {
    double a = 0.0;
    if (sys.mem_index(i) >= 0)
#pragma unroll
      for (int j = 0; j < MD; ++j)
        if (sys.mem_index(j) >= 0) a += __ldg(Q + i * D + j) * z[j];
    x[i] = a;
  }
}
template <class Sys, int MD>
CS_D void basis_out(const Sys &sys, const double *Q, int D, const double (&x)[MD], double (&z)[MD]) {
#pragma unroll
  for (int j = 0; j < MD; ++j) {
    double a = 0.0;
    if (sys.mem_index(j) >= 0)
#pragma unroll
      for (int i = 0; i < MD; ++i)
        if (sys.mem_index(i) >= 0) a += x[i] * __ldg(Q + i * D + j);
    z[j] = a;
  }
}
// NT tangents through the system, conjugated by the basis when one is set
template <int NT, typename TT, class Sys, int MD>
CS_D void jvp_basis(const Sys &sys, const double *Q, int D, const typename Sys::Aux &aux,
                    const double (&V)[NT][MD], double (&O)[NT][MD], int n, bool relaxed) {
  if (!Q) {
    sys.template jvp_many<NT, TT>(aux, V, O, n, relaxed);
    return;
  }
  double Vx[NT][MD], Ox[NT][MD];
#pragma unroll
  for (int k = 0; k < NT; ++k) basis_in<Sys, MD>(sys, Q, D, V[k], Vx[k]);
  sys.template jvp_many<NT, TT>(aux, Vx, Ox, n, relaxed);
#pragma unroll
  for (int k = 0; k < NT; ++k) basis_out<Sys, MD>(sys, Q, D, Ox[k], O[k]);
}

// Element for one step from the forward pass (deer.py:161-204).
template <class Sys, int MODE, int MD, typename ST>
CS_D void build_elem(const Sys &sys, const typename Sys::Aux &aux, const double (&prev)[MD],
                     const double (&f)[MD], int64_t t, int it, const SolveArgs<ST> &A,
                     Elem<MODE, MD> &e, bool &jac_ok) {
  jac_ok = true;
  if constexpr (MODE == CS_MODE_DIAG) {
    // Hutchinson: one probe at a time (deer.py:128-131), probes hashed on device
    double est[MD];
#pragma unroll
    for (int i = 0; i < MD; ++i) est[i] = 0.0;
    const uint64_t h3 = hash_t(probe_prefix(A.sys.seed, it), (uint64_t)t);
#pragma unroll 1
    for (int k = 0; k < A.nsamp; ++k) {
      double V[1][MD], O[1][MD];
#pragma unroll
      for (int i = 0; i < MD; ++i) {
        const int m = sys.mem_index(i);
        V[0][i] = m >= 0 ? probe_sign(h3, k, m) : 0.0;
      }
      jvp_basis<1, ST>(sys, A.sys.basis, A.D, aux, V, O, 1, false);
#pragma unroll
      for (int i = 0; i < MD; ++i) est[i] += V[0][i] * O[0][i];
    }
#pragma unroll
    for (int i = 0; i < MD; ++i) {
      const int m = sys.mem_index(i);
      if (m < 0) { e.j(i) = 0.0; e.u(i) = 0.0; continue; }
      double d = est[i] / (double)A.nsamp;
      jac_ok &= finite(d);
      if (A.pre) d = d * __ldg(A.pre + m);
      d = d * A.damping;
      if (isfinite(A.clip)) d = clipv(d, A.clip);
      e.j(i) = d;
      e.u(i) = f[i] - d * prev[i];
    }
  } else if constexpr (MODE == CS_MODE_DENSE) {
    // D unit tangents in one pass (core.py:125-134: column d = J e_d)
    double V[MD][MD], O[MD][MD];
    int nk = 0;
#pragma unroll
    for (int c = 0; c < MD; ++c) {
      if (sys.mem_index(c) >= 0) nk = c + 1;
#pragma unroll
      for (int i = 0; i < MD; ++i) V[c][i] = (i == c && sys.mem_index(c) >= 0) ? 1.0 : 0.0;
    }
    jvp_basis<MD, ST>(sys, A.sys.basis, A.D, aux, V, O, nk, false);
#pragma unroll
    for (int a = 0; a < MD; ++a) {
      const int ma = sys.mem_index(a);
      double acc = 0.0;
#pragma unroll
      for (int c = 0; c < MD; ++c) {
        const int mc = sys.mem_index(c);
        double J = O[c][a];
        if (ma >= 0 && mc >= 0) {
          jac_ok &= finite(J);
          if (A.pre) J = J * (__ldg(A.pre + mc) / __ldg(A.pre + ma));
          J = J * A.damping;
          if (isfinite(A.clip)) J = clipv(J, A.clip);
        } else {
          J = 0.0;
        }
        e.M(a, c) = J;
        acc += J * prev[c];
      }
      e.u(a) = ma >= 0 ? f[a] - acc : 0.0;
    }
  } else {
    if constexpr (HasBlock<Sys>::value) {
      constexpr int H = MD / 2;
      double ba[H], bb[H], bc[H], bd[H];
      sys.block(aux, t, A.nsamp, it, ba, bb, bc, bd);
      const int n = A.D / 2;
#pragma unroll
      for (int i = 0; i < H; ++i) {
        if (i >= n) {
          e.ba(i) = 0.0; e.bb(i) = 0.0; e.bc(i) = 0.0; e.bd(i) = 0.0;
          e.u(i) = 0.0; e.u(H + i) = 0.0;
          continue;
        }
        jac_ok &= finite(ba[i]) && finite(bb[i]) && finite(bc[i]) && finite(bd[i]);
        double a = ba[i], b = bb[i], c = bc[i], d = bd[i];
        if (A.pre) {
          const double px = __ldg(A.pre + i), pv = __ldg(A.pre + n + i);
          b = b * (pv / px);
          c = c * (px / pv);
        }
        a = A.damping * a; b = A.damping * b; c = A.damping * c; d = A.damping * d;
        if (isfinite(A.clip)) { a = clipv(a, A.clip); b = clipv(b, A.clip); c = clipv(c, A.clip); d = clipv(d, A.clip); }
        e.ba(i) = a; e.bb(i) = b; e.bc(i) = c; e.bd(i) = d;
        const double x = prev[i], v = prev[H + i];
        e.u(i) = f[i] - (a * x + b * v);
        e.u(H + i) = f[H + i] - (c * x + d * v);
      }
    }
  }
}

// exclusive prefix (excl) and CTA total of an ordered element sequence
template <class E>
CS_D void block_scan(const E &x, E &excl, E &total, E *s_warp) {
  constexpr int NW = kSolveThreads / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  E inc = x;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    E o;
    inc.shfl_up(d, o);
    if (lane >= d) {
      o.after(inc);
      inc = o;
    }
  }
  E ex;
  inc.shfl_up(1, ex);
  if (lane == 0) ex.ident();
  if (lane == 31) s_warp[wid] = inc;
  __syncthreads();
  if (threadIdx.x == 0) {
    E tot;
    tot.ident();
    for (int w = 0; w < NW; ++w) {
      E e = s_warp[w];
      s_warp[w] = tot;
      tot.after(e);
    }
    s_warp[NW] = tot;
  }
  __syncthreads();
  E r = s_warp[wid];
  r.after(ex);
  excl = r;
  total = s_warp[NW];
  __syncthreads();
}

// Every CTA's aggregate is written kAggReplicas times and CTA b folds copy
// b % kAggReplicas: right after the barrier all CTAs read the low CTAs'
// records at once, and one copy per line serialised those reads at its L2
// slice (the high CTAs, which read the most records, finished the fold last).
#ifndef CS_AGG_REPLICAS
#define CS_AGG_REPLICAS 4
#endif
constexpr int kAggReplicas = CS_AGG_REPLICAS;

// Grid barrier on a monotone arrival counter: every CTA adds 1 with release
// semantics and waits (acquire) until the counter reaches nblocks * generation.
// No reset and no last-arriver hand-off, so one L2 round trip per barrier.
CS_D void grid_sync(SolveCtl *c, unsigned nblocks, unsigned &target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    target += nblocks;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&c->arrive) : "memory");
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&c->arrive) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

template <typename T> CS_D T vload(const T *p) { return *((const volatile T *)p); }

// timing probe (cs_debug_probe): CTA 0 / thread 0 stamps %globaltimer at the
// phase boundaries of the first iterations; null = off
CS_D void probe_stamp(unsigned long long *buf, int n, int it, int k) {
  if (buf && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (blockIdx.x == 0 && it * 8 + k < n) buf[it * 8 + k] = t;
    // every CTA's phase stamps of iteration 4 (skew across the grid)
    const int slot = 1024 + blockIdx.x * 8 + k;
    if (it == 4 && slot < n) buf[slot] = t;
  }
}

// ---------------------------------------------------------------------------
#ifndef CS_SOLVE_MIN_BLOCKS
#define CS_SOLVE_MIN_BLOCKS 2
#endif
// Systems with a one-pass f_t + tangent (step_tangent): the diag quasi-Newton
// solve with one Hutchinson sample runs it instead of prepare + jvp_many.
template <class Sys> struct HasStepTangent { static constexpr bool value = false; };
template <int MD, typename ST, int TK> struct HasStepTangent<Hmc<MD, ST, TK>> { static constexpr bool value = true; };

// resident CTAs per SM the instance is compiled for: the fused-tangent HMC
// kernels fit 3 x 256 threads (one step per thread at T = 100K)
template <bool FT> struct SolveOcc { static constexpr int kMinBlocks = FT ? 3 : CS_SOLVE_MIN_BLOCKS; };

template <class Sys, int MODE, int MD, typename ST, bool KEEP, bool FT = false>
__global__ void __launch_bounds__(kSolveThreads, SolveOcc<FT>::kMinBlocks)
deer_persistent(SolveArgs<ST> A) {
  static_assert(!FT || (MODE == CS_MODE_DIAG && HasStepTangent<Sys>::value), "fused tangent: diag HMC only");
  using E = Elem<MODE, MD>;
  // KEEP: the segment's elements wait in shared memory across the grid sync,
  // laid out [k][w][thread] so every access is bank-conflict free
  extern __shared__ double s_keep[];
  __shared__ E s_warp[kSolveThreads / 32 + 1];
  __shared__ long long s_min[3];
  __shared__ unsigned s_cnt[2];
  __shared__ unsigned long long s_dm;
  __shared__ long long s_dec[6];  // the slot words every thread decides on, read once per CTA

  const Sys sys = SysFactory<Sys>::make(A.sys);
  const int b = blockIdx.x;
  const int D = A.D;
  if (b == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    A.out->t_start = t;
  }
  // balanced contiguous ranges: CTA b owns rows [lo_b, hi_b), thread i the
  // segment starting at lo_b + i * seg (every SM gets the same share of steps)
  const int64_t lo_b = (int64_t)b * A.T / A.nblocks, hi_b = (int64_t)(b + 1) * A.T / A.nblocks;
  const int seg = (int)((hi_b - lo_b + kSolveThreads - 1) / kSolveThreads);
  const int64_t row0 = lo_b + (int64_t)threadIdx.x * seg;
  const int64_t row_end = hi_b;
  double s0r[MD];
  load_row<Sys, MD, ST>(sys, A.s0, s0r);
  for (int k = 0; k < seg; ++k)
    if (row0 + k < row_end) A.last_fail[row0 + k] = 0;

  unsigned target = 0;
  double d0 = -1.0;
  bool have_d0 = false;
  int it = 0, cur = 0;
  int status = CS_RUN_MAXITERS, err_kind = CS_DIV_NONE, err_iter = -1, stop = CS_STOP_MAXITERS;
  long long err_step = -1;
  double g_dmax = 0.0;
  E excl;  // this thread's exclusive in-CTA prefix of the current pass

  for (;;) {
    SolveSlot *S = &A.ctl->slot[it & 3][b / kSlotGroup];  // this CTA's group slot
    const int ngroups = (A.nblocks + kSlotGroup - 1) / kSlotGroup;
    const ST *Gc = cur ? A.G1 : A.G0;
    if (threadIdx.x == 0) {
      s_min[0] = s_min[1] = s_min[2] = kNoStep;
      s_cnt[0] = s_cnt[1] = 0;
      s_dm = 0ull;
    }
    // ---------------- phase A(it): f, Picard, elements, segment fold -------
    // the halo row guess_it[row0-1] of CTA b's first thread was written by CTA b-1
    probe_stamp(A.probe, A.probe_n, it, 0);
    if (it > 0 && threadIdx.x == 0 && b > 0) {
      const int *rd = A.ready + (size_t)(b - 1) * kReadyStride;
      while (ld_acquire(rd) < it) {
      }
    }
    __syncthreads();
    probe_stamp(A.probe, A.probe_n, it, 1);
    E agg;
    agg.ident();
    long long bp = kNoStep, bf = kNoStep, bj = kNoStep;
    unsigned pf = 0;
    const bool want_elem = it < A.max_iters;
    double prev[MD];
    if (it == 0 || row0 == 0 || row0 >= row_end) {
#pragma unroll
      for (int i = 0; i < MD; ++i) prev[i] = s0r[i];
    } else {
      load_row<Sys, MD, ST>(sys, Gc + (row0 - 1) * D, prev);
    }
#pragma unroll 1
    for (int k = 0; k < seg; ++k) {
      const int64_t r = row0 + k;
      if (r >= row_end) break;
      const int64_t t = r + 1;
      double gr[MD];
      if (it == 0) {
#pragma unroll
        for (int i = 0; i < MD; ++i) gr[i] = s0r[i];
      } else {
        load_row<Sys, MD, ST>(sys, Gc + r * D, gr);
      }
      double f[MD];
      E e;
      bool jok = true;
      if constexpr (FT) {
        // f_t and the one Hutchinson tangent in a single integrator pass
        const uint64_t h3 = hash_t(probe_prefix(A.sys.seed, it), (uint64_t)t);
        double V[MD], O[MD];
#pragma unroll
        for (int i = 0; i < MD; ++i) {
          const int m = sys.mem_index(i);
          V[i] = m >= 0 ? probe_sign(h3, 0, m) : 0.0;
        }
        if (!sys.template step_tangent<ST>(t, prev, V, f, O)) bp = min(bp, (long long)t);
        if (want_elem) {
#pragma unroll
          for (int i = 0; i < MD; ++i) {
            const int m = sys.mem_index(i);
            if (m < 0) { e.j(i) = 0.0; e.u(i) = 0.0; continue; }
            double est = 0.0;
            est += V[i] * O[i];
            double d = est / 1.0;  // deer.py:131 mean over one sample, same bits as the general path
            jok &= finite(d);
            if (A.pre) d = d * __ldg(A.pre + m);
            d = d * A.damping;
            if (isfinite(A.clip)) d = clipv(d, A.clip);
            e.j(i) = d;
            e.u(i) = f[i] - d * prev[i];
          }
        }
      } else {
        typename Sys::Aux aux;
        if (!sys.prepare(t, prev, aux)) bp = min(bp, (long long)t);
        sys.f(aux, f);
        if (want_elem) build_elem<Sys, MODE, MD, ST>(sys, aux, prev, f, t, it, A, e, jok);
      }
      bool fin = true, pfail = false;
#pragma unroll
      for (int i = 0; i < MD; ++i) {
        if (sys.mem_index(i) < 0) continue;
        fin &= finite(f[i]);
        pfail |= !(fabs(f[i] - gr[i]) <= A.atol + A.rtol * fabs(f[i]));
      }
      if (!fin) bf = min(bf, (long long)t);
      pf += pfail ? 1u : 0u;
      if (want_elem) {
        if (!jok) bj = min(bj, (long long)t);
        agg.after(e);
        if constexpr (KEEP) {
#pragma unroll
          for (int w = 0; w < E::W; ++w) s_keep[(k * E::W + w) * kSolveThreads + threadIdx.x] = e.v[w];
        }
      }
#pragma unroll
      for (int i = 0; i < MD; ++i) prev[i] = gr[i];
    }
    probe_stamp(A.probe, A.probe_n, it, 2);
    E total;
    block_scan(agg, excl, total, s_warp);
    if (threadIdx.x < kAggReplicas) {  // one copy per replica: readers spread over kAggReplicas lines
      double *g = A.agg + (((size_t)(it & 1) * kAggReplicas + threadIdx.x) * A.nblocks + b) * E::W;
#pragma unroll
      for (int q = 0; q < E::W; ++q) g[q] = total.v[q];
    }
    bp = warp_min_nn64(bp);
    bf = warp_min_nn64(bf);
    bj = warp_min_nn64(bj);
    pf = warp_sum_u32(pf);
    if ((threadIdx.x & 31) == 0) {
      if (bp != kNoStep) atomicMin(&s_min[0], bp);
      if (bf != kNoStep) atomicMin(&s_min[1], bf);
      if (bj != kNoStep) atomicMin(&s_min[2], bj);
      if (pf) atomicAdd(&s_cnt[0], pf);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (s_min[0] != kNoStep) atomicMin(&S->bad_prop, s_min[0]);
      if (s_min[1] != kNoStep) atomicMin(&S->bad_f, s_min[1]);
      if (s_min[2] != kNoStep) atomicMin(&S->bad_jac, s_min[2]);
      if (s_cnt[0]) atomicAdd(&S->picard_fail, s_cnt[0]);
    }
    // the ONE grid barrier of the iteration: it publishes pass it's aggregates
    // and flags together with update it-1's fail count and delta_max
    probe_stamp(A.probe, A.probe_n, it, 3);
    grid_sync(A.ctl, (unsigned)A.nblocks, target);
    probe_stamp(A.probe, A.probe_n, it, 4);
    if (b == 0 && threadIdx.x < ngroups) {
      SolveSlot *O = &A.ctl->slot[(it + 2) & 3][threadIdx.x];
      O->bad_prop = O->bad_f = O->bad_jac = kNoStep;
      O->picard_fail = O->any_fail = 0;
      O->dmax_bits = 0ull;
    }

    // the predecessors' aggregates, loaded now so this L2 round trip overlaps
    // the decision reads below (used by phase B's carry-in)
    E fold;
    fold.ident();
    {
      const double *ag = A.agg + ((size_t)(it & 1) * kAggReplicas + (b % kAggReplicas)) * A.nblocks * E::W;
      const int per = (b + kSolveThreads - 1) / kSolveThreads;
      const int lo = threadIdx.x * per, hi = min(b, lo + per);
      for (int q = lo; q < hi; ++q) {
        E e;
        const double2 *src = (const double2 *)(ag + (size_t)q * E::W);  // W is even, records 16 B aligned
#pragma unroll
        for (int w = 0; w < E::W / 2; ++w) {
          const double2 p = __ldcg(src + w);
          e.v[2 * w] = p.x;
          e.v[2 * w + 1] = p.y;
        }
        fold.after(e);
      }
    }

    // ---------------- decisions (identical in every CTA) ------------------
    // one thread per CTA reads the slot words (not every thread: 100K readers
    // of one L2 line serialise at its slice and skew the grid by microseconds)
    if (threadIdx.x < 32) {  // warp 0 folds the group slots
      unsigned gaf = 0, gpf = 0;
      unsigned long long gdm = 0ull;
      long long gbp = kNoStep, gbf = kNoStep, gbj = kNoStep;
      for (int q = threadIdx.x; q < ngroups; q += 32) {
        // 16-byte loads: [bad_prop bad_f] [bad_jac picard|any_fail] [dmax]
        if (it > 0) {
          const longlong2 *P = (const longlong2 *)&A.ctl->slot[(it - 1) & 3][q];
          const longlong2 w1 = __ldcg(P + 1), w2 = __ldcg(P + 2);
          gaf += (unsigned)((unsigned long long)w1.y >> 32);
          const unsigned long long d = (unsigned long long)w2.x;
          gdm = d > gdm ? d : gdm;
        }
        const longlong2 *Q = (const longlong2 *)&A.ctl->slot[it & 3][q];
        const longlong2 w0 = __ldcg(Q), w1 = __ldcg(Q + 1);
        gbp = min(gbp, w0.x);
        gbf = min(gbf, w0.y);
        gbj = min(gbj, w1.x);
        gpf += (unsigned)w1.y;
      }
      gaf = warp_sum_u32(gaf);
      gpf = warp_sum_u32(gpf);
      gdm = warp_max_nn64(gdm);
      gbp = warp_min_nn64(gbp);
      gbf = warp_min_nn64(gbf);
      gbj = warp_min_nn64(gbj);
      if (threadIdx.x == 0) {
        s_dec[0] = (long long)gaf;
        s_dec[1] = (long long)gdm;
        s_dec[2] = gbp;
        s_dec[3] = gbf;
        s_dec[4] = gbj;
        s_dec[5] = (long long)gpf;
      }
    }
    __syncthreads();
    if (it > 0) {  // the update that produced guess_it (deer.py:273-286)
      const unsigned gaf = (unsigned)s_dec[0];
      const double dmax = __longlong_as_double(s_dec[1]);
      if (b == 0 && threadIdx.x == 0) A.hist[it - 1] = dmax;
      if (!have_d0) { d0 = dmax; have_d0 = true; }
      g_dmax = dmax;
      if (d0 > 0.0 && dmax > 1e6 * d0) {
        status = CS_RUN_DIVERGED; stop = CS_STOP_ERROR; err_kind = CS_DIV_GUARD; err_step = -1; err_iter = it;
        break;
      }
      if (gaf == 0) { status = CS_RUN_CONVERGED; stop = CS_STOP_NOFAIL; break; }
    }
    {
      const long long gbp = s_dec[2], gbf = s_dec[3], gbj = s_dec[4];
      const unsigned gpf = (unsigned)s_dec[5];
      if (gbp != kNoStep) { status = CS_RUN_DIVERGED; stop = CS_STOP_ERROR; err_kind = CS_DIV_PROPOSAL; err_step = gbp; err_iter = -1; break; }
      if (gbf != kNoStep) { status = CS_RUN_DIVERGED; stop = CS_STOP_ERROR; err_kind = CS_DIV_STEP; err_step = gbf; err_iter = it + 1; break; }
      if (gpf == 0) { status = CS_RUN_CONVERGED; stop = CS_STOP_PICARD; break; }
      if (it >= A.max_iters) { status = CS_RUN_MAXITERS; stop = CS_STOP_MAXITERS; break; }
      if (gbj != kNoStep) { status = CS_RUN_DIVERGED; stop = CS_STOP_ERROR; err_kind = CS_DIV_JACOBIAN; err_step = gbj; err_iter = it + 1; break; }
    }

    // ---------------- phase B(it): carry-in, replay, bookkeeping ----------
    ST *Gn = cur ? A.G0 : A.G1;
    {
      E fex, ftot;
      block_scan(fold, fex, ftot, s_warp);
      probe_stamp(A.probe, A.probe_n, it, 5);
      double x[MD];
#pragma unroll
      for (int i = 0; i < MD; ++i) x[i] = s0r[i];
      ftot.apply(x);      // state entering this CTA
      excl.apply(x);      // state entering this thread's segment
      unsigned af = 0;
      unsigned long long dmb = 0ull;
      double pv[MD];
      if (!KEEP) {
        if (it == 0 || row0 == 0 || row0 >= row_end) {
#pragma unroll
          for (int i = 0; i < MD; ++i) pv[i] = s0r[i];
        } else {
          load_row<Sys, MD, ST>(sys, Gc + (row0 - 1) * D, pv);
        }
      }
#pragma unroll 1
      for (int k = 0; k < seg; ++k) {
        const int64_t r = row0 + k;
        if (r >= row_end) break;
        double gr[MD];
        if (it == 0) {
#pragma unroll
          for (int i = 0; i < MD; ++i) gr[i] = s0r[i];
        } else {
          load_row<Sys, MD, ST>(sys, Gc + r * D, gr);
        }
        E e;
        if constexpr (KEEP) {
#pragma unroll
          for (int w = 0; w < E::W; ++w) e.v[w] = s_keep[(k * E::W + w) * kSolveThreads + threadIdx.x];
        } else {
          const int64_t t = r + 1;
          typename Sys::Aux aux;
          sys.prepare(t, pv, aux);
          double f[MD];
          sys.f(aux, f);
          bool jok;
          build_elem<Sys, MODE, MD, ST>(sys, aux, pv, f, t, it, A, e, jok);
#pragma unroll
          for (int i = 0; i < MD; ++i) pv[i] = gr[i];
        }
        e.apply(x);
        bool fail = false;
#pragma unroll
        for (int i = 0; i < MD; ++i) {
          const int m = sys.mem_index(i);
          if (m < 0) continue;
          const ST xs = (ST)x[i];
          Gn[r * D + m] = xs;
          const double xd = (double)xs;
          const double gap = fabs(xd - gr[i]);
          fail |= gap > A.atol + A.rtol * fabs(xd);
          const unsigned long long gb = (unsigned long long)__double_as_longlong(gap);
          dmb = gb > dmb ? gb : dmb;
        }
        if (fail) {
          A.last_fail[r] = it + 1;
          ++af;
        }
      }
      af = warp_sum_u32(af);
      dmb = warp_max_nn64(dmb);
      if ((threadIdx.x & 31) == 0) {
        if (af) atomicAdd(&s_cnt[1], af);
        atomicMax(&s_dm, dmb);
      }
      // the CTA barrier orders every thread's stores before thread 0's fence +
      // release (cumulativity), so one fence per CTA publishes the whole segment
      __syncthreads();
      if (threadIdx.x == 0) {
        if (s_cnt[1]) atomicAdd(&S->any_fail, s_cnt[1]);
        atomicMax(&S->dmax_bits, s_dm);
        __threadfence();
        st_release(A.ready + (size_t)b * kReadyStride, it + 1);  // rows of guess_{it+1} from this CTA are visible
      }
    }
    probe_stamp(A.probe, A.probe_n, it, 6);
    ++it;
    cur ^= 1;
  }

  // trace <- final iterate, per_step_converged_at = last_fail + 1
  // (deer.py:321-328), each CTA over its own rows (written only by itself)
  {
    const int fb = it == 0 ? -1 : cur;
    for (int64_t r = lo_b + threadIdx.x; r < hi_b; r += kSolveThreads) {
      if (fb == 1) {
        for (int d = 0; d < D; ++d) A.G0[r * D + d] = A.G1[r * D + d];
      } else if (fb == -1) {
        for (int d = 0; d < D; ++d) A.G0[r * D + d] = A.s0[d];
      }
      A.last_fail[r] = A.last_fail[r] + 1;
    }
  }
  if (b == 0 && threadIdx.x == 0) {
    SolveOut *o = A.out;
    o->iterations = it;
    o->status = status;
    o->stop = stop;
    o->err_kind = err_kind;
    o->err_step = err_step;
    o->err_iter = err_iter;
    o->final_buf = it == 0 ? -1 : cur;
    o->guard_dmax = g_dmax;
    o->guard_d0 = d0;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    o->t_end = t;
    __threadfence_system();  // the record and the delta history before the signal
    *(volatile unsigned *)&o->seq = A.seq;
  }
  // leave the control block zeroed for the next solve on this stream: the last
  // CTA out (every other CTA is past its last read of it) resets it
  __shared__ unsigned s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&A.ctl->exit_count, 1u) == (unsigned)A.nblocks - 1u;
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    for (int i = threadIdx.x; i < A.nblocks; i += kSolveThreads) A.ready[(size_t)i * kReadyStride] = 0;
    for (int i = threadIdx.x; i < 4 * kMaxSlotGroups; i += kSolveThreads) {
      SolveSlot *O = &A.ctl->slot[i / kMaxSlotGroups][i % kMaxSlotGroups];
      O->bad_prop = O->bad_f = O->bad_jac = kNoStep;
      O->picard_fail = O->any_fail = 0;
      O->dmax_bits = 0ull;
    }
    if (threadIdx.x == 0) {
      A.ctl->arrive = 0;
      A.ctl->gen = 0;
      A.ctl->exit_count = 0;
    }
  }
}

}  // namespace cs
