// Affine scans s_t = J_t s_{t-1} + u_t on B200 (pscan.py:273-354).
//
// Three element carriers (pscan.py:100-173):
//   diag      j,u (T,D)                       -> scan_rows<DIAG>  (D <= 64)
//   block2x2  a,b,c,d (T,D), u (T,2D) [x|v]   -> scan_rows<BLOCK> (D <= 64)
//   both, wide D > 64                         -> scan_cols<...>
//   dense     J (T,D,D), u (T,D), D <= 8      -> scan_dense_small<MD>
// The column and dense scans are single-pass: each tile is read from HBM once,
// reduced, linked to its predecessors by decoupled look-back, replayed and
// written once (12 B/element diag f32).  Long plain row scans (T >= 2^19) take
// the local scan + fix-up (scan_local / scan_local_blk): every CTA scans its own
// range from zero in one streaming pass and only each range's leading tiles are
// corrected by P e -- j, u read once.  The bookkeeping update scans below 2^22
// and short scans use the two-pass chunk scan (A: reduce, C: re-read and replay
// a round later, see scan_rows): 20 B/element of HBM traffic.
// Carries and composition run in f64 regardless of storage type; every
// chunk's entry state is the fixed chain exit(k) = A_k(exit(k-1)) from s0
// (lookback_cta applies aggregates one at a time), so results are bit-
// identical run to run however the look-back races resolve.
#include <cstdlib>

#include "cs_lookback.cuh"
#include "cs_scan.cuh"
#include "cs_tma.cuh"

namespace cs {

constexpr int kScanThreads = 256;
constexpr int kHalf = kScanThreads / 2;

// A thread group that cooperates on one phase: the whole CTA, or one half of
// a warp-specialised CTA synchronised with a named barrier.
template <int BASE, int NT, int BAR>
struct Grp {
  static constexpr int kN = NT;
  static constexpr int kBase = BASE;
  CS_D static int tid() { return (int)threadIdx.x - BASE; }
  CS_D static void sync() {
    if constexpr (BAR == 0) __syncthreads();
    else asm volatile("bar.sync %0, %1;" ::"n"(BAR), "n"(NT) : "memory");
  }
};
using CtaGrp = Grp<0, kScanThreads, 0>;

// ---------------------------------------------------------------------------
// per-column affine monoid, diag and block2x2
template <int VAR> struct ColElem;

template <> struct ColElem<SCAN_DIAG> {
  static constexpr int W = 2;  // j, u
  double j, u;
  CS_D void ident() { j = 1.0; u = 0.0; }
  // this <- e o this  (apply this first, then e)
  CS_D void push(double ej, double eu) { u = ej * u + eu; j = ej * j; }
  CS_D void push(const ColElem &e) { push(e.j, e.u); }
  // this <- this o e  (apply e first)
  CS_D void pre(const ColElem &e) { u = j * e.u + u; j = j * e.j; }
  CS_D void apply(double &x) const { x = j * x + u; }
  CS_D void store(double *p) const { p[0] = j; p[1] = u; }
  CS_D void load(const double *p) { j = p[0]; u = p[1]; }
  CS_D void load_cg(const double *p) { j = ld_cg(p); u = ld_cg(p + 1); }
  CS_D ColElem down(int off) const {
    ColElem o;
    o.j = __shfl_down_sync(0xffffffffu, j, off);
    o.u = __shfl_down_sync(0xffffffffu, u, off);
    return o;
  }
  CS_D ColElem up(int off) const {
    ColElem o;
    o.j = __shfl_up_sync(0xffffffffu, j, off);
    o.u = __shfl_up_sync(0xffffffffu, u, off);
    return o;
  }
};

template <> struct ColElem<SCAN_BLOCK> {
  static constexpr int W = 6;
  double A, B, C, E, ux, uv;
  CS_D void ident() { A = 1.0; B = 0.0; C = 0.0; E = 1.0; ux = 0.0; uv = 0.0; }
  CS_D void push(double a, double b, double c, double d, double px, double pv) {
    // compose(e_t, run): (a,b;c,d) * (A,B;C,E), u = M_t u + u_t  (_scan_kernels.py:118-126)
    double An = a * A + b * C, Bn = a * B + b * E, Cn = c * A + d * C, En = c * B + d * E;
    double xn = a * ux + b * uv + px, vn = c * ux + d * uv + pv;
    A = An; B = Bn; C = Cn; E = En; ux = xn; uv = vn;
  }
  CS_D void push(const ColElem &e) { push(e.A, e.B, e.C, e.E, e.ux, e.uv); }
  CS_D void pre(const ColElem &e) {
    double An = A * e.A + B * e.C, Bn = A * e.B + B * e.E, Cn = C * e.A + E * e.C,
           En = C * e.B + E * e.E;
    double xn = A * e.ux + B * e.uv + ux, vn = C * e.ux + E * e.uv + uv;
    A = An; B = Bn; C = Cn; E = En; ux = xn; uv = vn;
  }
  CS_D void apply(double &x, double &v) const {
    double xn = A * x + B * v + ux, vn = C * x + E * v + uv;
    x = xn; v = vn;
  }
  CS_D void store(double *p) const { p[0] = A; p[1] = B; p[2] = C; p[3] = E; p[4] = ux; p[5] = uv; }
  CS_D void load(const double *p) { A = p[0]; B = p[1]; C = p[2]; E = p[3]; ux = p[4]; uv = p[5]; }
  CS_D void load_cg(const double *p) {
    A = ld_cg(p); B = ld_cg(p + 1); C = ld_cg(p + 2); E = ld_cg(p + 3); ux = ld_cg(p + 4); uv = ld_cg(p + 5);
  }
  CS_D ColElem down(int off) const {
    ColElem o;
    o.A = __shfl_down_sync(0xffffffffu, A, off);
    o.B = __shfl_down_sync(0xffffffffu, B, off);
    o.C = __shfl_down_sync(0xffffffffu, C, off);
    o.E = __shfl_down_sync(0xffffffffu, E, off);
    o.ux = __shfl_down_sync(0xffffffffu, ux, off);
    o.uv = __shfl_down_sync(0xffffffffu, uv, off);
    return o;
  }
  CS_D ColElem up(int off) const {
    ColElem o;
    o.A = __shfl_up_sync(0xffffffffu, A, off);
    o.B = __shfl_up_sync(0xffffffffu, B, off);
    o.C = __shfl_up_sync(0xffffffffu, C, off);
    o.E = __shfl_up_sync(0xffffffffu, E, off);
    o.ux = __shfl_up_sync(0xffffffffu, ux, off);
    o.uv = __shfl_up_sync(0xffffffffu, uv, off);
    return o;
  }
};

// The same monoid in the storage precision T, for in-stage segment work.
template <int VAR, typename T> struct SegE;
template <typename T> struct SegE<SCAN_DIAG, T> {
  static constexpr int W = 2;
  T j, u;
  CS_D void ident() { j = 1; u = 0; }
  CS_D void push(const SegE &e) { u = e.j * u + e.u; j = e.j * j; }  // this <- e o this
  CS_D void store(T *p) const { p[0] = j; p[1] = u; }
  CS_D void load(const T *p) { j = p[0]; u = p[1]; }
  CS_D void apply(double &x) const { x = (double)j * x + (double)u; }
  CS_D ColElem<SCAN_DIAG> wide() const { ColElem<SCAN_DIAG> o; o.j = (double)j; o.u = (double)u; return o; }
  CS_D SegE up(int off) const {
    SegE o;
    o.j = __shfl_up_sync(0xffffffffu, j, off);
    o.u = __shfl_up_sync(0xffffffffu, u, off);
    return o;
  }
};
template <typename T> struct SegE<SCAN_BLOCK, T> {
  static constexpr int W = 6;
  T A, B, C, E, ux, uv;
  CS_D void ident() { A = 1; B = 0; C = 0; E = 1; ux = 0; uv = 0; }
  CS_D void push(const SegE &e) {
    const T An = e.A * A + e.B * C, Bn = e.A * B + e.B * E, Cn = e.C * A + e.E * C, En = e.C * B + e.E * E;
    const T xn = e.A * ux + e.B * uv + e.ux, vn = e.C * ux + e.E * uv + e.uv;
    A = An; B = Bn; C = Cn; E = En; ux = xn; uv = vn;
  }
  CS_D void store(T *p) const { p[0] = A; p[1] = B; p[2] = C; p[3] = E; p[4] = ux; p[5] = uv; }
  CS_D void load(const T *p) { A = p[0]; B = p[1]; C = p[2]; E = p[3]; ux = p[4]; uv = p[5]; }
  CS_D void apply(double &x, double &v) const {
    const double xn = (double)A * x + (double)B * v + (double)ux, vn = (double)C * x + (double)E * v + (double)uv;
    x = xn; v = vn;
  }
  CS_D ColElem<SCAN_BLOCK> wide() const {
    ColElem<SCAN_BLOCK> o;
    o.A = A; o.B = B; o.C = C; o.E = E; o.ux = ux; o.uv = uv;
    return o;
  }
  CS_D SegE up(int off) const {
    SegE o;
    o.A = __shfl_up_sync(0xffffffffu, A, off);
    o.B = __shfl_up_sync(0xffffffffu, B, off);
    o.C = __shfl_up_sync(0xffffffffu, C, off);
    o.E = __shfl_up_sync(0xffffffffu, E, off);
    o.ux = __shfl_up_sync(0xffffffffu, ux, off);
    o.uv = __shfl_up_sync(0xffffffffu, uv, off);
    return o;
  }
};

// CTA-wide decoupled look-back over a window of 32 predecessors at a time:
// warp 0 waits until every predecessor in the window has published at least
// its aggregate and finds the nearest exit state; then the 8 warps fold the
// window's aggregates column by column (lane = tile, ordered tree reduction)
// into the running prefix s_acc.  One L2 round trip covers kLbWindow tiles.
//   status(p) -> const int*     agg(p, c) -> const double*
//   exit_x(p, c), exit_v(p, c)  the published exit state of tile p
//   s0x(c), s0v(c)              the chain's initial state
constexpr int kLbPerLane = 4;                    // tiles per lane in a look-back window
constexpr int kLbWindow = 32 * kLbPerLane;          // 128 predecessors per round trip

template <int VAR, class G = CtaGrp, int KB = 8, class StatusF, class AggF, class ExitF, class ExitVF, class S0F,
          class S0VF>
CS_D void lookback_cta(int64_t pos, int ncol, StatusF status, AggF agg, ExitF exit_x, ExitVF exit_v,
                       S0F s0x, S0VF s0v, double *s_acc, double *s_entry, int *s_ctl) {
  (void)s_acc;
  const int tid = G::tid(), lane = tid & 31, wid = tid >> 5;
  // (1) the nearest published exit state at or before pos - 1, scanning back
  // window by window; every tile between it and pos has its aggregate out
  int64_t hi = pos - 1, pe = -1;
  for (;;) {
    G::sync();
    if (wid == 0) {
      // lane l watches tiles hi - l*K - j, j < K (lane 0 holds the latest)
      int st[kLbPerLane];
#pragma unroll
      for (int j = 0; j < kLbPerLane; ++j) {  // K independent loads: one round trip
        const int64_t p = hi - lane * kLbPerLane - j;
        st[j] = p >= 0 ? ld_acquire(status(p)) : 2;  // p < 0: the chain start (s0) acts as an exit
      }
      int first = kLbWindow;
#pragma unroll
      for (int j = 0; j < kLbPerLane; ++j) {
        const int64_t p = hi - lane * kLbPerLane - j;
        while (st[j] == 0) st[j] = ld_acquire(status(p));
        if (st[j] == 2 && first == kLbWindow) first = lane * kLbPerLane + j;
      }
      // nearest exit in the window = the smallest index over lanes
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, off));
      if (lane == 0) s_ctl[0] = first;
    }
    G::sync();
    const int stop = s_ctl[0];
    if (stop < kLbWindow) {
      pe = hi - stop;
      break;
    }
    hi -= kLbWindow;
  }
  // (2) apply the aggregates pe+1 .. pos-1 to that exit ONE AT A TIME, oldest
  // first.  Every published exit is itself exit(k) = A_k(exit(k-1)) from s0,
  // so whichever exit the scan found, the entry is the same chain of single
  // applications -- the same bits run to run (the reference's fixed-chunk
  // property, _scan_kernels.py:3-8), independent of publication timing.
  // (Composing the aggregates first and applying the product once would round
  // differently depending on where the look-back stopped.)
  constexpr int kB = KB;  // aggregates in flight per round trip (a register budget, set by the caller)
  for (int c = tid; c < ncol; c += G::kN) {
    double x = pe < 0 ? s0x(c) : exit_x(pe, c);
    double v = 0.0;
    if (VAR == SCAN_BLOCK) v = pe < 0 ? s0v(c) : exit_v(pe, c);
    for (int64_t k0 = pe + 1; k0 < pos; k0 += kB) {
      ColElem<VAR> e[kB];
#pragma unroll
      for (int j = 0; j < kB; ++j)
        if (k0 + j < pos) e[j].load_cg(agg(k0 + j, c));  // a batch of loads in flight, then the chain
#pragma unroll
      for (int j = 0; j < kB; ++j) {
        if (k0 + j >= pos) break;
        if constexpr (VAR == SCAN_DIAG) e[j].apply(x);
        else e[j].apply(x, v);
      }
    }
    s_entry[c] = x;
    if (VAR == SCAN_BLOCK) s_entry[ncol + c] = v;
  }
  G::sync();
}

// Two-level look-back for row tiles (see cs_lookback.cuh).  On return
// s_entry holds the chain state entering tile b.
template <int VAR, class G = CtaGrp, int KB = 8, class S0F, class S0VF, class StampF>
CS_D void lookback_grouped(int64_t b, int ncol, const LookbackWs &ws, S0F s0x, S0VF s0v, double *s_acc,
                           double *s_acc2, double *s_entry, double *s_gentry, int *s_ctl, StampF stamp) {
  constexpr int W = ColElem<VAR>::W;
  const int SW = VAR == SCAN_DIAG ? ncol : 2 * ncol;
  const int tid = G::tid();
  const int64_t g = b / kGroupTiles;
  const int i = (int)(b % kGroupTiles);
  const int64_t t0 = g * kGroupTiles;
  // The two levels are independent: the first half of the group folds the
  // in-group prefix while the second half looks back over groups.
  using H0 = Grp<G::kBase, G::kN / 2, 3>;
  using H1 = Grp<G::kBase + G::kN / 2, G::kN / 2, 4>;
  if (tid < G::kN / 2) {
    // (1) in-group exclusive prefix over tiles t0 .. b-1 (lane l <-> tile t0+l)
    const int ht = H0::tid(), lane = ht & 31, wid = ht >> 5;
    if (wid == 0 && lane < i)
      while (ld_acquire(ws.status + t0 + lane) == 0) {
      }
    H0::sync();
    for (int c = wid; c < ncol; c += H0::kN / 32) {
      ColElem<VAR> e;
      e.ident();
      if (lane < i) e.load_cg(ws.agg + ((t0 + lane) * ncol + c) * W);
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        ColElem<VAR> o = e.down(off);
        if (lane + off < 32) e.push(o);  // later lanes hold later tiles
      }
      if (lane == 0) e.store(s_acc + c * W);
    }
    H0::sync();
    if (ht == 0) stamp(6);
  } else {
    // (2) state entering the group: decoupled look-back over group aggregates
    lookback_cta<VAR, H1, KB>(
        g, ncol, [&](int64_t p) { return ws.gstatus + p; },
        [&](int64_t p, int cc) { return ws.gagg + (p * ncol + cc) * W; },
        [&](int64_t p, int cc) { return ld_cg(ws.exit + p * SW + cc); },
        [&](int64_t p, int cc) { return ld_cg(ws.exit + p * SW + ncol + cc); }, s0x, s0v, s_acc2, s_gentry,
        s_ctl);
    if (H1::tid() == 0) stamp(7);
  }
  G::sync();
  // (3) tile entry = in-group prefix applied to the group entry
  for (int c = tid; c < ncol; c += G::kN) {
    ColElem<VAR> acc;
    acc.load(s_acc + c * W);
    double x = s_gentry[c], v = VAR == SCAN_BLOCK ? s_gentry[ncol + c] : 0.0;
    if constexpr (VAR == SCAN_DIAG) acc.apply(x);
    else acc.apply(x, v);
    s_entry[c] = x;
    if (VAR == SCAN_BLOCK) s_entry[ncol + c] = v;
  }
  G::sync();
  // the first tile of a group publishes the group's entry as the previous
  // group's exit (second half only; the first half goes on to the replay)
  if (i == 0 && g > 0 && tid >= G::kN / 2) {
    const int ht = H1::tid();
    for (int c = ht; c < SW; c += H1::kN) ws.exit[(g - 1) * SW + c] = s_gentry[c];
    __threadfence();
    H1::sync();
    if (ht == 0) st_release(ws.gstatus + g - 1, 2);
  }
}

// Producer side of the two-level scheme: count this tile's aggregate into its
// group; the producer completing the group folds and publishes the group
// aggregate (status 1).
template <int VAR, class G>
CS_D void group_aggregate_publish(int64_t b, int ncol, const LookbackWs &ws, int *s_flag) {
  constexpr int W = ColElem<VAR>::W;
  constexpr int NW = G::kN / 32;
  const int tid = G::tid(), lane = tid & 31, wid = tid >> 5;
  const int64_t g = b / kGroupTiles;
  if (tid == 0) {
    __threadfence();
    const int old = atomicAdd(ws.gcount + g, 1);
    __threadfence();
    *s_flag = old == kGroupTiles - 1;
  }
  G::sync();
  if (!*s_flag) return;
  const int64_t t0 = g * kGroupTiles;
  for (int c = wid; c < ncol; c += NW) {
    ColElem<VAR> e;
    e.load_cg(ws.agg + ((t0 + lane) * ncol + c) * W);
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      ColElem<VAR> o = e.down(off);
      if (lane + off < 32) e.push(o);
    }
    if (lane == 0) {
      double tmp[W];
      e.store(tmp);
#pragma unroll
      for (int q = 0; q < W; ++q) ws.gagg[(g * ncol + c) * W + q] = tmp[q];
      __threadfence();
    }
  }
  G::sync();
  if (tid == 0) st_release(ws.gstatus + g, 1);
}

// ---------------------------------------------------------------------------
// One-warp look-back (the dedicated look-back warp of scan_rows).  The same
// two-level scheme as lookback_grouped, arranged so a lookup costs a handful
// of L2 round trips whatever D is: statuses are polled one per lane, and the
// aggregate records a fold needs are contiguous in the workspace, so they are
// staged into shared memory with every 16-byte copy in flight at once
// (cp.async), then folded lane-per-column from shared memory.
constexpr int kLbwStage = 2048;     // doubles of look-back staging buffer (16 KB)
constexpr int kLbwPubStage = 1024;  // doubles of the publisher's staging buffer (8 KB)

// acc(c) <- acc(c) o (rec[n-1] o ... o rec[0]) for every column c, where
// rec[p] = src + p * ncol * W (earliest record first).
template <int VAR>
CS_D void lbw_fold_records(const double *src, int n, int ncol, double *stage, double *s_acc, int cap = kLbwStage) {
  constexpr int W = ColElem<VAR>::W;
  constexpr int U = W / 2;  // 16-byte units per (record, column)
  const int lane = threadIdx.x & 31;
  if (n <= 0) return;
  const int nbmax = min(32, cap / (32 * W));
  for (int c0 = 0; c0 < ncol; c0 += nbmax) {
    const int nb = min(nbmax, ncol - c0);
    const int units = n * nb * U;
    for (int k = lane; k < units; k += 32) {
      const int p = k / (nb * U), rem = k - p * nb * U;  // rem = column-in-batch * U + unit
      cp_async16(stage + (p * nb) * W + rem * 2, src + ((int64_t)p * ncol + c0) * W + rem * 2);
    }
    cp_async_wait_all();
    __syncwarp();
    if (lane < nb) {
      ColElem<VAR> e;
      e.ident();
      for (int p = 0; p < n; ++p) {
        ColElem<VAR> r;
        r.load(stage + (p * nb + lane) * W);
        e.push(r);
      }
      ColElem<VAR> acc;
      acc.load(s_acc + (c0 + lane) * W);
      acc.pre(e);
      acc.store(s_acc + (c0 + lane) * W);
    }
    __syncwarp();
  }
}

// Entry state of chunk b into s_entry (SW doubles).  s_acc, s_acc2: ncol*W
// doubles each; stage: kLbwStage doubles.  Publishes the previous group's exit
// when b opens a group.
template <int VAR, class S0F, class S0VF, class StampF>
CS_D void lookback_warp(int64_t b, int ncol, const LookbackWs &ws, S0F s0x, S0VF s0v, double *s_acc,
                        double *s_acc2, double *stage, double *s_entry, StampF stamp) {
  constexpr int W = ColElem<VAR>::W;
  const int SW = VAR == SCAN_DIAG ? ncol : 2 * ncol;
  const int lane = threadIdx.x & 31;
  const int64_t g = b / kGroupTiles;
  const int i = (int)(b % kGroupTiles);
  const int64_t t0 = g * kGroupTiles;
  for (int c = lane; c < ncol; c += 32) {
    ColElem<VAR> id;
    id.ident();
    id.store(s_acc + c * W);
    id.store(s_acc2 + c * W);
  }
  // (1) state entering the group: look back over group aggregates, one
  // window of 32 groups per round trip (lane l watches group hi - l)
  int64_t hi = g - 1;
  for (;;) {
    const int64_t p = hi - lane;
    int st = p >= 0 ? ld_acquire(ws.gstatus + p) : 2;  // p < 0: the chain start acts as an exit
    unsigned exits = __ballot_sync(0xffffffffu, st == 2);
    int stop = exits ? __ffs(exits) - 1 : 32;
    for (;;) {  // every group nearer than the exit must have its aggregate
      const unsigned below = stop == 32 ? 0xffffffffu : ((1u << stop) - 1u);
      if (!(__ballot_sync(0xffffffffu, st == 0) & below)) break;
      __nanosleep(200);  // a spinning warp would steal issue slots from the streaming warps
      if (st == 0) st = ld_acquire(ws.gstatus + p);
      exits = __ballot_sync(0xffffffffu, st == 2);
      stop = exits ? __ffs(exits) - 1 : 32;
    }
    if (lane == 0) stamp(10);
    // groups hi-stop+1 .. hi, earliest first, folded after what is already in s_acc2
    lbw_fold_records<VAR>(ws.gagg + (hi - stop + 1) * ncol * W, stop, ncol, stage, s_acc2);
    if (lane == 0) stamp(11);
    if (stop < 32) {
      const int64_t pe = hi - stop;
      for (int c = lane; c < ncol; c += 32) {
        double x = pe < 0 ? s0x(c) : ld_cg(ws.exit + pe * SW + c);
        double v = 0.0;
        if (VAR == SCAN_BLOCK) v = pe < 0 ? s0v(c) : ld_cg(ws.exit + pe * SW + ncol + c);
        ColElem<VAR> acc;
        acc.load(s_acc2 + c * W);
        if constexpr (VAR == SCAN_DIAG) acc.apply(x);
        else acc.apply(x, v);
        s_entry[c] = x;
        if (VAR == SCAN_BLOCK) s_entry[ncol + c] = v;
      }
      break;
    }
    hi -= 32;
  }
  __syncwarp();
  // the first chunk of a group publishes the group's entry as the previous group's exit
  if (i == 0 && g > 0) {
    for (int c = lane; c < SW; c += 32) ws.exit[(g - 1) * SW + c] = s_entry[c];
    __threadfence();
    __syncwarp();
    if (lane == 0) st_release(ws.gstatus + g - 1, 2);
  }
  // (2) in-group prefix over chunks t0 .. b-1, applied to the group entry
  if (i > 0) {
    if (lane == 0) stamp(12);
    if (lane < i)
      while (ld_acquire(ws.status + t0 + lane) == 0) __nanosleep(200);
    __syncwarp();
    if (lane == 0) stamp(13);
    lbw_fold_records<VAR>(ws.agg + t0 * ncol * W, i, ncol, stage, s_acc);
    if (lane == 0) stamp(14);
    for (int c = lane; c < ncol; c += 32) {
      ColElem<VAR> acc;
      acc.load(s_acc + c * W);
      double x = s_entry[c], v = VAR == SCAN_BLOCK ? s_entry[ncol + c] : 0.0;
      if constexpr (VAR == SCAN_DIAG) acc.apply(x);
      else acc.apply(x, v);
      s_entry[c] = x;
      if (VAR == SCAN_BLOCK) s_entry[ncol + c] = v;
    }
  }
  __syncwarp();
}

// One-warp group publication (the publisher warp of scan_rows): count chunk
// b's aggregate into its group; the chunk completing the group folds the 32
// aggregates (staged, one round trip) and publishes the group aggregate.
template <int VAR>
CS_D void group_publish_warp(int64_t b, int ncol, const LookbackWs &ws, double *stage, double *s_acc) {
  constexpr int W = ColElem<VAR>::W;
  const int lane = threadIdx.x & 31;
  const int64_t g = b / kGroupTiles;
  int last = 0;
  if (lane == 0) {
    const int old = atomicAdd(ws.gcount + g, 1);
    __threadfence();
    last = old == kGroupTiles - 1;
  }
  if (!__shfl_sync(0xffffffffu, last, 0)) return;
  for (int c = lane; c < ncol; c += 32) {
    ColElem<VAR> id;
    id.ident();
    id.store(s_acc + c * W);
  }
  __syncwarp();
  lbw_fold_records<VAR>(ws.agg + g * kGroupTiles * ncol * W, kGroupTiles, ncol, stage, s_acc, kLbwPubStage);
  for (int k = lane; k < ncol * W; k += 32) ws.gagg[g * ncol * W + k] = s_acc[k];
  __threadfence();
  __syncwarp();
  if (lane == 0) st_release(ws.gstatus + g, 1);
}

// ---------------------------------------------------------------------------
// narrow rows: tile = R consecutive rows x all columns, staged in smem.
// Persistent CTAs (grid = resident capacity) claim tiles in ticket order and
// double-buffer them: the bulk (TMA) load of the next tile is in flight while
// the current one is reduced, linked and replayed, so HBM never idles behind
// a wave of CTAs that all sit in look-back at the same time.
template <typename ST, int VAR>
CS_D bool rows_tile_tma(const ScanArgs<ST> &a, int64_t b, int R) {
  const int ncol = a.D;
  const int64_t row0 = b * R;
  const int rows = (int)(a.T - row0 < (int64_t)R ? a.T - row0 : (int64_t)R);
  const unsigned bytes = (unsigned)(sizeof(ST) * rows * ncol);
  const ST *u_src = a.u + (VAR == SCAN_BLOCK ? 2 : 1) * row0 * ncol;
  return (bytes % 16 == 0) && aligned16(a.e0 + row0 * ncol) && aligned16(u_src) &&
         (VAR == SCAN_DIAG || (aligned16(a.e1 + row0 * ncol) && aligned16(a.e2 + row0 * ncol) &&
                               aligned16(a.e3 + row0 * ncol)));
}

template <typename ST, int VAR>
CS_D void rows_tile_issue(const ScanArgs<ST> &a, int64_t b, int R, ST *tile, uint64_t *bar, uint64_t pol) {
  const int ncol = a.D;
  const int64_t row0 = b * R;
  const int rows = (int)(a.T - row0 < (int64_t)R ? a.T - row0 : (int64_t)R);
  const unsigned bytes = (unsigned)(sizeof(ST) * rows * ncol);
  const int64_t g0 = row0 * ncol;
  if constexpr (VAR == SCAN_DIAG) {
    mbar_expect_tx(bar, 2 * bytes);
    bulk_g2s_hint(tile, a.e0 + g0, bytes, bar, pol);
    bulk_g2s_hint(tile + R * ncol, a.u + g0, bytes, bar, pol);
  } else {
    mbar_expect_tx(bar, 6 * bytes);
    bulk_g2s_hint(tile, a.e0 + g0, bytes, bar, pol);
    bulk_g2s_hint(tile + R * ncol, a.e1 + g0, bytes, bar, pol);
    bulk_g2s_hint(tile + 2 * R * ncol, a.e2 + g0, bytes, bar, pol);
    bulk_g2s_hint(tile + 3 * R * ncol, a.e3 + g0, bytes, bar, pol);
    bulk_g2s_hint(tile + 4 * R * ncol, a.u + 2 * g0, 2 * bytes, bar, pol);
  }
}

CS_D unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
CS_D unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %smid;" : "=r"(r));
  return r;
}
template <typename ST>
CS_D void scan_stamp(const ScanArgs<ST> &a, int64_t b, int k) {
  if (a.probe && b * 16 + 16 <= a.probe_n) a.probe[b * 16 + k] = k == 0 ? smid() : gtimer();
}

// Chained-chunk row scan.  A persistent grid of G CTAs (3 per SM) walks the
// sequence in rounds: chunk q = r*G + j (CS stages of R rows) belongs to CTA
// j.  Each CTA alternates two passes over its chunks, stage by stage, with
// every thread loading its own column segment of the stage straight into
// registers (all of a stage's loads in flight before the FMA chain starts):
//   A(r)    read chunk (r, j), reduce it, publish its aggregate
//   C(r-1)  look back for chunk (r-1, j)'s entry state, re-read the chunk,
//           replay it and stream the states out
// The look-back for a chunk runs a full round after its predecessors
// published, so it resolves in a few L2 round trips instead of waiting on a
// chain of in-flight tiles.  Loads carry L2 eviction hints (A: evict_last,
// C: evict_first) so the re-read hits L2 when a round fits in it.  Chunks are
// linked with the two-level (group) look-back.  HBM traffic is 20 B/element
// (diag f32: j,u read twice, s written once) against 12 B/element for a
// single pass; see DESIGN.md for why the single-pass variants lost.

struct RowsJob {  // position in a CTA's job stream: A(0) .. A(L-1) A(L) C(0) A(L+1) C(1) ... C(nr-1)
  int64_t r;
  int ph;  // 0: A(r), 1: C(r-L)
  int s, ns;
  int64_t q;
};

struct RowsGeom {
  int64_t T, nchunks, nr;
  int R, CS, G, j;
  int L;  // rounds between a chunk's A pass and its C pass
  bool agg_only;
  int64_t nstages;  // ceil(T / R)
  // balanced partition: chunk q covers stages [c0(q), c0(q+1)), at most CS of
  // them, so the last round of the grid is as full as the others
  CS_D int64_t c0(int64_t q) const { return q * nstages / nchunks; }
  CS_D int stages_in(int64_t q) const { return (int)(c0(q + 1) - c0(q)); }
  CS_D void settle(RowsJob &it) const {
    while (it.r < nr + L) {
      const int64_t rr = it.ph == 0 ? it.r : it.r - L;
      const bool ok = (it.ph == 0 ? it.r < nr : (it.r >= L && !agg_only)) && rr * G + j < nchunks;
      if (ok) {
        it.q = rr * G + j;
        it.ns = stages_in(it.q);
        it.s = 0;
        return;
      }
      if (it.ph == 0) it.ph = 1;
      else { it.ph = 0; ++it.r; }
    }
  }
  CS_D RowsJob first() const {
    RowsJob it{0, 0, 0, 0, 0};
    settle(it);
    return it;
  }
  CS_D void next(RowsJob &it) const {
    if (++it.s < it.ns) return;
    if (it.ph == 0) it.ph = 1;
    else { it.ph = 0; ++it.r; }
    settle(it);
  }
  CS_D bool valid(const RowsJob &it) const { return it.r < nr + L; }
};

// rows per thread segment per stage: the thread's loads for a stage are all
// issued before its FMA chain starts (registers: NA * kSegRows values)
// Per-thread rows per stage and resident CTAs per SM, by scan kind (measured,
// tools/build_scan_variants.sh, T = 4M, D = 18 fp32): the plain diag scan runs
// best at 24 rows x 2 CTAs/SM (2.29 -> 2.50 TB/s against 16 x 3; 2.58 -> 2.83
// at T = 16M), block2x2 at 6 rows x 3 CTAs/SM (1.90 -> 2.39 TB/s), and the
// diag scan with the fused Newton bookkeeping (UPDATE: it also reads the
// previous iterate) at 16 x 3 -- 24 x 2 made it 30% slower at cfg 5's T = 1M.
#ifndef CS_ROWS_PREFETCH
#define CS_ROWS_PREFETCH 0  // software-pipelined stage loads (needs 2x registers)
#endif
#ifndef CS_ROWS_DIAG_KR
#define CS_ROWS_DIAG_KR 24  // plain diag: fp32 rows per thread per stage (tools/build_scan_variants.sh)
#endif
#ifndef CS_ROWS_DIAG_MINB
#define CS_ROWS_DIAG_MINB 2
#endif
template <int VAR, bool UPD>
struct RowsTune {
  static constexpr int kRows32 = VAR == SCAN_DIAG ? (UPD ? 16 : CS_ROWS_DIAG_KR) : 6;  // fp32 rows per thread per stage
  static constexpr int kMinBlocks = VAR == SCAN_DIAG && !UPD ? CS_ROWS_DIAG_MINB : 3;
};
template <typename ST, int VAR, bool UPD = false>
struct RowsSeg {
  static constexpr int kRows = sizeof(ST) == 4 ? RowsTune<VAR, UPD>::kRows32
                                               : (RowsTune<VAR, UPD>::kRows32 / 2 > 0 ? RowsTune<VAR, UPD>::kRows32 / 2 : 1);
};
#ifndef CS_ROWS_LBW_MINB
#define CS_ROWS_LBW_MINB 2
#endif

template <typename T>
CS_D T ld_hint(const T *p, uint64_t pol) {
  if constexpr (sizeof(T) == 4) {
    float v;
    asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    return v;
  } else {
    double v;
    asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
  }
}
// 16-byte variant for the small-D diag scan's coalesced stage loads
CS_D float4 ld_hint_v4(const float *p, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p), "l"(pol));
  return v;
}
// small-D diag (D | 256, D <= 4, fp32): each thread owns KR rows of one column, so a
// warp's per-row loads touch 32 / D rows KR rows apart (D = 2: 8 useful bytes per
// 32-byte sector per request, LSU-bound).  Instead the CTA loads the stage block
// with coalesced 16-byte loads and redistributes it through shared memory
// (segments padded by 4 floats: 16-byte stores, <= 2-way read conflicts).
#ifndef CS_ROWS_TX_UPDATE
#define CS_ROWS_TX_UPDATE 1  // the fused-bookkeeping (streamed engine) variant too
#endif
template <typename ST, int VAR, bool UPDATE, bool LBW>
struct RowsTx {
  static constexpr bool kOn = sizeof(ST) == 4 && VAR == SCAN_DIAG && (!UPDATE || CS_ROWS_TX_UPDATE) && !LBW && !CS_ROWS_PREFETCH;
};
CS_HD bool rows_tx_dim(int D) { return D == 1 || D == 2 || D == 4; }

template <typename ST, int VAR, bool AGG_ONLY = false, bool UPDATE = false, bool LBW = false>
__global__ void __launch_bounds__(kScanThreads + (LBW ? 64 : 0),
                                  LBW ? CS_ROWS_LBW_MINB : RowsTune<VAR, UPDATE>::kMinBlocks)
scan_rows(ScanArgs<ST> a, LookbackWs ws, int R, int CS, int64_t nchunks, int lag, int NS) {
  (void)NS;
  // LBW: two helper warps take every global hand-off off the eight streaming
  // warps.  Warp 8 computes the entry state of each of the CTA's C chunks
  // while the main warps stream the A pass before it (lookback_warp); warp 9
  // publishes each chunk aggregate and its group's (group_publish_warp), so
  // the memory fences a publication needs never wait on the main warps'
  // in-flight state stores.
  using MG = Grp<0, kScanThreads, LBW ? 1 : 0>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int W = ColElem<VAR>::W;
  constexpr int KR = RowsSeg<ST, VAR, UPDATE>::kRows;
  using CT = ST;  // in-segment arithmetic type; everything crossing segments is f64
  const int ncol = a.D;
  const int SW = VAR == SCAN_DIAG ? ncol : 2 * ncol;
  const int nseg = kScanThreads / ncol;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int c = tid % ncol, sg = tid / ncol;
  const bool active = sg < nseg;
  __shared__ double s_chunk2[(LBW ? 2 : 1) * 64 * W];  // A: running chunk aggregate (LBW: two slots)
  __shared__ double s_run[2 * 2 * 64];  // C: running chain state, double-buffered by stage parity
  __shared__ double s_entry[2 * 64];
  __shared__ double s_acc[64 * W];
  __shared__ double s_acc2[64 * W];
  __shared__ double s_acc3[LBW ? 64 * W : 1];
  __shared__ double s_gentry[2 * 64];
  __shared__ int s_ctl[1];
  __shared__ int s_gflag;
  __shared__ unsigned long long s_dm;
  CT *segagg = (CT *)smem_raw;                                // [2][nseg+1][ncol][W], by stage parity
  int *s_fail = (int *)(segagg + 2 * (nseg + 1) * ncol * W);  // UPDATE: one flag per stage row
  // LBW: look-back staging buffer and the two-slot entry hand-off
  double *lb_stage = (double *)(((uintptr_t)(s_fail + R) + 15) & ~(uintptr_t)15);
  // small-D transposition buffer (same spot as lb_stage: the two never coexist)
  float *txb = (float *)lb_stage;
  constexpr bool kTx = RowsTx<ST, VAR, UPDATE, LBW>::kOn;
  static_assert(!kTx || KR % 4 == 0, "coalesced stage loads move 4 rows' floats at a time");
  const int txw = R * ncol + 4 * nseg;  // floats per array in txb
  const bool tx = kTx && rows_tx_dim(ncol) && ((((uintptr_t)a.e0) | ((uintptr_t)a.u)) & 15) == 0;
  __shared__ double s_lbe[2 * 128];
  __shared__ __align__(8) uint64_t s_full[2], s_empty[2], s_aggfull[2], s_aggempty[2];
  double *pub_stage = lb_stage + kLbwStage;  // kLbwPubStage doubles
  if constexpr (UPDATE)
    for (int r = tid; r < R; r += kScanThreads) s_fail[r] = 0;
  if constexpr (LBW) {
    if (tid == 0) {
      mbar_init(&s_full[0], 1);
      mbar_init(&s_full[1], 1);
      mbar_init(&s_empty[0], 1);
      mbar_init(&s_empty[1], 1);
      mbar_init(&s_aggfull[0], 1);
      mbar_init(&s_aggfull[1], 1);
      mbar_init(&s_aggempty[0], 1);
      mbar_init(&s_aggempty[1], 1);
      fence_mbar_init();
    }
  }

  RowsGeom geo;
  geo.T = a.T;
  geo.nchunks = nchunks;
  geo.G = gridDim.x;
  geo.j = blockIdx.x;
  geo.R = R;
  geo.CS = CS;
  geo.nr = (nchunks + geo.G - 1) / geo.G;
  geo.nstages = (a.T + R - 1) / R;
  geo.agg_only = AGG_ONLY;
  geo.L = LBW ? (lag > 0 ? lag : 1) : 1;
  // A keeps what it reads in L2 for C (one round later); C's reads are the last use
  const uint64_t pol_a = l2_policy_evict_last(), pol_c = l2_policy_evict_first();
  __syncthreads();
  if constexpr (LBW) {
    if (wid == kScanThreads / 32) {  // the look-back warp: one entry per C chunk, in job order
      int64_t k = 0;
      for (int64_t q = geo.j; q < nchunks; q += geo.G, ++k) {
        const int slot = (int)(k & 1);
        if (k >= 2) mbar_wait(&s_empty[slot], (unsigned)(((k >> 1) - 1) & 1));
        if (lane == 0) scan_stamp(a, q, 6);
        lookback_warp<VAR>(
            q, ncol, ws, [&](int cc) { return (double)a.s0[cc]; }, [&](int cc) { return (double)a.s0[ncol + cc]; },
            s_acc, s_acc2, lb_stage, s_lbe + slot * 128, [&](int kk) { scan_stamp(a, q, kk); });
        if (lane == 0) {
          scan_stamp(a, q, 7);
          mbar_arrive(&s_full[slot]);
        }
      }
      return;
    }
    if (wid == kScanThreads / 32 + 1) {  // the publisher warp: chunk and group aggregates, in job order
      int64_t k = 0;
      for (int64_t q = geo.j; q < nchunks; q += geo.G, ++k) {
        const int slot = (int)(k & 1);
        mbar_wait(&s_aggfull[slot], (unsigned)((k >> 1) & 1));
        const double *src = s_chunk2 + slot * 64 * W;
        for (int cc = lane; cc < ncol * W; cc += 32) ws.agg[q * ncol * W + cc] = src[cc];
        __syncwarp();
        if (lane == 0) {
          __threadfence();
          st_release(ws.status + q, 1);
          scan_stamp(a, q, 4);
          mbar_arrive(&s_aggempty[slot]);
        }
        group_publish_warp<VAR>(q, ncol, ws, pub_stage, s_acc3);
        if (lane == 0) scan_stamp(a, q, 3);
      }
      return;
    }
  }
  int64_t kc = 0;  // C jobs started (LBW hand-off slot/parity)
  int64_t ka = 0;  // A jobs started (LBW publication slot/parity)

  constexpr int NA = VAR == SCAN_DIAG ? 2 : 6;
  // issue one stage's loads (this thread's KR rows of its column) into ev
  auto load_stage = [&](const RowsJob &job, CT (&ev)[NA][KR]) {
    const int64_t row0 = (geo.c0(job.q) + job.s) * R;
    const int rows = (int)(a.T - row0 < (int64_t)R ? a.T - row0 : (int64_t)R);
    const uint64_t pol = job.ph == 0 ? pol_a : pol_c;
    const int r0 = sg * KR, r1 = min(rows, r0 + KR);
    if constexpr (kTx) {
      if (tx) {  // ev[.][4m + e] <- float 4 * (tid + m * 256) + e of the stage block
        const int nv = rows * ncol;
        const float *b0 = (const float *)a.e0 + row0 * ncol, *bu = (const float *)a.u + row0 * ncol;
#pragma unroll
        for (int m = 0; m < KR / 4; ++m) {
          const int f = 4 * (tid + m * kScanThreads);
          float4 x0, xu;
          if (f + 4 <= nv) {
            x0 = ld_hint_v4(b0 + f, pol);
            xu = ld_hint_v4(bu + f, pol);
          } else {  // ragged last stage: identity past the end
            x0.x = f + 0 < nv ? ld_hint(b0 + f + 0, pol) : 1.f; xu.x = f + 0 < nv ? ld_hint(bu + f + 0, pol) : 0.f;
            x0.y = f + 1 < nv ? ld_hint(b0 + f + 1, pol) : 1.f; xu.y = f + 1 < nv ? ld_hint(bu + f + 1, pol) : 0.f;
            x0.z = f + 2 < nv ? ld_hint(b0 + f + 2, pol) : 1.f; xu.z = f + 2 < nv ? ld_hint(bu + f + 2, pol) : 0.f;
            x0.w = f + 3 < nv ? ld_hint(b0 + f + 3, pol) : 1.f; xu.w = f + 3 < nv ? ld_hint(bu + f + 3, pol) : 0.f;
          }
          ev[0][4 * m + 0] = (CT)x0.x; ev[0][4 * m + 1] = (CT)x0.y; ev[0][4 * m + 2] = (CT)x0.z; ev[0][4 * m + 3] = (CT)x0.w;
          ev[1][4 * m + 0] = (CT)xu.x; ev[1][4 * m + 1] = (CT)xu.y; ev[1][4 * m + 2] = (CT)xu.z; ev[1][4 * m + 3] = (CT)xu.w;
        }
        return;
      }
    }
    if (!active) return;
    // per-stage 64-bit bases, 32-bit offsets inside the stage
    const int64_t g0 = row0 * ncol;
    const ST *p0 = a.e0 + g0 + c, *pu = a.u + (VAR == SCAN_BLOCK ? 2 : 1) * g0 + c;
    const ST *p1 = VAR == SCAN_BLOCK ? a.e1 + g0 + c : nullptr, *p2 = VAR == SCAN_BLOCK ? a.e2 + g0 + c : nullptr;
    const ST *p3 = VAR == SCAN_BLOCK ? a.e3 + g0 + c : nullptr;
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      const int r = r0 + k;
      if (r < r1) {
        const int i = r * ncol;
        if constexpr (VAR == SCAN_DIAG) {
          ev[0][k] = (CT)ld_hint(p0 + i, pol);
          ev[1][k] = (CT)ld_hint(pu + i, pol);
        } else {
          ev[0][k] = (CT)ld_hint(p0 + i, pol);
          ev[1][k] = (CT)ld_hint(p1 + i, pol);
          ev[2][k] = (CT)ld_hint(p2 + i, pol);
          ev[3][k] = (CT)ld_hint(p3 + i, pol);
          ev[4][k] = (CT)ld_hint(pu + 2 * i, pol);
          ev[5][k] = (CT)ld_hint(pu + 2 * i + ncol, pol);
        }
      } else {  // identity rows
        if constexpr (VAR == SCAN_DIAG) {
          ev[0][k] = 1;
          ev[1][k] = 0;
        } else {
          ev[0][k] = 1; ev[1][k] = 0; ev[2][k] = 0; ev[3][k] = 1; ev[4][k] = 0; ev[5][k] = 0;
        }
      }
    }
  };

  // process one stage whose loads are in ev (the next stage's loads are
  // already in flight in the other register set)
  auto body = [&](const RowsJob &cur, int64_t n, const CT (&ev)[NA][KR]) {
    const int64_t q = cur.q;
    const int64_t stg = geo.c0(q) + cur.s;
    const int64_t row0 = stg * R;
    const int rows = (int)(a.T - row0 < (int64_t)R ? a.T - row0 : (int64_t)R);
    double *s_chunk = s_chunk2 + (LBW ? (ka & 1) * 64 * W : 0);
    if (cur.s == 0) {
      if (cur.ph == 0) {
        if constexpr (LBW)
          if (ka >= 2) mbar_wait(&s_aggempty[ka & 1], (unsigned)(((ka >> 1) - 1) & 1));
        if (tid == 0) scan_stamp(a, q, 1);
        for (int cc = tid; cc < ncol; cc += kScanThreads) {
          ColElem<VAR> id;
          id.ident();
          id.store(s_chunk + cc * W);
        }
      } else {
        if (tid == 0) {
          scan_stamp(a, q, 5);
          s_dm = 0ull;
        }
        if constexpr (LBW) {
          mbar_wait(&s_full[kc & 1], (unsigned)((kc >> 1) & 1));
          for (int cc = tid; cc < SW; cc += kScanThreads) s_run[(n & 1) * 2 * 64 + cc] = s_lbe[(kc & 1) * 128 + cc];
        } else {
          // the 80-register instances (block2x2, the bookkeeping scan) fetch fewer
          // aggregates per round trip so the look-back does not spill the stage loop
          lookback_grouped<VAR, CtaGrp, (VAR == SCAN_BLOCK ? 1 : UPDATE ? 2 : 8)>(
              q, ncol, ws, [&](int cc) { return (double)a.s0[cc]; },
              [&](int cc) { return (double)a.s0[ncol + cc]; }, s_acc, s_acc2, s_entry, s_gentry, s_ctl,
              [&](int k) { scan_stamp(a, q, k); });
          for (int cc = tid; cc < SW; cc += kScanThreads) s_run[(n & 1) * 2 * 64 + cc] = s_entry[cc];
        }
        if (tid == 0) scan_stamp(a, q, 8);
      }
    }
    const int r0 = sg * KR, r1 = min(rows, r0 + KR);
    // ---- segment aggregate (CT) -> segagg[par]
    CT *sa = segagg + (n & 1) * (nseg + 1) * ncol * W;
    if (active) {
      SegE<VAR, CT> run;
      run.ident();
#pragma unroll
      for (int k = 0; k < KR; ++k) {
        SegE<VAR, CT> e;
        if constexpr (VAR == SCAN_DIAG) {
          e.j = ev[0][k];
          e.u = ev[1][k];
        } else {
          e.A = ev[0][k]; e.B = ev[1][k]; e.C = ev[2][k]; e.E = ev[3][k]; e.ux = ev[4][k]; e.uv = ev[5][k];
        }
        run.push(e);
      }
      run.store(sa + (sg * ncol + c) * W);
    }
    MG::sync();
    if constexpr (LBW) {
      if (cur.ph == 1 && cur.s == 0) {
        if (tid == 0) mbar_arrive(&s_empty[kc & 1]);  // every main thread has copied the entry
        ++kc;
      }
    }
    if (nseg > 32) {
      // narrow D: many segments per column -- warp scan per column (lane q
      // holds segments [q*K, q*K+K)), exclusive prefixes in place, total in slot nseg
      const int K = (nseg + 31) / 32;
      for (int cc = wid; cc < ncol; cc += kScanThreads / 32) {
        SegE<VAR, CT> e;
        e.ident();
        for (int qq = lane * K; qq < lane * K + K && qq < nseg; ++qq) {
          SegE<VAR, CT> x;
          x.load(sa + (qq * ncol + cc) * W);
          e.push(x);
        }
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          SegE<VAR, CT> o = e.up(off);
          if (lane >= off) { o.push(e); e = o; }  // earlier lanes hold earlier segments
        }
        SegE<VAR, CT> ex = e.up(1);
        if (lane == 0) ex.ident();
        if (lane == 31) e.store(sa + (nseg * ncol + cc) * W);
        for (int qq = lane * K; qq < lane * K + K && qq < nseg; ++qq) {
          SegE<VAR, CT> x;
          x.load(sa + (qq * ncol + cc) * W);
          ex.store(sa + (qq * ncol + cc) * W);
          ex.push(x);
        }
      }
      MG::sync();
    }

    if (cur.ph == 0) {
      // ---- A: fold the stage into the chunk aggregate (f64); segagg is
      // double-buffered, so the next stage does not wait for this
      for (int cc = tid; cc < ncol; cc += kScanThreads) {
        ColElem<VAR> ch;
        ch.load(s_chunk + cc * W);
        if (nseg > 32) {
          SegE<VAR, CT> x;
          x.load(sa + (nseg * ncol + cc) * W);
          ch.push(x.wide());
        } else {
          for (int qq = 0; qq < nseg; ++qq) {
            SegE<VAR, CT> x;
            x.load(sa + (qq * ncol + cc) * W);
            ch.push(x.wide());
          }
        }
        ch.store(s_chunk + cc * W);
      }
      if (cur.s == cur.ns - 1) {  // publish the chunk aggregate after its last stage
        MG::sync();
        if constexpr (LBW) {  // hand it to the publisher warp
          if (tid == 0) {
            scan_stamp(a, q, 2);
            mbar_arrive(&s_aggfull[ka & 1]);
          }
          ++ka;
          return;
        }
        for (int cc = tid; cc < ncol * W; cc += kScanThreads) ws.agg[q * ncol * W + cc] = s_chunk[cc];
        __threadfence();
        MG::sync();
        if (tid == 0) {
          st_release(ws.status + q, 1);
          scan_stamp(a, q, 4);
        }
        if constexpr (!AGG_ONLY) group_aggregate_publish<VAR, MG>(q, ncol, ws, &s_gflag);
      }
      return;
    }

    // ---- C: entry state of each segment = (segments before it) o running state
    double *run_in = s_run + (n & 1) * 2 * 64, *run_out = s_run + ((n + 1) & 1) * 2 * 64;
    if (active) {
      // UPDATE: this thread's previous-guess values, loaded before the entry
      // fold (the replay's stores may alias them, so loads issued at the point
      // of use would serialise behind every store)
      constexpr int NG = UPDATE ? (VAR == SCAN_BLOCK ? 2 : 1) : 0;
      ST gv[NG > 0 ? NG : 1][UPDATE ? KR : 1];
      if constexpr (UPDATE) {
        const ST *gb0 = a.guess + row0 * SW + c;
#pragma unroll
        for (int k = 0; k < KR; ++k) {
          if (r0 + k < r1) {
            gv[0][k] = gb0[(r0 + k) * SW];
            if constexpr (NG == 2) gv[NG - 1][k] = gb0[(r0 + k) * SW + ncol];
          }
        }
      }
      SegE<VAR, CT> pre;
      pre.ident();
      if (nseg <= 32) {
        for (int qq = 0; qq < sg; ++qq) {
          SegE<VAR, CT> x;
          x.load(sa + (qq * ncol + c) * W);
          pre.push(x);
        }
      } else {
        pre.load(sa + (sg * ncol + c) * W);  // exclusive prefix from the warp scan
      }
      double xe = run_in[c], ve = VAR == SCAN_BLOCK ? run_in[ncol + c] : 0.0;
      if (sg == nseg - 1) {  // the last segment carries the running state to the next stage
        SegE<VAR, CT> tot = pre;
        if (nseg <= 32) {
          SegE<VAR, CT> own;
          own.load(sa + (sg * ncol + c) * W);
          tot.push(own);
        } else {
          tot.load(sa + (nseg * ncol + c) * W);
        }
        double xo = xe, vo = ve;
        if constexpr (VAR == SCAN_DIAG) tot.apply(xo);
        else tot.apply(xo, vo);
        run_out[c] = xo;
        if constexpr (VAR == SCAN_BLOCK) run_out[ncol + c] = vo;
      }
      if constexpr (VAR == SCAN_DIAG) pre.apply(xe);
      else pre.apply(xe, ve);

      // ---- replay from registers; states stream straight out (lanes of a warp
      // cover whole rows, so each store instruction writes contiguous runs)
      unsigned long long dmb = 0ull;
      auto check = [&](int r, double g, double xv) {  // deer.py:273-275 on the stored value
        if constexpr (UPDATE) {
          const double gap = fabs(xv - g);
          if (gap > a.atol + a.rtol * fabs(xv)) s_fail[r] = 1;
          const unsigned long long gb = (unsigned long long)__double_as_longlong(gap);
          dmb = gb > dmb ? gb : dmb;
        }
      };
      ST *o = a.out + row0 * SW + c;
      if constexpr (VAR == SCAN_DIAG) {
        CT x = (CT)xe;
#pragma unroll
        for (int k = 0; k < KR; ++k) {
          x = ev[0][k] * x + ev[1][k];
          if (r0 + k < r1) {
            __stcs(o + (r0 + k) * SW, (ST)x);
            check(r0 + k, (double)gv[0][k], (double)x);
          }
        }
      } else {
        CT x = (CT)xe, v = (CT)ve;
#pragma unroll
        for (int k = 0; k < KR; ++k) {
          const CT xa = ev[0][k] * x + ev[1][k] * v + ev[4][k];
          const CT va = ev[2][k] * x + ev[3][k] * v + ev[5][k];
          x = xa;
          v = va;
          if (r0 + k < r1) {
            __stcs(o + (r0 + k) * SW, (ST)x);
            __stcs(o + (r0 + k) * SW + ncol, (ST)v);
            check(r0 + k, (double)gv[0][k], (double)x);
            check(r0 + k, (double)gv[NG > 1 ? 1 : 0][k], (double)v);
          }
        }
      }
      if constexpr (UPDATE) {
        dmb = warp_max_u64(dmb);
        if (lane == 0) atomicMax(&s_dm, dmb);
      }
    } else if constexpr (UPDATE) {
      const unsigned long long z = warp_max_u64(0ull);
      if (lane == 0) atomicMax(&s_dm, z);
    }
    if constexpr (UPDATE) {
      MG::sync();  // every row's flag is final
      unsigned nf = 0;
      for (int r = tid; r < rows; r += kScanThreads)
        if (s_fail[r]) {
          a.last_fail[row0 + r] = a.it;
          s_fail[r] = 0;
          ++nf;
        }
      nf = (unsigned)warp_sum_i((int)nf);
      if (lane == 0 && nf) atomicAdd(&a.stats->fail_rows, nf);
      if (tid == 0 && cur.s == cur.ns - 1) atomicMax((unsigned long long *)&a.stats->dmax, s_dm);
    }
    if (tid == 0 && cur.s == cur.ns - 1) scan_stamp(a, q, 9);
  };

#if CS_ROWS_PREFETCH
  // two register sets, swapped by unrolling the stage loop by two
  CT evA[NA][KR], evB[NA][KR];
  RowsJob cur = geo.first();
  if (geo.valid(cur)) load_stage(cur, evA);
  int64_t n = 0;
  while (geo.valid(cur)) {
    RowsJob nx = cur;
    geo.next(nx);
    if (geo.valid(nx)) load_stage(nx, evB);
    body(cur, n++, evA);
    cur = nx;
    if (!geo.valid(cur)) break;
    nx = cur;
    geo.next(nx);
    if (geo.valid(nx)) load_stage(nx, evA);
    body(cur, n++, evB);
    cur = nx;
  }
#else
  // one register set: occupancy hides the load latency better than a second
  // set would (measured); a bulk-copy (TMA) ring of stage slots measured
  // 0.8-1.4 TB/s here against 2.3-2.4 TB/s for register-streamed loads
  CT ev[NA][KR];
  int64_t n = 0;
  for (RowsJob cur = geo.first(); geo.valid(cur); geo.next(cur)) {
    load_stage(cur, ev);
    if constexpr (kTx) {
      if (tx) {  // flat (coalesced) order -> this thread's KR rows of column c
        const int KD = KR * ncol;
#pragma unroll
        for (int m = 0; m < KR / 4; ++m) {
          const int f = 4 * (tid + m * kScanThreads);
          const int pf = f + 4 * (f / KD);  // segment pad: 4 floats
          *(float4 *)(txb + pf) = make_float4(ev[0][4 * m], ev[0][4 * m + 1], ev[0][4 * m + 2], ev[0][4 * m + 3]);
          *(float4 *)(txb + txw + pf) = make_float4(ev[1][4 * m], ev[1][4 * m + 1], ev[1][4 * m + 2], ev[1][4 * m + 3]);
        }
        __syncthreads();
        const int base = sg * (KD + 4) + c;
#pragma unroll
        for (int k = 0; k < KR; ++k) {
          ev[0][k] = txb[base + k * ncol];
          ev[1][k] = txb[txw + base + k * ncol];
        }
        __syncthreads();
      }
    }
    body(cur, n++, ev);
  }
#endif
}

// ---------------------------------------------------------------------------
// wide rows (D > 64): tile = 64 rows x 32 columns, one column per lane,
// 8 row segments of 8 rows kept in registers.
constexpr int kWideSeg = 8;
template <typename ST, int VAR, bool AGG_ONLY = false, bool UPDATE = false>
__global__ void __launch_bounds__(kScanThreads)
scan_cols(ScanArgs<ST> a, LookbackWs ws) {
  constexpr int W = ColElem<VAR>::W;
  const int ncol = a.D;
  const int SW = VAR == SCAN_DIAG ? ncol : 2 * ncol;
  const int ncb = (ncol + 31) / 32;
  __shared__ int64_t s_tile;
  __shared__ double segagg[9][32][W];
  __shared__ double s_entry[2 * 32];
  __shared__ double s_acc[32 * W];
  __shared__ int s_ctl[1];
  if (threadIdx.x == 0) s_tile = atomicAdd(ws.ticket, 1u);
  __syncthreads();
  const int64_t tk = s_tile;
  const int64_t rb = tk / ncb;
  const int cb = (int)(tk % ncb);
  const int lane = threadIdx.x & 31, s = threadIdx.x >> 5;
  const int c = cb * 32 + lane;
  const bool colok = c < ncol;
  const int64_t rbase = rb * 64 + s * kWideSeg;
  double ej[kWideSeg], eu[kWideSeg], eb[kWideSeg], ec[kWideSeg], ed[kWideSeg], ev[kWideSeg];
  // UPDATE: the previous guess of this thread's rows, loaded up front so the
  // look-back hides them (loaded at the check they cost a round trip per row)
  // (diag only: the block variant has no registers to spare and reads them at the check)
  ST gx[(UPDATE && VAR == SCAN_DIAG) ? kWideSeg : 1];
  if constexpr (UPDATE && VAR == SCAN_DIAG) {
#pragma unroll
    for (int k = 0; k < kWideSeg; ++k) {
      const int64_t r = rbase + k;
      gx[k] = (colok && r < a.T) ? __ldg(a.guess + r * ncol + c) : (ST)0;
    }
  }
  ColElem<VAR> run;
  run.ident();
#pragma unroll
  for (int k = 0; k < kWideSeg; ++k) {
    const int64_t r = rbase + k;
    const bool ok = colok && r < a.T;
    if constexpr (VAR == SCAN_DIAG) {
      ej[k] = ok ? (double)a.e0[r * ncol + c] : 1.0;
      eu[k] = ok ? (double)a.u[r * ncol + c] : 0.0;
      run.push(ej[k], eu[k]);
    } else {
      ej[k] = ok ? (double)a.e0[r * ncol + c] : 1.0;
      eb[k] = ok ? (double)a.e1[r * ncol + c] : 0.0;
      ec[k] = ok ? (double)a.e2[r * ncol + c] : 0.0;
      ed[k] = ok ? (double)a.e3[r * ncol + c] : 1.0;
      eu[k] = ok ? (double)a.u[r * 2 * ncol + c] : 0.0;
      ev[k] = ok ? (double)a.u[r * 2 * ncol + ncol + c] : 0.0;
      run.push(ej[k], eb[k], ec[k], ed[k], eu[k], ev[k]);
    }
  }
  run.store(segagg[s][lane]);
  __syncthreads();
  if (threadIdx.x < 32) {
    ColElem<VAR> tot;
    tot.ident();
    for (int q = 0; q < 8; ++q) {
      ColElem<VAR> e;
      e.load(segagg[q][lane]);
      tot.store(segagg[q][lane]);
      tot.push(e);
    }
    tot.store(segagg[8][lane]);
    double tmp[W];
    tot.store(tmp);
    double *g = ws.agg + (tk * 32 + lane) * W;
#pragma unroll
    for (int k = 0; k < W; ++k) g[k] = tmp[k];
    __threadfence();
  }
  __syncthreads();
  if (threadIdx.x == 0) st_release(ws.status + tk, 1);
  if constexpr (AGG_ONLY) return;

  lookback_cta<VAR>(
      rb, 32, [&](int64_t p) { return ws.status + p * ncb + cb; },
      [&](int64_t p, int cc) { return ws.agg + ((p * ncb + cb) * 32 + cc) * W; },
      [&](int64_t p, int cc) { return cb * 32 + cc < ncol ? ld_cg(ws.exit + p * SW + cb * 32 + cc) : 0.0; },
      [&](int64_t p, int cc) { return cb * 32 + cc < ncol ? ld_cg(ws.exit + p * SW + ncol + cb * 32 + cc) : 0.0; },
      [&](int cc) { return cb * 32 + cc < ncol ? (double)a.s0[cb * 32 + cc] : 0.0; },
      [&](int cc) { return cb * 32 + cc < ncol ? (double)a.s0[ncol + cb * 32 + cc] : 0.0; }, s_acc, s_entry,
      s_ctl);

  if (threadIdx.x < 32) {
    ColElem<VAR> tot;
    tot.load(segagg[8][lane]);
    double x = s_entry[lane], v = VAR == SCAN_BLOCK ? s_entry[32 + lane] : 0.0;
    if constexpr (VAR == SCAN_DIAG) tot.apply(x);
    else tot.apply(x, v);
    if (colok) {
      ws.exit[rb * SW + c] = x;
      if (VAR == SCAN_BLOCK) ws.exit[rb * SW + ncol + c] = v;
    }
    __threadfence();
  }
  __syncthreads();
  if (threadIdx.x == 0) st_release(ws.status + tk, 2);

  __shared__ int s_fail[64];
  if constexpr (UPDATE) {
    if (threadIdx.x < 64) s_fail[threadIdx.x] = 0;
    __syncthreads();
  }
  unsigned long long dmb = 0ull;
  auto check = [&](int k, double g, double xv) {
    if constexpr (UPDATE) {
      const double xd = (double)(ST)xv;
      const double gap = fabs(xd - g);
      if (gap > a.atol + a.rtol * fabs(xd)) s_fail[s * kWideSeg + k] = 1;
      const unsigned long long gb = (unsigned long long)__double_as_longlong(gap);
      dmb = gb > dmb ? gb : dmb;
    }
  };
  ColElem<VAR> pre;
  pre.load(segagg[s][lane]);
  double x = s_entry[lane], v = VAR == SCAN_BLOCK ? s_entry[32 + lane] : 0.0;
  if constexpr (VAR == SCAN_DIAG) pre.apply(x);
  else pre.apply(x, v);
#pragma unroll
  for (int k = 0; k < kWideSeg; ++k) {
    const int64_t r = rbase + k;
    if (!(colok && r < a.T)) continue;
    if constexpr (VAR == SCAN_DIAG) {
      x = ej[k] * x + eu[k];
      a.out[r * ncol + c] = (ST)x;
      check(k, (double)gx[k], x);
    } else {
      const double xa = ej[k] * x + eb[k] * v + eu[k];
      const double va = ec[k] * x + ed[k] * v + ev[k];
      x = xa;
      v = va;
      a.out[r * 2 * ncol + c] = (ST)x;
      a.out[r * 2 * ncol + ncol + c] = (ST)v;
      if constexpr (UPDATE) {
        check(k, (double)__ldg(a.guess + r * 2 * ncol + c), x);
        check(k, (double)__ldg(a.guess + r * 2 * ncol + ncol + c), v);
      }
    }
  }
  if constexpr (UPDATE) {
    __shared__ unsigned s_nf;
    __shared__ unsigned long long s_dm;
    if (threadIdx.x == 0) { s_nf = 0; s_dm = 0ull; }
    __syncthreads();
    if (threadIdx.x < 64) {
      const int64_t r = rb * 64 + threadIdx.x;
      if (r < a.T && s_fail[threadIdx.x]) {
        a.last_fail[r] = a.it;
        atomicAdd(&s_nf, 1u);
      }
    }
    dmb = warp_max_u64(dmb);
    if ((threadIdx.x & 31) == 0) atomicMax(&s_dm, dmb);
    __syncthreads();
    if (threadIdx.x == 0) {
      if (s_nf) atomicAdd(&a.stats->fail_rows, s_nf);
      atomicMax((unsigned long long *)&a.stats->dmax, s_dm);
    }
  }
}

// ---------------------------------------------------------------------------
// wide rows, short sequences (D > 64, T <= 128; e.g. the leapfrog inside one HMC
// proposal, L = 100, state 2 x 1000): one CTA per 32 columns holds the whole
// sequence -- 16 warps x up to 8 rows in registers -- so there is no look-back
// between row tiles at all: segment aggregates meet in shared memory, each
// warp folds its predecessors' and replays.  Same arithmetic (f64) and the same
// bookkeeping as scan_cols.
constexpr int kSmallWarps = 16, kSmallRows = 8, kSmallT = kSmallWarps * kSmallRows;

template <typename ST, int VAR, bool UPDATE>
__global__ void __launch_bounds__(kSmallWarps * 32)
scan_cols_small(ScanArgs<ST> a) {
  constexpr int W = ColElem<VAR>::W;
  const int ncol = a.D;
  const int lane = threadIdx.x & 31, s = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  const bool colok = c < ncol;
  const int rpt = (int)((a.T + kSmallWarps - 1) / kSmallWarps);
  const int64_t rbase = (int64_t)s * rpt;
  __shared__ double segagg[kSmallWarps][32][W];
  __shared__ int s_fail[kSmallT];
  __shared__ unsigned s_nf;
  __shared__ unsigned long long s_dm;
  double ej[kSmallRows], eu[kSmallRows], eb[kSmallRows], ec[kSmallRows], ed[kSmallRows], ev[kSmallRows];
  ColElem<VAR> run;
  run.ident();
#pragma unroll
  for (int k = 0; k < kSmallRows; ++k) {
    const int64_t r = rbase + k;
    const bool ok = colok && k < rpt && r < a.T;
    if constexpr (VAR == SCAN_DIAG) {
      ej[k] = ok ? (double)a.e0[r * ncol + c] : 1.0;
      eu[k] = ok ? (double)a.u[r * ncol + c] : 0.0;
      run.push(ej[k], eu[k]);
    } else {
      ej[k] = ok ? (double)a.e0[r * ncol + c] : 1.0;
      eb[k] = ok ? (double)a.e1[r * ncol + c] : 0.0;
      ec[k] = ok ? (double)a.e2[r * ncol + c] : 0.0;
      ed[k] = ok ? (double)a.e3[r * ncol + c] : 1.0;
      eu[k] = ok ? (double)a.u[r * 2 * ncol + c] : 0.0;
      ev[k] = ok ? (double)a.u[r * 2 * ncol + ncol + c] : 0.0;
      run.push(ej[k], eb[k], ec[k], ed[k], eu[k], ev[k]);
    }
  }
  run.store(segagg[s][lane]);
  if constexpr (UPDATE) {
    for (int i = threadIdx.x; i < kSmallT; i += blockDim.x) s_fail[i] = 0;
    if (threadIdx.x == 0) { s_nf = 0; s_dm = 0ull; }
  }
  __syncthreads();
  // state entering this warp's rows: s0, then the earlier warps' segments
  double x = colok ? (double)a.s0[c] : 0.0, v = (VAR == SCAN_BLOCK && colok) ? (double)a.s0[ncol + c] : 0.0;
  for (int q = 0; q < s; ++q) {
    ColElem<VAR> e;
    e.load(segagg[q][lane]);
    if constexpr (VAR == SCAN_DIAG) e.apply(x);
    else e.apply(x, v);
  }
  unsigned long long dmb = 0ull;
  auto check = [&](int k, double g, double xv) {
    if constexpr (UPDATE) {
      const double xd = (double)(ST)xv;
      const double gap = fabs(xd - g);
      if (gap > a.atol + a.rtol * fabs(xd)) s_fail[s * rpt + k] = 1;
      const unsigned long long gb = (unsigned long long)__double_as_longlong(gap);
      dmb = gb > dmb ? gb : dmb;
    }
  };
  // replay (stores only), then the bookkeeping on the stored values with the
  // guess loads issued together (at the point of use they serialised, one L2
  // round trip per row)
  double xo[kSmallRows], vo[kSmallRows];
#pragma unroll
  for (int k = 0; k < kSmallRows; ++k) {
    const int64_t r = rbase + k;
    xo[k] = vo[k] = 0.0;
    if (!(colok && k < rpt && r < a.T)) continue;
    if constexpr (VAR == SCAN_DIAG) {
      x = ej[k] * x + eu[k];
      a.out[r * ncol + c] = (ST)x;
      xo[k] = x;
    } else {
      const double xa = ej[k] * x + eb[k] * v + eu[k];
      const double va = ec[k] * x + ed[k] * v + ev[k];
      x = xa;
      v = va;
      a.out[r * 2 * ncol + c] = (ST)x;
      a.out[r * 2 * ncol + ncol + c] = (ST)v;
      xo[k] = x;
      vo[k] = v;
    }
  }
  if constexpr (UPDATE) {
    double gx[kSmallRows], gw[kSmallRows];
#pragma unroll
    for (int k = 0; k < kSmallRows; ++k) {
      const int64_t r = rbase + k;
      const bool ok = colok && k < rpt && r < a.T;
      if constexpr (VAR == SCAN_DIAG) {
        gx[k] = ok ? (double)__ldg(a.guess + r * ncol + c) : 0.0;
      } else {
        gx[k] = ok ? (double)__ldg(a.guess + r * 2 * ncol + c) : 0.0;
        gw[k] = ok ? (double)__ldg(a.guess + r * 2 * ncol + ncol + c) : 0.0;
      }
    }
#pragma unroll
    for (int k = 0; k < kSmallRows; ++k) {
      const int64_t r = rbase + k;
      if (!(colok && k < rpt && r < a.T)) continue;
      check(k, gx[k], xo[k]);
      if constexpr (VAR == SCAN_BLOCK) check(k, gw[k], vo[k]);
    }
  }
  if constexpr (UPDATE) {
    dmb = warp_max_u64(dmb);
    if (lane == 0) atomicMax(&s_dm, dmb);
    __syncthreads();
    for (int i = threadIdx.x; i < a.T; i += blockDim.x)
      if (s_fail[i]) {
        a.last_fail[i] = a.it;
        atomicAdd(&s_nf, 1u);  // per column block, like scan_cols: only "any row failed" is used
      }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (s_nf) atomicAdd(&a.stats->fail_rows, s_nf);
      atomicMax((unsigned long long *)&a.stats->dmax, s_dm);
    }
  }
}

// ---------------------------------------------------------------------------
// dense, D <= MD <= 8: each thread folds SEG consecutive steps into (M, w) in
// registers; warp shuffles + smem give the block scan; look-back on the
// D-vector exit state.
template <int MD> struct DenseElem {
  double M[MD][MD], w[MD];
  CS_D void ident(int D) {
#pragma unroll
    for (int r = 0; r < MD; ++r) {
      w[r] = 0.0;
#pragma unroll
      for (int k = 0; k < MD; ++k) M[r][k] = (r == k) ? 1.0 : 0.0;
    }
  }
  // this <- e o this
  CS_D void push(const DenseElem &e) {
    double Mn[MD][MD], wn[MD];
#pragma unroll
    for (int r = 0; r < MD; ++r) {
      double aw = e.w[r];
#pragma unroll
      for (int k = 0; k < MD; ++k) aw += e.M[r][k] * w[k];
      wn[r] = aw;
#pragma unroll
      for (int cc = 0; cc < MD; ++cc) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < MD; ++k) acc += e.M[r][k] * M[k][cc];
        Mn[r][cc] = acc;
      }
    }
#pragma unroll
    for (int r = 0; r < MD; ++r) {
      w[r] = wn[r];
#pragma unroll
      for (int k = 0; k < MD; ++k) M[r][k] = Mn[r][k];
    }
  }
  CS_D void apply(double (&x)[MD]) const {
    double y[MD];
#pragma unroll
    for (int r = 0; r < MD; ++r) {
      double acc = w[r];
#pragma unroll
      for (int k = 0; k < MD; ++k) acc += M[r][k] * x[k];
      y[r] = acc;
    }
#pragma unroll
    for (int r = 0; r < MD; ++r) x[r] = y[r];
  }
  CS_D void shfl_up(const DenseElem &src, int delta, DenseElem &dst) const {
#pragma unroll
    for (int r = 0; r < MD; ++r) {
      dst.w[r] = __shfl_up_sync(0xffffffffu, src.w[r], delta);
#pragma unroll
      for (int k = 0; k < MD; ++k) dst.M[r][k] = __shfl_up_sync(0xffffffffu, src.M[r][k], delta);
    }
  }
};

template <typename ST, int MD>
CS_D void load_dense_elem(const ScanArgs<ST> &a, int64_t t, DenseElem<MD> &e) {
  const int D = a.D;
#pragma unroll
  for (int r = 0; r < MD; ++r) {
    e.w[r] = (r < D) ? (double)a.u[t * D + r] : 0.0;
#pragma unroll
    for (int k = 0; k < MD; ++k)
      e.M[r][k] = (r < D && k < D) ? (double)a.e0[(t * D + r) * D + k] : (r == k ? 1.0 : 0.0);
  }
}

template <typename ST, int MD, int SEG, bool AGG_ONLY = false>
__global__ void __launch_bounds__(kScanThreads)
scan_dense_small(ScanArgs<ST> a, LookbackWs ws) {
  __shared__ int64_t s_tile;
  __shared__ DenseElem<MD> warp_tot[kScanThreads / 32];
  __shared__ double s_entry[MD];
  if (threadIdx.x == 0) s_tile = atomicAdd(ws.ticket, 1u);
  __syncthreads();
  const int64_t b = s_tile;
  const int D = a.D;
  const int64_t t0 = (b * kScanThreads + threadIdx.x) * SEG;
  DenseElem<MD> run;
  run.ident(D);
  for (int k = 0; k < SEG; ++k) {
    const int64_t t = t0 + k;
    if (t < a.T) {
      DenseElem<MD> e;
      load_dense_elem(a, t, e);
      run.push(e);
    }
  }
  // inclusive warp scan: lane l gets e_l o ... o e_0
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  DenseElem<MD> inc = run;
#pragma unroll
  for (int dlt = 1; dlt < 32; dlt <<= 1) {
    DenseElem<MD> o;
    inc.shfl_up(inc, dlt, o);
    if (lane >= dlt) {
      DenseElem<MD> tmp = o;   // earlier part
      tmp.push(inc);           // inc o earlier
      inc = tmp;
    }
  }
  if (lane == 31) warp_tot[wid] = inc;
  __syncthreads();
  if (threadIdx.x == 0) {
    DenseElem<MD> tot;
    tot.ident(D);
    for (int q = 0; q < kScanThreads / 32; ++q) {
      DenseElem<MD> e = warp_tot[q];
      warp_tot[q] = tot;   // exclusive warp prefix
      tot.push(e);
    }
    // publish aggregate (M row-major then w)
    double *g = ws.agg + b * (MD * MD + MD);
#pragma unroll
    for (int r = 0; r < MD; ++r) {
      g[MD * MD + r] = tot.w[r];
#pragma unroll
      for (int k = 0; k < MD; ++k) g[r * MD + k] = tot.M[r][k];
    }
    __threadfence();
    st_release(ws.status + b, 1);
  }
  if constexpr (AGG_ONLY) return;
  if (threadIdx.x == 0) {
    // the tile total, as just published by this thread
    DenseElem<MD> tot;
    const double *g = ws.agg + b * (MD * MD + MD);
#pragma unroll
    for (int r = 0; r < MD; ++r) {
      tot.w[r] = g[MD * MD + r];
#pragma unroll
      for (int k = 0; k < MD; ++k) tot.M[r][k] = g[r * MD + k];
    }
    // look-back
    DenseElem<MD> acc;
    acc.ident(D);
    double x[MD];
    int64_t p = b - 1;
    while (p >= 0) {
      int st;
      do { st = ld_acquire(ws.status + p); } while (st == 0);
      if (st == 2) {
#pragma unroll
        for (int r = 0; r < MD; ++r) x[r] = (r < D) ? ld_cg(ws.exit + p * MD + r) : 0.0;
        break;
      }
      DenseElem<MD> e;
      const double *q = ws.agg + p * (MD * MD + MD);
#pragma unroll
      for (int r = 0; r < MD; ++r) {
        e.w[r] = ld_cg(q + MD * MD + r);
#pragma unroll
        for (int k = 0; k < MD; ++k) e.M[r][k] = ld_cg(q + r * MD + k);
      }
      // acc <- acc o e
      DenseElem<MD> tmp = e;
      tmp.push(acc);
      acc = tmp;
      --p;
    }
    if (p < 0) {
#pragma unroll
      for (int r = 0; r < MD; ++r) x[r] = (r < D) ? (double)a.s0[r] : 0.0;
    }
    acc.apply(x);
#pragma unroll
    for (int r = 0; r < MD; ++r) s_entry[r] = x[r];
    tot.apply(x);
#pragma unroll
    for (int r = 0; r < MD; ++r) ws.exit[b * MD + r] = x[r];
    __threadfence();
    st_release(ws.status + b, 2);
  }
  __syncthreads();
  // entry of this thread = (inclusive-warp-prefix of lanes < l) o warp prefix applied to tile entry
  double x[MD];
#pragma unroll
  for (int r = 0; r < MD; ++r) x[r] = s_entry[r];
  warp_tot[wid].apply(x);
  DenseElem<MD> exl;
  inc.shfl_up(inc, 1, exl);
  if (lane > 0) exl.apply(x);
  for (int k = 0; k < SEG; ++k) {
    const int64_t t = t0 + k;
    if (t >= a.T) break;
    DenseElem<MD> e;
    load_dense_elem(a, t, e);
    e.apply(x);
#pragma unroll
    for (int r = 0; r < MD; ++r)
      if (r < D) a.out[t * D + r] = (ST)x[r];
  }
}

// ---------------------------------------------------------------------------
// whole-sequence aggregate (the composed affine map of all T elements), used
// by the T-sharded driver to exchange one carry per shard: tile aggregates
// from the AGG_ONLY scans, then an ordered fold here.  Output layout (f64):
//   diag  [j(D) | u(D)]   block [A|B|C|E|ux|uv] each (D)   dense [M (DxD) | w(D)]
template <int VAR>
__global__ void __launch_bounds__(kScanThreads)
k_agg_compose_cols(const double *agg, int64_t nrt, int ncol, int ncb, double *out) {
  constexpr int W = ColElem<VAR>::W;
  __shared__ double part[kScanThreads][W];
  const int per_pass = ncol < kScanThreads ? ncol : kScanThreads;
  for (int c0 = 0; c0 < ncol; c0 += per_pass) {
    const int nc = min(per_pass, ncol - c0);
    const int nparts = kScanThreads / nc;
    const int t = threadIdx.x, c = c0 + t % nc, p = t / nc;
    if (p < nparts) {
      ColElem<VAR> run;
      run.ident();
      const int64_t per = (nrt + nparts - 1) / nparts;
      const int64_t lo = p * per, hi = lo + per < nrt ? lo + per : nrt;
      for (int64_t r = lo; r < hi; ++r) {
        const int64_t idx = ncb ? ((r * ncb + c / 32) * 32 + (c % 32)) : (r * ncol + c);
        ColElem<VAR> e;
        e.load(agg + idx * W);
        run.push(e);
      }
      run.store(part[t]);
    }
    __syncthreads();
    if (t < nc) {
      ColElem<VAR> tot;
      tot.ident();
      for (int q = 0; q < nparts; ++q) {
        ColElem<VAR> e;
        e.load(part[q * nc + t]);
        tot.push(e);
      }
      double v[W];
      tot.store(v);
#pragma unroll
      for (int k = 0; k < W; ++k) out[k * ncol + c0 + t] = v[k];
    }
    __syncthreads();
  }
}

template <int MD>
__global__ void k_agg_compose_dense(const double *agg, int64_t ntiles, int D, double *out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  DenseElem<MD> tot;
  tot.ident(D);
  for (int64_t q = 0; q < ntiles; ++q) {
    DenseElem<MD> e;
    const double *g = agg + q * (MD * MD + MD);
    for (int r = 0; r < MD; ++r) {
      e.w[r] = g[MD * MD + r];
      for (int k = 0; k < MD; ++k) e.M[r][k] = g[r * MD + k];
    }
    tot.push(e);
  }
  for (int r = 0; r < D; ++r) {
    out[D * D + r] = tot.w[r];
    for (int k = 0; k < D; ++k) out[r * D + k] = tot.M[r][k];
  }
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
// Single-pass row scan (plain diag, D <= 64).  Persistent CTAs claim tiles of
// R rows in order through the ticket (every predecessor of a claimed tile has
// been claimed, and its aggregate is published before its claimer waits on
// anything: forward progress without co-residency).  A tile's j and u arrive
// in shared memory by two 1-D bulk copies (TMA engine); each thread reduces its
// column segment (storage precision) and the tile aggregate (f64, fixed fold)
// is published and counted into its group.  The tile's look-back (two-level,
// the same fixed chain of single applications as scan_rows: bit-identical run
// to run), replay in place and bulk store run one claim later, while the next
// tile's copies are in flight -- the look-back is a round behind its
// predecessors instead of racing them.  HBM traffic is the algorithmic 12 B per
// f32 element: j and u read once, s written once.
constexpr int kRows1pMinB = 2;

template <typename ST>
__global__ void __launch_bounds__(kScanThreads, kRows1pMinB)
scan_rows_1p(ScanArgs<ST> a, LookbackWs ws, int R, int64_t ntiles) {
  using CT = ST;
  constexpr int W = 2;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ double s_acc[64 * W];
  __shared__ double s_acc2[64 * W];
  __shared__ double s_entry[2 * 64];
  __shared__ double s_gentry[2 * 64];
  __shared__ int s_ctl[1];
  __shared__ int s_gflag;
  __shared__ unsigned s_tile;
  __shared__ __align__(8) uint64_t s_bar[2];
  const int D = a.D, tid = threadIdx.x;
  const size_t tile_elems = (size_t)R * D;
  ST *buf = (ST *)smem_raw;  // [2][j | u] tiles
  const int nseg = kScanThreads / D, c = tid % D, sg = tid / D;
  const bool active = sg < nseg;
  CT *sa_base = (CT *)(buf + 4 * tile_elems);  // [2][nseg][D][2] segment aggregates
  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    fence_mbar_init();
  }
  unsigned use[2] = {0u, 0u};  // mbarrier phases per buffer
  auto claim = [&]() -> int64_t {
    if (tid == 0) s_tile = atomicAdd(ws.ticket, 1u);
    __syncthreads();
    const int64_t t = s_tile;
    __syncthreads();  // s_tile is rewritten by the next claim
    return t;
  };
  auto rows_of = [&](int64_t t) { return (int)(a.T - t * R < R ? a.T - t * R : R); };
  auto bulk_of = [&](int64_t t) { return (unsigned)(((size_t)rows_of(t) * D * sizeof(ST)) & ~(size_t)15); };
  // issue tile t's copies into buffer k (thread 0) and the ragged tail (all)
  auto load = [&](int64_t t, int k) {
    ST *jt = buf + (size_t)k * 2 * tile_elems, *ut = jt + tile_elems;
    const int64_t row0 = t * R;
    const unsigned bulk = bulk_of(t);
    if (tid == 0) {
      bulk_wait_read();  // the previous store out of this buffer has read it
      if (bulk) {
        mbar_expect_tx(&s_bar[k], 2 * bulk);
        bulk_g2s(jt, a.e0 + row0 * D, bulk, &s_bar[k]);
        bulk_g2s(ut, a.u + row0 * D, bulk, &s_bar[k]);
      }
    }
    const int n = rows_of(t) * D, nb = (int)(bulk / sizeof(ST));
    for (int i = nb + tid; i < n; i += kScanThreads) {
      jt[i] = a.e0[row0 * D + i];
      ut[i] = a.u[row0 * D + i];
    }
  };
  // wait for buffer k, reduce its segments, publish the tile aggregate
  auto reduce_publish = [&](int64_t t, int k) {
    ST *jt = buf + (size_t)k * 2 * tile_elems, *ut = jt + tile_elems;
    CT *sa = sa_base + (size_t)k * nseg * D * W;
    if (bulk_of(t)) mbar_wait(&s_bar[k], use[k]++ & 1);
    __syncthreads();
    const int rows = rows_of(t), rs = (rows + nseg - 1) / nseg, r0 = sg * rs, r1 = min(rows, r0 + rs);
    if (active) {
      SegE<SCAN_DIAG, CT> run;
      run.ident();
      for (int r = r0; r < r1; ++r) {
        SegE<SCAN_DIAG, CT> e;
        e.j = jt[r * D + c];
        e.u = ut[r * D + c];
        run.push(e);
      }
      run.store(sa + (sg * D + c) * W);
    }
    __syncthreads();
    if (tid < D) {
      ColElem<SCAN_DIAG> ch;
      ch.ident();
      for (int q = 0; q < nseg; ++q) {
        SegE<SCAN_DIAG, CT> x;
        x.load(sa + (q * D + tid) * W);
        ch.push(x.wide());
      }
      ch.store(ws.agg + (t * D + tid) * W);
      __threadfence();
    }
    __syncthreads();
    if (tid == 0) st_release(ws.status + t, 1);
    group_aggregate_publish<SCAN_DIAG, CtaGrp>(t, D, ws, &s_gflag);
  };
  // look back for tile t's entry, replay buffer k in place, store it
  auto finish = [&](int64_t t, int k) {
    ST *jt = buf + (size_t)k * 2 * tile_elems, *ut = jt + tile_elems;
    CT *sa = sa_base + (size_t)k * nseg * D * W;
    lookback_grouped<SCAN_DIAG, CtaGrp, 4>(
        t, D, ws, [&](int cc) { return (double)a.s0[cc]; }, [&](int) { return 0.0; }, s_acc, s_acc2, s_entry,
        s_gentry, s_ctl, [&](int) {});
    const int rows = rows_of(t), rs = (rows + nseg - 1) / nseg, r0 = sg * rs, r1 = min(rows, r0 + rs);
    if (active) {
      SegE<SCAN_DIAG, CT> pre;
      pre.ident();
      for (int q = 0; q < sg; ++q) {
        SegE<SCAN_DIAG, CT> x;
        x.load(sa + (q * D + c) * W);
        pre.push(x);
      }
      double xe = s_entry[c];
      pre.apply(xe);
      CT x = (CT)xe;
      for (int r = r0; r < r1; ++r) {
        x = jt[r * D + c] * x + ut[r * D + c];
        ut[r * D + c] = (ST)x;
      }
    }
    fence_proxy_async_smem();  // every thread's writes -> visible to the bulk store
    __syncthreads();
    const int64_t row0 = t * R;
    const unsigned bulk = bulk_of(t);
    if (tid == 0 && bulk) {
      bulk_s2g(a.out + row0 * D, ut, bulk);
      bulk_commit();
    }
    const int n = rows * D, nb = (int)(bulk / sizeof(ST));
    for (int i = nb + tid; i < n; i += kScanThreads) a.out[row0 * D + i] = ut[i];
  };
  int64_t cur = claim();
  if (cur >= ntiles) return;
  int kc = 0;
  load(cur, kc);
  reduce_publish(cur, kc);
  for (;;) {
    const int64_t nxt = claim();
    if (nxt < ntiles) {
      // the next tile's aggregate goes out before this tile's look-back, so
      // aggregates never wait on look-backs; the look-back then runs a tile behind
      load(nxt, kc ^ 1);
      reduce_publish(nxt, kc ^ 1);
    }
    finish(cur, kc);
    if (nxt >= ntiles) break;
    cur = nxt;
    kc ^= 1;
  }
  if (tid == 0) bulk_wait_read();
}

// ---------------------------------------------------------------------------
// Local-scan + fix-up row scan (plain diag, D <= 64; CS_SCAN_1P=3).  Every CTA
// owns one contiguous range of rows and scans it from a zero state in one
// streaming pass (j, u in by bulk copy, the local states s~ out by bulk
// store), recording the range aggregate (P = prod a, s~ at the end) and, per
// tile while P is not yet exactly zero, P at the tile start.  One CTA chains
// the ranges' entries (e_g, a fixed sequential walk), and a fix-up pass adds
// P_t e_g to the rows of each range's leading tiles: x_t = s~_t + P_t e_g.  P
// is carried in f64, so for a contracting map it reaches exactly zero after a
// few thousand rows and every later row is already final -- HBM moves j, u
// once and s once plus the fixed-up prefix of each range.
struct LocalWs {
  double *ragg;    // [G][D][2]  (P, s~ at the range end)
  double *rentry;  // [G][D]
  int *nfix;       // [G]       leading tiles with some P != 0
  double *tileP;   // [G][tmax][D]  P at each such tile's start
};

template <typename ST>
struct LocalStream {  // double-buffered bulk-copy stream of row tiles through shared memory
  ST *buf;
  size_t be;
  uint64_t *bar;
  unsigned use[2];
  int D;
  bool aligned;  // 16-byte aligned arrays: bulk copies, else plain loads / stores
  const ST *gsrc = nullptr;  // optional third stream (the previous guess), two slots at gbuf
  ST *gbuf = nullptr;
  CS_D ST *jt(int k) const { return buf + (size_t)k * 2 * be; }
  CS_D ST *ut(int k) const { return buf + (size_t)k * 2 * be + be; }
  CS_D ST *gt(int k) const { return gbuf + (size_t)k * be; }
  CS_D unsigned issue(const ST *j, const ST *u, int64_t row0, int rows, int k) const {
    const unsigned bulk = aligned ? (unsigned)(((size_t)rows * D * sizeof(ST)) & ~(size_t)15) : 0u;
    if (threadIdx.x == 0 && bulk) {
      mbar_expect_tx(&bar[k], (gsrc ? 3 : 2) * bulk);
      bulk_g2s(jt(k), j + row0 * D, bulk, &bar[k]);
      bulk_g2s(ut(k), u + row0 * D, bulk, &bar[k]);
      if (gsrc) bulk_g2s(gt(k), gsrc + row0 * D, bulk, &bar[k]);
    }
    return bulk;
  }
  CS_D void land(const ST *j, const ST *u, int64_t row0, int rows, int k, unsigned bulk) {
    const int n = rows * D, nb = (int)(bulk / sizeof(ST));
    for (int i = nb + threadIdx.x; i < n; i += kScanThreads) {
      jt(k)[i] = j[row0 * D + i];
      ut(k)[i] = u[row0 * D + i];
      if (gsrc) gt(k)[i] = gsrc[row0 * D + i];
    }
    if (bulk) mbar_wait(&bar[k], use[k]++ & 1);
    __syncthreads();
  }
  CS_D void store(ST *out, int64_t row0, int rows, int k, unsigned bulk) const {
    fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0 && bulk) {
      bulk_s2g(out + row0 * D, ut(k), bulk);
      bulk_commit();
    }
    const int n = rows * D, nb = (int)(bulk / sizeof(ST));
    for (int i = nb + threadIdx.x; i < n; i += kScanThreads) out[row0 * D + i] = ut(k)[i];
  }
};

// fused Newton bookkeeping (deer.py:273-277) on a tile whose states are final:
// rows with any |x - guess| > atol + rtol |x| get last_fail = it; fail-row count
// and max gap into the stats record (the scan_rows UPDATE semantics)
template <typename ST>
CS_D void local_bookkeep(const ScanArgs<ST> &a, const ST *xt, int64_t row0, int rows, int *s_fail,
                         unsigned long long *s_dm, const ST *gtile = nullptr) {  // gtile: the guess rows staged in smem
  const int D = a.D, tid = threadIdx.x, lane = tid & 31;
  for (int r = tid; r < rows; r += kScanThreads) s_fail[r] = 0;
  if (tid == 0) *s_dm = 0ull;
  __syncthreads();
  unsigned long long dmb = 0ull;
  const ST *gb = gtile ? gtile : a.guess + row0 * D;
  for (int i = tid; i < rows * D; i += kScanThreads) {
    const double xv = (double)xt[i];
    const double gap = fabs(xv - (double)gb[i]);
    if (gap > a.atol + a.rtol * fabs(xv)) s_fail[i / D] = 1;
    const unsigned long long bits = (unsigned long long)__double_as_longlong(gap);
    dmb = bits > dmb ? bits : dmb;
  }
  dmb = warp_max_u64(dmb);
  if (lane == 0) atomicMax(s_dm, dmb);
  __syncthreads();
  unsigned nf = 0;
  for (int r = tid; r < rows; r += kScanThreads)
    if (s_fail[r]) {
      a.last_fail[row0 + r] = a.it;
      ++nf;
    }
  nf = (unsigned)warp_sum_i((int)nf);
  if (lane == 0 && nf) atomicAdd(&a.stats->fail_rows, nf);
  if (tid == 0) atomicMax((unsigned long long *)&a.stats->dmax, *s_dm);
  __syncthreads();
}

CS_D void local_range(int64_t T, int G, int g, int64_t &lo, int64_t &hi) {  // 4-row aligned balanced split
  lo = (T * g / G) & ~(int64_t)3;
  hi = g == G - 1 ? T : (T * (g + 1) / G) & ~(int64_t)3;
}

template <typename ST, bool UPD = false>
__global__ void __launch_bounds__(kScanThreads, 2)
scan_local(ScanArgs<ST> a, LocalWs ws, int B, int tmax, bool aligned) {
  using CT = ST;
  constexpr int W = 2;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ double s_x[64], s_P[64];
  __shared__ int s_nz;
  __shared__ unsigned long long s_dm;
  __shared__ __align__(8) uint64_t s_bar[2];
  const int D = a.D, tid = threadIdx.x, G = gridDim.x, g = blockIdx.x;
  const size_t be = (size_t)B * D;
  LocalStream<ST> S{(ST *)smem_raw, be, s_bar, {0u, 0u}, D, aligned};
  double *sa = (double *)(S.buf + 4 * be);  // f64 segment aggregates: P and the range exits stay exact products
  int *s_fail = (int *)(sa + 2 * (kScanThreads / D) * D);  // UPD: one flag per tile row
  const int nseg = kScanThreads / D, c = tid % D, sg = tid / D;
  const bool active = sg < nseg;
  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    fence_mbar_init();
  }
  if (tid < D) {
    s_x[tid] = 0.0;
    s_P[tid] = 1.0;
  }
  __syncthreads();
  int64_t lo, hi;
  local_range(a.T, G, g, lo, hi);
  const int nblk = (int)((hi - lo + B - 1) / B);
  int nfix = 0;
  bool nz = true;  // some column's P is still nonzero
  unsigned bk[2] = {0u, 0u};
  if (nblk > 0) bk[0] = S.issue(a.e0, a.u, lo, (int)(hi - lo < B ? hi - lo : B), 0);
  for (int k = 0; k < nblk; ++k) {
    const int64_t row0 = lo + (int64_t)k * B;
    const int rows = (int)(hi - row0 < B ? hi - row0 : B);
    const int kb = k & 1;
    if (k + 1 < nblk) {
      if (tid == 0) bulk_wait_read();
      __syncthreads();
      const int64_t rn = row0 + B;
      bk[kb ^ 1] = S.issue(a.e0, a.u, rn, (int)(hi - rn < B ? hi - rn : B), kb ^ 1);
    }
    const bool fixed_later = nz;  // this tile's states get P e added by the fix-up pass
    if (nz) {
      if (tid < D) ws.tileP[((size_t)g * tmax + k) * D + tid] = s_P[tid];
      nfix = k + 1;
    }
    S.land(a.e0, a.u, row0, rows, kb, bk[kb]);
    ST *jt = S.jt(kb), *ut = S.ut(kb);
    const int rs = (rows + nseg - 1) / nseg, r0 = sg * rs, r1 = min(rows, r0 + rs);
    if (active) {
      SegE<SCAN_DIAG, double> run;
      run.ident();
      for (int r = r0; r < r1; ++r) {
        SegE<SCAN_DIAG, double> e;
        e.j = (double)jt[r * D + c];
        e.u = (double)ut[r * D + c];
        run.push(e);
      }
      run.store(sa + (sg * D + c) * W);
    }
    __syncthreads();
    if (active) {  // replay from the local running state
      double xe = s_x[c];
      for (int q = 0; q < sg; ++q) {  // the segments before this one, in order (f64)
        SegE<SCAN_DIAG, double> x;
        x.load(sa + (q * D + c) * W);
        x.apply(xe);
      }
      CT x = (CT)xe;
      for (int r = r0; r < r1; ++r) {
        x = jt[r * D + c] * x + ut[r * D + c];
        ut[r * D + c] = (ST)x;
      }
    }
    __syncthreads();
    if (tid == 0) s_nz = 0;
    __syncthreads();
    if (tid < D) {  // the tile's exit (segments in order, f64) and P through it
      double xv = s_x[tid], P = s_P[tid];
      for (int q = 0; q < nseg; ++q) {
        SegE<SCAN_DIAG, double> e;
        e.load(sa + (q * D + tid) * W);
        e.apply(xv);
        P *= e.j;
      }
      s_x[tid] = xv;
      s_P[tid] = P;
      if (P != 0.0) s_nz = 1;
    }
    if constexpr (UPD) {
      if (!fixed_later) local_bookkeep(a, (const ST *)ut, row0, rows, s_fail, &s_dm);  // these states are final
    }
    S.store(a.out, row0, rows, kb, bk[kb]);
    __syncthreads();
    nz = s_nz != 0;
  }
  if (tid == 0) bulk_wait_read();
  if (tid < D) {
    ws.ragg[((size_t)g * D + tid) * W] = s_P[tid];
    ws.ragg[((size_t)g * D + tid) * W + 1] = s_x[tid];
  }
  if (tid == 0) ws.nfix[g] = nfix;
}

// entries of the ranges: e_0 = s0, e_{g+1} = P_g e_g + s~_g (one thread per column, in order)
template <typename ST>
__global__ void scan_local_carry(const ST *s0, LocalWs ws, int G, int D) {
  constexpr int KB = 32;  // range aggregates in flight per round trip, then applied in order
  for (int c = threadIdx.x; c < D; c += blockDim.x) {
    double e = (double)s0[c];
    for (int g0 = 0; g0 < G; g0 += KB) {
      double A[KB], Bv[KB];
#pragma unroll
      for (int k = 0; k < KB; ++k)
        if (g0 + k < G) {
          A[k] = ws.ragg[((size_t)(g0 + k) * D + c) * 2];
          Bv[k] = ws.ragg[((size_t)(g0 + k) * D + c) * 2 + 1];
        }
#pragma unroll
      for (int k = 0; k < KB; ++k)
        if (g0 + k < G) {
          ws.rentry[(size_t)(g0 + k) * D + c] = e;
          e = A[k] * e + Bv[k];
        }
    }
  }
}

// x_t = s~_t + P_t e_g over each range's leading tiles (P_t = P at the tile start
// times the a's of the rows up to t, f64)
template <typename ST, bool UPD = false>
__global__ void __launch_bounds__(kScanThreads, 2)
scan_local_fixup(ScanArgs<ST> a, LocalWs ws, int B, int tmax, bool aligned) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t s_bar[2];
  __shared__ unsigned long long s_dm;
  __shared__ double s_pre[kScanThreads];  // [seg][col] P at the segment start (nseg * D <= 256)
  const int D = a.D, tid = threadIdx.x, G = gridDim.x, g = blockIdx.x;
  const size_t be = (size_t)B * D;
  LocalStream<ST> S{(ST *)smem_raw, be, s_bar, {0u, 0u}, D, aligned};
  const int nseg = kScanThreads / D, c = tid % D, sg = tid / D;
  const bool active = sg < nseg;
  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  int64_t lo, hi;
  local_range(a.T, G, g, lo, hi);
  const int nblk = ws.nfix[g];
  const double e = active ? ws.rentry[(size_t)g * D + c] : 0.0;
  unsigned bk[2] = {0u, 0u};
  // j in, the local states (a.out) in the u slot, fixed states back out
  if (nblk > 0) bk[0] = S.issue(a.e0, a.out, lo, (int)(hi - lo < B ? hi - lo : B), 0);
  for (int k = 0; k < nblk; ++k) {
    const int64_t row0 = lo + (int64_t)k * B;
    const int rows = (int)(hi - row0 < B ? hi - row0 : B);
    const int kb = k & 1;
    if (k + 1 < nblk) {
      if (tid == 0) bulk_wait_read();
      __syncthreads();
      const int64_t rn = row0 + B;
      bk[kb ^ 1] = S.issue(a.e0, a.out, rn, (int)(hi - rn < B ? hi - rn : B), kb ^ 1);
    }
    S.land(a.e0, a.out, row0, rows, kb, bk[kb]);
    ST *jt = S.jt(kb), *xt = S.ut(kb);
    const int rs = (rows + nseg - 1) / nseg, r0 = sg * rs, r1 = min(rows, r0 + rs);
    double pseg = 1.0;
    if (active)
      for (int r = r0; r < r1; ++r) pseg *= (double)jt[r * D + c];
    if (active) s_pre[sg * D + c] = pseg;
    __syncthreads();
    if (tid < D) {  // exclusive products over the segments, from the tile's recorded start
      double P = ws.tileP[((size_t)g * tmax + k) * D + tid];
      for (int q = 0; q < nseg; ++q) {
        const double v = s_pre[q * D + tid];
        s_pre[q * D + tid] = P;
        P *= v;
      }
    }
    __syncthreads();
    if (active) {
      double P = s_pre[sg * D + c];
      for (int r = r0; r < r1; ++r) {
        P *= (double)jt[r * D + c];
        if (e != 0.0) xt[r * D + c] = (ST)((double)xt[r * D + c] + P * e);  // e = 0: nothing to add (even if P overflowed)
      }
    }
    if constexpr (UPD) {
      __syncthreads();
      local_bookkeep(a, (const ST *)xt, row0, rows, (int *)(S.buf + 4 * be), &s_dm);
    }
    S.store(a.out, row0, rows, kb, bk[kb]);
    __syncthreads();
  }
  if (tid == 0) bulk_wait_read();
}

// ---------------------------------------------------------------------------
// Reduce-then-replay row scan with the fused Newton bookkeeping (diag, moderate
// T): the local scan's ranges, but the first pass only forms each range's map
// (tiles walked last to first, so the replay's first tiles are the ones still
// in L2), and the replay scans every
// range from its true entry (each CTA folds the maps of the ranges before its
// own while its first tile lands).  No fix-up, however slowly the maps contract (the
// Newton iterates of cfg 5 do): j, u are read twice, guess once, s written once.
constexpr int kRrMaxD = 256;  // one thread per column at least (nseg = 256 / D >= 1)
CS_HD size_t rr_guess_off(int B, int D, size_t esz) {  // after the j/u slots, segment aggregates, row flags
  const size_t o = 4 * (size_t)B * D * esz + (size_t)(kScanThreads / D) * D * 2 * sizeof(double) + sizeof(int) * (size_t)B;
  return (o + 127) & ~(size_t)127;
}
template <typename ST>
__global__ void __launch_bounds__(kScanThreads, 2)
scan_rr_reduce(ScanArgs<ST> a, LocalWs ws, int B, bool aligned) {
  constexpr int W = 2;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ double s_x[kRrMaxD], s_P[kRrMaxD];  // map of the tiles after the current one
  __shared__ __align__(8) uint64_t s_bar[2];
  const int D = a.D, tid = threadIdx.x, G = gridDim.x, g = blockIdx.x;
  const size_t be = (size_t)B * D;
  LocalStream<ST> S{(ST *)smem_raw, be, s_bar, {0u, 0u}, D, aligned};
  double *sa = (double *)(S.buf + 4 * be);
  const int nseg = kScanThreads / D, c = tid % D, sg = tid / D;
  const bool active = sg < nseg;
  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    fence_mbar_init();
  }
  if (tid < D) {
    s_x[tid] = 0.0;
    s_P[tid] = 1.0;
  }
  __syncthreads();
  int64_t lo, hi;
  local_range(a.T, G, g, lo, hi);
  const int nblk = (int)((hi - lo + B - 1) / B);
  unsigned bk[2] = {0u, 0u};
  if (nblk > 0) {
    const int64_t rl = lo + (int64_t)(nblk - 1) * B;
    bk[(nblk - 1) & 1] = S.issue(a.e0, a.u, rl, (int)(hi - rl), (nblk - 1) & 1);
  }
  for (int k = nblk - 1; k >= 0; --k) {
    const int64_t row0 = lo + (int64_t)k * B;
    const int rows = (int)(hi - row0 < B ? hi - row0 : B);
    const int kb = k & 1;
    if (k > 0) {
      __syncthreads();  // the slot the previous tile lands in is free
      bk[kb ^ 1] = S.issue(a.e0, a.u, row0 - B, B, kb ^ 1);
    }
    S.land(a.e0, a.u, row0, rows, kb, bk[kb]);
    const ST *jt = S.jt(kb), *ut = S.ut(kb);
    const int rs = (rows + nseg - 1) / nseg, r0 = sg * rs, r1 = min(rows, r0 + rs);
    if (active) {
      SegE<SCAN_DIAG, double> run;
      run.ident();
      for (int r = r0; r < r1; ++r) {
        SegE<SCAN_DIAG, double> e;
        e.j = (double)jt[r * D + c];
        e.u = (double)ut[r * D + c];
        run.push(e);
      }
      run.store(sa + (sg * D + c) * W);
    }
    __syncthreads();
    if (tid < D) {  // (tiles after) o (this tile), the tile's segments in order
      double xv = 0.0, P = 1.0;
      for (int q = 0; q < nseg; ++q) {
        SegE<SCAN_DIAG, double> e;
        e.load(sa + (q * D + tid) * W);
        e.apply(xv);
        P *= e.j;
      }
      const double Pl = s_P[tid];
      s_x[tid] = (xv != 0.0 ? Pl * xv : 0.0) + s_x[tid];
      s_P[tid] = Pl * P;
    }
  }
  __syncthreads();
  if (tid < D) {
    ws.ragg[((size_t)g * D + tid) * W] = s_P[tid];
    ws.ragg[((size_t)g * D + tid) * W + 1] = s_x[tid];
  }
}

template <typename ST, bool UPD>
__global__ void __launch_bounds__(kScanThreads, 2)
scan_rr_replay(ScanArgs<ST> a, LocalWs ws, int B, bool aligned) {
  using CT = ST;
  constexpr int W = 2;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ double s_x[kRrMaxD];
  __shared__ unsigned long long s_dm;
  __shared__ unsigned s_nf;
  __shared__ __align__(8) uint64_t s_bar[2];
  const int D = a.D, tid = threadIdx.x, lane = tid & 31, G = gridDim.x, g = blockIdx.x;
  const size_t be = (size_t)B * D;
  LocalStream<ST> S{(ST *)smem_raw, be, s_bar, {0u, 0u}, D, aligned};
  double *sa = (double *)(S.buf + 4 * be);
  int *s_fail = (int *)(sa + 2 * (kScanThreads / D) * D);
  if constexpr (UPD) {  // the guess rows ride the same bulk copies (two more slots after the row flags)
    S.gsrc = a.guess;
    S.gbuf = (ST *)((unsigned char *)smem_raw + rr_guess_off(B, D, sizeof(ST)));
  }
  const int nseg = kScanThreads / D, c = tid % D, sg = tid / D;
  const bool active = sg < nseg;
  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    fence_mbar_init();
    s_dm = 0ull;
    s_nf = 0u;
  }
  for (int r = tid; r < B; r += kScanThreads) s_fail[r] = 0;
  __syncthreads();
  int64_t lo, hi;
  local_range(a.T, G, g, lo, hi);
  const int nblk = (int)((hi - lo + B - 1) / B);
  unsigned bk[2] = {0u, 0u};
  if (nblk > 0) bk[0] = S.issue(a.e0, a.u, lo, (int)(hi - lo < B ? hi - lo : B), 0);
  // this range's entry while the first tile lands: s0 through ranges 0..g-1 in
  // order (f64) -- each of a column's threads composes a contiguous run of the
  // range maps, then one thread per column chains the runs
  if (active) {
    constexpr int KP = 8;
    const int per = (g + nseg - 1) / nseg, q0 = min(g, sg * per), q1 = min(g, q0 + per);
    double P = 1.0, X = 0.0;
    for (int qb = q0; qb < q1; qb += KP) {
      double pa[KP], xa[KP];
#pragma unroll
      for (int i = 0; i < KP; ++i)
        if (qb + i < q1) {
          pa[i] = ws.ragg[((size_t)(qb + i) * D + c) * 2];
          xa[i] = ws.ragg[((size_t)(qb + i) * D + c) * 2 + 1];
        }
#pragma unroll
      for (int i = 0; i < KP; ++i)
        if (qb + i < q1) {
          X = (X != 0.0 ? pa[i] * X : 0.0) + xa[i];
          P *= pa[i];
        }
    }
    sa[(sg * D + c) * W] = P;
    sa[(sg * D + c) * W + 1] = X;
  }
  __syncthreads();
  if (tid < D) {
    double e = (double)a.s0[tid];
    for (int q = 0; q < nseg; ++q) {
      const double P = sa[(q * D + tid) * W], X = sa[(q * D + tid) * W + 1];
      e = (e != 0.0 ? P * e : 0.0) + X;
    }
    s_x[tid] = e;
  }
  __syncthreads();
  unsigned long long dmb = 0ull;  // bookkeeping partials over all of this thread's rows
  unsigned nf = 0;
  for (int k = 0; k < nblk; ++k) {
    const int64_t row0 = lo + (int64_t)k * B;
    const int rows = (int)(hi - row0 < B ? hi - row0 : B);
    const int kb = k & 1;
    if (k + 1 < nblk) {
      if (tid == 0) bulk_wait_read();
      __syncthreads();
      const int64_t rn = row0 + B;
      bk[kb ^ 1] = S.issue(a.e0, a.u, rn, (int)(hi - rn < B ? hi - rn : B), kb ^ 1);
    }
    S.land(a.e0, a.u, row0, rows, kb, bk[kb]);
    ST *jt = S.jt(kb), *ut = S.ut(kb);
    const int rs = (rows + nseg - 1) / nseg, r0 = sg * rs, r1 = min(rows, r0 + rs);
    if (active) {  // segment maps in the storage precision (no exact-zero P needed here)
      SegE<SCAN_DIAG, CT> run;
      run.ident();
      for (int r = r0; r < r1; ++r) {
        SegE<SCAN_DIAG, CT> e;
        e.j = jt[r * D + c];
        e.u = ut[r * D + c];
        run.push(e);
      }
      sa[(sg * D + c) * W] = (double)run.j;
      sa[(sg * D + c) * W + 1] = (double)run.u;
    }
    __syncthreads();
    if (active) {  // replay from the tile's entry and the segments before this one (f64)
      double xe = s_x[c];
      for (int q = 0; q < sg; ++q) {
        SegE<SCAN_DIAG, double> x;
        x.load(sa + (q * D + c) * W);
        x.apply(xe);
      }
      CT x = (CT)xe;
      const ST *gt = UPD ? S.gt(kb) : nullptr;
      for (int r = r0; r < r1; ++r) {
        x = jt[r * D + c] * x + ut[r * D + c];
        ut[r * D + c] = (ST)x;
        if constexpr (UPD) {  // deer.py:273-275 on the stored value
          const double xv = (double)(ST)x, gap = fabs(xv - (double)gt[r * D + c]);
          if (gap > a.atol + a.rtol * fabs(xv)) s_fail[r] = 1;
          const unsigned long long bits = (unsigned long long)__double_as_longlong(gap);
          dmb = bits > dmb ? bits : dmb;
        }
      }
    }
    __syncthreads();
    if (tid < D) {  // the tile's exit
      double xv = s_x[tid];
      for (int q = 0; q < nseg; ++q) {
        SegE<SCAN_DIAG, double> e;
        e.load(sa + (q * D + tid) * W);
        e.apply(xv);
      }
      s_x[tid] = xv;
    }
    if constexpr (UPD) {
      for (int r = tid; r < rows; r += kScanThreads)
        if (s_fail[r]) {
          a.last_fail[row0 + r] = a.it;
          s_fail[r] = 0;
          ++nf;
        }
    }
    S.store(a.out, row0, rows, kb, bk[kb]);
    __syncthreads();
  }
  if constexpr (UPD) {
    dmb = warp_max_u64(dmb);
    nf = (unsigned)warp_sum_i((int)nf);
    if (lane == 0) {
      atomicMax(&s_dm, dmb);
      if (nf) atomicAdd(&s_nf, nf);
    }
    __syncthreads();
    if (tid == 0) {
      if (s_nf) atomicAdd(&a.stats->fail_rows, s_nf);
      atomicMax((unsigned long long *)&a.stats->dmax, s_dm);
    }
  }
  if (tid == 0) bulk_wait_read();
}

// ---------------------------------------------------------------------------
// Block2x2 version of the local scan + fix-up (plain block scans): per column
// the state is (x, v), the map M_t = (a b; c d) with u_t = (ux, uv); P is the
// 2 x 2 product of the range's maps (f64), x_t = s~_t + P_t e_g.  Tiles carry
// a, b, c, d (B x D each) and u (B x 2D, rows [x | v]); the states replace u.
template <typename ST>
struct BlkTile {  // the five input slots of one ring buffer
  ST *a, *b, *c, *d, *u;
};

template <typename ST>
CS_D BlkTile<ST> blk_tile(ST *buf, size_t be, int k) {
  ST *base = buf + (size_t)k * 6 * be;
  return BlkTile<ST>{base, base + be, base + 2 * be, base + 3 * be, base + 4 * be};
}

template <typename ST>
CS_D unsigned blk_issue(const ScanArgs<ST> &a, BlkTile<ST> t, int64_t row0, int rows, uint64_t *bar, bool aligned,
                        const ST *usrc) {
  const int D = a.D;
  const unsigned bh = aligned ? (unsigned)(((size_t)rows * D * sizeof(ST)) & ~(size_t)15) : 0u;
  const unsigned bu = aligned ? (unsigned)(((size_t)rows * 2 * D * sizeof(ST)) & ~(size_t)15) : 0u;
  if (threadIdx.x == 0 && bh) {
    mbar_expect_tx(bar, 4 * bh + bu);
    bulk_g2s(t.a, a.e0 + row0 * D, bh, bar);
    bulk_g2s(t.b, a.e1 + row0 * D, bh, bar);
    bulk_g2s(t.c, a.e2 + row0 * D, bh, bar);
    bulk_g2s(t.d, a.e3 + row0 * D, bh, bar);
    bulk_g2s(t.u, usrc + row0 * 2 * D, bu, bar);
  }
  return bh;
}

template <typename ST>
CS_D void blk_land(const ScanArgs<ST> &a, BlkTile<ST> t, int64_t row0, int rows, unsigned bh, uint64_t *bar,
                   unsigned &use, const ST *usrc) {
  const int D = a.D;
  const int n = rows * D, nb = (int)(bh / sizeof(ST));
  const int nbu = bh ? (int)((((size_t)rows * 2 * D * sizeof(ST)) & ~(size_t)15) / sizeof(ST)) : 0;
  for (int i = nb + threadIdx.x; i < n; i += kScanThreads) {
    t.a[i] = a.e0[row0 * D + i];
    t.b[i] = a.e1[row0 * D + i];
    t.c[i] = a.e2[row0 * D + i];
    t.d[i] = a.e3[row0 * D + i];
  }
  for (int i = nbu + threadIdx.x; i < 2 * n; i += kScanThreads) t.u[i] = usrc[row0 * 2 * D + i];
  if (bh) mbar_wait(bar, use++ & 1);
  __syncthreads();
}

template <typename ST>
CS_D void blk_store(const ScanArgs<ST> &a, BlkTile<ST> t, int64_t row0, int rows, bool aligned) {
  const int D = a.D;
  const unsigned bu = aligned ? (unsigned)(((size_t)rows * 2 * D * sizeof(ST)) & ~(size_t)15) : 0u;
  fence_proxy_async_smem();
  __syncthreads();
  if (threadIdx.x == 0 && bu) {
    bulk_s2g(a.out + row0 * 2 * D, t.u, bu);
    bulk_commit();
  }
  const int nb = (int)(bu / sizeof(ST));
  for (int i = nb + threadIdx.x; i < rows * 2 * D; i += kScanThreads) a.out[row0 * 2 * D + i] = t.u[i];
}

template <typename ST>
__global__ void __launch_bounds__(kScanThreads, 2)
scan_local_blk(ScanArgs<ST> a, LocalWs ws, int B, int tmax, bool aligned) {
  using CT = ST;
  constexpr int W = 6;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ double s_x[64], s_v[64], s_P[4 * 64];
  __shared__ int s_nz;
  __shared__ __align__(8) uint64_t s_bar[2];
  const int D = a.D, tid = threadIdx.x, G = gridDim.x, g = blockIdx.x;
  const size_t be = (size_t)B * D;
  ST *buf = (ST *)smem_raw;
  double *sa = (double *)(buf + 12 * be);  // [nseg][D][6] f64
  const int nseg = kScanThreads / D, c = tid % D, sg = tid / D;
  const bool active = sg < nseg;
  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    fence_mbar_init();
  }
  if (tid < D) {
    s_x[tid] = 0.0;
    s_v[tid] = 0.0;
    s_P[4 * tid] = 1.0;
    s_P[4 * tid + 1] = 0.0;
    s_P[4 * tid + 2] = 0.0;
    s_P[4 * tid + 3] = 1.0;
  }
  __syncthreads();
  unsigned use[2] = {0u, 0u};
  int64_t lo, hi;
  local_range(a.T, G, g, lo, hi);
  const int nblk = (int)((hi - lo + B - 1) / B);
  int nfix = 0;
  bool nz = true;
  unsigned bk[2] = {0u, 0u};
  if (nblk > 0) bk[0] = blk_issue(a, blk_tile(buf, be, 0), lo, (int)(hi - lo < B ? hi - lo : B), &s_bar[0], aligned, a.u);
  for (int k = 0; k < nblk; ++k) {
    const int64_t row0 = lo + (int64_t)k * B;
    const int rows = (int)(hi - row0 < B ? hi - row0 : B);
    const int kb = k & 1;
    if (k + 1 < nblk) {
      if (tid == 0) bulk_wait_read();
      __syncthreads();
      const int64_t rn = row0 + B;
      bk[kb ^ 1] = blk_issue(a, blk_tile(buf, be, kb ^ 1), rn, (int)(hi - rn < B ? hi - rn : B), &s_bar[kb ^ 1],
                             aligned, a.u);
    }
    if (nz) {
      if (tid < 4 * D) ws.tileP[((size_t)g * tmax + k) * 4 * D + tid] = s_P[tid];
      nfix = k + 1;
    }
    BlkTile<ST> t = blk_tile(buf, be, kb);
    blk_land(a, t, row0, rows, bk[kb], &s_bar[kb], use[kb], a.u);
    const int rs = (rows + nseg - 1) / nseg, r0 = sg * rs, r1 = min(rows, r0 + rs);
    if (active) {
      SegE<SCAN_BLOCK, double> run;
      run.ident();
      for (int r = r0; r < r1; ++r) {
        SegE<SCAN_BLOCK, double> e;
        e.A = (double)t.a[r * D + c];
        e.B = (double)t.b[r * D + c];
        e.C = (double)t.c[r * D + c];
        e.E = (double)t.d[r * D + c];
        e.ux = (double)t.u[r * 2 * D + c];
        e.uv = (double)t.u[r * 2 * D + D + c];
        run.push(e);
      }
      run.store(sa + (sg * D + c) * W);
    }
    __syncthreads();
    if (active) {
      double xe = s_x[c], ve = s_v[c];
      for (int q = 0; q < sg; ++q) {
        SegE<SCAN_BLOCK, double> e;
        e.load(sa + (q * D + c) * W);
        e.apply(xe, ve);
      }
      CT x = (CT)xe, v = (CT)ve;
      for (int r = r0; r < r1; ++r) {
        const CT xa = t.a[r * D + c] * x + t.b[r * D + c] * v + t.u[r * 2 * D + c];
        const CT va = t.c[r * D + c] * x + t.d[r * D + c] * v + t.u[r * 2 * D + D + c];
        x = xa;
        v = va;
        t.u[r * 2 * D + c] = (ST)x;
        t.u[r * 2 * D + D + c] = (ST)v;
      }
    }
    __syncthreads();
    if (tid == 0) s_nz = 0;
    __syncthreads();
    if (tid < D) {
      double xv = s_x[tid], vv = s_v[tid];
      double p0 = s_P[4 * tid], p1 = s_P[4 * tid + 1], p2 = s_P[4 * tid + 2], p3 = s_P[4 * tid + 3];
      for (int q = 0; q < nseg; ++q) {
        SegE<SCAN_BLOCK, double> e;
        e.load(sa + (q * D + tid) * W);
        e.apply(xv, vv);
        const double n0 = e.A * p0 + e.B * p2, n1 = e.A * p1 + e.B * p3;
        const double n2 = e.C * p0 + e.E * p2, n3 = e.C * p1 + e.E * p3;
        p0 = n0;
        p1 = n1;
        p2 = n2;
        p3 = n3;
      }
      s_x[tid] = xv;
      s_v[tid] = vv;
      s_P[4 * tid] = p0;
      s_P[4 * tid + 1] = p1;
      s_P[4 * tid + 2] = p2;
      s_P[4 * tid + 3] = p3;
      if (p0 != 0.0 || p1 != 0.0 || p2 != 0.0 || p3 != 0.0) s_nz = 1;
    }
    blk_store(a, t, row0, rows, aligned);
    __syncthreads();
    nz = s_nz != 0;
  }
  if (tid == 0) bulk_wait_read();
  if (tid < D) {
    double *o = ws.ragg + ((size_t)g * D + tid) * 6;
    o[0] = s_P[4 * tid];
    o[1] = s_P[4 * tid + 1];
    o[2] = s_P[4 * tid + 2];
    o[3] = s_P[4 * tid + 3];
    o[4] = s_x[tid];
    o[5] = s_v[tid];
  }
  if (tid == 0) ws.nfix[g] = nfix;
}

template <typename ST>
__global__ void scan_local_carry_blk(const ST *s0, LocalWs ws, int G, int D) {
  constexpr int KB = 8;  // range aggregates in flight per round trip, then applied in order
  for (int c = threadIdx.x; c < D; c += blockDim.x) {
    double ex = (double)s0[c], ev = (double)s0[D + c];
    for (int g0 = 0; g0 < G; g0 += KB) {
      double r[KB][6];
#pragma unroll
      for (int k = 0; k < KB; ++k)
        if (g0 + k < G)
#pragma unroll
          for (int q = 0; q < 6; ++q) r[k][q] = ws.ragg[((size_t)(g0 + k) * D + c) * 6 + q];
#pragma unroll
      for (int k = 0; k < KB; ++k)
        if (g0 + k < G) {
          ws.rentry[((size_t)(g0 + k) * D + c) * 2] = ex;
          ws.rentry[((size_t)(g0 + k) * D + c) * 2 + 1] = ev;
          const double nx = r[k][0] * ex + r[k][1] * ev + r[k][4], nv = r[k][2] * ex + r[k][3] * ev + r[k][5];
          ex = nx;
          ev = nv;
        }
    }
  }
}

template <typename ST>
__global__ void __launch_bounds__(kScanThreads, 2)
scan_local_fixup_blk(ScanArgs<ST> a, LocalWs ws, int B, int tmax, bool aligned) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t s_bar[2];
  __shared__ double s_pre[4 * kScanThreads];  // [seg][col][4] P at the segment start
  const int D = a.D, tid = threadIdx.x, G = gridDim.x, g = blockIdx.x;
  const size_t be = (size_t)B * D;
  ST *buf = (ST *)smem_raw;
  const int nseg = kScanThreads / D, c = tid % D, sg = tid / D;
  const bool active = sg < nseg;
  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  unsigned use[2] = {0u, 0u};
  int64_t lo, hi;
  local_range(a.T, G, g, lo, hi);
  const int nblk = ws.nfix[g];
  const double ex = active ? ws.rentry[((size_t)g * D + c) * 2] : 0.0;
  const double ev = active ? ws.rentry[((size_t)g * D + c) * 2 + 1] : 0.0;
  unsigned bk[2] = {0u, 0u};
  // the local states (a.out) ride in the u slot
  if (nblk > 0)
    bk[0] = blk_issue(a, blk_tile(buf, be, 0), lo, (int)(hi - lo < B ? hi - lo : B), &s_bar[0], aligned,
                      (const ST *)a.out);
  for (int k = 0; k < nblk; ++k) {
    const int64_t row0 = lo + (int64_t)k * B;
    const int rows = (int)(hi - row0 < B ? hi - row0 : B);
    const int kb = k & 1;
    if (k + 1 < nblk) {
      if (tid == 0) bulk_wait_read();
      __syncthreads();
      const int64_t rn = row0 + B;
      bk[kb ^ 1] = blk_issue(a, blk_tile(buf, be, kb ^ 1), rn, (int)(hi - rn < B ? hi - rn : B), &s_bar[kb ^ 1],
                             aligned, (const ST *)a.out);
    }
    BlkTile<ST> t = blk_tile(buf, be, kb);
    blk_land(a, t, row0, rows, bk[kb], &s_bar[kb], use[kb], (const ST *)a.out);
    const int rs = (rows + nseg - 1) / nseg, r0 = sg * rs, r1 = min(rows, r0 + rs);
    double m0 = 1.0, m1 = 0.0, m2 = 0.0, m3 = 1.0;  // the segment's map product
    if (active) {
      for (int r = r0; r < r1; ++r) {
        const double A = (double)t.a[r * D + c], Bq = (double)t.b[r * D + c];
        const double C = (double)t.c[r * D + c], E = (double)t.d[r * D + c];
        const double n0 = A * m0 + Bq * m2, n1 = A * m1 + Bq * m3, n2 = C * m0 + E * m2, n3 = C * m1 + E * m3;
        m0 = n0;
        m1 = n1;
        m2 = n2;
        m3 = n3;
      }
      double *sp = s_pre + (sg * D + c) * 4;
      sp[0] = m0;
      sp[1] = m1;
      sp[2] = m2;
      sp[3] = m3;
    }
    __syncthreads();
    if (tid < D) {  // exclusive products over the segments, from the tile's recorded start
      const double *tp = ws.tileP + ((size_t)g * tmax + k) * 4 * D + 4 * tid;
      double p0 = tp[0], p1 = tp[1], p2 = tp[2], p3 = tp[3];
      for (int q = 0; q < nseg; ++q) {
        double *sp = s_pre + (q * D + tid) * 4;
        const double a0 = sp[0], a1 = sp[1], a2 = sp[2], a3 = sp[3];
        sp[0] = p0;
        sp[1] = p1;
        sp[2] = p2;
        sp[3] = p3;
        const double n0 = a0 * p0 + a1 * p2, n1 = a0 * p1 + a1 * p3, n2 = a2 * p0 + a3 * p2, n3 = a2 * p1 + a3 * p3;
        p0 = n0;
        p1 = n1;
        p2 = n2;
        p3 = n3;
      }
    }
    __syncthreads();
    if (active && (ex != 0.0 || ev != 0.0)) {
      const double *sp = s_pre + (sg * D + c) * 4;
      double p0 = sp[0], p1 = sp[1], p2 = sp[2], p3 = sp[3];
      for (int r = r0; r < r1; ++r) {
        const double A = (double)t.a[r * D + c], Bq = (double)t.b[r * D + c];
        const double C = (double)t.c[r * D + c], E = (double)t.d[r * D + c];
        const double n0 = A * p0 + Bq * p2, n1 = A * p1 + Bq * p3, n2 = C * p0 + E * p2, n3 = C * p1 + E * p3;
        p0 = n0;
        p1 = n1;
        p2 = n2;
        p3 = n3;
        t.u[r * 2 * D + c] = (ST)((double)t.u[r * 2 * D + c] + p0 * ex + p1 * ev);
        t.u[r * 2 * D + D + c] = (ST)((double)t.u[r * 2 * D + D + c] + p2 * ex + p3 * ev);
      }
    }
    blk_store(a, t, row0, rows, aligned);
    __syncthreads();
  }
  if (tid == 0) bulk_wait_read();
}

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

static int env_int(const char *name, int lo, int hi, int dflt) {
  const char *e = getenv(name);
  const int v = e ? atoi(e) : 0;
  return v >= lo && v <= hi ? v : dflt;
}
// cap on stages per chunk (measured, tools/sweep_scan.sh): diag 16 (T = 4M: 2.51
// TB/s vs 2.27 at 32), block2x2 32 (T = 4M D = 18: 2.56 vs 2.38 at 16)
static bool rows_balanced() {  // CS_SCAN_BALANCED=0: uniform chunks with a partial last round (A/B experiments)
  static const bool v = [] {
    const char *e = getenv("CS_SCAN_BALANCED");
    return e ? atoi(e) != 0 : true;
  }();
  return v;
}
static int rows_chunk_stages(int var) {
  static const int v = env_int("CS_SCAN_CHUNK_STAGES", 1, 256, 0);  // tuning override for experiments
  // with whole rounds (rows_balanced) the >= 2-rounds rule sets the chunk length
  // at every T that fills the grid; the cap only binds at very long chains
  // (tools/sweep_chunk_stages.sh, T = 16M D = 18: diag 16 -> 64+ stages 2.85 -> 3.08 TB/s,
  // block2x2 32 -> 128 2.53 -> 2.66)
  (void)var;
  return v ? v : 128;
}
static int rows_resident_ctas(int minb) {  // persistent grid of scan_rows (launch bounds: minb CTAs per SM)
  static const int sms = [] {
    int dev = 0, n = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
  }();
  return minb * sms;
}
static bool rows_lbw() {  // dedicated look-back warp (CS_SCAN_LBW=0 selects the in-line look-back)
  static const bool v = [] {
    const char *e = getenv("CS_SCAN_LBW");
    return e ? atoi(e) != 0 : false;
  }();
  return v;
}
static int rows_round_kb() {  // LBW: input bytes per round of the grid, sized so the C pass re-reads from L2
  static const int v = env_int("CS_SCAN_ROUND_KB", 1024, 1 << 20, 24 * 1024);
  return v;
}
static int rows_lag() {  // LBW: rounds between a chunk's A and C passes
  static const int v = env_int("CS_SCAN_LAG", 1, 8, 2);
  return v;
}

static int rows_per_tile(int var, int dtype, int D) {
  const int esz = dtype == CS_F64 ? 8 : 4;
  const int per = (var == SCAN_DIAG ? 2 : 6) * esz;
  static const int tile_kb = env_int("CS_SCAN_TILE_KB", 4, 96, 16);
  int E = (tile_kb * 1024) / per;
  int R = E / D;
  if (R > 8192) R = 8192;
  const int q = dtype == CS_F64 ? 2 : 4;  // R*D*esize % 16 == 0 for any D
  R = (R / q) * q;
  if (R < q) R = q;
  return R;
}

// CS_SCAN_1P=1 selects the single-pass kernel for plain diag scans.  Off by
// default: at T = 2^24, D = 18 it measured 1.50 ms (36.8 % of HBM) against the
// two-pass scan's 1.21 ms -- with j, u moved once (0.83 ms without the
// look-back, 67 %), each tile's look-back (~5 L2 round trips) is exposed per
// CTA; see DESIGN.md section 8.
size_t scan_local_ws_bytes(int dtype, int64_t T, int D);
bool scan_rr_eligible(int var, int64_t T, int D);
size_t scan_rr_ws_bytes(int dtype, int64_t T, int D);
bool scan_1p_eligible(int var, int64_t T, int D) { return scan_1p_mode() == 1 && var == SCAN_DIAG && D >= 1 && D <= 64 && T > 0; }
// long scans only: each range's fixed-up prefix (until P underflows) and the
// three launches are amortised from ~2M steps on (T = 1M, D = 18: two-pass
// 0.127 ms vs 0.164; T = 4M: 0.344 vs 0.287; T = 16M: 1.21 vs 0.77)
bool scan_local_eligible(int var, int64_t T, int D) {
  static const int64_t min_t = [] {
    const char *e = getenv("CS_SCAN_LOCAL_MIN_T");
    return e ? (int64_t)atoll(e) : ((int64_t)1 << 19);
  }();
  return scan_1p_mode() == 3 && (var == SCAN_DIAG || var == SCAN_BLOCK) && D >= 1 && D <= 64 && T >= min_t && T > 0;
}

// tiles of ~kB KB of j + u, R a multiple of 4 so every full tile is whole 16-byte lines
ScanPlan scan_plan_1p(int var, int dtype, int64_t T, int D) {
  ScanPlan p{};
  p.var = var;
  p.kind = 3;
  const int esz = dtype == CS_F64 ? 8 : 4;
  static const int kb = env_int("CS_SCAN_1P_KB", 8, 100, 48);
  int R = (kb * 1024) / (2 * esz * D);
  R = R / 4 * 4;
  if (R < 4) R = 4;
  p.R = R;
  p.ntiles = (T + R - 1) / R;
  p.agg_w = 2 * D;
  p.state_w = D;
  const int nseg = kScanThreads / D;
  p.smem = (size_t)4 * R * D * esz + (size_t)2 * nseg * D * 2 * esz;  // two tiles in flight
  const int64_t ngroups = (p.ntiles + kGroupTiles - 1) / kGroupTiles;
  p.ws_bytes = align_up(sizeof(unsigned)) + align_up(sizeof(int) * (p.ntiles + 2 * ngroups)) +
               align_up(sizeof(double) * (p.ntiles + ngroups) * p.agg_w) + align_up(sizeof(double) * p.ntiles * p.state_w);
  return p;
}

size_t scan_ws_bytes(int var, int dtype, int64_t T, int D) {
  size_t a = scan_plan(var, dtype, T, D, false).ws_bytes, b = scan_plan(var, dtype, T, D, true).ws_bytes;
  if (scan_1p_eligible(var, T, D)) {
    const size_t c = scan_plan_1p(var, dtype, T, D).ws_bytes;
    a = a > c ? a : c;
  }
  if (scan_local_eligible(var, T, D)) {
    const size_t c = var == SCAN_BLOCK ? scan_local_blk_ws_bytes(dtype, T, D) : scan_local_ws_bytes(dtype, T, D);
    a = a > c ? a : c;
  }
  if (scan_rr_eligible(var, T, D)) {
    const size_t c = scan_rr_ws_bytes(dtype, T, D);
    a = a > c ? a : c;
  }
  return a > b ? a : b;
}

template <typename ST>
cudaError_t launch_scan_1p_t(const ScanPlan &p, ScanArgs<ST> a, void *ws, cudaStream_t st) {
  LookbackWs w = carve_ws(p, ws, a.D);
  cudaError_t e = cudaMemsetAsync(ws, 0, (unsigned char *)w.agg - (unsigned char *)ws, st);
  if (e != cudaSuccess) return e;
  if (p.ntiles == 0) return cudaSuccess;
  e = cudaFuncSetAttribute(scan_rows_1p<ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148, occ = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, scan_rows_1p<ST>, kScanThreads, p.smem);
  if (occ < 1) occ = 1;
  const int64_t g = (int64_t)occ * sms;
  scan_rows_1p<ST><<<(unsigned)(p.ntiles < g ? p.ntiles : g), kScanThreads, p.smem, st>>>(a, w, p.R, p.ntiles);
  return cudaGetLastError();
}
static void local_geom(int dtype, int64_t T, int D, int &G, int &B, int &tmax, size_t &smem, int kb = 0, int cps = 2) {
  const int esz = dtype == CS_F64 ? 8 : 4;
  static const int blk_kb = env_int("CS_SCAN_BLOCK_KB", 4, 48, 48);  // j + u per tile (T = 2^24, D = 18: 24 KB 0.92 ms, 40-48 KB 0.74-0.77 ms)
  B = ((kb ? kb : blk_kb) * 1024) / (2 * esz * D);
  B = B / 4 * 4;
  if (B < 4) B = 4;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // two ranges per SM, each at least four tiles long (short scans: fewer, longer ranges)
  G = cps * sms;
  if ((int64_t)G * 4 * B > T) G = (int)(T / (4 * (int64_t)B));
  if (G < 1) G = 1;
  const int64_t maxrows = T / G + 8;
  tmax = (int)((maxrows + B - 1) / B) + 1;
  const int nseg = kScanThreads / D;
  smem = (size_t)4 * B * D * esz + (size_t)nseg * D * 2 * sizeof(double) + sizeof(int) * (size_t)B;  // + UPD row flags
}
size_t scan_local_ws_bytes(int dtype, int64_t T, int D) {
  int G, B, tmax;
  size_t smem;
  local_geom(dtype, T, D, G, B, tmax, smem);
  return align_up(sizeof(double) * (size_t)G * D * 2) + align_up(sizeof(double) * (size_t)G * D) +
         align_up(sizeof(int) * (size_t)G) + align_up(sizeof(double) * (size_t)G * tmax * D);
}
template <typename ST, bool UPD>
cudaError_t launch_scan_local_t(ScanArgs<ST> a, void *ws, cudaStream_t st) {
  int G, B, tmax;
  size_t smem;
  local_geom(sizeof(ST) == 8 ? CS_F64 : CS_F32, a.T, a.D, G, B, tmax, smem);
  unsigned char *b = (unsigned char *)ws;
  LocalWs w;
  w.ragg = (double *)b;
  b += align_up(sizeof(double) * (size_t)G * a.D * 2);
  w.rentry = (double *)b;
  b += align_up(sizeof(double) * (size_t)G * a.D);
  w.nfix = (int *)b;
  b += align_up(sizeof(int) * (size_t)G);
  w.tileP = (double *)b;
  for (auto k : {(const void *)scan_local<ST, UPD>, (const void *)scan_local_fixup<ST, UPD>}) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  const bool al = ((((uintptr_t)a.e0) | ((uintptr_t)a.u) | ((uintptr_t)a.out)) & 15) == 0;
  scan_local<ST, UPD><<<G, kScanThreads, smem, st>>>(a, w, B, tmax, al);
  scan_local_carry<ST><<<1, 64, 0, st>>>(a.s0, w, G, a.D);
  scan_local_fixup<ST, UPD><<<G, kScanThreads, smem, st>>>(a, w, B, tmax, al);
  return cudaGetLastError();
}
static void local_geom_blk(int dtype, int64_t T, int D, int &G, int &B, int &tmax, size_t &smem) {
  const int esz = dtype == CS_F64 ? 8 : 4;
  static const int blk_kb = env_int("CS_SCAN_BLOCK_KB", 4, 48, 48);
  B = (blk_kb * 1024) / (6 * esz * D);  // a, b, c, d, u (2 D): 6 D values per row
  B = B / 4 * 4;
  if (B < 4) B = 4;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  G = 2 * sms;
  if ((int64_t)G * 4 * B > T) G = (int)(T / (4 * (int64_t)B));
  if (G < 1) G = 1;
  tmax = (int)((T / G + 8 + B - 1) / B) + 1;
  const int nseg = kScanThreads / D;
  smem = (size_t)12 * B * D * esz + (size_t)nseg * D * 6 * sizeof(double);
}
size_t scan_local_blk_ws_bytes(int dtype, int64_t T, int D) {
  int G, B, tmax;
  size_t smem;
  local_geom_blk(dtype, T, D, G, B, tmax, smem);
  return align_up(sizeof(double) * (size_t)G * D * 6) + align_up(sizeof(double) * (size_t)G * D * 2) +
         align_up(sizeof(int) * (size_t)G) + align_up(sizeof(double) * (size_t)G * tmax * D * 4);
}
template <typename ST>
cudaError_t launch_scan_local_blk_t(ScanArgs<ST> a, void *ws, cudaStream_t st) {
  int G, B, tmax;
  size_t smem;
  local_geom_blk(sizeof(ST) == 8 ? CS_F64 : CS_F32, a.T, a.D, G, B, tmax, smem);
  unsigned char *b = (unsigned char *)ws;
  LocalWs w;
  w.ragg = (double *)b;
  b += align_up(sizeof(double) * (size_t)G * a.D * 6);
  w.rentry = (double *)b;
  b += align_up(sizeof(double) * (size_t)G * a.D * 2);
  w.nfix = (int *)b;
  b += align_up(sizeof(int) * (size_t)G);
  w.tileP = (double *)b;
  for (auto k : {(const void *)scan_local_blk<ST>, (const void *)scan_local_fixup_blk<ST>}) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  const bool al = ((((uintptr_t)a.e0) | ((uintptr_t)a.e1) | ((uintptr_t)a.e2) | ((uintptr_t)a.e3) |
                    ((uintptr_t)a.u) | ((uintptr_t)a.out)) & 15) == 0;
  scan_local_blk<ST><<<G, kScanThreads, smem, st>>>(a, w, B, tmax, al);
  scan_local_carry_blk<ST><<<1, 64, 0, st>>>(a.s0, w, G, a.D);
  scan_local_fixup_blk<ST><<<G, kScanThreads, smem, st>>>(a, w, B, tmax, al);
  return cudaGetLastError();
}
template cudaError_t launch_scan_local_blk_t<float>(ScanArgs<float>, void *, cudaStream_t);
template cudaError_t launch_scan_local_blk_t<double>(ScanArgs<double>, void *, cudaStream_t);

// reduce-then-replay (scan_rr_*): the local scan's ranges, no tile records
bool scan_rr_eligible(int var, int64_t T, int D) {
  static const int64_t min_t = [] {
    const char *e = getenv("CS_SCAN_RR_MIN_T");
    return e ? (int64_t)atoll(e) : ((int64_t)1 << 16);
  }();
  return var == SCAN_DIAG && D >= 1 && D <= kRrMaxD && T >= min_t;
}
static int rr_kb() {  // j + u per tile
  static const int v = env_int("CS_SCAN_RR_KB", 4, 48, 32);  // cfg 5: 48 KB 64.5 ms, 32 KB 59.6 (tools/sweep_rr.sh)
  return v;
}
static int rr_cps() {  // ranges (CTAs) per SM
  static const int v = env_int("CS_SCAN_RR_CPS", 1, 8, 2);
  return v;
}
size_t scan_rr_ws_bytes(int dtype, int64_t T, int D) {
  int G, B, tmax;
  size_t smem;
  local_geom(dtype, T, D, G, B, tmax, smem, rr_kb(), rr_cps());
  return align_up(sizeof(double) * (size_t)G * D * 2) + align_up(sizeof(double) * (size_t)G * D);
}
template <typename ST, bool UPD>
cudaError_t launch_scan_rr_t(ScanArgs<ST> a, void *ws, cudaStream_t st) {
  int G, B, tmax;
  size_t smem;
  local_geom(sizeof(ST) == 8 ? CS_F64 : CS_F32, a.T, a.D, G, B, tmax, smem, rr_kb(), rr_cps());
  unsigned char *b = (unsigned char *)ws;
  LocalWs w{};
  w.ragg = (double *)b;
  b += align_up(sizeof(double) * (size_t)G * a.D * 2);
  w.rentry = (double *)b;
  const size_t smem_r = UPD ? rr_guess_off(B, a.D, sizeof(ST)) + 2 * (size_t)B * a.D * sizeof(ST) : smem;
  cudaError_t e = cudaFuncSetAttribute(scan_rr_reduce<ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(scan_rr_replay<ST, UPD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_r);
  if (e != cudaSuccess) return e;
  const bool al = ((((uintptr_t)a.e0) | ((uintptr_t)a.u) | ((uintptr_t)a.out)) & 15) == 0 &&
                  (!UPD || (((uintptr_t)a.guess) & 15) == 0);
  scan_rr_reduce<ST><<<G, kScanThreads, smem, st>>>(a, w, B, al);
  scan_rr_replay<ST, UPD><<<G, kScanThreads, smem_r, st>>>(a, w, B, al);
  return cudaGetLastError();
}
template cudaError_t launch_scan_rr_t<float, true>(ScanArgs<float>, void *, cudaStream_t);
template cudaError_t launch_scan_rr_t<double, true>(ScanArgs<double>, void *, cudaStream_t);
template cudaError_t launch_scan_rr_t<float, false>(ScanArgs<float>, void *, cudaStream_t);
template cudaError_t launch_scan_rr_t<double, false>(ScanArgs<double>, void *, cudaStream_t);

template cudaError_t launch_scan_local_t<float, false>(ScanArgs<float>, void *, cudaStream_t);
template cudaError_t launch_scan_local_t<double, false>(ScanArgs<double>, void *, cudaStream_t);
template cudaError_t launch_scan_local_t<float, true>(ScanArgs<float>, void *, cudaStream_t);
template cudaError_t launch_scan_local_t<double, true>(ScanArgs<double>, void *, cudaStream_t);
int scan_1p_mode() {  // plain diag scans: 3 local scan + fix-up (default), 1 single-pass tiles, 0 two-pass chunks
  static const int v = [] {
    const char *e = getenv("CS_SCAN_1P");
    return e ? atoi(e) : 3;
  }();
  return v;
}

template cudaError_t launch_scan_1p_t<float>(const ScanPlan &, ScanArgs<float>, void *, cudaStream_t);
template cudaError_t launch_scan_1p_t<double>(const ScanPlan &, ScanArgs<double>, void *, cudaStream_t);

ScanPlan scan_plan(int var, int dtype, int64_t T, int D, bool update) {
  ScanPlan p{};
  p.var = var;
  if (var == SCAN_DENSE) {
    p.kind = 2;
    p.md = D <= 1 ? 1 : D <= 2 ? 2 : D <= 4 ? 4 : 8;
    p.seg = p.md <= 2 ? 4 : 1;
    const int64_t per_tile = (int64_t)kScanThreads * p.seg;
    p.ntiles = (T + per_tile - 1) / per_tile;
    p.agg_w = p.md * p.md + p.md;
    p.state_w = p.md;
  } else if (D <= 64) {
    p.kind = 0;
    const int nseg = kScanThreads / D;
    const bool u = update;
    const int kr = dtype == CS_F64
                       ? (var == SCAN_DIAG ? (u ? RowsSeg<double, SCAN_DIAG, true>::kRows : RowsSeg<double, SCAN_DIAG>::kRows)
                                           : (u ? RowsSeg<double, SCAN_BLOCK, true>::kRows : RowsSeg<double, SCAN_BLOCK>::kRows))
                       : (var == SCAN_DIAG ? (u ? RowsSeg<float, SCAN_DIAG, true>::kRows : RowsSeg<float, SCAN_DIAG>::kRows)
                                           : (u ? RowsSeg<float, SCAN_BLOCK, true>::kRows : RowsSeg<float, SCAN_BLOCK>::kRows));
    const int minb = rows_lbw() ? CS_ROWS_LBW_MINB
                                : var == SCAN_DIAG ? (u ? RowsTune<SCAN_DIAG, true>::kMinBlocks : RowsTune<SCAN_DIAG, false>::kMinBlocks)
                                                   : RowsTune<SCAN_BLOCK, false>::kMinBlocks;
    p.R = nseg * kr;                      // rows per stage
    // stages per chunk: large chunks amortise the per-chunk look-back, but
    // every resident CTA needs chunks -- aim for >= 2 rounds of the grid
    {
      const int64_t stages = (T + p.R - 1) / p.R;
      const int64_t g = (int64_t)rows_resident_ctas(minb);
      int64_t cs = stages / (2 * g);
      const int cmax = rows_chunk_stages(var);
      if (cs > cmax) cs = cmax;
      if (rows_lbw()) {
        // the look-back is off the critical path, so chunks only need to be
        // large enough to amortise the per-chunk fold: size a round of the
        // grid to stay L2-resident until its C pass (one round later)
        const int esz0 = dtype == CS_F64 ? 8 : 4;
        const int64_t stage_bytes = (int64_t)p.R * D * (var == SCAN_DIAG ? 2 : 6) * esz0;
        const int64_t cl = ((int64_t)rows_round_kb() * 1024) / (g * stage_bytes);
        if (cs > cl) cs = cl;
      }
      if (cs < 1) cs = 1;
      p.seg = (int)cs;
    }
    p.ntiles = (T + (int64_t)p.R * p.seg - 1) / ((int64_t)p.R * p.seg);  // chunks
    {
      // round the chunk count up to whole rounds of the grid (chunks then hold
      // seg or seg-1 stages): a partial last round leaves most CTAs idle while
      // the rest finish it (T = 16M diag: 10.5 rounds -> 11 full ones)
      const int64_t nst = (T + p.R - 1) / p.R;
      const int64_t g = (int64_t)rows_resident_ctas(minb);
      if (rows_balanced() && p.ntiles > g) {
        const int64_t nb = (p.ntiles + g - 1) / g * g;
        if (nb <= nst) p.ntiles = nb;
      }
    }
    p.agg_w = D * (var == SCAN_DIAG ? 2 : 6);
    p.state_w = var == SCAN_DIAG ? D : 2 * D;
    const int esz = dtype == CS_F64 ? 8 : 4;
    const int W = var == SCAN_DIAG ? 2 : 6;
    p.win = rows_lbw() ? rows_lag() : 1;
    p.md = 0;
    p.smem = (size_t)esz * 2 * (nseg + 1) * D * W + sizeof(int) * p.R + 16;
    if (rows_lbw()) {
      p.smem += 16 + sizeof(double) * (kLbwStage + kLbwPubStage);
    }
    if (!rows_lbw() && (!update || CS_ROWS_TX_UPDATE) && var == SCAN_DIAG && dtype == CS_F32 && rows_tx_dim(D))
      p.smem += 16 + sizeof(float) * 2 * ((size_t)p.R * D + 4 * nseg);  // small-D transposition buffer
  } else {
    p.kind = 1;
    const int ncb = (D + 31) / 32;
    p.ntiles = ((T + 63) / 64) * ncb;
    p.agg_w = 32 * (var == SCAN_DIAG ? 2 : 6);
    p.state_w = var == SCAN_DIAG ? D : 2 * D;
  }
  const int64_t ngroups = (p.kind == 0 || p.kind == 3) ? (p.ntiles + kGroupTiles - 1) / kGroupTiles : 0;
  p.ws_bytes = align_up(sizeof(unsigned)) + align_up(sizeof(int) * (p.ntiles + 2 * ngroups)) +
               align_up(sizeof(double) * (p.ntiles + ngroups) * p.agg_w) +
               align_up(sizeof(double) * (p.kind == 1 ? (p.ntiles / ((D + 31) / 32) + 1) : p.ntiles) * p.state_w);
  return p;
}

LookbackWs carve_ws(const ScanPlan &p, void *ws, int D) {
  unsigned char *b = (unsigned char *)ws;
  LookbackWs w;
  w.ticket = (unsigned *)b;
  b += align_up(sizeof(unsigned));
  const int64_t ngroups = (p.kind == 0 || p.kind == 3) ? (p.ntiles + kGroupTiles - 1) / kGroupTiles : 0;
  w.status = (int *)b;
  w.gstatus = w.status + p.ntiles;
  w.gcount = w.gstatus + ngroups;
  b += align_up(sizeof(int) * (p.ntiles + 2 * ngroups));
  w.agg = (double *)b;
  w.gagg = w.agg + p.ntiles * p.agg_w;
  b += align_up(sizeof(double) * (p.ntiles + ngroups) * p.agg_w);
  w.exit = (double *)b;
  (void)D;
  return w;
}

// persistent grid for scan_rows: every CTA must be co-resident (look-back
// waits on tiles held by other CTAs), so never launch more than fit at once
static unsigned rows_grid(const ScanPlan &p, const void *k, int threads = kScanThreads) {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
  int dev = 0, sms = 148, occ = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, threads, p.smem);
  if (occ < 1) occ = 1;
  const int64_t cap = (int64_t)occ * sms;
  return (unsigned)(p.ntiles < cap ? p.ntiles : cap);
}

// scan_rows maps chunks to CTAs statically and its look-back waits on chunks of
// other CTAs, so the whole grid must be resident at once: launched cooperative,
// the launch waits for (or fails without) co-residency instead of hanging when
// another stream or process holds part of the device
template <typename ST, int VAR, bool AGG, bool UPD, bool LBW>
static void launch_rows_coop(const ScanPlan &p, const ScanArgs<ST> &a, LookbackWs w, int md, cudaStream_t st) {
  auto k = scan_rows<ST, VAR, AGG, UPD, LBW>;
  const int threads = LBW ? kScanThreads + 64 : kScanThreads;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(rows_grid(p, (const void *)k, threads));
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, a, w, p.R, p.seg, p.ntiles, p.win, md);
}

template <typename ST, int VAR, bool UPD>
static void launch_rows(const ScanPlan &p, const ScanArgs<ST> &a, LookbackWs w, cudaStream_t st) {
  if (rows_lbw()) launch_rows_coop<ST, VAR, false, UPD, true>(p, a, w, 0, st);
  else launch_rows_coop<ST, VAR, false, UPD, false>(p, a, w, p.md, st);
}

template <typename ST>
cudaError_t launch_scan_t(const ScanPlan &p, ScanArgs<ST> a, void *ws, cudaStream_t st, bool update) {
  LookbackWs w = carve_ws(p, ws, a.D);
  // ticket + status must start at zero for every launch
  cudaError_t e = cudaMemsetAsync(ws, 0, (unsigned char *)w.agg - (unsigned char *)ws, st);
  if (e != cudaSuccess) return e;
  if (p.ntiles == 0) return cudaSuccess;
  const unsigned grid = (unsigned)p.ntiles;
  if (p.kind == 0) {
    if (p.var == SCAN_DIAG) {
      if (update) launch_rows<ST, SCAN_DIAG, true>(p, a, w, st);
      else launch_rows<ST, SCAN_DIAG, false>(p, a, w, st);
    } else {
      if (update) launch_rows<ST, SCAN_BLOCK, true>(p, a, w, st);
      else launch_rows<ST, SCAN_BLOCK, false>(p, a, w, st);
    }
  } else if (p.kind == 1 && a.T <= kSmallT) {  // the whole sequence fits one CTA per column block
    const unsigned g = (unsigned)((a.D + 31) / 32);
    if (p.var == SCAN_DIAG) {
      if (update) scan_cols_small<ST, SCAN_DIAG, true><<<g, kSmallWarps * 32, 0, st>>>(a);
      else scan_cols_small<ST, SCAN_DIAG, false><<<g, kSmallWarps * 32, 0, st>>>(a);
    } else {
      if (update) scan_cols_small<ST, SCAN_BLOCK, true><<<g, kSmallWarps * 32, 0, st>>>(a);
      else scan_cols_small<ST, SCAN_BLOCK, false><<<g, kSmallWarps * 32, 0, st>>>(a);
    }
  } else if (p.kind == 1) {
    if (p.var == SCAN_DIAG) {
      if (update) scan_cols<ST, SCAN_DIAG, false, true><<<grid, kScanThreads, 0, st>>>(a, w);
      else scan_cols<ST, SCAN_DIAG><<<grid, kScanThreads, 0, st>>>(a, w);
    } else {
      if (update) scan_cols<ST, SCAN_BLOCK, false, true><<<grid, kScanThreads, 0, st>>>(a, w);
      else scan_cols<ST, SCAN_BLOCK><<<grid, kScanThreads, 0, st>>>(a, w);
    }
  } else {
    switch (p.md) {
      case 1: scan_dense_small<ST, 1, 4><<<grid, kScanThreads, 0, st>>>(a, w); break;
      case 2: scan_dense_small<ST, 2, 4><<<grid, kScanThreads, 0, st>>>(a, w); break;
      case 4: scan_dense_small<ST, 4, 1><<<grid, kScanThreads, 0, st>>>(a, w); break;
      default: scan_dense_small<ST, 8, 1><<<grid, kScanThreads, 0, st>>>(a, w); break;
    }
  }
  return cudaGetLastError();
}

template <typename ST>
cudaError_t launch_aggregate_t(const ScanPlan &p, ScanArgs<ST> a, void *ws, double *out, cudaStream_t st) {
  LookbackWs w = carve_ws(p, ws, a.D);
  cudaError_t e = cudaMemsetAsync(ws, 0, (unsigned char *)w.agg - (unsigned char *)ws, st);
  if (e != cudaSuccess) return e;
  const unsigned grid = (unsigned)p.ntiles;
  if (p.kind == 0) {
    if (p.var == SCAN_DIAG) {
      launch_rows_coop<ST, SCAN_DIAG, true, false, false>(p, a, w, p.md, st);
      k_agg_compose_cols<SCAN_DIAG><<<1, kScanThreads, 0, st>>>(w.agg, p.ntiles, a.D, 0, out);
    } else {
      launch_rows_coop<ST, SCAN_BLOCK, true, false, false>(p, a, w, p.md, st);
      k_agg_compose_cols<SCAN_BLOCK><<<1, kScanThreads, 0, st>>>(w.agg, p.ntiles, a.D, 0, out);
    }
  } else if (p.kind == 1) {
    const int ncb = (a.D + 31) / 32;
    if (p.var == SCAN_DIAG) {
      scan_cols<ST, SCAN_DIAG, true><<<grid, kScanThreads, 0, st>>>(a, w);
      k_agg_compose_cols<SCAN_DIAG><<<1, kScanThreads, 0, st>>>(w.agg, p.ntiles / ncb, a.D, ncb, out);
    } else {
      scan_cols<ST, SCAN_BLOCK, true><<<grid, kScanThreads, 0, st>>>(a, w);
      k_agg_compose_cols<SCAN_BLOCK><<<1, kScanThreads, 0, st>>>(w.agg, p.ntiles / ncb, a.D, ncb, out);
    }
  } else {
    switch (p.md) {
      case 1: scan_dense_small<ST, 1, 4, true><<<grid, kScanThreads, 0, st>>>(a, w);
              k_agg_compose_dense<1><<<1, 32, 0, st>>>(w.agg, p.ntiles, a.D, out); break;
      case 2: scan_dense_small<ST, 2, 4, true><<<grid, kScanThreads, 0, st>>>(a, w);
              k_agg_compose_dense<2><<<1, 32, 0, st>>>(w.agg, p.ntiles, a.D, out); break;
      case 4: scan_dense_small<ST, 4, 1, true><<<grid, kScanThreads, 0, st>>>(a, w);
              k_agg_compose_dense<4><<<1, 32, 0, st>>>(w.agg, p.ntiles, a.D, out); break;
      default: scan_dense_small<ST, 8, 1, true><<<grid, kScanThreads, 0, st>>>(a, w);
               k_agg_compose_dense<8><<<1, 32, 0, st>>>(w.agg, p.ntiles, a.D, out); break;
    }
  }
  return cudaGetLastError();
}

template cudaError_t launch_scan_t<float>(const ScanPlan &, ScanArgs<float>, void *, cudaStream_t, bool);
template cudaError_t launch_aggregate_t<float>(const ScanPlan &, ScanArgs<float>, void *, double *, cudaStream_t);
template cudaError_t launch_aggregate_t<double>(const ScanPlan &, ScanArgs<double>, void *, double *, cudaStream_t);
template cudaError_t launch_scan_t<double>(const ScanPlan &, ScanArgs<double>, void *, cudaStream_t, bool);

}  // namespace cs
