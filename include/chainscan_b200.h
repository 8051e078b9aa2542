/* chainscan_b200 -- C-ABI of the B200-native parallel-in-time MCMC hot path.
 *
 * The drop-in boundary for arXiv 2508.18413's chainscan package
 * (/root/reference/pkg/src/chainscan).  Every entry point replaces one call
 * the reference makes on its hot path; the replaced interface is cited as
 * file:line beside each declaration.  Plain pointers and sizes only: device
 * buffers are caller-owned, every call is ordered on the given CUDA stream
 * (`stream` is a cudaStream_t, NULL = legacy default stream), and nothing is
 * allocated except inside cs_deer_solve's caller-sized workspace.
 *
 * Status codes map onto the reference's exceptions in the Python host layer
 * (paper_2508_18413_b200/_lib.py): CS_ERR_STRUCTURAL -> StructuralError
 * (core.py:30), CS_ERR_CONFIG -> ConfigurationError (noise.py:30),
 * CS_ERR_DIVERGED -> ChainDivergedError(step, iteration) (core.py:34-44).
 * cs_last_error() returns a thread-local message for the last failure.
 *
 * dtype: CS_F32 / CS_F64 is the storage type of states and scan elements.
 * Gate margins, noise transforms and scan carries are always computed in f64.
 */
#ifndef CHAINSCAN_B200_H
#define CHAINSCAN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { CS_OK = 0, CS_ERR_STRUCTURAL = 1, CS_ERR_CONFIG = 2, CS_ERR_DIVERGED = 3,
       CS_ERR_CUDA = 4, CS_ERR_INDEX = 5 };
enum { CS_F32 = 0, CS_F64 = 1 };
/* noise.py:83-104 distribution kinds */
enum { CS_NOISE_NORMAL = 0, CS_NOISE_UNIFORM = 1, CS_NOISE_CHI2 = 2, CS_NOISE_LOG_UNIFORM = 3 };
/* targets.py:46 model kinds */
enum { CS_TARGET_STD_NORMAL = 0, CS_TARGET_GAUSSIAN = 1, CS_TARGET_ROSENBROCK = 2,
       CS_TARGET_MOG = 3, CS_TARGET_BLR = 4 };
/* samplers.py kernels */
enum { CS_SYS_MALA = 0, CS_SYS_HMC = 1, CS_SYS_LEAPFROG = 2, CS_SYS_GIBBS = 3 };
/* core.py:27 JACOBIAN_MODES */
enum { CS_MODE_DENSE = 0, CS_MODE_DIAG = 1, CS_MODE_BLOCK = 2 };
/* cs_deer_result.status */
enum { CS_RUN_MAXITERS = 0, CS_RUN_CONVERGED = 1, CS_RUN_DIVERGED = 2 };
/* why the Newton loop stopped (deer.py:265-286) */
enum { CS_STOP_MAXITERS = 0, CS_STOP_PICARD = 1, CS_STOP_NOFAIL = 2, CS_STOP_ERROR = 3 };
/* divergence kinds reported in cs_deer_result.err_kind */
enum { CS_DIV_NONE = 0, CS_DIV_PROPOSAL = 1, CS_DIV_STEP = 2, CS_DIV_JACOBIAN = 3, CS_DIV_GUARD = 4 };

/* A compiled target model (targets.py:290-308, model_logp_grad_hvp).
 * All parameter arrays are device pointers to f64. */
typedef struct cs_target {
  int32_t kind;
  int32_t dim;
  double a, b, scale1, scale2;   /* rosenbrock (targets.py:92-104)           */
  const double *mu;              /* gaussian mean (dim)                      */
  const double *chol;            /* gaussian L, precision = L L^T (dim x dim) */
  const double *prec;            /* gaussian P = L L^T (dim x dim)           */
  int32_t n_comp;                /* mog K (targets.py:107-127)               */
  const double *means;           /* (K, dim)                                 */
  const double *variances;       /* (K)                                      */
  const double *logw;            /* (K) log weights                          */
  const double *lognorm;         /* (K) -dim/2 log(2 pi var_k)               */
  int64_t n_data;                /* blr N (targets.py:130-146)               */
  const double *X;               /* (N, dim)                                 */
  const double *y;               /* (N)                                      */
  double prior_precision;
} cs_target;

/* A transition system (core.py:61-160 TransitionSystem and its subclasses in
 * samplers.py).  Noise is the pre-drawn sequence, one row per step t = 0..T
 * (noise.py:107-113: step t reads index t): `noise_vec` is xi (MALA) or
 * momentum (HMC), shape (T+1, model dim), in the call's dtype; `noise_logu`
 * is log(u) of the gate uniform, shape (T+1), f64.  Gibbs reads
 * g_tau (T+1), xi_mu (T+1), xi_theta (T+1, S), g_sigma (T+1, S) in the
 * call's dtype and `gibbs` = [nu0, tau0_sq, mu0, kappa0, alpha0, sigma0_sq,
 * S, n, xbar[S], ss[S]] in f64 (samplers.py:416-461). */
typedef struct cs_system {
  int32_t kind;
  int32_t dim;                   /* state dimension (leapfrog: 2 x model dim) */
  cs_target target;
  double eps;
  int32_t L;                     /* leapfrog steps per HMC proposal          */
  const double *mass;            /* (model dim) or NULL for ones             */
  uint64_t seed;                 /* NoiseTable seed = diag Hutchinson probe seed
                                    (deer.py:172-175 uses system.noise.seed)   */
  uint64_t probe_seed;           /* LeapfrogSystem.probe_seed for the block
                                    estimate (samplers.py:213-214, 290-293)     */
  int64_t T;
  const void *noise_vec;
  const double *noise_logu;
  const void *g_tau, *xi_mu, *xi_theta, *g_sigma;
  const double *gibbs;
  const double *basis;           /* NULL, or an orthogonal Q (dim x dim, row-
                                    major, device f64): the system runs in z =
                                    Q' s coordinates, z -> Q' f(Q z), jvp
                                    V -> Q' J Q V (targets.py:473-517
                                    transform_system), fused into the MALA /
                                    HMC kernels                               */
} cs_system;

/* DeerConfig (deer.py:55-93), validated on the host. */
typedef struct cs_deer_config {
  int32_t mode;
  double atol, rtol;
  int32_t max_iters;
  int32_t hutchinson_samples;
  double damping;
  double clip;                   /* +inf = no clipping                       */
  const double *preconditioner;  /* device (dim) or NULL                     */
} cs_deer_config;

typedef struct cs_deer_result {
  int32_t iterations;            /* counted Newton updates (deer.py:272)     */
  int32_t status;                /* CS_RUN_*                                 */
  int32_t err_kind;              /* CS_DIV_*                                 */
  int64_t err_step;              /* first offending step (1-based), -1 none  */
  int32_t err_iteration;         /* ChainDivergedError.iteration, -1 = None  */
  int32_t launches;              /* kernels launched by the call             */
  double guard_dmax, guard_d0;
  int32_t stop_reason;           /* CS_STOP_*                                */
  int32_t grid_blocks;           /* persistent CTAs used                     */
  int32_t steps_per_thread;      /* contiguous steps folded per thread       */
  int32_t kept_in_registers;     /* 1 = elements kept across the grid sync   */
  int32_t fused_tangent;         /* 1 = f_t and its one Hutchinson tangent in
                                    a single integrator pass (diag HMC)       */
  double device_ms;              /* device time of the solve (CUDA events on
                                    the caller's stream around the launch)   */
} cs_deer_result;

const char *cs_last_error(void);
int cs_version(void);
/* Development timing hook: the persistent solver stamps %globaltimer (ns) at
 * 8 phase boundaries of each of its first n/8 iterations into dev_buf (NULL off). */
int cs_debug_probe(unsigned long long *dev_buf, int n);
/* Test hook for the tcgen05 weighted Gram kernel: H_out[t] (128 x 128 f32,
 * zero padded) = X^T diag(W[t]) X for X (N x D, D <= 128) and W (T x N), f64
 * device inputs.  The Hessian term of the dense logistic-regression builder. */
int cs_debug_gram(const double *X, int32_t N, int32_t D, const double *W, int64_t T, float *H_out,
                  void *stream);
/* The same product through the pair-Gram GEMM (all steps at once: W Q^T over
 * the data-row pairs, tcgen05 + bulk-copy operand tiles), unpacked into the
 * same 128 x 128 zero-padded layout. */
int cs_debug_pair_gram(const double *X, int32_t N, int32_t D, const double *W, int64_t T, float *H_out,
                       void *stream);
int cs_device_sm_count(int *out);
/* Target model functions for a batch of n states (targets.py:160-287, the
 * ModelFns a model_logp_grad_hvp returns), f64 device arrays: what = 0 log
 * density (out: n), 1 gradient (out: n x dim), 2 Hessian-vector product with
 * v (out: n x dim).  Logistic regression and dense Gaussians (any dim) run on
 * the library's DMMA GEMM; other kinds return CS_ERR_CONFIG. */
int cs_target_eval(const cs_target *target, int what, int64_t n, const double *x, const double *v, double *out,
                   void *stream);
/* Wait for the work queued on `stream` (the host-engine read-backs). */
int cs_stream_sync(void *stream);

/* ---- counter-based noise (noise.py:50-80, 140-156, 159-171) ------------- */
/* out[(i*count + k)] = value k of the slot at step t0+i; f64 always except
 * dtype-typed variants below.  CS_NOISE_LOG_UNIFORM writes log(u) (the gate's
 * log u, samplers.py:116). */
int cs_noise_fill(int kind, uint64_t seed, uint64_t slot_id, int64_t t0, int64_t nt,
                  int32_t count, double df, int dtype, void *out, void *stream);
/* z[i, d] = rademacher_probe(seed, iteration, ts[i], sample, dim)[i, d];
 * ts == NULL means ts[i] = t0 + i. */
int cs_rademacher_fill(uint64_t seed, int64_t iteration, const int64_t *ts, int64_t t0,
                       int64_t n, int32_t sample, int32_t dim, int dtype, void *out,
                       void *stream);

/* ---- affine scans (pscan.py:273-354 parallel_affine_solve) -------------- */
size_t cs_scan_workspace_bytes(int mode, int dtype, int64_t T, int32_t D);
int cs_scan_diag(int dtype, const void *j, const void *u, const void *s0, void *out,
                 int64_t T, int32_t D, void *ws, size_t ws_bytes, void *stream);
int cs_scan_block(int dtype, const void *a, const void *b, const void *c, const void *d,
                  const void *u, const void *s0, void *out, int64_t T, int32_t D,
                  void *ws, size_t ws_bytes, void *stream);
/* dense: D <= 8 single-pass register kernel; 8 < D <= 128 chunked reduce /
 * two-level f64 carry / replay; D > 128 chunk maps composed by strided-batched
 * library GEMMs (storage type), f64 carry, CTA-per-chunk replay
 * (pscan.py:196-213, _scan_kernels.py:47-99; any D like the reference). */
int cs_scan_dense(int dtype, const void *J, const void *u, const void *s0, void *out,
                  int64_t T, int32_t D, void *ws, size_t ws_bytes, void *stream);

/* Composed affine map of the whole sequence (the shard carry exchanged by the
 * T-sharded driver): agg_out f64 = diag [j|u] (2D), block
 * [A|B|C|E|ux|uv] (6D), dense [M row-major | w] (D*D + D; for D > 8 the chunk
 * maps are folded as a tree of f64 GEMMs on augmented (D+1)^2 matrices).  Same
 * workspace as the scan of that mode. */
int cs_scan_aggregate(int mode, int dtype, const void *e0, const void *e1, const void *e2,
                      const void *e3, const void *u, int64_t T, int32_t D, double *agg_out,
                      void *ws, size_t ws_bytes, void *stream);

/* ---- Newton-update building blocks (deer.py:107-208, 273-277) ----------- */
/* The three reductions below write into caller-owned DEVICE scalars (the host
 * reads them once per iteration, after the stream work it needs is queued).
 * First row (0-based) with a non-finite entry, INT64_MAX if none (deer.py:135-144). */
/* First row r < n with last_fail[r] == iteration into *d_first (device,
 * INT64_MAX if none): the sliding window's advance to the first step that
 * failed the update test (deer.py:318, w = lo + argmax(fail)). */
int cs_first_stamped_row(const int32_t *last_fail, int64_t n, int32_t iteration, int64_t *d_first, void *stream);
int cs_first_nonfinite_row(int dtype, const void *x, int64_t n, int64_t width,
                           int64_t *d_first, void *stream);
/* converged(prev, next): *d_notok = #entries with !(|next-prev| <= atol + rtol|next|),
 * *d_dmax = max |next-prev| (NaN propagates) (deer.py:107-115). */
int cs_converged(int dtype, const void *prev, const void *next, int64_t n, double atol,
                 double rtol, uint32_t *d_notok, double *d_dmax, void *stream);
/* Post-update bookkeeping (deer.py:273-277): rows with any |next-guess| > atol +
 * rtol|next| get last_fail[t] = iteration; *d_fail_rows counts them, *d_dmax as above. */
int cs_update_bookkeeping(int dtype, const void *guess, const void *next, int64_t T, int32_t D,
                          double atol, double rtol, int32_t iteration, int32_t *last_fail,
                          uint32_t *d_fail_rows, double *d_dmax, void *stream);
/* Element formation with preconditioner, damping and clip in the reference's
 * order; u = f - Jhat prev (deer.py:161-204).  prev = [s0; guess[:-1]]. */
int cs_form_diag(int dtype, const void *est, const void *f, const void *s0, const void *guess,
                 int64_t T, int32_t D, const double *pre, double damping, double clip,
                 void *j, void *u, void *stream);
int cs_form_dense(int dtype, const void *J_in, const void *f, const void *s0, const void *guess,
                  int64_t T, int32_t D, const double *pre, double damping, double clip,
                  void *J, void *u, void *stream);
int cs_form_block(int dtype, const void *a_in, const void *b_in, const void *c_in,
                  const void *d_in, const void *f, const void *s0, const void *guess,
                  int64_t T, int32_t D, const double *pre, double damping, double clip,
                  void *a, void *b, void *c, void *d, void *u, void *stream);
/* est = (first ? 0 : est) + z * jz, then est /= final_div when final_div > 0
 * (hutchinson_diag, deer.py:127-132). */
int cs_hutchinson_accumulate(int dtype, void *est, const void *z, const void *jz, int64_t n,
                             int32_t first, double final_div, void *stream);

/* ---- fused transition systems (samplers.py) ----------------------------- */
/* 1 if the register-resident fused kernels below cover this system (small
 * state dimension, non-GEMM target), else 0 (the host layer then evaluates
 * the system with cuBLAS GEMMs, e.g. logistic regression, D = 1000 Gaussians). */
int cs_system_supported(const cs_system *sys, int dtype);
/* f_t for rows ts[i] (or t0+i) at states S (n, dim) -> out (n, dim).
 * *bad_step receives the first step whose proposal / trajectory was
 * non-finite (samplers.py:101-105, 332-336) or -1. */
int cs_system_step(const cs_system *sys, int dtype, const int64_t *ts, int64_t t0, int64_t n,
                   const void *S, void *out, int64_t *bad_step, void *stream);
/* Solver-form JVP (hard gate + sigmoid' bend), samplers.py:129-145, 353-384,
 * 194-200, 593-627.  relaxed != 0 uses the sigmoid gate (relaxed_jvp_batch). */
int cs_system_jvp(const cs_system *sys, int dtype, const int64_t *ts, int64_t t0, int64_t n,
                  const void *S, const void *V, void *out, int32_t relaxed, void *stream);
/* relaxed_step_batch (samplers.py:124-127, 348-351). */
int cs_system_relaxed_step(const cs_system *sys, int dtype, const int64_t *ts, int64_t t0,
                           int64_t n, const void *S, void *out, void *stream);
/* LeapfrogSystem.block_jacobian_batch (samplers.py:202-222). */
int cs_system_block_jacobian(const cs_system *sys, int dtype, const int64_t *ts, int64_t t0,
                             int64_t n, const void *S, int32_t n_samples, int64_t iteration,
                             void *a, void *b, void *c, void *d, void *stream);
/* sequential_evaluate (core.py:163-184) as one device-resident chain walk. */
int cs_system_sequential(const cs_system *sys, int dtype, const void *s0, int64_t T,
                         void *out, int64_t *bad_step, void *stream);

/* Per-iteration flags of the fused element builder (device struct). */
typedef struct cs_elem_stats {
  int64_t bad_proposal;          /* first step with a non-finite proposal, INT64_MAX none */
  int64_t bad_step;              /* first step with non-finite f_t                       */
  int64_t bad_jacobian;          /* first step with a non-finite Jacobian estimate        */
  uint32_t picard_fail;          /* rows failing |f - guess| <= atol + rtol|f|             */
  uint32_t fail_rows;            /* filled by cs_scan_*_update                             */
  double dmax;                   /* filled by cs_scan_*_update (max |next - guess|)        */
} cs_elem_stats;

/* One fused pass over all T steps (deer.py:262-271 + 157-204): f_t at
 * prev = [s0; guess[:-1]], finite checks, the Picard residual against guess,
 * the Jacobian estimate for cfg->mode at `iteration` (Hutchinson probes hashed
 * in-kernel), preconditioner / damping / clip and u = f - Jhat prev.  Writes
 * the elements (diag: e0 = j; dense: e0 = J; block: e0..e3 = a,b,c,d; u) and
 * resets/fills *d_stats (device). */
int cs_system_elements(const cs_system *sys, const cs_deer_config *cfg, int dtype, int64_t iteration,
                       const void *s0, const void *guess, void *e0, void *e1, void *e2, void *e3,
                       void *u, cs_elem_stats *d_stats, void *stream);
/* cs_system_elements for the step range t0+1 .. t0+n of the chain -- one rank's
 * T shard in the sharded driver: guess holds the shard's n rows,
 * s0 the state before step t0+1 (the halo row); noise and probes are indexed by
 * the absolute step, so the shard's elements equal rows t0 .. t0+n-1 of the
 * whole chain's.  Register-kernel systems (incl. Gibbs) and logistic-regression
 * MALA; CS_ERR_CONFIG for the wide leapfrog builder unless the range is the
 * whole chain.  Replaces the
 * per-shard _iterate_range (deer.py:147-208) of a T-sharded run. */
int cs_system_elements_range(const cs_system *sys, const cs_deer_config *cfg, int dtype, int64_t iteration,
                             int64_t t0, int64_t n, const void *s0, const void *guess, void *e0, void *e1,
                             void *e2, void *e3, void *u, cs_elem_stats *d_stats, void *stream);
/* 1 when cs_system_elements_range can build this system's elements for a step
 * range under cfg (register-kernel systems, Gibbs, logistic-regression MALA in
 * dense mode or diag with <= 7 probes), else 0.  The sharded driver's test for
 * its streamed shard path (replaces the per-shard _iterate_range dispatch). */
int cs_system_elements_range_supported(const cs_system *sys, const cs_deer_config *cfg, int dtype);
/* 1 when cs_system_elements can build elements for (sys, mode, dtype): the
 * register builders (narrow built-in systems); for a leapfrog system on a
 * dense Gaussian target in block2x2 mode at any dimension, the GEMM-backed
 * builder (samplers.py:165-222; one cuBLAS DGEMM per iteration); for MALA on
 * the logistic-regression target (D <= 128) in diag mode the four-GEMM
 * Hutchinson builder, and in dense mode the closed-form Jacobian builder
 * (samplers.py:129-145 collapsed: A = I + eps H(S), per-step Hessian on the
 * tensor cores for f32 storage). */
int cs_system_elements_supported(const cs_system *sys, int32_t mode, int dtype);
/* B independent inner leapfrog solves at once (samplers.py:301-320: the
 * parallel-leapfrog HMC proposal, one run_deer per chain row in the reference):
 * one CTA per proposal runs the whole Newton loop of deer.py:259-286 for its
 * L-step trajectory in block2x2 mode.  s0s / finals: (B, dim) device rows in the
 * call's dtype (finals = the last trajectory state); info (B, 4) int32 =
 * {CS_RUN_* status, Newton iterations, CS_DIV_* kind, error iteration};
 * err_step (B) = offending step or -1.  Supported for leapfrog systems on the
 * register targets with L <= 256 and dim <= 4. */
int cs_leapfrog_batch_supported(const cs_system *sys, int32_t mode, int dtype);
int cs_leapfrog_batch_solve(const cs_system *sys, const cs_deer_config *cfg, int dtype, int32_t B,
                            const void *s0s, void *finals, int32_t *info, int64_t *err_step,
                            void *stream);
/* Scans with the post-update bookkeeping fused into the replay (deer.py:273-277):
 * rows of `out` that moved more than atol + rtol|out| from `guess` get
 * last_fail[t] = iteration; d_stats->fail_rows / dmax are accumulated.
 * `out` must not overlap `guess` (CS_ERR_CONFIG otherwise): the kernels read
 * guess through the read-only path while they write out. */
int cs_scan_diag_update(int dtype, const void *j, const void *u, const void *s0, void *out, int64_t T,
                        int32_t D, void *ws, size_t ws_bytes, const void *guess, double atol, double rtol,
                        int32_t iteration, int32_t *last_fail, cs_elem_stats *d_stats, void *stream);
int cs_scan_block_update(int dtype, const void *a, const void *b, const void *c, const void *d,
                         const void *u, const void *s0, void *out, int64_t T, int32_t D, void *ws,
                         size_t ws_bytes, const void *guess, double atol, double rtol, int32_t iteration,
                         int32_t *last_fail, cs_elem_stats *d_stats, void *stream);

/* ---- whole-chain Newton solve (deer.py:230-328, run_deer, no window) ---- */
/* One cooperative persistent kernel runs every Newton iteration on device:
 * fused f_t + Jacobian estimate + element formation, block scan with grid-wide
 * carry, convergence test and bookkeeping; one host sync at the end. */
size_t cs_deer_workspace_bytes(const cs_system *sys, int dtype, int32_t max_iters);
int cs_deer_supported(const cs_system *sys, int mode, int dtype);
int cs_deer_solve(const cs_system *sys, const cs_deer_config *cfg, int dtype, const void *s0,
                  void *trace, int32_t *per_step_converged_at, double *delta_history,
                  void *ws, size_t ws_bytes, cs_deer_result *res, void *stream);

#ifdef __cplusplus
}
#endif
#endif
