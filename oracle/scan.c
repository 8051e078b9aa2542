/* CPU oracle scans -- TEST INFRASTRUCTURE ONLY (never linked into the product).
 *
 * Restates the blocked two-pass affine scans of the reference
 * (chainscan/_scan_kernels.py:16-149) in C99 + pthreads, with the same
 * association order, so that for a fixed chunk the f64 results equal the
 * reference's bit-for-bit:
 *   phase 1 (parallel over chunks): fold each chunk into one summary,
 *            element t composed onto the running summary;
 *   phase 2 (serial): exclusive scan of the chunk summaries from s0;
 *   phase 3 (parallel over chunks): replay each chunk from its entry state.
 * Layout is time-major, C-contiguous: j,u,out (T,D); dense J (T,D,D) row-major
 * J[t][r][k]; block a,b,c,d (T,D), u/out (T,2D) as [x | v].
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

/* Static partition of [0, n) over the worker threads (CHAINSCAN_THREADS or
 * the online core count), like numba's prange: results do not depend on the
 * thread count because chunks own disjoint outputs. */
typedef void (*body_fn)(int64_t c, void *ctx);
typedef struct { body_fn fn; void *ctx; int64_t lo, hi; } span_t;

static void *run_span(void *p) {
  span_t *s = (span_t *)p;
  for (int64_t c = s->lo; c < s->hi; ++c) s->fn(c, s->ctx);
  return NULL;
}

int oracle_num_threads(void) {
  const char *env = getenv("CHAINSCAN_THREADS");
  if (env && atoi(env) > 0) return atoi(env);
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}

static void par_for(int64_t n, body_fn fn, void *ctx) {
  int64_t nt = oracle_num_threads();
  if (nt > 256) nt = 256;
  if (nt > n) nt = n;
  if (nt <= 1) { for (int64_t c = 0; c < n; ++c) fn(c, ctx); return; }
  pthread_t th[256];
  span_t sp[256];
  for (int64_t i = 0; i < nt; ++i) {
    sp[i].fn = fn; sp[i].ctx = ctx;
    sp[i].lo = n * i / nt; sp[i].hi = n * (i + 1) / nt;
    pthread_create(&th[i], NULL, run_span, &sp[i]);
  }
  for (int64_t i = 0; i < nt; ++i) pthread_join(th[i], NULL);
}

typedef struct {
  const double *j, *u, *a, *b, *c, *d;   /* elements (diag: j,u; dense: j=J) */
  int64_t T, D, chunk;
  double *sum, *entry, *out;            /* per-chunk summaries and entry states */
} job_t;

static inline int64_t hi_of(const job_t *q, int64_t c) {
  int64_t hi = (c + 1) * q->chunk;
  return hi < q->T ? hi : q->T;
}

/* ---------------- diag ---------------- */
static void diag_reduce(int64_t c, void *p) {
  job_t *q = (job_t *)p;
  int64_t D = q->D;
  double *jr = q->sum + c * 2 * D, *ur = jr + D;
  for (int64_t k = 0; k < D; ++k) { jr[k] = 1.0; ur[k] = 0.0; }
  for (int64_t t = c * q->chunk; t < hi_of(q, c); ++t)
    for (int64_t k = 0; k < D; ++k) {
      double jt = q->j[t * D + k];
      ur[k] = jt * ur[k] + q->u[t * D + k];
      jr[k] = jt * jr[k];
    }
}

static void diag_replay(int64_t c, void *p) {
  job_t *q = (job_t *)p;
  int64_t D = q->D;
  for (int64_t k = 0; k < D; ++k) {
    double run = q->entry[c * D + k];
    for (int64_t t = c * q->chunk; t < hi_of(q, c); ++t) {
      run = q->j[t * D + k] * run + q->u[t * D + k];
      q->out[t * D + k] = run;
    }
  }
}

void oracle_scan_diag(const double *j, const double *u, const double *s0,
                      int64_t T, int64_t D, int64_t chunk, double *out) {
  int64_t nc = (T + chunk - 1) / chunk;
  job_t q = {j, u, 0, 0, 0, 0, T, D, chunk,
             malloc(sizeof(double) * nc * 2 * D), malloc(sizeof(double) * nc * D), out};
  par_for(nc, diag_reduce, &q);
  double *carry = malloc(sizeof(double) * D);
  memcpy(carry, s0, sizeof(double) * D);
  for (int64_t c = 0; c < nc; ++c) {
    const double *jr = q.sum + c * 2 * D, *ur = jr + D;
    for (int64_t k = 0; k < D; ++k) {
      q.entry[c * D + k] = carry[k];
      carry[k] = jr[k] * carry[k] + ur[k];
    }
  }
  par_for(nc, diag_replay, &q);
  free(q.sum); free(q.entry); free(carry);
}

/* ---------------- dense ---------------- */
static void dense_reduce(int64_t c, void *p) {
  job_t *q = (job_t *)p;
  int64_t D = q->D;
  double *M = malloc(sizeof(double) * D * D), *Mn = malloc(sizeof(double) * D * D);
  double *w = malloc(sizeof(double) * D), *wn = malloc(sizeof(double) * D);
  for (int64_t r = 0; r < D; ++r) {
    w[r] = 0.0;
    for (int64_t k = 0; k < D; ++k) M[r * D + k] = (r == k) ? 1.0 : 0.0;
  }
  for (int64_t t = c * q->chunk; t < hi_of(q, c); ++t) {
    const double *Jt = q->j + t * D * D;
    for (int64_t r = 0; r < D; ++r) {
      double aw = q->u[t * D + r];
      for (int64_t k = 0; k < D; ++k) aw += Jt[r * D + k] * w[k];
      wn[r] = aw;
      for (int64_t col = 0; col < D; ++col) {
        double acc = 0.0;
        for (int64_t k = 0; k < D; ++k) acc += Jt[r * D + k] * M[k * D + col];
        Mn[r * D + col] = acc;
      }
    }
    double *tm = M; M = Mn; Mn = tm;
    double *tw = w; w = wn; wn = tw;
  }
  double *dst = q->sum + c * (D * D + D);
  memcpy(dst, M, sizeof(double) * D * D);
  memcpy(dst + D * D, w, sizeof(double) * D);
  free(M); free(Mn); free(w); free(wn);
}

static void dense_replay(int64_t c, void *p) {
  job_t *q = (job_t *)p;
  int64_t D = q->D;
  double *run = malloc(sizeof(double) * D), *st = malloc(sizeof(double) * D);
  memcpy(run, q->entry + c * D, sizeof(double) * D);
  for (int64_t t = c * q->chunk; t < hi_of(q, c); ++t) {
    const double *Jt = q->j + t * D * D;
    for (int64_t r = 0; r < D; ++r) {
      double acc = q->u[t * D + r];
      for (int64_t k = 0; k < D; ++k) acc += Jt[r * D + k] * run[k];
      st[r] = acc;
    }
    double *tmp = run; run = st; st = tmp;
    memcpy(q->out + t * D, run, sizeof(double) * D);
  }
  free(run); free(st);
}

void oracle_scan_dense(const double *J, const double *u, const double *s0,
                       int64_t T, int64_t D, int64_t chunk, double *out) {
  int64_t nc = (T + chunk - 1) / chunk;
  job_t q = {J, u, 0, 0, 0, 0, T, D, chunk,
             malloc(sizeof(double) * nc * (D * D + D)), malloc(sizeof(double) * nc * D), out};
  par_for(nc, dense_reduce, &q);
  double *carry = malloc(sizeof(double) * D), *nx = malloc(sizeof(double) * D);
  memcpy(carry, s0, sizeof(double) * D);
  for (int64_t c = 0; c < nc; ++c) {
    const double *Mc = q.sum + c * (D * D + D), *wc = Mc + D * D;
    for (int64_t k = 0; k < D; ++k) q.entry[c * D + k] = carry[k];
    for (int64_t r = 0; r < D; ++r) {
      double acc = wc[r];
      for (int64_t k = 0; k < D; ++k) acc += Mc[r * D + k] * carry[k];
      nx[r] = acc;
    }
    double *tmp = carry; carry = nx; nx = tmp;
  }
  par_for(nc, dense_replay, &q);
  free(q.sum); free(q.entry); free(carry); free(nx);
}

/* ---------------- block 2x2 ---------------- */
static void block_reduce(int64_t c, void *p) {
  job_t *q = (job_t *)p;
  int64_t D = q->D;
  double *A = q->sum + c * 6 * D, *B = A + D, *C = B + D, *E = C + D, *ux = E + D, *uv = ux + D;
  for (int64_t i = 0; i < D; ++i) { A[i] = 1.0; B[i] = 0.0; C[i] = 0.0; E[i] = 1.0; ux[i] = 0.0; uv[i] = 0.0; }
  for (int64_t t = c * q->chunk; t < hi_of(q, c); ++t)
    for (int64_t i = 0; i < D; ++i) {
      double at = q->a[t * D + i], bt = q->b[t * D + i], ct = q->c[t * D + i], dt = q->d[t * D + i];
      double An = at * A[i] + bt * C[i];
      double Bn = at * B[i] + bt * E[i];
      double Cn = ct * A[i] + dt * C[i];
      double Dn = ct * B[i] + dt * E[i];
      double uxn = at * ux[i] + bt * uv[i] + q->u[t * 2 * D + i];
      double uvn = ct * ux[i] + dt * uv[i] + q->u[t * 2 * D + D + i];
      A[i] = An; B[i] = Bn; C[i] = Cn; E[i] = Dn; ux[i] = uxn; uv[i] = uvn;
    }
}

static void block_replay(int64_t c, void *p) {
  job_t *q = (job_t *)p;
  int64_t D = q->D;
  double *run = malloc(sizeof(double) * 2 * D);
  memcpy(run, q->entry + c * 2 * D, sizeof(double) * 2 * D);
  for (int64_t t = c * q->chunk; t < hi_of(q, c); ++t) {
    for (int64_t i = 0; i < D; ++i) {
      double x = run[i], v = run[D + i];
      run[i] = q->a[t * D + i] * x + q->b[t * D + i] * v + q->u[t * 2 * D + i];
      run[D + i] = q->c[t * D + i] * x + q->d[t * D + i] * v + q->u[t * 2 * D + D + i];
    }
    memcpy(q->out + t * 2 * D, run, sizeof(double) * 2 * D);
  }
  free(run);
}

void oracle_scan_block(const double *a, const double *b, const double *cc,
                       const double *d, const double *u, const double *s0,
                       int64_t T, int64_t D, int64_t chunk, double *out) {
  int64_t nc = (T + chunk - 1) / chunk;
  job_t q = {0, u, a, b, cc, d, T, D, chunk,
             malloc(sizeof(double) * nc * 6 * D), malloc(sizeof(double) * nc * 2 * D), out};
  par_for(nc, block_reduce, &q);
  double *carry = malloc(sizeof(double) * 2 * D);
  memcpy(carry, s0, sizeof(double) * 2 * D);
  for (int64_t c = 0; c < nc; ++c) {
    const double *A = q.sum + c * 6 * D, *B = A + D, *C = B + D, *E = C + D, *ux = E + D, *uv = ux + D;
    memcpy(q.entry + c * 2 * D, carry, sizeof(double) * 2 * D);
    for (int64_t i = 0; i < D; ++i) {
      double x = carry[i], v = carry[D + i];
      carry[i] = A[i] * x + B[i] * v + ux[i];
      carry[D + i] = C[i] * x + E[i] * v + uv[i];
    }
  }
  par_for(nc, block_replay, &q);
  free(q.sum); free(q.entry); free(carry);
}
