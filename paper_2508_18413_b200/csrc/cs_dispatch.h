// Dispatch declarations shared by the generated instantiation units.
#pragma once
#include "cs_apikern.cuh"

namespace cs {
cudaError_t syscall_gibbs(const cs_system &, int dtype, int md, const SysCall &, cudaStream_t);
cudaError_t solve_gibbs(int dtype, int md, int mode, void *args, int sms, cudaStream_t, SolvePick *);
cudaError_t elements_gibbs(int dtype, int md, int mode, void *args, int it, const void *g, void *e0, void *e1,
                           void *e2, void *e3, void *u, cs_elem_stats *stats, cudaStream_t st);
bool wide_leapfrog_ok(const cs_system &s, int mode);
cudaError_t elements_wide(const cs_system &sys, const cs_deer_config &cfg, int dtype, int64_t iteration,
                          const void *s0, const void *guess, void *e0, void *e1, void *e2, void *e3, void *u,
                          cs_elem_stats *stats, cudaStream_t st);
bool blr_mala_ok(const cs_system &s, int mode);
bool blr_fused_ok(const cs_system &s, const cs_deer_config &cfg);
cudaError_t blr_sequential(const cs_system &sys, int dtype, const void *s0, int64_t T, void *out, long long *bad,
                           cudaStream_t st);
cudaError_t elements_blr_fused(const cs_system &sys, const cs_deer_config &cfg, int dtype, int64_t iteration,
                               int64_t t0, int64_t n, const void *s0, const void *guess, void *j, void *u,
                               cs_elem_stats *stats, cudaStream_t st);
bool leapfrog_batch_ok(const cs_system &s, int mode);
cudaError_t wide_batch_solve(const cs_system &sys, const cs_deer_config &cfg, int dtype, int B, const void *s0s,
                             void *finals, int32_t *info, long long *err_step, cudaStream_t st);
cudaError_t leapfrog_batch_solve(const cs_system &sys, const cs_deer_config &cfg, int dtype, int B, const void *s0s,
                                 void *finals, int32_t *info, long long *err_step, cudaStream_t st);
cudaError_t debug_gram(const double *X, int N, int D, const double *W, int64_t T, float *H, cudaStream_t st);
cudaError_t debug_pair_gram(const double *X, int N, int D, const double *W, int64_t T, float *H, cudaStream_t st);
cudaError_t target_eval_gemm(const cs_target &tg, int what, int64_t n, const double *x, const double *v,
                             double *out, cudaStream_t st);
cudaError_t elements_blr(const cs_system &sys, const cs_deer_config &cfg, int dtype, int64_t iteration,
                         const void *s0, const void *guess, void *e0, void *u, cs_elem_stats *stats,
                         cudaStream_t st);
}  // namespace cs
