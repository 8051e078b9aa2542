// Eight-schools GibbsKernel (samplers.py:464-668): batched API kernels + fused solver.
#include "cs_dispatch.h"

namespace cs {
cudaError_t syscall_gibbs(const cs_system &s, int dtype, int md, const SysCall &c, cudaStream_t st) {
  if (md != 18) return cudaErrorNotSupported;
  return dtype == CS_F64 ? run_syscall<Gibbs<18, double>, 18, double>(s, c, st)
                         : run_syscall<Gibbs<18, float>, 18, float>(s, c, st);
}
cudaError_t solve_gibbs(int dtype, int md, int mode, void *args, int sms, cudaStream_t st, SolvePick *pick) {
  if (md != 18) return cudaErrorNotSupported;
  if (mode == CS_MODE_DIAG)
    return dtype == CS_F64 ? launch_solve<Gibbs<18, double>, CS_MODE_DIAG, 18, double>(*(SolveArgs<double> *)args, sms, st, pick)
                           : launch_solve<Gibbs<18, float>, CS_MODE_DIAG, 18, float>(*(SolveArgs<float> *)args, sms, st, pick);
  return cudaErrorNotSupported;
}
cudaError_t elements_gibbs(int dtype, int md, int mode, void *args, int it, const void *g, void *e0, void *e1,
                           void *e2, void *e3, void *u, cs_elem_stats *stats, cudaStream_t st) {
  if (md != 18) return cudaErrorNotSupported;
  if (mode == CS_MODE_DIAG)
    return dtype == CS_F64 ? launch_elements<Gibbs<18, double>, CS_MODE_DIAG, 18, double>(*(SolveArgs<double> *)args, it, g, e0, e1, e2, e3, u, stats, st)
                           : launch_elements<Gibbs<18, float>, CS_MODE_DIAG, 18, float>(*(SolveArgs<float> *)args, it, g, e0, e1, e2, e3, u, stats, st);
  return cudaErrorNotSupported;
}
}  // namespace cs
