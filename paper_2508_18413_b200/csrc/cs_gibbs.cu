// Eight-schools GibbsKernel (samplers.py:464-668): batched API kernels + fused solver.
#include "cs_dispatch.h"

namespace cs {

// ---------------------------------------------------------------------------
// The eight-schools element builder with one 8-lane team per chain step
// (lane = school).  The sweep (samplers.py:551-587) and its JVP (593-627) couple
// schools only through sums over schools, which become 3-level xor butterflies
// -- the same pairwise order numpy uses for 8 terms.  Each lane holds one
// school's state, so 8x more threads carry the f64 dependency chains than in the
// one-thread-per-step kernel, at a fraction of the registers.
template <typename V>
CS_D V team_sum(V v) {
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  v += __shfl_xor_sync(0xffffffffu, v, 4);
  return v;
}
#ifndef CS_GIBBS_TT_SUMS  // tangent team sums + probe shuffles in the tangent type (fp32: 89.3 -> 87 ms at cfg 5, same 135 iterations)
#define CS_GIBBS_TT_SUMS 1
#endif

// fp32 storage: compiled for 4 resident CTAs per SM (64 registers, 4 B of
// spill): cfg 5 T = 1M 92.8 -> 88.8 ms against the unconstrained 80-register
// build (tools/build_gibbs_variants.sh); f64 keeps 80 (64 would spill 24 B)
#ifndef CS_GIBBS_MINB
#define CS_GIBBS_MINB 4
#endif

template <typename ST>
__global__ void __launch_bounds__(256, sizeof(ST) == 4 ? CS_GIBBS_MINB : 1)
k_gibbs_elements_team(SolveArgs<ST> A, int iteration, const ST *guess, ST *jout, ST *uout, cs_elem_stats *stats) {
  constexpr int S = 8, D = 18;
  constexpr double kFloor = 1e-8;
  __shared__ long long smin[3];
  __shared__ unsigned scnt;
  __shared__ uint64_t s_h2;  // the iteration's probe prefix (two hash rounds), once per CTA
  if (threadIdx.x == 0) {
    smin[0] = smin[1] = smin[2] = kNoStep;
    scnt = 0;
    s_h2 = probe_prefix(A.sys.seed, iteration);
  }
  __syncthreads();
  const double *prm = A.sys.gibbs;
  const double nu0 = __ldg(prm + 0), tau0_sq = __ldg(prm + 1), mu0 = __ldg(prm + 2);
  const double kappa0 = __ldg(prm + 3), alpha0 = __ldg(prm + 4), sigma0_sq = __ldg(prm + 5), n = __ldg(prm + 7);
  const int sub = threadIdx.x & 7;
  const int64_t r = ((int64_t)blockIdx.x * 256 + threadIdx.x) >> 3;
  const bool valid = r < A.T;
  const int64_t rr = valid ? r : 0;
  const int64_t t = A.t0 + rr + 1;
  const ST *prow = rr == 0 ? A.s0 : guess + (rr - 1) * D;
  const ST *grow = guess + rr * D;
  const ST *g_tau = (const ST *)A.sys.g_tau, *xi_mu = (const ST *)A.sys.xi_mu;
  const ST *xi_theta = (const ST *)A.sys.xi_theta, *g_sigma = (const ST *)A.sys.g_sigma;
  const double xbar = __ldg(prm + 8 + sub), ss = __ldg(prm + 8 + S + sub);
  // prev state (tau^2 is never read by the sweep, samplers.py:543-548)
  const double mu = (double)prow[1], th = (double)prow[2 + sub], sgraw = (double)prow[2 + S + sub];
  const double gt = (double)g_tau[t], xm = (double)xi_mu[t];
  const double xt = (double)xi_theta[t * S + sub], gs = (double)g_sigma[t * S + sub];
  const bool raw_ok = sgraw > kFloor;
  const double sg = fmax(sgraw, kFloor);
  // ---- forward sweep
  const double dm = th - mu;
  const double q = team_sum(dm * dm);
  const double sth = team_sum(th);
  const double dmu0 = mu - mu0;
  const double q_tau = (nu0 * tau0_sq + kappa0 * (dmu0 * dmu0)) + q;
  const double tau2n = q_tau / gt;
  const double kS = kappa0 + (double)S;
  double mun, prec, mean, thn, inv_t = 0, inv_sg = 0, rq = 0, rsq = 0;
  if constexpr (sizeof(ST) == 4) {
    // fp32 storage: the f64 sweep with shared reciprocals (1/tau^2, 1/sigma^2,
    // 1/kS, rsqrt(prec)) -- a few f64 ulps against the quotients, far below the
    // fp32 rounding of the stored states; f64 storage keeps the exact quotients
    const double inv_kS = 1.0 / kS;
    inv_t = 1.0 / tau2n;
    inv_sg = 1.0 / sg;
    mun = (kappa0 * mu0 + sth) * inv_kS + sqrt(tau2n * inv_kS) * xm;
    prec = inv_t + n * inv_sg;
    rq = rsqrt(prec);
    mean = (mun * inv_t + (n * xbar) * inv_sg) * (rq * rq);
    thn = mean + xt * rq;
  } else {
    mun = (kappa0 * mu0 + sth) / kS + sqrt(tau2n / kS) * xm;
    prec = 1.0 / tau2n + n / sg;
    mean = (mun / tau2n + (n * xbar) / sg) / prec;
    rsq = sqrt(prec);
    thn = mean + xt / rsq;
  }
  const double res = xbar - thn;
  const double sgn = ((alpha0 * sigma0_sq + ss) + n * (res * res)) / gs;
  // finite / Picard on the coordinates this lane owns (lane 0 also tau^2, mu)
  auto tol_fail = [&](double f, double g) { return !(fabs(f - g) <= A.atol + A.rtol * fabs(f)); };
  bool fin = isfinite(thn) && isfinite(sgn);
  bool pfail = tol_fail(thn, (double)grow[2 + sub]) || tol_fail(sgn, (double)grow[2 + S + sub]);
  if (sub == 0) {
    fin &= isfinite(tau2n) && isfinite(mun);
    pfail |= tol_fail(tau2n, (double)grow[0]) || tol_fail(mun, (double)grow[1]);
  }
  // ---- Hutchinson over nsamp probes (deer.py:118-132).  The tangent map is
  // linear in the probe, so every per-step quotient is hoisted into a
  // reciprocal once; the tangents run in the storage precision TT (the estimate
  // only steers convergence, the step values above stay f64).
  using TT = ST;
  const uint64_t h3 = hash_t(s_h2, (uint64_t)t);
  // coefficients of the tangent map, formed in TT: in fp32 storage mode these
  // are fp32 reciprocals (the f64 forward values above are only rounded once)
  TT inv_gt, inv_kS, inv_tau2n, inv_t2sq, n_sg2, inv_prec, c_mu, c_th, c_sg;
  if constexpr (sizeof(TT) == 4) {
    const float gt_t = (float)gt, kS_t = (float)kS, t2_t = (float)tau2n, n_t = (float)n;
    inv_gt = 1.0f / gt_t;
    inv_kS = 1.0f / kS_t;
    inv_tau2n = (float)inv_t;
    inv_t2sq = inv_tau2n * inv_tau2n;
    n_sg2 = (float)(n * inv_sg * inv_sg);
    inv_prec = (float)(rq * rq);
    c_mu = (float)xm / (2.0f * sqrtf(t2_t * kS_t));
    c_th = 0.5f * (float)xt * inv_prec * (float)rq;
    c_sg = (-2.0f * n_t * (float)(xbar - thn)) / (float)gs;
  } else {
    inv_gt = 1.0 / gt; inv_kS = 1.0 / kS; inv_tau2n = 1.0 / tau2n;
    inv_t2sq = 1.0 / (tau2n * tau2n); n_sg2 = n / (sg * sg); inv_prec = 1.0 / prec;
    c_mu = xm / (2.0 * sqrt(tau2n * kS)); c_th = 0.5 * xt / (prec * rsq);
    c_sg = (-2.0 * n * (xbar - thn)) / gs;
  }
  const TT mun_t = (TT)mun, mean_t = (TT)mean;
  const TT xbar_t = (TT)xbar, two_dm = (TT)(2.0 * (th - mu)), mu_c = (TT)(2.0 * kappa0 * (mu - mu0));
  TT e_tau = 0, e_mu = 0, e_th = 0, e_sg = 0;
#if CS_GIBBS_TT_SUMS
  using SU = TT;
#else
  using SU = double;
#endif
  const int team0 = (threadIdx.x & 31) & ~7;
  SU zpre = 0;  // z_tau / z_mu are shared by the team: lane j hashes (probe j/2, coordinate j%2) of 4 probes
  for (int k = 0; k < A.nsamp; ++k) {
    if ((k & 3) == 0) zpre = (SU)probe_sign_fast(h3, k + (sub >> 1), sub & 1);
    const TT z_tau = (TT)__shfl_sync(0xffffffffu, zpre, team0 + 2 * (k & 3));
    const TT z_mu = (TT)__shfl_sync(0xffffffffu, zpre, team0 + 2 * (k & 3) + 1);
    const TT z_th = (TT)probe_sign_fast(h3, k, 2 + sub), z_sg = (TT)probe_sign_fast(h3, k, 2 + S + sub);
    const TT dsg = raw_ok ? z_sg : (TT)0;
    const TT dq = mu_c * z_mu + (TT)team_sum((SU)(two_dm * (z_th - z_mu)));
    const TT dtau2 = dq * inv_gt;
    const TT dmu = (TT)team_sum((SU)z_th) * inv_kS + c_mu * dtau2;
    const TT dprec = -dtau2 * inv_t2sq - n_sg2 * dsg;
    const TT damean = (dmu * inv_tau2n - mun_t * dtau2 * inv_t2sq) - xbar_t * n_sg2 * dsg;
    const TT dmean = (damean - mean_t * dprec) * inv_prec;
    const TT dth = dmean - c_th * dprec;
    const TT dsgo = c_sg * dth;
    e_tau += z_tau * dtau2;
    e_mu += z_mu * dmu;
    e_th += z_th * dth;
    e_sg += z_sg * dsgo;
  }
  const double ns = (double)A.nsamp, inv_ns = 1.0 / ns;
  bool jok = true;
  auto elem = [&](int d, double est, double f, double p, int64_t off) {
    // est / n_samples as deer.py:131 (fp32 storage: times the reciprocal -- the
    // f64 quotient is rounded to fp32 anyway)
    double v = sizeof(ST) == 4 ? est * inv_ns : est / ns;
    jok &= isfinite(v);
    if (A.pre) v = v * __ldg(A.pre + d);
    v = v * A.damping;
    if (isfinite(A.clip)) v = clipv(v, A.clip);
    if (valid) {
      jout[off] = (ST)v;
      uout[off] = (ST)(f - v * p);
    }
  };
  elem(2 + sub, (double)e_th, thn, th, rr * D + 2 + sub);
  elem(2 + S + sub, (double)e_sg, sgn, sgraw, rr * D + 2 + S + sub);
  if (sub < 2)  // tau^2 on lane 0, mu on lane 1 (every lane holds both team values)
    elem(sub, sub == 0 ? (double)e_tau : (double)e_mu, sub == 0 ? tau2n : mun, sub == 0 ? (double)prow[0] : mu,
         rr * D + sub);
  // team flags -> block -> stats
  const unsigned bad_fin = __ballot_sync(0xffffffffu, valid && !fin);
  const unsigned bad_jac = __ballot_sync(0xffffffffu, valid && !jok);
  const unsigned pf = __ballot_sync(0xffffffffu, valid && pfail);
  const int lane = threadIdx.x & 31;
  if (lane == 0) {
    const int64_t r0 = ((int64_t)blockIdx.x * 256 + (threadIdx.x & ~31)) >> 3;
    unsigned cnt = 0;
    for (int tm = 0; tm < 4; ++tm) {
      const unsigned m = 0xFFu << (8 * tm);
      const long long step = r0 + tm + 1;
      if (bad_fin & m) atomicMin(&smin[1], step);
      if (bad_jac & m) atomicMin(&smin[2], step);
      if (pf & m) ++cnt;
    }
    if (cnt) atomicAdd(&scnt, cnt);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (smin[1] != kNoStep) atomicMin((long long *)&stats->bad_step, smin[1]);
    if (smin[2] != kNoStep) atomicMin((long long *)&stats->bad_jacobian, smin[2]);
    if (scnt) atomicAdd(&stats->picard_fail, scnt);
  }
}

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
  if (md != 18 || mode != CS_MODE_DIAG) return cudaErrorNotSupported;
  (void)e1; (void)e2; (void)e3;
  if (dtype == CS_F64) {
    const SolveArgs<double> &A = *(SolveArgs<double> *)args;
    const unsigned grid = (unsigned)((A.T * 8 + 255) / 256);
    k_gibbs_elements_team<double><<<grid, 256, 0, st>>>(A, it, (const double *)g, (double *)e0, (double *)u, stats);
  } else {
    const SolveArgs<float> &A = *(SolveArgs<float> *)args;
    const unsigned grid = (unsigned)((A.T * 8 + 255) / 256);
    k_gibbs_elements_team<float><<<grid, 256, 0, st>>>(A, it, (const float *)g, (float *)e0, (float *)u, stats);
  }
  return cudaGetLastError();
}
}  // namespace cs
