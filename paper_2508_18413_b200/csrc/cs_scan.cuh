// Scan launch plans shared by the standalone C-ABI scans and the generic driver.
#pragma once
#include "cs_common.cuh"

namespace cs {

enum { SCAN_DIAG = 0, SCAN_BLOCK = 1, SCAN_DENSE = 2 };

template <typename ST>
struct ScanArgs {
  const ST *e0, *e1, *e2, *e3;  // diag: j | block: a b c d | dense: J
  const ST *u, *s0;
  ST *out;
  int64_t T;
  int D;                        // diag/dense: state dim; block: half (position) dim
  // fused post-update bookkeeping (deer.py:273-277), used by the *_update scans
  const ST *guess;
  double atol, rtol;
  int it;
  int32_t *last_fail;
  cs_elem_stats *stats;
  // debug timeline (cs_debug_probe): per tile 8 x u64 {sm, claim, data, agg,
  // linked, replayed, -, -} globaltimer stamps; null in production
  unsigned long long *probe;
  int64_t probe_n;
};

struct ScanPlan {
  int var, kind, R, md, seg, win;
  int64_t ntiles;
  int agg_w, state_w;
  size_t smem, ws_bytes;
};

ScanPlan scan_plan(int var, int dtype, int64_t T, int D, bool update = false);
// workspace for either the plain or the bookkeeping (update) scan of a shape
size_t scan_ws_bytes(int var, int dtype, int64_t T, int D);
// single-pass row scan for plain diag scans (scan_rows_1p): eligibility, plan, launch
bool scan_1p_eligible(int var, int64_t T, int D);
bool scan_local_eligible(int var, int64_t T, int D);
ScanPlan scan_plan_1p(int var, int dtype, int64_t T, int D);
template <typename ST>
cudaError_t launch_scan_1p_t(const ScanPlan &p, ScanArgs<ST> a, void *ws, cudaStream_t st);
// local-scan + fix-up row scan (CS_SCAN_1P=3)
int scan_1p_mode();
size_t scan_local_ws_bytes(int dtype, int64_t T, int D);
template <typename ST, bool UPD>
cudaError_t launch_scan_local_t(ScanArgs<ST> a, void *ws, cudaStream_t st);
// reduce-then-replay row scan (diag; the update scans at moderate T)
bool scan_rr_eligible(int var, int64_t T, int D);
size_t scan_rr_ws_bytes(int dtype, int64_t T, int D);
template <typename ST, bool UPD>
cudaError_t launch_scan_rr_t(ScanArgs<ST> a, void *ws, cudaStream_t st);
size_t scan_local_blk_ws_bytes(int dtype, int64_t T, int D);
template <typename ST>
cudaError_t launch_scan_local_blk_t(ScanArgs<ST> a, void *ws, cudaStream_t st);
template <typename ST>
cudaError_t launch_scan_t(const ScanPlan &p, ScanArgs<ST> a, void *ws, cudaStream_t st, bool update = false);
// wide dense scans, 8 < D <= 128 (cs_dense.cu)
size_t dense_wide_ws_bytes(int64_t T, int D, int esize);  // esize: storage bytes (4 adds the f32 tree levels)
// agg_out != null: write the whole-sequence map [M (D x D) | w (D)] (f64) instead of scanning
template <typename ST>
cudaError_t launch_dense_wide_t(ScanArgs<ST> a, void *ws, cudaStream_t st, double *agg_out = nullptr);
// dense scans and aggregates for D > 128 (cs_dense_xl.cu)
size_t dense_xl_ws_bytes(int64_t T, int D, int elem_bytes);
template <typename ST>
cudaError_t launch_dense_xl_t(ScanArgs<ST> a, void *ws, double *agg_out, cudaStream_t st);
size_t dense_tree_bytes(int64_t n, int D);
cudaError_t dense_fold_aggregates(const double *aggM, const double *aggw, int64_t n, int D, double *tree,
                                  double *out, cudaStream_t st);
template <typename ST>
cudaError_t launch_aggregate_t(const ScanPlan &p, ScanArgs<ST> a, void *ws, double *out, cudaStream_t st);

}  // namespace cs
