// Decoupled look-back across row tiles for the affine scans.
//
// Tiles are claimed in order through an atomic ticket, so every predecessor of
// a running tile has already started (forward progress without co-residency).
// Tile b publishes its aggregate (status 1) as soon as its local reduce is
// done, looks back composing predecessors' aggregates until it meets an
// inclusive exit state (status 2) or s0, then publishes its own exit state.
// For the affine monoid the "inclusive prefix" is simply the chain state at
// the end of the tile, so the hand-off is a D-vector, not a D x D matrix.
#pragma once
#include "cs_common.cuh"

namespace cs {

struct LookbackWs {
  unsigned *ticket;   // [1]
  int *status;        // [ntiles]   0 none, 1 aggregate, 2 exit state
  double *agg;        // [ntiles * agg_width]
  double *exit;       // [ntiles * state_width]
};

CS_D int ld_acquire(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
CS_D void st_release(int *p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
CS_D double ld_cg(const double *p) { return __ldcg(p); }

}  // namespace cs
