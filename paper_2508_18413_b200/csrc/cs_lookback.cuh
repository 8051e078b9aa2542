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
  double *exit;       // [ntiles * state_width]   (rows scan: group exits)
  // rows scan only: groups of kGroupTiles consecutive tiles
  int *gstatus;       // [ngroups]  0 none, 1 group aggregate, 2 group exit
  int *gcount;        // [ngroups]  tile aggregates published so far
  double *gagg;       // [ngroups * agg_width]
};

// Row tiles are linked in two levels.  The producer that publishes the last
// missing tile aggregate of a group (atomic count) folds the group's 32
// aggregates into the group aggregate at once, so group aggregates never wait
// on any look-back.  A tile then folds its own group's predecessors (<= 31,
// one round trip) and runs a decoupled look-back over group aggregates for
// the state entering its group; the first tile of a group publishes that
// state as the previous group's exit.  Look-back reads per tile stay
// O(group + groups in flight) instead of O(tiles in flight).
constexpr int kGroupTiles = 32;

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
