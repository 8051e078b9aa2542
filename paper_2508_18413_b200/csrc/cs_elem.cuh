// Affine elements held in registers, one per chain step, for the fused solver.
//
//   DIAG   j[MD], u[MD]                 (DiagElements,      pscan.py:100-116)
//   DENSE  J[MD][MD] row-major, u[MD]   (DenseElements,     pscan.py:119-136)
//   BLOCK  a,b,c,d[H], u[2H] = [x | v]  (Block2x2Elements,  pscan.py:139-170)
// stored flat in v[W] so warp shuffles and smem moves are generic.
#pragma once
#include "cs_common.cuh"

namespace cs {

template <int MODE, int MD> struct ElemShape;
template <int MD> struct ElemShape<CS_MODE_DIAG, MD> { static constexpr int W = 2 * MD; };
template <int MD> struct ElemShape<CS_MODE_DENSE, MD> { static constexpr int W = MD * MD + MD; };
template <int MD> struct ElemShape<CS_MODE_BLOCK, MD> { static constexpr int W = 3 * MD; };

template <int MODE, int MD>
struct Elem {
  static constexpr int W = ElemShape<MODE, MD>::W;
  static constexpr int H = MD / 2;
  double v[W];

  // diag accessors
  CS_D double &j(int i) { return v[i]; }
  CS_D double j(int i) const { return v[i]; }
  // dense accessors
  CS_D double &M(int r, int c) { return v[r * MD + c]; }
  CS_D double M(int r, int c) const { return v[r * MD + c]; }
  // block accessors
  CS_D double &ba(int i) { return v[i]; }
  CS_D double &bb(int i) { return v[H + i]; }
  CS_D double &bc(int i) { return v[2 * H + i]; }
  CS_D double &bd(int i) { return v[3 * H + i]; }
  CS_D double ba(int i) const { return v[i]; }
  CS_D double bb(int i) const { return v[H + i]; }
  CS_D double bc(int i) const { return v[2 * H + i]; }
  CS_D double bd(int i) const { return v[3 * H + i]; }
  // offset vector (all modes): last MD entries
  CS_D double &u(int i) { return v[W - MD + i]; }
  CS_D double u(int i) const { return v[W - MD + i]; }

  CS_D void ident() {
#pragma unroll
    for (int k = 0; k < W; ++k) v[k] = 0.0;
    if constexpr (MODE == CS_MODE_DIAG) {
#pragma unroll
      for (int i = 0; i < MD; ++i) v[i] = 1.0;
    } else if constexpr (MODE == CS_MODE_DENSE) {
#pragma unroll
      for (int i = 0; i < MD; ++i) v[i * MD + i] = 1.0;
    } else {
#pragma unroll
      for (int i = 0; i < H; ++i) { v[i] = 1.0; v[3 * H + i] = 1.0; }
    }
  }

  // this <- L o this (L applied after this)
  CS_D void after(const Elem &L) {
    Elem r;
    if constexpr (MODE == CS_MODE_DIAG) {
#pragma unroll
      for (int i = 0; i < MD; ++i) {
        r.v[MD + i] = L.v[i] * v[MD + i] + L.v[MD + i];
        r.v[i] = L.v[i] * v[i];
      }
    } else if constexpr (MODE == CS_MODE_DENSE) {
#pragma unroll
      for (int a = 0; a < MD; ++a) {
        double aw = L.u(a);
#pragma unroll
        for (int k = 0; k < MD; ++k) aw += L.M(a, k) * u(k);
        r.u(a) = aw;
#pragma unroll
        for (int c = 0; c < MD; ++c) {
          double acc = 0.0;
#pragma unroll
          for (int k = 0; k < MD; ++k) acc += L.M(a, k) * M(k, c);
          r.M(a, c) = acc;
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < H; ++i) {
        const double A = ba(i), B = bb(i), C = bc(i), E = bd(i), ux = u(i), uv = u(H + i);
        const double a = L.ba(i), b = L.bb(i), c = L.bc(i), d = L.bd(i);
        r.ba(i) = a * A + b * C;
        r.bb(i) = a * B + b * E;
        r.bc(i) = c * A + d * C;
        r.bd(i) = c * B + d * E;
        r.u(i) = a * ux + b * uv + L.u(i);
        r.u(H + i) = c * ux + d * uv + L.u(H + i);
      }
    }
    *this = r;
  }

  CS_D void apply(double (&x)[MD]) const {
    if constexpr (MODE == CS_MODE_DIAG) {
#pragma unroll
      for (int i = 0; i < MD; ++i) x[i] = j(i) * x[i] + u(i);
    } else if constexpr (MODE == CS_MODE_DENSE) {
      double y[MD];
#pragma unroll
      for (int a = 0; a < MD; ++a) {
        double acc = u(a);
#pragma unroll
        for (int k = 0; k < MD; ++k) acc += M(a, k) * x[k];
        y[a] = acc;
      }
#pragma unroll
      for (int a = 0; a < MD; ++a) x[a] = y[a];
    } else {
#pragma unroll
      for (int i = 0; i < H; ++i) {
        const double xi = x[i], vi = x[H + i];
        x[i] = ba(i) * xi + bb(i) * vi + u(i);
        x[H + i] = bc(i) * xi + bd(i) * vi + u(H + i);
      }
    }
  }

  CS_D void shfl_up(int delta, Elem &o) const {
#pragma unroll
    for (int k = 0; k < W; ++k) o.v[k] = __shfl_up_sync(0xffffffffu, v[k], delta);
  }
};

}  // namespace cs
