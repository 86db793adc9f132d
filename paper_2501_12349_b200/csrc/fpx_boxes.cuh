// fpx_boxes.cuh -- candidate filter arithmetic shared by the exact TU
// (prefilter) and the FMA TU (overflow scan of the rest kernel).
//
// Every multiply and add is an explicit round-to-nearest intrinsic, so the
// result does not depend on the TU's --fmad policy and is bit-identical to
// the oracle (aabb_contains / obb_contains, bounds.py:387-396; best-first
// value of DESIGN.md §3 "Candidate order").
#pragma once
#include <math.h>

#include "fpx_common.cuh"

namespace fpx {

__device__ __forceinline__ bool aabb_in(int d, const double* __restrict__ bx, const double* x) {
  for (int c = 0; c < d; ++c)
    if (!(__dmul_rn(__dsub_rn(x[c], bx[c]), __dsub_rn(bx[d + c], x[c])) >= 0.0)) return false;
  return true;
}

__device__ __forceinline__ bool obb_in(int d, const double* __restrict__ cen,
                                       const double* __restrict__ inv, const double* x) {
  double dx[3];
  for (int c = 0; c < d; ++c) dx[c] = __dsub_rn(x[c], cen[c]);
  for (int c = 0; c < d; ++c) {
    double y = 0.0;
    for (int b = 0; b < d; ++b) y = __dadd_rn(y, __dmul_rn(inv[c * d + b], dx[b]));
    if (!(fabs(y) <= 1.0)) return false;
  }
  return true;
}

// Best-first value of candidate e at x: |J_c^{-1}(x - x_c)|_inf, with
// fr = frame[e] = (x_c[d], J_c^{-1}[d][d]).
__device__ __forceinline__ double bestfirst_value(int d, const double* __restrict__ fr,
                                                  const double* x) {
  double dx[3];
  for (int c = 0; c < d; ++c) dx[c] = __dsub_rn(x[c], fr[c]);
  double v = 0.0;
  for (int c = 0; c < d; ++c) {
    double y = 0.0;
    for (int b = 0; b < d; ++b) y = __dadd_rn(y, __dmul_rn(fr[d + c * d + b], dx[b]));
    v = fabs(y) > v ? fabs(y) : v;
  }
  return v;
}

// Full filter of candidate e (AABB, then OBB unless the frame is singular).
__device__ __forceinline__ bool candidate_passes(const fpx_mesh_t& m, int e, const double* x) {
  const int d = m.d;
  if (!aabb_in(d, m.aabb + (int64_t)e * 2 * d, x)) return false;
  if (m.obb_ok[e] && !obb_in(d, m.obb_c + (int64_t)e * d, m.obb_inv + (int64_t)e * d * d, x))
    return false;
  return true;
}

// cell_of; returns -1 outside, per-axis coords in ax.
__device__ __forceinline__ int64_t cell_of(int d, const double* grid, int n, const double* x,
                                           int* ax) {
  int64_t idx = 0, mul = 1;
  for (int c = 0; c < d; ++c) {
    if (!(x[c] >= grid[c] && x[c] <= grid[3 + c])) return -1;
    double t = __ddiv_rn(__dsub_rn(x[c], grid[c]), grid[6 + c]);
    int64_t q = (int64_t)floor(t);
    q = q > n - 1 ? n - 1 : q;
    q = q < 0 ? 0 : q;
    ax[c] = (int)q;
    idx += q * mul;
    mul *= n;
  }
  return idx;
}

template <int D>
__device__ __forceinline__ bool candidate_passes_t(const fpx_mesh_t& m, int e, const double* x) {
  if (!aabb_in(D, m.aabb + (int64_t)e * 2 * D, x)) return false;
  if (m.obb_ok[e] && !obb_in(D, m.obb_c + (int64_t)e * D, m.obb_inv + (int64_t)e * D * D, x))
    return false;
  return true;
}

// Doubles [A, B) of element e's filter record (16-byte loads).
template <int D, int A, int B>
__device__ __forceinline__ void frec_range(const double* __restrict__ frec, int64_t e, double* v) {
  const double2* p = reinterpret_cast<const double2*>(frec + e * FPX_FREC);
#pragma unroll
  for (int i = A / 2; i < (B + 1) / 2; ++i) {
    const double2 t = __ldg(p + i);
    v[2 * i] = t.x;
    v[2 * i + 1] = t.y;
  }
}

// The candidate filter (D4) with the record loaded in stages: the AABB
// (48 B), the OBB and its flag only if the AABB passes, the affine frame
// only if the OBB passes (then *v = the best-first value).
template <int D>
__device__ __forceinline__ bool frec_filter(const double* __restrict__ frec, int64_t e,
                                            const double* x, double* v) {
  double R[FPX_FREC];
  frec_range<D, 0, 2 * D>(frec, e, R);
  if (!aabb_in(D, R, x)) return false;
  frec_range<D, 2 * D, 3 * D + D * D>(frec, e, R);
  frec_range<D, FPX_FREC - 1, FPX_FREC>(frec, e, R);
  if (!(R[FPX_FREC - 1] == 0.0 || obb_in(D, R + 2 * D, R + 3 * D, x))) return false;
  if (v) {
    frec_range<D, 3 * D + D * D, 4 * D + 2 * D * D>(frec, e, R);
    *v = bestfirst_value(D, R + 3 * D + D * D, x);
  }
  return true;
}

// (v, e) lexicographic order of the best-first ranking (ties -> lower id).
__device__ __forceinline__ bool bf_less(double v1, int e1, double v2, int e2) {
  return v1 < v2 || (v1 == v2 && e1 < e2);
}

}  // namespace fpx
