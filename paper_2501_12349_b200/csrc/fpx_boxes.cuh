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

// ---- float pre-tests (include/fpx.h, mesh.fbox) -------------------------
// Outcome 0 = the double test fails, 1 = it passes, 2 = undecided here (the
// double record decides).  Either way the filter's outcome is the double
// test's, bit for bit; the pre-tests only spare most candidates the double
// record's loads (16 B + 8 B of box row instead of 48 B, 48 B of OBB row
// instead of 104 B) -- the prefilter is bound by L1 wavefronts.
constexpr int kFboxMode = 6;  // OBB mode slot of the box row

// Box row: lo rounded down, hi rounded up.  xd = x rounded down, xu = up:
// xu < lo' => x < lo; xd > lo' => xd >= nextup(lo') >= lo => x >= lo (same
// for hi).  A failed test is exact whatever the magnitudes: x < lo' <= lo
// leaves x - lo at least one float spacing away from 0, so the product in
// aabb_in cannot underflow to -0.
template <int D>
__device__ __forceinline__ int fbox_aabb(const float* b, const double* x) {
  int res = 1;
#pragma unroll
  for (int c = 0; c < D; ++c) {
    const float xd = __double2float_rd(x[c]), xu = __double2float_ru(x[c]);
    if (xu < b[c] || xd > b[D + c]) return 0;
    if (!(xd > b[c] && xu < b[D + c])) res = 2;
  }
  return res;
}

// OBB row (mode 1): cen', inv' = cen, inv rounded to nearest, every value 0
// or normal with 24 bits kept.  y' = inv'(x - cen') differs from obb_in's y
// by at most sum_b |inv_b - inv'_b||dx_b| + |inv'_b||cen_b - cen'_b| plus the
// rounding of both sums, <= 2^-23 sum_b |inv'_b| (|dx'_b| + |cen'_b|); the
// bound used is twice that (covering its own rounding).  NaN / inf -> 2.
template <int D>
__device__ __forceinline__ int fobb_in(const float* o, const double* x) {
  double dx[D], ab[D];
#pragma unroll
  for (int b = 0; b < D; ++b) {
    const double cb = (double)o[b];
    dx[b] = x[b] - cb;
    ab[b] = fabs(dx[b]) + fabs(cb);
  }
  int res = 1;
#pragma unroll
  for (int c = 0; c < D; ++c) {
    double y = 0.0, bnd = 0.0;
#pragma unroll
    for (int b = 0; b < D; ++b) {
      const double iv = (double)o[D + c * D + b];
      y = fma(iv, dx[b], y);
      bnd = fma(fabs(iv), ab[b], bnd);
    }
    bnd *= 0x1p-21;
    const double ay = fabs(y);
    if (ay - bnd > 1.0) return 0;
    if (!(ay + bnd < 1.0)) res = 2;
  }
  return res;
}

template <int D>
__device__ __forceinline__ void fbox_row(const float* __restrict__ fbox, int64_t e, float* b) {
  const float4* p = reinterpret_cast<const float4*>(fbox + e * FPX_FBOX);
  const float4 t0 = __ldg(p), t1 = __ldg(p + 1);
  b[0] = t0.x, b[1] = t0.y, b[2] = t0.z, b[3] = t0.w;
  b[4] = t1.x, b[5] = t1.y, b[6] = t1.z, b[7] = t1.w;
}

// OBB stage of the filter given the box row's mode (0, 1, 2).
template <int D>
__device__ __forceinline__ bool obb_stage(const fpx_mesh_t& m, int64_t e, float mode,
                                          const double* x) {
  if (mode == 0.0f) return true;
  if (mode == 1.0f) {
    const float4* p = reinterpret_cast<const float4*>(m.fbox + m.E * FPX_FBOX + e * FPX_FOBB);
    float o[FPX_FOBB];
#pragma unroll
    for (int i = 0; i < (D + D * D + 3) / 4; ++i) {
      const float4 t = __ldg(p + i);
      o[4 * i] = t.x, o[4 * i + 1] = t.y, o[4 * i + 2] = t.z, o[4 * i + 3] = t.w;
    }
    const int r = fobb_in<D>(o, x);
    if (r != 2) return r == 1;
  }
  double R[FPX_FREC];
  frec_range<D, 2 * D, 3 * D + D * D>(m.frec, e, R);
  return obb_in(D, R + 2 * D, R + 3 * D, x);
}

// The candidate filter (D4) with the records loaded in stages: the float
// box row, the OBB row only if the box passes, the affine frame only if the
// OBB passes (then *v = the best-first value); the double rows only where
// a float pre-test is undecided.
template <int D>
__device__ __forceinline__ bool frec_filter(const fpx_mesh_t& m, int64_t e, const double* x,
                                            double* v) {
  float b[FPX_FBOX];
  fbox_row<D>(m.fbox, e, b);
  int a = fbox_aabb<D>(b, x);
  if (a == 2) {
    double R[2 * D];
    frec_range<D, 0, 2 * D>(m.frec, e, R);
    a = aabb_in(D, R, x) ? 1 : 0;
  }
  if (a == 0 || !obb_stage<D>(m, e, b[kFboxMode], x)) return false;
  if (v) {
    double R[FPX_FREC];
    frec_range<D, 3 * D + D * D, 4 * D + 2 * D * D>(m.frec, e, R);
    *v = bestfirst_value(D, R + 3 * D + D * D, x);
  }
  return true;
}

// (v, e) lexicographic order of the best-first ranking (ties -> lower id).
__device__ __forceinline__ bool bf_less(double v1, int e1, double v2, int e2) {
  return v1 < v2 || (v1 == v2 && e1 < e2);
}

}  // namespace fpx
