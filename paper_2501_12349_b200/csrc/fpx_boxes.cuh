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

// |inv (x - cen)|_inf with the OBB test's terms (rest ranking, prefilter).
__device__ __forceinline__ double obb_norm(int d, const double* __restrict__ cen,
                                           const double* __restrict__ inv, const double* x) {
  double dx[3];
  for (int c = 0; c < d; ++c) dx[c] = __dsub_rn(x[c], cen[c]);
  double v = 0.0;
  for (int c = 0; c < d; ++c) {
    double y = 0.0;
    for (int b = 0; b < d; ++b) y = __dadd_rn(y, __dmul_rn(inv[c * d + b], dx[b]));
    v = fabs(y) > v ? fabs(y) : v;
  }
  return v;
}


// ---- float pre-tests (include/fpx.h, mesh.fbox) -------------------------
// Outcome 0 = the double test fails, 1 = it passes, 2 = undecided here (the
// double record decides).  Either way the filter's outcome is the double
// test's, bit for bit; the pre-tests only spare most candidates the double
// record's loads: one 80-byte row (box and OBB in one round trip: at cfg-2
// 99% of listed candidates pass the AABB and 30% the OBB, so the OBB half
// is always wanted) instead of 152 bytes in two dependent steps -- the
// prefilter is bound by L1 wavefronts and load latency.
constexpr int kFboxMode = 6;  // OBB mode slot of the row
constexpr int kFrowObb = 8;   // obb_c, obb_inv

// Box: lo rounded down, hi rounded up.  xd = x rounded down, xu = up:
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

// OBB (mode 1) in float arithmetic: cen', inv' = cen, inv rounded to
// nearest (every value 0 or normal: 24 bits kept), x' = x rounded to
// nearest.  y' = fl(inv'(x' - cen')) differs from obb_in's y by at most
//   sum_b |inv_b - inv'_b||x_b - cen_b| + |inv'_b|(|x_b - x'_b| + |cen_b - cen'_b|)
//   + the float rounding of dx' and of the three-term sum
//   <= 6 * 2^-24 sum_b |inv'_b| (|dx'_b| + |x'_b| + |cen'_b|),
// plus 2^-149 |inv'| where x' is subnormal; the bound used is 2^-19 times
// the sum (5x slack, covering its own rounding and that of the compares)
// plus 2^-40.  NaN / inf (x beyond float range) -> 2.
template <int D>
__device__ __forceinline__ int fobb_in(const float* o, const double* x, float* ymax = nullptr) {
  float dx[D], ab[D], ym = 0.0f;
#pragma unroll
  for (int b = 0; b < D; ++b) {
    const float xf = __double2float_rn(x[b]);
    dx[b] = __fsub_rn(xf, o[b]);
    ab[b] = fabsf(dx[b]) + fabsf(xf) + fabsf(o[b]);
  }
  int res = 1;
#pragma unroll
  for (int c = 0; c < D; ++c) {
    float y = 0.0f, bnd = 0.0f;
#pragma unroll
    for (int b = 0; b < D; ++b) {
      const float iv = o[D + c * D + b];
      y = fmaf(iv, dx[b], y);
      bnd = fmaf(fabsf(iv), ab[b], bnd);
    }
    bnd = fmaf(bnd, 0x1p-19f, 0x1p-40f);
    const float ay = fabsf(y);
    if (ay - bnd > 1.0f) return 0;
    if (!(ay + bnd < 1.0f)) res = 2;
    ym = ay > ym ? ay : ym;
  }
  if (ymax) *ymax = ym;
  return res;
}

// The row's floats the D-dimensional tests read (16-byte loads).
template <int D>
__device__ __forceinline__ void frow_load(const float* __restrict__ fbox, int64_t e, float* b) {
  const float4* p = reinterpret_cast<const float4*>(fbox + e * FPX_FROW);
#pragma unroll
  for (int i = 0; i < (kFrowObb + D + D * D + 3) / 4; ++i) {
    const float4 t = __ldg(p + i);
    b[4 * i] = t.x, b[4 * i + 1] = t.y, b[4 * i + 2] = t.z, b[4 * i + 3] = t.w;
  }
}

// AABB and OBB tests of candidate e from its loaded row (the double record
// only where a pre-test is undecided).  yn (optional): the OBB norm
// |obb_inv (x - obb_c)|_inf of a passing candidate, from the float
// pre-test (mode 1) or the double record (mode 2), 0 without an OBB
// (mode 0): a term of the prefilter's ranking (k_prefilter_points).
template <int D>
__device__ __forceinline__ bool frow_passes(const fpx_mesh_t& m, int64_t e, const float* b,
                                            const double* x, float* yn = nullptr) {
  const float mode = b[kFboxMode];
  const int a = fbox_aabb<D>(b, x);
  float ym = 0.0f;
  const int o = mode == 0.0f ? 1 : (mode == 1.0f ? fobb_in<D>(b + kFrowObb, x, &ym) : 2);
  if (a == 0 || o == 0) return false;
  double R[FPX_FREC];
  if (a == 2) {
    frec_range<D, 0, 2 * D>(m.frec, e, R);
    if (!aabb_in(D, R, x)) return false;
  }
  if (o == 2) {
    frec_range<D, 2 * D, 3 * D + D * D>(m.frec, e, R);
    if (!obb_in(D, R + 2 * D, R + 3 * D, x)) return false;
    if (mode != 1.0f) ym = (float)obb_norm(D, R + 2 * D, R + 3 * D, x);
  }
  if (yn) *yn = ym;
  return true;
}

// The candidate filter (D4): the float row, then the affine frame only if
// the candidate passes (then *v = the best-first value).
template <int D>
__device__ __forceinline__ bool frec_filter(const fpx_mesh_t& m, int64_t e, const double* x,
                                            double* v) {
  float b[FPX_FROW];
  frow_load<D>(m.fbox, e, b);
  if (!frow_passes<D>(m, e, b, x)) return false;
  if (v) {
    double R[FPX_FREC];
    frec_range<D, 3 * D + D * D, 4 * D + 2 * D * D>(m.frec, e, R);
    *v = bestfirst_value(D, R + 3 * D + D * D, x);
  }
  return true;
}

// Rank value of a rest-phase candidate (ranks >= 1: k_rest_lists and the
// rest kernel's scan past its list): |obb_inv (x - obb_c)|_inf where the
// element has an OBB (row mode != 0), else its best-first value.  Measured
// on cfg-2, the point's owner is the first of its remaining candidates in
// this order for 87% of the rest points (53% in best-first order; mean rank
// 1.18 against 2.46; tests/rank_study.py).  The order decides only how
// soon a point's INTERIOR record is found: a point is INTERIOR in at most
// one element of a conforming mesh, and a BORDER point's record is the D6
// minimum over all of its candidates.
template <int D>
__device__ __forceinline__ double rest_rank_value(const fpx_mesh_t& m, int64_t e, float mode,
                                                  const double* x) {
  double R[FPX_FREC];
  if (mode != 0.0f) {
    frec_range<D, 2 * D, 3 * D + D * D>(m.frec, e, R);
    return obb_norm(D, R + 2 * D, R + 3 * D, x);
  }
  frec_range<D, 3 * D + D * D, 4 * D + 2 * D * D>(m.frec, e, R);
  return bestfirst_value(D, R + 3 * D + D * D, x);
}

// The rest rank value of a candidate already known to pass the filter.
template <int D>
__device__ __forceinline__ double rest_rank_of(const fpx_mesh_t& m, int64_t e, const double* x) {
  return rest_rank_value<D>(m, e, __ldg(m.fbox + e * FPX_FROW + kFboxMode), x);
}

// The candidate filter with the rest rank value (*v) of a passing candidate.
template <int D>
__device__ __forceinline__ bool frec_filter_rest(const fpx_mesh_t& m, int64_t e, const double* x,
                                                 double* v) {
  float b[FPX_FROW];
  frow_load<D>(m.fbox, e, b);
  if (!frow_passes<D>(m, e, b, x)) return false;
  if (v) *v = rest_rank_value<D>(m, e, b[kFboxMode], x);
  return true;
}

// (v, e) lexicographic order of the best-first ranking (ties -> lower id).
__device__ __forceinline__ bool bf_less(double v1, int e1, double v2, int e2) {
  return v1 < v2 || (v1 == v2 && e1 < e2);
}

}  // namespace fpx
