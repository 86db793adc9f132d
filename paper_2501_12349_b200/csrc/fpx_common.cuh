// fpx_common.cuh -- shared device helpers for the sm_100a findpts kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/fpx.h"

#define FPX_WARP 32
#define FPX_FULL 0xffffffffu

// Record-code constants mirrored for device code.
enum { kInterior = FPX_INTERIOR, kBorder = FPX_BORDER, kNotFound = FPX_NOT_FOUND };

// SPEC.md:311,434 strict-interior tolerance; literal shared with the oracle.
#define FPX_INTERIOR_TOL 1e-12
// D8 resolvability floor of the predicted decrease (oracle UNRES_REL/ABS)
#define FPX_UNRES_REL 1e-13
#define FPX_UNRES_ABS 1e-14
#define FPX_ZERO_EXTENT_REL 1e-12  // bounds.py:43

// Newton settings copied by value into kernels.
struct NewtonParams {
  int max_iters;
  double tol, grow, keep, accept, shrink, alpha0;
};

__host__ __device__ inline NewtonParams newton_of(const fpx_mesh_t& m) {
  NewtonParams p;
  p.max_iters = m.max_iters;
  p.tol = m.tol;
  p.grow = m.grow;
  p.keep = m.keep;
  p.accept = m.accept;
  p.shrink = m.shrink;
  p.alpha0 = m.alpha0;
  return p;
}

template <int DR, int N>
struct Pow {
  static constexpr int K = DR == 1 ? N : (DR == 2 ? N * N : N * N * N);
};

// Lagrange values / first / second derivatives at r for all N GLL basis
// functions, prefix/suffix products (basis.py:138-198).  z, scale live in
// shared memory (warp-uniform reads broadcast).
template <int N, bool SECOND>
__device__ __forceinline__ void lagrange(const double* __restrict__ z,
                                         const double* __restrict__ scale, double r, double* v,
                                         double* g, double* h) {
  double u[N];
#pragma unroll
  for (int k = 0; k < N; ++k) u[k] = r - z[k];
  double pv[N + 1], pd[N + 1], ps[N + 1];
  double sv[N + 1], sd[N + 1], ss[N + 1];
  pv[0] = 1.0;
  pd[0] = 0.0;
  ps[0] = 0.0;
  sv[N] = 1.0;
  sd[N] = 0.0;
  ss[N] = 0.0;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    if (SECOND) ps[k + 1] = ps[k] * u[k] + 2.0 * pd[k];
    pd[k + 1] = pd[k] * u[k] + pv[k];
    pv[k + 1] = pv[k] * u[k];
  }
#pragma unroll
  for (int k = N - 1; k >= 0; --k) {
    if (SECOND) ss[k] = ss[k + 1] * u[k] + 2.0 * sd[k + 1];
    sd[k] = sd[k + 1] * u[k] + sv[k + 1];
    sv[k] = sv[k + 1] * u[k];
  }
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const double a = pv[i], b = sv[i + 1], da = pd[i], db = sd[i + 1];
    v[i] = (a * b) * scale[i];
    g[i] = (da * b + a * db) * scale[i];
    if (SECOND) h[i] = (ps[i] * b + 2.0 * da * db + a * ss[i + 1]) * scale[i];
  }
}

// Thread-local error helpers are in fpx_abi.cu.
