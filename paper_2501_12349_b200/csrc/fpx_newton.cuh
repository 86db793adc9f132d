// fpx_newton.cuh -- element-major FP64 trust-region Newton (findpts) and
// tensor-product evaluation (findpts_eval) for sm_100a.
//
// Scheduling: the (point, candidate-element) units of a
// find are grouped by element; one warp owns a work item = one element and
// up to 32 units.  The warp stages the element's nodal geometry (and, for the
// fused find+eval, its field block) into shared memory with cp.async, then
// every lane runs the full Newton solve of its own unit, reading the
// geometry by warp-uniform (broadcast) shared loads.  All FP64 work is done
// by all 32 lanes; the only inefficiency is divergence in iteration count.
//
// Arithmetic follows the oracle (oracle/fpx_oracle.c, fpxo_invert) operation
// by operation except that products and sums contract into FMAs; the seed
// distance uses explicit non-FMA intrinsics so the seed node is bit-identical.
#pragma once
#include <math.h>
#include <stdlib.h>

#include "fpx_common.cuh"
#include "fpx_kernels.cuh"
#include "fpx_boxes.cuh"

#ifndef FPX_KUNROLL
#define FPX_KUNROLL 1  // k-planes of the contraction per loop trip (ILP vs registers)
#endif

#ifndef FPX_NEWTON_MINB
#define FPX_NEWTON_MINB 2  // CTAs of 128 threads per SM the Newton kernels are built for
#endif

namespace fpx {

constexpr int kUnrollK = FPX_KUNROLL;

template <int D, int DR, int N>
struct Lay {
  static constexpr int K = Pow<DR, N>::K;
  static constexpr int NP = (N % 2 == 0) ? N : N + 1;  // rows padded to 16 B
  static constexpr int ROWS = K / N;
  static constexpr int CS = ROWS * NP;                 // doubles per component
  static constexpr int GEO = D * CS;
};

__device__ __forceinline__ void cp_async8(void* sdst, const void* gsrc) {
  unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

// Stage `comps` components of a lexicographic [comps][K] block into the
// padded shared layout [comps][ROWS][NP].
template <int DR, int N>
__device__ __forceinline__ void stage_block(double* sdst, const double* __restrict__ gsrc,
                                            int comps, int lane) {
  constexpr int K = Pow<DR, N>::K;
  constexpr int NP = (N % 2 == 0) ? N : N + 1;
  constexpr int CS = (K / N) * NP;
  const int total = comps * K;
  for (int t = lane; t < total; t += FPX_WARP) {
    const int c = t / K, q = t - c * K;
    const int row = q / N, i = q - row * N;
    cp_async8(sdst + c * CS + row * NP + i, gsrc + t);
  }
}

// Per-lane Newton state at one iterate: f = |dx|^2, J = -G^T dx,
// H0 = G^T G, Q = sum_c dx_c d2x_c (symmetric order 00,11,22,01,02,12).
struct NState {
  double f;
  double J[3];
  double H0[6];
  double Q[6];
};

// Per-lane basis scratch in shared memory: slot (axis-1, kind, j) of lane
// at sb[((axis-1)*3 + kind)*N + j)*32 + lane]; axes 1..DR-1 only (axis 0 is
// used in the innermost loop and stays in registers).
template <int DR, int N>
struct Scratch {
  static constexpr int SLOTS = (DR - 1) * 3 * N + 16;  // + 16: Newton state stash
  static constexpr int STASH = (DR - 1) * 3 * N;       // first stash slot
};

// Sum-factorised forward map x(r), G (+ second derivatives when W2), reduced
// on the fly into the Newton state (Eqs. 28-29).
template <int D, int DR, int N, bool W2, int LAY = 0>
__device__ __forceinline__ void eval_state(const double* __restrict__ sX,
                                           const double* __restrict__ z,
                                           const double* __restrict__ scale, const double* r,
                                           const double* xs, NState& S, double* sb) {
  // LAY 0: geometry staged in shared memory, rows padded to NP;
  // LAY 1: read in place from global memory ([d][N^dr]);
  // LAY 2: a per-lane shared slot holding [d][N^dr] unpadded.
  using Lp = Lay<D, DR, N>;
  // LAY 3: global memory, rows padded to NP (mesh.nodes_pad)
  constexpr bool GEO = LAY == 1;
  constexpr int GCS = (LAY == 1 || LAY == 2) ? Lp::K : Lp::CS;
  constexpr int GNP = (LAY == 1 || LAY == 2) ? N : Lp::NP;
  double v0[N], g0[N], h0[N];
  lagrange<N, W2>(z, scale, r[0], v0, g0, h0);
#pragma unroll
  for (int a = 1; a < DR; ++a) {
    double v[N], g[N], h[N];
    lagrange<N, W2>(z, scale, r[a], v, g, h);
#pragma unroll
    for (int j = 0; j < N; ++j) {
      sb[(((a - 1) * 3 + 0) * N + j) * FPX_WARP] = v[j];
      sb[(((a - 1) * 3 + 1) * N + j) * FPX_WARP] = g[j];
      if (W2) sb[(((a - 1) * 3 + 2) * N + j) * FPX_WARP] = h[j];
    }
  }
#define SB(a, kind, j) sb[((((a)-1) * 3 + (kind)) * N + (j)) * FPX_WARP]
  S.f = 0.0;
#pragma unroll
  for (int m = 0; m < 3; ++m) S.J[m] = 0.0;
#pragma unroll
  for (int m = 0; m < 6; ++m) {
    S.H0[m] = 0.0;
    S.Q[m] = 0.0;
  }
#pragma unroll 1
  for (int c = 0; c < D; ++c) {
    const double* Xc = sX + c * GCS;
    double xv = 0.0, G[3] = {0.0, 0.0, 0.0}, H2[6] = {0, 0, 0, 0, 0, 0};
    if constexpr (DR == 3) {
#pragma unroll kUnrollK
      for (int k = 0; k < N; ++k) {
        double t00 = 0.0, t10 = 0.0, t01 = 0.0, t20 = 0.0, t11 = 0.0, t02 = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) {
          const double* row = Xc + (j + N * k) * GNP;
          double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
          for (int i = 0; i < N; i += 2) {
            double2 p;
            if (GEO) p = make_double2(__ldg(row + i), i + 1 < N ? __ldg(row + i + 1) : 0.0);
            else if (LAY == 2) p = make_double2(row[i], i + 1 < N ? row[i + 1] : 0.0);
            else if (LAY == 3) p = __ldg(reinterpret_cast<const double2*>(row + i));
            else if (i + 1 < N) p = *reinterpret_cast<const double2*>(row + i);
            else p = make_double2(row[i], 0.0);
            s0 = fma(p.x, v0[i], s0);
            s1 = fma(p.x, g0[i], s1);
            if (W2) s2 = fma(p.x, h0[i], s2);
            if (i + 1 < N) {
              s0 = fma(p.y, v0[i + 1], s0);
              s1 = fma(p.y, g0[i + 1], s1);
              if (W2) s2 = fma(p.y, h0[i + 1], s2);
            }
          }
          const double vj = SB(1, 0, j), gj = SB(1, 1, j);
          t00 = fma(s0, vj, t00);
          t10 = fma(s1, vj, t10);
          t01 = fma(s0, gj, t01);
          if (W2) {
            const double hj = SB(1, 2, j);
            t20 = fma(s2, vj, t20);
            t11 = fma(s1, gj, t11);
            t02 = fma(s0, hj, t02);
          }
        }
        const double vk = SB(2, 0, k), gk = SB(2, 1, k);
        xv = fma(t00, vk, xv);
        G[0] = fma(t10, vk, G[0]);
        G[1] = fma(t01, vk, G[1]);
        G[2] = fma(t00, gk, G[2]);
        if (W2) {
          const double hk = SB(2, 2, k);
          H2[0] = fma(t20, vk, H2[0]);
          H2[1] = fma(t02, vk, H2[1]);
          H2[2] = fma(t00, hk, H2[2]);
          H2[3] = fma(t11, vk, H2[3]);
          H2[4] = fma(t10, gk, H2[4]);
          H2[5] = fma(t01, gk, H2[5]);
        }
      }
    } else if constexpr (DR == 2) {
#pragma unroll
      for (int j = 0; j < N; ++j) {
        const double* row = Xc + j * GNP;
        double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
        for (int i = 0; i < N; ++i) {
          const double p = row[i];
          s0 = fma(p, v0[i], s0);
          s1 = fma(p, g0[i], s1);
          if (W2) s2 = fma(p, h0[i], s2);
        }
        const double vj = SB(1, 0, j), gj = SB(1, 1, j);
        xv = fma(s0, vj, xv);
        G[0] = fma(s1, vj, G[0]);
        G[1] = fma(s0, gj, G[1]);
        if (W2) {
          const double hj = SB(1, 2, j);
          H2[0] = fma(s2, vj, H2[0]);
          H2[1] = fma(s0, hj, H2[1]);
          H2[3] = fma(s1, gj, H2[3]);
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const double p = Xc[i];
        xv = fma(p, v0[i], xv);
        G[0] = fma(p, g0[i], G[0]);
        if (W2) H2[0] = fma(p, h0[i], H2[0]);
      }
    }
#undef SB
    const double dx = (c == 0 ? xs[0] : (c == 1 ? xs[1] : xs[D - 1])) - xv;
    S.f = fma(dx, dx, S.f);
#pragma unroll
    for (int a = 0; a < DR; ++a) S.J[a] = fma(-G[a], dx, S.J[a]);
    S.H0[0] = fma(G[0], G[0], S.H0[0]);
    if (DR > 1) {
      S.H0[1] = fma(G[1], G[1], S.H0[1]);
      S.H0[3] = fma(G[0], G[1], S.H0[3]);
    }
    if (DR > 2) {
      S.H0[2] = fma(G[2], G[2], S.H0[2]);
      S.H0[4] = fma(G[0], G[2], S.H0[4]);
      S.H0[5] = fma(G[1], G[2], S.H0[5]);
    }
    if (W2) {
#pragma unroll
      for (int m = 0; m < 6; ++m) S.Q[m] = fma(dx, H2[m], S.Q[m]);
    }
  }
}

// eval_state with the second-derivative switch as a runtime (warp-uniform)
// flag: one copy of the contraction in the streamed kernels, whose lone
// warps at the end of a launch are bound by instruction fetch (the flag is
// set in ~90% of their evaluations, so the predicated-off FMAs are rare).
template <int D, int DR, int N, int LAY = 0, int W2C = -1>
__device__ __forceinline__ void eval_state_rt(const double* __restrict__ sX,
                                           const double* __restrict__ z,
                                           const double* __restrict__ scale, const double* r,
                                           const double* xs, NState& S, double* sb, const bool W2) {
  // W2C = 1 / 0: second derivatives accumulated / not (compile time; round
  // 1 picks the body per warp evaluation).  W2C = -1: accumulated always,
  // the runtime flag W2 gates only their use in S.Q (the rest kernel: nearly
  // all of its evaluations need them, and a select per FMA cost more)
  // LAY 0: geometry staged in shared memory, rows padded to NP;
  // LAY 1: read in place from global memory ([d][N^dr]);
  // LAY 2: a per-lane shared slot holding [d][N^dr] unpadded.
  using Lp = Lay<D, DR, N>;
  // LAY 3: global memory, rows padded to NP (mesh.nodes_pad)
  constexpr bool GEO = LAY == 1;
  constexpr int GCS = (LAY == 1 || LAY == 2) ? Lp::K : Lp::CS;
  constexpr int GNP = (LAY == 1 || LAY == 2) ? N : Lp::NP;
  double v0[N], g0[N], h0[N];
  lagrange<N, W2C != 0>(z, scale, r[0], v0, g0, h0);
  // axes 1..dr-1 to the scratch: one rolled copy of the basis recursion
  // (instruction footprint of the hot loop; r[a] by selects, not indexing)
#pragma unroll 1
  for (int a = 1; a < DR; ++a) {
    double v[N], g[N], h[N];
    lagrange<N, W2C != 0>(z, scale, a == 1 ? r[1] : r[DR - 1], v, g, h);
    double* sa = sb + (a - 1) * 3 * N * FPX_WARP;
#pragma unroll
    for (int j = 0; j < N; ++j) {
      sa[(0 * N + j) * FPX_WARP] = v[j];
      sa[(1 * N + j) * FPX_WARP] = g[j];
      if (W2C != 0) sa[(2 * N + j) * FPX_WARP] = h[j];
    }
  }
#define SB(a, kind, j) sb[((((a)-1) * 3 + (kind)) * N + (j)) * FPX_WARP]
  S.f = 0.0;
#pragma unroll
  for (int m = 0; m < 3; ++m) S.J[m] = 0.0;
#pragma unroll
  for (int m = 0; m < 6; ++m) {
    S.H0[m] = 0.0;
    S.Q[m] = 0.0;
  }
#pragma unroll 1
  for (int c = 0; c < D; ++c) {
    const double* Xc = sX + c * GCS;
    double xv = 0.0, G[3] = {0.0, 0.0, 0.0}, H2[6] = {0, 0, 0, 0, 0, 0};
    if constexpr (DR == 3) {
#pragma unroll kUnrollK
      for (int k = 0; k < N; ++k) {
        double t00 = 0.0, t10 = 0.0, t01 = 0.0, t20 = 0.0, t11 = 0.0, t02 = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) {
          const double* row = Xc + (j + N * k) * GNP;
          double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
          for (int i = 0; i < N; i += 2) {
            double2 p;
            if (GEO) p = make_double2(__ldg(row + i), i + 1 < N ? __ldg(row + i + 1) : 0.0);
            else if (LAY == 2) p = make_double2(row[i], i + 1 < N ? row[i + 1] : 0.0);
            else if (LAY == 3) p = __ldg(reinterpret_cast<const double2*>(row + i));
            else if (i + 1 < N) p = *reinterpret_cast<const double2*>(row + i);
            else p = make_double2(row[i], 0.0);
            s0 = fma(p.x, v0[i], s0);
            s1 = fma(p.x, g0[i], s1);
            if (W2C != 0) s2 = fma(p.x, h0[i], s2);
            if (i + 1 < N) {
              s0 = fma(p.y, v0[i + 1], s0);
              s1 = fma(p.y, g0[i + 1], s1);
              if (W2C != 0) s2 = fma(p.y, h0[i + 1], s2);
            }
          }
          const double vj = SB(1, 0, j), gj = SB(1, 1, j);
          t00 = fma(s0, vj, t00);
          t10 = fma(s1, vj, t10);
          t01 = fma(s0, gj, t01);
          if (W2C != 0) {
            const double hj = SB(1, 2, j);
            t20 = fma(s2, vj, t20);
            t11 = fma(s1, gj, t11);
            t02 = fma(s0, hj, t02);
          }
        }
        const double vk = SB(2, 0, k), gk = SB(2, 1, k);
        xv = fma(t00, vk, xv);
        G[0] = fma(t10, vk, G[0]);
        G[1] = fma(t01, vk, G[1]);
        G[2] = fma(t00, gk, G[2]);
        if (W2C != 0) {
          const double hk = SB(2, 2, k);
          H2[0] = fma(t20, vk, H2[0]);
          H2[1] = fma(t02, vk, H2[1]);
          H2[2] = fma(t00, hk, H2[2]);
          H2[3] = fma(t11, vk, H2[3]);
          H2[4] = fma(t10, gk, H2[4]);
          H2[5] = fma(t01, gk, H2[5]);
        }
      }
    } else if constexpr (DR == 2) {
#pragma unroll
      for (int j = 0; j < N; ++j) {
        const double* row = Xc + j * GNP;
        double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
        for (int i = 0; i < N; ++i) {
          const double p = row[i];
          s0 = fma(p, v0[i], s0);
          s1 = fma(p, g0[i], s1);
          if (W2C != 0) s2 = fma(p, h0[i], s2);
        }
        const double vj = SB(1, 0, j), gj = SB(1, 1, j);
        xv = fma(s0, vj, xv);
        G[0] = fma(s1, vj, G[0]);
        G[1] = fma(s0, gj, G[1]);
        if (W2C != 0) {
          const double hj = SB(1, 2, j);
          H2[0] = fma(s2, vj, H2[0]);
          H2[1] = fma(s0, hj, H2[1]);
          H2[3] = fma(s1, gj, H2[3]);
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const double p = Xc[i];
        xv = fma(p, v0[i], xv);
        G[0] = fma(p, g0[i], G[0]);
        if (W2C != 0) H2[0] = fma(p, h0[i], H2[0]);
      }
    }
#undef SB
    const double dx = (c == 0 ? xs[0] : (c == 1 ? xs[1] : xs[D - 1])) - xv;
    S.f = fma(dx, dx, S.f);
#pragma unroll
    for (int a = 0; a < DR; ++a) S.J[a] = fma(-G[a], dx, S.J[a]);
    S.H0[0] = fma(G[0], G[0], S.H0[0]);
    if (DR > 1) {
      S.H0[1] = fma(G[1], G[1], S.H0[1]);
      S.H0[3] = fma(G[0], G[1], S.H0[3]);
    }
    if (DR > 2) {
      S.H0[2] = fma(G[2], G[2], S.H0[2]);
      S.H0[4] = fma(G[0], G[2], S.H0[4]);
      S.H0[5] = fma(G[1], G[2], S.H0[5]);
    }
    if (W2C == 1 || (W2C < 0 && W2)) {
#pragma unroll
      for (int m = 0; m < 6; ++m) S.Q[m] = fma(dx, H2[m], S.Q[m]);
    }
  }
}

__device__ __forceinline__ int symi(int a, int b) {
  return a == b ? a : (a + b == 1 ? 3 : (a + b == 2 ? 4 : 5));
}

// Cholesky solve on the active principal submatrix (oracle chol_solve):
// pivot must exceed 1e-14 |trace|.  A is symmetric-packed.
template <int DR>
__device__ __forceinline__ bool chol_solve(const double* A, const bool* act, const double* b,
                                           double* x) {
  // The active principal submatrix as the block-diagonal matrix with the
  // held axes' rows and columns replaced by the identity (and zero right-
  // hand side): the unconditional factorisation then computes exactly the
  // masked one's values on the active axes (the identity block contributes
  // exact zeros) and x = 0 on the held axes, without per-entry branches.
  double Ap[6], bp[3], L[3][3], y[3], iL[3];
  double tr = 0.0;
#pragma unroll
  for (int k = 0; k < DR; ++k) {
    if (act[k]) tr += A[k];
    Ap[k] = act[k] ? A[k] : 1.0;
    bp[k] = act[k] ? b[k] : 0.0;
  }
#pragma unroll
  for (int i = 1; i < DR; ++i)
#pragma unroll
    for (int k = 0; k < i; ++k) Ap[symi(i, k)] = act[i] && act[k] ? A[symi(i, k)] : 0.0;
  const double thr = 1e-14 * fabs(tr);
#pragma unroll
  for (int k = 0; k < DR; ++k) {
    double s = Ap[k];
#pragma unroll
    for (int m = 0; m < k; ++m) s -= L[k][m] * L[k][m];
    if (act[k] && !(s > thr)) return false;
    // 1/L[k][k] (L[k][k] itself is never used): one rsqrt instead of a
    // sqrt and a division (round 1 654 -> 635 us); within 1 ulp of the
    // oracle's 1/sqrt
    iL[k] = rsqrt(s);
#pragma unroll
    for (int i = k + 1; i < DR; ++i) {
      double t = Ap[symi(i, k)];
#pragma unroll
      for (int m = 0; m < k; ++m) t -= L[i][m] * L[k][m];
      L[i][k] = t * iL[k];
    }
  }
#pragma unroll
  for (int k = 0; k < DR; ++k) {
    double t = bp[k];
#pragma unroll
    for (int m = 0; m < k; ++m) t -= L[k][m] * y[m];
    y[k] = t * iL[k];
  }
#pragma unroll
  for (int k = DR - 1; k >= 0; --k) {
    double t = y[k];
#pragma unroll
    for (int m = k + 1; m < DR; ++m) t -= L[m][k] * x[m];
    x[k] = t * iL[k];
  }
  return true;
}

// Projected trust-region Newton step (oracle constrained_step, decision D8):
// the Newton direction on the free axes (free axes on a face that the
// direction would leave become active, re-solve), truncated at the trust
// radius and at the first face it reaches.  `hit` marks the axes whose face
// limits the step.  Returns false if the free block is not positive definite.
template <int DR>
__device__ __forceinline__ bool constrained_step(const double* Hm, const double* J,
                                                 const double* r, bool* freem, double alpha,
                                                 double* s, int& hit) {
  double x[3] = {0.0, 0.0, 0.0};
  hit = 0;
#pragma unroll
  for (int a = 0; a < DR; ++a) s[a] = 0.0;
#pragma unroll 1
  for (int pass = 0; pass <= DR; ++pass) {
    int nf = 0;
#pragma unroll
    for (int a = 0; a < DR; ++a) nf += freem[a] ? 1 : 0;
    if (nf == 0) return true;
    double rhs[3], y[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int a = 0; a < DR; ++a) rhs[a] = -J[a];
    if (!chol_solve<DR>(Hm, freem, rhs, y)) return false;
    bool blocked = false;
#pragma unroll
    for (int a = 0; a < DR; ++a) {
      x[a] = freem[a] ? y[a] : 0.0;
      // on a face with the direction leaving it: |r| = 1 and r y > 0 (exact)
      if (freem[a] && fabs(r[a]) == 1.0 && r[a] * y[a] > 0.0) {
        freem[a] = false;
        blocked = true;
      }
    }
    if (!blocked) break;
    if (pass == DR) return true;
  }
  double m = 0.0;
#pragma unroll
  for (int a = 0; a < DR; ++a)
    if (freem[a]) m = fabs(x[a]) > m ? fabs(x[a]) : m;
  if (m == 0.0) return true;
  double t = m > alpha ? alpha / m : 1.0;
  double ta[3] = {INFINITY, INFINITY, INFINITY};
#pragma unroll
  for (int a = 0; a < DR; ++a) {
    if (!freem[a] || x[a] == 0.0) continue;
    ta[a] = x[a] > 0.0 ? (1.0 - r[a]) / x[a] : (-1.0 - r[a]) / x[a];
    t = ta[a] < t ? ta[a] : t;
  }
#pragma unroll
  for (int a = 0; a < DR; ++a) {
    if (!freem[a]) continue;
    s[a] = t * x[a];
    if (ta[a] == t) hit |= 1 << a;
  }
  return true;
}

// |x*|_inf: the scale of the rounding noise in dx = x* - x(r) (D8)
template <int D>
__device__ __forceinline__ double xscale(const double* xs) {
  double m = fabs(xs[0]);
#pragma unroll
  for (int c = 1; c < D; ++c) m = fmax(m, fabs(xs[c]));
  return m;
}

// D7' seed of a volume element: r0 = clamp(J_c^-1 (x* - x_c)) from its centre
// frame fr = (x_c[D], J_c^-1[D][D]) (zero matrix when the frame is unusable),
// with separate multiply and add in the oracle's order (candidate_solve).
template <int D>
__device__ __forceinline__ void affine_seed(const double* fr, const double* xs, double* r0) {
  double dx[3];
#pragma unroll
  for (int c = 0; c < D; ++c) dx[c] = __dsub_rn(xs[c], fr[c]);
#pragma unroll
  for (int a = 0; a < D; ++a) {
    double y = 0.0;
#pragma unroll
    for (int b = 0; b < D; ++b) y = __dadd_rn(y, __dmul_rn(fr[D + a * D + b], dx[b]));
    r0[a] = fabs(y) < INFINITY ? fmin(1.0, fmax(-1.0, y)) : 0.0;  // inf / NaN -> 0
  }
}

template <int DR>
__device__ __forceinline__ bool on_boundary(const double* r) {
  bool b = false;
#pragma unroll
  for (int a = 0; a < DR; ++a) b |= fabs(r[a]) == 1.0;
  return b;
}

struct NewtonOut {
  double r[3];
  double dist;
  int iters;
  bool conv;
};

__device__ __forceinline__ void stash_state(double* sb, const NState& S) {
#pragma unroll
  for (int m = 0; m < 3; ++m) sb[m * FPX_WARP] = S.J[m];
#pragma unroll
  for (int m = 0; m < 6; ++m) {
    sb[(3 + m) * FPX_WARP] = S.H0[m];
    sb[(9 + m) * FPX_WARP] = S.Q[m];
  }
}
__device__ __forceinline__ void unstash_state(const double* sb, NState& S) {
#pragma unroll
  for (int m = 0; m < 3; ++m) S.J[m] = sb[m * FPX_WARP];
#pragma unroll
  for (int m = 0; m < 6; ++m) {
    S.H0[m] = sb[(3 + m) * FPX_WARP];
    S.Q[m] = sb[(9 + m) * FPX_WARP];
  }
}

// invert_point for every active lane of the warp (SPEC.md:298-307,
// PAPER.md:414-451, decision D8).  Inactive lanes follow along (warp-uniform
// evaluation) but do not update.  One Newton state lives in registers: the
// predicted decrease is formed before the trial evaluation, the current
// state is stashed in the lane's shared scratch and restored only when the
// step is rejected.  sb: this lane's scratch (stride 32 doubles).
template <int D, int DR, int N, int LAY = 0>
__device__ __forceinline__ NewtonOut newton_warp(const double* __restrict__ sX,
                                                 const double* __restrict__ z,
                                                 const double* __restrict__ scale,
                                                 const double* xs, bool active,
                                                 const NewtonParams& P, double* sb,
                                                 int64_t* nev = nullptr,
                                                 const double* r0 = nullptr) {
  using L = Lay<D, DR, N>;
  double* stash = sb + Scratch<DR, N>::STASH * FPX_WARP;
  // seed: nearest GLL node, ties -> lowest lexicographic index (D7); the
  // distance is accumulated with fma exactly as the oracle does.  An
  // explicit initial guess r0 (invert_point's r0; warp-uniform
  // presence) replaces it, clamped to [-1, 1].
  double best = INFINITY;
  int bi = 0;
#pragma unroll 1
  for (int row = 0; row < (r0 ? 0 : L::ROWS); ++row) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double dd = 0.0;
#pragma unroll
      for (int c = 0; c < D; ++c) {
        const double xn = LAY == 1   ? __ldg(sX + c * L::K + row * N + i)
                          : LAY == 2 ? sX[c * L::K + row * N + i]
                                     : sX[c * L::CS + row * L::NP + i];
        const double t = __dsub_rn(xs[c], xn);
        dd = __fma_rn(t, t, dd);
      }
      if (dd < best) {
        best = dd;
        bi = row * N + i;
      }
    }
  }
  double r[3] = {0.0, 0.0, 0.0};
  r[0] = z[bi % N];
  if (DR > 1) r[1] = z[(bi / N) % N];
  if (DR > 2) r[2] = z[bi / (N * N)];
  if (r0)
#pragma unroll
    for (int a = 0; a < DR; ++a) r[a] = fmin(1.0, fmax(-1.0, r0[a]));
  // One evaluation site (the seed is evaluated as the first "trial") and one
  // constrained_step site (the Hessian fallbacks loop over it) keep the
  // kernel's code small: instruction fetch was the top stall when inlined.
  NState st;
  double rn[3] = {r[0], r[1], r[2]};
  double alpha = P.alpha0, fcur = 0.0, pred = 0.0, smax = 0.0;
  const double xsc = xscale<D>(xs);
  int it = 0;
  bool done = !active, conv = false, first = true, step = active;
  while (true) {
    const bool w2 = __any_sync(FPX_FULL, step && on_boundary<DR>(rn));
    if (nev) {
      nev[0] += 1;
      nev[1] += w2 ? 1 : 0;
    }
    if (w2)
      eval_state<D, DR, N, true, LAY>(sX, z, scale, rn, xs, st, sb);
    else
      eval_state<D, DR, N, false, LAY>(sX, z, scale, rn, xs, st, sb);
    // lanes not stepping evaluated at rn == r: their state is recomputed
    // bit-identically (eval_state is a pure function of r)
    if (first) {
      first = false;
    } else if (step) {
      const double decr = fcur - st.f;
      if (decr >= P.accept * pred) {
        if (decr >= P.keep * pred) alpha *= P.grow;
#pragma unroll
        for (int a = 0; a < DR; ++a) r[a] = rn[a];
      } else {
        alpha *= P.shrink;
        unstash_state(stash, st);
        st.f = fcur;
      }
      if (smax < P.tol) {
        conv = true;
        done = true;
      } else if (it >= P.max_iters) {
        done = true;
      }
    }
    step = false;
#pragma unroll
    for (int a = 0; a < 3; ++a) rn[a] = r[a];
    if (!__any_sync(FPX_FULL, !done)) break;
    if (!done) {
      fcur = st.f;
      const bool beta = it > 0 && on_boundary<DR>(r);
      bool freem[3] = {true, true, true};
#pragma unroll
      for (int a = 0; a < DR; ++a)
        if (fabs(r[a]) == 1.0 && r[a] * st.J[a] < 0.0) freem[a] = false;  // descent leaves the face
      double Hm[6], s[3] = {0.0, 0.0, 0.0};
      int hit = 0;
      bool ok = false;
      // model Hessians in order: beta=1 (faces), Gauss-Newton, regularised
#pragma unroll 1
      for (int att = beta ? 0 : 1; att < 3 && !ok; ++att) {
        double lam = 0.0;
        if (att == 2) {
          double tr = 0.0;
#pragma unroll
          for (int a = 0; a < DR; ++a) tr += st.H0[a];
          lam = 1e-10 * tr / DR;
          if (!(lam > 0.0)) lam = 1e-300;
        }
#pragma unroll
        for (int m = 0; m < 6; ++m)
          Hm[m] = att == 0 ? st.H0[m] - st.Q[m] : st.H0[m] + (m < DR ? lam : 0.0);
        bool fr[3] = {freem[0], freem[1], freem[2]};
        ok = constrained_step<DR>(Hm, st.J, r, fr, alpha, s, hit);
      }
      if (!ok) {
        hit = 0;
#pragma unroll
        for (int a = 0; a < DR; ++a) s[a] = 0.0;
      }
      ++it;
      double js = 0.0, shs = 0.0;
      smax = 0.0;
#pragma unroll
      for (int a = 0; a < DR; ++a) {
        js += st.J[a] * s[a];
        double t = 0.0;
#pragma unroll
        for (int b = 0; b < DR; ++b) t += Hm[symi(a, b)] * s[b];
        shs += s[a] * t;
        smax = fabs(s[a]) > smax ? fabs(s[a]) : smax;
      }
      pred = -(2.0 * js + shs);
#pragma unroll
      for (int a = 0; a < DR; ++a) {
        double v = r[a] + s[a];
        if (hit & (1 << a)) v = s[a] > 0.0 ? 1.0 : -1.0;  // lands on the face
        v = v < -1.0 ? -1.0 : (v > 1.0 ? 1.0 : v);
        rn[a] = v;
      }
      // D8 resolvability: below the rounding floor of |dx|^2 the step is
      // taken on the model's word (pred = -inf); such a step below tol is
      // the last one, applied without a trial evaluation (oracle fpxo_invert)
      const bool unres = !(pred > FPX_UNRES_REL * fcur + FPX_UNRES_ABS * sqrt(fcur) * xsc);
      if (unres) pred = -INFINITY;
      if (unres && smax < P.tol) {
        conv = true;
        done = true;
#pragma unroll
        for (int a = 0; a < DR; ++a) r[a] = rn[a];
      } else {
        step = true;
        stash_state(stash, st);
      }
    }
    if (!__any_sync(FPX_FULL, step)) break;
  }
  NewtonOut o;
  o.r[0] = r[0];
  o.r[1] = r[1];
  o.r[2] = r[2];
  o.dist = sqrt(st.f);
  o.iters = it;
  o.conv = conv;
  return o;
}

// classify (surfaces SPEC.md:329).
template <int D, int DR>
__device__ __forceinline__ int classify(const double* r, double dist, double eps_d) {
  bool in = true;
#pragma unroll
  for (int a = 0; a < DR; ++a) in &= fabs(r[a]) < 1.0 - FPX_INTERIOR_TOL;
  if (DR < D) in &= dist < eps_d;
  return in ? kInterior : kBorder;
}

__device__ __forceinline__ double eps_d_of(const fpx_mesh_t& m, int e) {
  if (m.eps_d_abs >= 0.0) return m.eps_d_abs;
  const double* bx = m.aabb + (int64_t)e * 2 * m.d;
  double s = 0.0;
  for (int c = 0; c < m.d; ++c) s += (bx[m.d + c] - bx[c]) * (bx[m.d + c] - bx[c]);
  return m.eps_d_rel * sqrt(s);
}

// Field value at r from a staged block in shared memory (eval_tensor_product
// order: axis 0 first).
template <int DR, int N>
__device__ __forceinline__ double contract_smem(const double* __restrict__ sU,
                                                const double (*v)[N]) {
  constexpr int NP = (N % 2 == 0) ? N : N + 1;
  if constexpr (DR == 3) {
    double q = 0.0;
#pragma unroll
    for (int k = 0; k < N; ++k) {
      double t = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) {
        const double* row = sU + (j + N * k) * NP;  // 16-byte aligned, NP even
        double s = 0.0, s1 = 0.0;
#pragma unroll
        for (int i = 0; i + 1 < N; i += 2) {
          const double2 p = *reinterpret_cast<const double2*>(row + i);
          s = fma(p.x, v[0][i], s);
          s1 = fma(p.y, v[0][i + 1], s1);
        }
        if (N % 2) s = fma(row[N - 1], v[0][N - 1], s);
        t = fma(s + s1, v[1][j], t);
      }
      q = fma(t, v[2][k], q);
    }
    return q;
  } else if constexpr (DR == 2) {
    double t = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) {
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) s = fma(sU[j * NP + i], v[0][i], s);
      t = fma(s, v[1][j], t);
    }
    return t;
  } else {
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) s = fma(sU[i], v[0][i], s);
    return s;
  }
}

// Field value at r from a lexicographic unpadded block [K] (a slot's staged
// field in shared memory, or global memory): generic loads.
template <int DR, int N>
__device__ __forceinline__ double contract_flat(const double* __restrict__ U,
                                               const double (*v)[N]) {
  if constexpr (DR == 3) {
    double q = 0.0;
#pragma unroll
    for (int k = 0; k < N; ++k) {
      double t = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) {
        const double* row = U + N * (j + N * k);
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int i = 0; i < N; i += 2) {
          s0 = fma(row[i], v[0][i], s0);
          if (i + 1 < N) s1 = fma(row[i + 1], v[0][i + 1], s1);
        }
        t = fma(s0 + s1, v[1][j], t);
      }
      q = fma(t, v[2][k], q);
    }
    return q;
  } else if constexpr (DR == 2) {
    double t = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) {
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int i = 0; i < N; i += 2) {
        s0 = fma(U[j * N + i], v[0][i], s0);
        if (i + 1 < N) s1 = fma(U[j * N + i + 1], v[0][i + 1], s1);
      }
      t = fma(s0 + s1, v[1][j], t);
    }
    return t;
  } else {
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) s = fma(U[i], v[0][i], s);
    return s;
  }
}

// contract_flat for d_r = 3 with the outer (k) loop rolled: the axis-2
// weights are read from the lane's shared scratch `w` (stride 32 doubles).
// Runs once per located point inside the round-1 loop, whose instruction
// footprint matters (the unrolled form is ~300 instructions at N = 5).
template <int N>
__device__ __forceinline__ double contract_flat_k(const double* __restrict__ U,
                                                  const double* v0, const double* v1,
                                                  const double* w) {
  double q = 0.0;
#pragma unroll 1
  for (int k = 0; k < N; ++k) {
    double t = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) {
      const double* row = U + N * (j + N * k);
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int i = 0; i < N; i += 2) {
        s0 = fma(row[i], v0[i], s0);
        if (i + 1 < N) s1 = fma(row[i + 1], v0[i + 1], s1);
      }
      t = fma(s0 + s1, v1[j], t);
    }
    q = fma(t, w[k * FPX_WARP], q);
  }
  return q;
}

// Same contraction from global memory (lexicographic, unpadded).
template <int DR, int N>
__device__ __forceinline__ double contract_gmem(const double* __restrict__ U,
                                                const double (*v)[N]) {
  if constexpr (DR == 3) {
    double q = 0.0;
#pragma unroll
    for (int k = 0; k < N; ++k) {
      double t = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) {
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < N; ++i) s = fma(__ldg(U + i + N * (j + N * k)), v[0][i], s);
        t = fma(s, v[1][j], t);
      }
      q = fma(t, v[2][k], q);
    }
    return q;
  } else if constexpr (DR == 2) {
    double t = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) {
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) s = fma(__ldg(U + i + N * j), v[0][i], s);
      t = fma(s, v[1][j], t);
    }
    return t;
  } else {
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) s = fma(__ldg(U + i), v[0][i], s);
    return s;
  }
}

template <int DR, int N>
__device__ __forceinline__ void basis_values(const double* z, const double* scale,
                                             const double* r, double (*v)[N]) {
  double g[N], h[N];
#pragma unroll
  for (int a = 0; a < DR; ++a) lagrange<N, false>(z, scale, r[a], v[a], g, h);
}

__device__ __forceinline__ int64_t warp_sum64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FPX_FULL, v, o);
  return v;
}

// Round 2 (and fpx_invert_pairs): Newton per explicit (point, element) pair.
template <int D, int DR, int N>
__global__ void __launch_bounds__(128, FPX_NEWTON_MINB)
    k_newton_pairs(fpx_mesh_t m, const double* __restrict__ x, const int32_t* __restrict__ pair_pt,
                   const int32_t* __restrict__ sorted, const Item* __restrict__ items,
                   const int64_t* __restrict__ nitems_dev, const double* __restrict__ r0,
                   int32_t* pcode, double* pr, double* pdist, int32_t* piters, int32_t* pconv,
                   int64_t* stats) {
  using L = Lay<D, DR, N>;
  extern __shared__ __align__(16) double smem[];
  double* z = smem;
  double* scale = smem + N;
  const int warp = threadIdx.x / FPX_WARP, lane = threadIdx.x % FPX_WARP;
  const int wpb = blockDim.x / FPX_WARP;
  constexpr int SCR = Scratch<DR, N>::SLOTS * FPX_WARP;
  double* sX = smem + 2 * ((N + 1) & ~1) + warp * (L::GEO + SCR);
  double* sb = sX + L::GEO + lane;
  if (threadIdx.x < N) {
    z[threadIdx.x] = m.basis[FPX_BASIS_NODES(N, m.M) + threadIdx.x];
    scale[threadIdx.x] = m.basis[FPX_BASIS_SCALE(N, m.M) + threadIdx.x];
  }
  __syncthreads();
  const NewtonParams P = newton_of(m);
  const int64_t nitems = *nitems_dev;
  int64_t s_newton = 0, s_iters = 0;
  for (int64_t w = (int64_t)blockIdx.x * wpb + warp; w < nitems; w += (int64_t)gridDim.x * wpb) {
    const Item itm = items[w];
    const int e = itm.elem;
    stage_block<DR, N>(sX, m.nodes + (int64_t)e * D * L::K, D, lane);
    cp_async_wait_all();
    __syncwarp();
    const bool active = lane < itm.count;
    const int pair = active ? sorted[itm.start + lane] : 0;
    const int pt = active ? (pair_pt ? pair_pt[pair] : pair) : 0;
    double xs[3] = {0.0, 0.0, 0.0}, rs[3] = {0.0, 0.0, 0.0};
    if (active) {
#pragma unroll
      for (int c = 0; c < D; ++c) xs[c] = x[(int64_t)pt * D + c];
      if (r0)
#pragma unroll
        for (int a = 0; a < DR; ++a) rs[a] = r0[(int64_t)pair * DR + a];
    }
    NewtonOut o = newton_warp<D, DR, N>(sX, z, scale, xs, active, P, sb, nullptr,
                                        r0 ? rs : nullptr);
    if (active) {
      s_newton += 1;
      s_iters += o.iters;
      const double epsd = DR < D ? eps_d_of(m, e) : 0.0;
      if (pcode) pcode[pair] = classify<D, DR>(o.r, o.dist, epsd);
#pragma unroll
      for (int a = 0; a < DR; ++a) pr[(int64_t)pair * DR + a] = o.r[a];
      pdist[pair] = o.dist;
      if (piters) piters[pair] = o.iters;
      if (pconv) pconv[pair] = o.conv ? 1 : 0;
    }
    __syncwarp();
  }
  if (stats) {
    s_newton = warp_sum64(s_newton);
    s_iters = warp_sum64(s_iters);
    if (lane == 0) {
      atomicAdd((unsigned long long*)&stats[FPX_STAT_NEWTON], (unsigned long long)s_newton);
      atomicAdd((unsigned long long*)&stats[FPX_STAT_ITERS], (unsigned long long)s_iters);
    }
  }
}

// The projected trust-region step from state st at r (D8; the same
// arithmetic as newton_warp): the trial point rn.  Returns false when the
// solve has converged (an unresolvable step below tol): rn is then the final
// iterate, taken without evaluation.
template <int DR>
__device__ __forceinline__ bool propose_step(const NState& st, const double* r, int it,
                                             double alpha, double xsc, double tol,
                                             double* rn, double& pred, double& smax) {
  const double fcur = st.f;
  const bool beta = it > 0 && on_boundary<DR>(r);
  bool freem[3] = {true, true, true};
#pragma unroll
  for (int a = 0; a < DR; ++a)
    if (fabs(r[a]) == 1.0 && r[a] * st.J[a] < 0.0) freem[a] = false;  // descent leaves the face
  double Hm[6], s[3] = {0.0, 0.0, 0.0};
  int hit = 0;
  bool ok = false;
#pragma unroll 1
  for (int att = beta ? 0 : 1; att < 3 && !ok; ++att) {
    double lam = 0.0;
    if (att == 2) {
      double tr = 0.0;
#pragma unroll
      for (int a = 0; a < DR; ++a) tr += st.H0[a];
      lam = 1e-10 * tr / DR;
      if (!(lam > 0.0)) lam = 1e-300;
    }
#pragma unroll
    for (int m = 0; m < 6; ++m)
      Hm[m] = att == 0 ? st.H0[m] - st.Q[m] : st.H0[m] + (m < DR ? lam : 0.0);
    bool fr[3] = {freem[0], freem[1], freem[2]};
    ok = constrained_step<DR>(Hm, st.J, r, fr, alpha, s, hit);
  }
  if (!ok) {
    hit = 0;
#pragma unroll
    for (int a = 0; a < DR; ++a) s[a] = 0.0;
  }
  double js = 0.0, shs = 0.0;
  smax = 0.0;
#pragma unroll
  for (int a = 0; a < DR; ++a) {
    js += st.J[a] * s[a];
    double t = 0.0;
#pragma unroll
    for (int b = 0; b < DR; ++b) t += Hm[symi(a, b)] * s[b];
    shs += s[a] * t;
    smax = fabs(s[a]) > smax ? fabs(s[a]) : smax;
  }
  pred = -(2.0 * js + shs);
#pragma unroll
  for (int a = 0; a < DR; ++a) {
    double v = r[a] + s[a];
    if (hit & (1 << a)) v = s[a] > 0.0 ? 1.0 : -1.0;  // lands on the face
    v = v < -1.0 ? -1.0 : (v > 1.0 ? 1.0 : v);
    rn[a] = v;
  }
  // D8 resolvability (newton_warp): below the floor the step is accepted
  // unchecked (pred = -inf); such a step below tol is the last one, applied
  // by the caller without a trial evaluation
  if (!(pred > FPX_UNRES_REL * fcur + FPX_UNRES_ABS * sqrt(fcur) * xsc)) {
    if (smax < tol) return false;
    pred = -INFINITY;
  }
  return true;
}

// ---------------------------------------------------------------- rest kernel
// Points left unresolved by round 1 (~5%: their best-first candidate ended
// BORDER or was stopped by rule R2) visit their remaining candidates in
// best-first order, stop at the first INTERIOR and otherwise keep the D6
// winner.  These (point, candidate) pairs hit ~1 pair per element, so the
// element-major mapping of round 1 would run warps with one live lane:
// k_rest_l1 gives every lane one pair and reads that element's geometry in
// place through L1 (mesh.nodes_pad).  Pass 1 solves from the affine seed
// (D7', rule R2); a BORDER or aborted result goes to the redo list, whose
// pairs the second launch solves from the nearest-node seed (D7, the
// warp-cooperative node search) only if their point found no INTERIOR.

__device__ __forceinline__ void mbar_init(uint64_t* mb, unsigned count) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(mb);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* mb) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(mb);
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(a) : "memory");
}
// One elected lane: expect `bytes` on the slot's mbarrier (its single
// arrival), then 1D TMA bulk copies global -> shared that complete_tx on it.
// The proxy fence orders the lanes' earlier generic reads of the slot before
// the async-proxy refill.
__device__ __forceinline__ void mbar_expect_tx(uint64_t* mb, unsigned bytes) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(mb);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(a), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, unsigned bytes,
                                         uint64_t* mb) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(sdst);
  const unsigned b = (unsigned)__cvta_generic_to_shared(mb);
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(d),
      "l"(gsrc), "r"(bytes), "r"(b)
      : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t* mb, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(mb);
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(a), "r"(parity)
      : "memory");
  return ok != 0;
}

// Warp argmin of (d, i) over all lanes, d >= 0 (a distance; +inf allowed):
// non-negative doubles order like their bit patterns, so three redux.sync
// minima suffice -- the high word, the low word among the high-word winners,
// the index among the exact ties.  Every lane gets the winning index.
__device__ __forceinline__ int warp_argmin(double d, int i) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(d);
  const unsigned hi = (unsigned)(b >> 32), lo = (unsigned)b;
  const bool c1 = hi == __reduce_min_sync(FPX_FULL, hi);
  const unsigned ml = __reduce_min_sync(FPX_FULL, c1 ? lo : 0xffffffffu);
  const bool c2 = c1 && lo == ml;
  return (int)__reduce_min_sync(FPX_FULL, c2 ? (unsigned)i : 0xffffffffu);
}

// Warp minimum of a non-negative double (bit patterns order like the values).
__device__ __forceinline__ double warp_min_nonneg(double d) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(d);
  const unsigned hi = __reduce_min_sync(FPX_FULL, (unsigned)(b >> 32));
  const unsigned lo =
      __reduce_min_sync(FPX_FULL, (unsigned)(b >> 32) == hi ? (unsigned)b : 0xffffffffu);
  return __longlong_as_double((long long)(((unsigned long long)hi << 32) | lo));
}

// Best-first ranked candidate lists of the rest points: the passing
// entries of the hash list sorted by (v, e), FPX_RK per point
// kept; beyond that the rest kernel scans the list itself.
#define FPX_LISTMAX 128
constexpr int kRlLanes = 16;                   // lanes per rest point (lists hold ~9 entries)
constexpr int kRlGroups = 128 / kRlLanes;      // points per 128-thread block at a time
template <int D>
__global__ void __launch_bounds__(128)
    k_rest_lists(fpx_mesh_t m, const double* __restrict__ x, const int64_t* __restrict__ nun_dev,
                 const int32_t* __restrict__ upts, int32_t* best, const int32_t* __restrict__ npass,
                 int32_t* clist, int32_t* cnum, int32_t* nps, int32_t* hist) {
  // kRlLanes lanes per rest point: they test the hash-list entries (one
  // float row each), (v, e) of the passing ones go to shared memory, and the
  // rank of each is the number of passing entries before it in (v, e) order
  // (v: rest_rank_value, fpx_boxes.cuh)
  __shared__ double s_v[kRlGroups][FPX_LISTMAX];
  __shared__ int s_e[kRlGroups][FPX_LISTMAX];
  __shared__ int s_hist[FPX_HMAX];  // block histogram of the pass counts
  const int grp = threadIdx.x / kRlLanes, gl = threadIdx.x % kRlLanes;
  for (int t = threadIdx.x; t < FPX_HMAX; t += blockDim.x) s_hist[t] = 0;
  __syncthreads();
  const int64_t nun = *nun_dev;
  // the loop runs on the block's first point (uniform), so the groups of a
  // warp stay together for the shuffles; a group past the end idles
  for (int64_t u0 = (int64_t)blockIdx.x * kRlGroups; u0 < nun;
       u0 += (int64_t)gridDim.x * kRlGroups) {
    const int64_t u = u0 + grp;
    const bool valid = u < nun;
    const int64_t k = valid ? upts[u] : 0;
    double xs[D];
#pragma unroll
    for (int c = 0; c < D; ++c) xs[c] = valid ? x[k * D + c] : 0.0;
    int ax[3];
    const int64_t cell = valid ? cell_of(D, m.grid, m.ncell, xs, ax) : -1;
    const int qs = cell >= 0 ? m.offsets[cell] : 0, qe = cell >= 0 ? m.offsets[cell + 1] : 0;
    const int L = qe - qs < FPX_LISTMAX ? qe - qs : FPX_LISTMAX;
    for (int q = gl; q < L; q += kRlLanes) {
      const int e = m.elems[qs + q];
      double v = INFINITY;
      const bool pass = frec_filter_rest<D>(m, e, xs, &v);
      s_v[grp][q] = pass ? v : INFINITY;
      s_e[grp][q] = pass ? e : -1;
    }
    __syncwarp();
    // rank 0 is the candidate round 1 solved (the prefilter's choice);
    // the others follow in (v, e) order of the rest rank value.  A hinted
    // point (npass < 0) has no rank-0 candidate: all of its passing
    // candidates are ranked from 1.
    const bool hinted = valid && npass[k] < 0;
    const int e0 = hinted || !valid ? -1 : best[k];
    __syncwarp();
    if (hinted && gl == 0) best[k] = -1;
    int np = 0;
    for (int q = gl; q < L; q += kRlLanes) {
      const int e = s_e[grp][q];
      if (e < 0) continue;
      ++np;
      const double v = s_v[grp][q];
      int rank = 0;
      if (e != e0) {
        rank = 1;
        for (int j = 0; j < L; ++j) {
          const int ej = s_e[grp][j];
          rank += (ej >= 0 && ej != e0 && bf_less(s_v[grp][j], ej, v, e)) ? 1 : 0;
        }
      }
      if (rank < FPX_RK) clist[u * FPX_RK + rank] = e;
    }
    for (int o = kRlLanes / 2; o > 0; o >>= 1) np += __shfl_xor_sync(FPX_FULL, np, o);
    // more than FPX_RK passing: the rest kernel scans after the last listed
    // one; lists longer than FPX_LISTMAX: it scans everything after rank 0
    const bool over = qe - qs > L;  // list longer than the buffer: count the rest
    if (__any_sync(FPX_FULL, over)) {
      int extra = 0;
      for (int q = qs + L + gl; q < qe; q += kRlLanes)
        extra += frec_filter<D>(m, m.elems[q], xs, nullptr) ? 1 : 0;
      for (int o = kRlLanes / 2; o > 0; o >>= 1) extra += __shfl_xor_sync(FPX_FULL, extra, o);
      np += extra;
    }
    if (valid && gl == 0) {
      const int npv = np + (hinted ? 1 : 0);  // ranks 0..npv-1 (rank 0 virtual when hinted)
      cnum[u] = over ? -1 : (npv > FPX_RK ? -FPX_RK : npv);
      nps[u] = npv;
      atomicAdd(&s_hist[npv < FPX_HMAX - 1 ? npv : FPX_HMAX - 1], 1);
    }
    __syncwarp();
  }
  __syncthreads();
  for (int t = threadIdx.x; t < FPX_HMAX; t += blockDim.x)
    if (s_hist[t]) atomicAdd(&hist[t], s_hist[t]);
}

// Nearest-node seeds (D7: smallest physical distance, ties -> lowest
// lexicographic index; the distance accumulates exactly as in newton_warp)
// for up to 4 lanes of the warp at once: every lane scans K/32 nodes of each
// of the seeded points' slots and the four argmin reductions run
// interleaved.  PAD: slot rows padded to Lay::NP (round-1 ring slots).
// Returns the seeded node index to lane js[s] (and -1 to the others).
template <int D, int DR, int N, bool PAD>
__device__ __forceinline__ int seed_batch(const unsigned* js, int cnt, const double* const* sj,
                                          const double (*xj)[3], int lane) {
  using L = Lay<D, DR, N>;
  constexpr int K = L::K;
  constexpr int CS = PAD ? L::CS : K;
  double best[4];
  int bi[4];
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    best[s] = INFINITY;
    bi[s] = 0x7fffffff;
  }
  for (int t = lane; t < K; t += FPX_WARP) {
    const int row = t / N, i = t - row * N;
    const int off = PAD ? row * L::NP + i : t;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      if (s < cnt) {
        double dd = 0.0;
#pragma unroll
        for (int c = 0; c < D; ++c) {
          const double tt = __dsub_rn(xj[s][c], sj[s][c * CS + off]);
          dd = __fma_rn(tt, tt, dd);
        }
        if (dd < best[s]) {
          best[s] = dd;
          bi[s] = t;
        }
      }
    }
  }
  int mine = -1;
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    if (s < cnt) {  // cnt is warp-uniform
      const int mi = warp_argmin(best[s], bi[s]);
      if ((unsigned)lane == js[s]) mine = mi;
    }
  }
  return mine;
}

// The abort rule (round 1 and rest pass 1): some axis of r is on a face and
// the descent direction -J leaves the element through it.
template <int DR>
__device__ __forceinline__ bool held_on_face(const double* r, const double* J) {
  bool held = false;
#pragma unroll
  for (int a = 0; a < DR; ++a) held |= fabs(r[a]) == 1.0 && r[a] * J[a] < 0.0;
  return held;
}

// Block-wide inclusive sum over FPX_HMAX threads (one value per thread).
__device__ __forceinline__ int64_t block_incl_sum(int64_t v, int64_t* ws) {
  const int lane = threadIdx.x % FPX_WARP, warp = threadIdx.x / FPX_WARP;
#pragma unroll
  for (int o = 1; o < FPX_WARP; o <<= 1) {
    const int64_t y = __shfl_up_sync(FPX_FULL, v, o);
    if (lane >= o) v += y;
  }
  if (lane == FPX_WARP - 1) ws[warp] = v;
  __syncthreads();
  if (warp == 0) {
    int64_t w = lane < (int)(blockDim.x / FPX_WARP) ? ws[lane] : 0;
#pragma unroll
    for (int o = 1; o < FPX_WARP; o <<= 1) {
      const int64_t y = __shfl_up_sync(FPX_FULL, w, o);
      if (lane >= o) w += y;
    }
    ws[lane] = w;
  }
  __syncthreads();
  if (warp > 0) v += ws[warp - 1];
  __syncthreads();
  return v;
}

// Pair enumeration of the rest kernel: rest points sorted by candidate count
// (descending) so that the points with a rank-r candidate are a prefix;
// cum[r] = number of pairs of rank < r (r >= 1).  One block.
static __global__ void __launch_bounds__(FPX_HMAX)
    k_rest_order(const int32_t* __restrict__ hist, int32_t* bstart, int64_t* cum,
                 int32_t* maxnp, int64_t* npairs) {
  // one thread per bucket, two block scans:
  //   bstart[v] = #(points with npass > v)          (descending bucket order)
  //   cum[r+1]  = sum_{1<=r'<=r} #(npass > r')       (pairs of rank <= r)
  __shared__ int64_t ws[FPX_WARP];
  __shared__ int64_t gt[FPX_HMAX];
  __shared__ int smx;
  const int t = threadIdx.x;
  if (t == 0) smx = 0;
  const int v = FPX_HMAX - 1 - t;
  const int hv = hist[v];
  __syncthreads();
  if (hv) atomicMax(&smx, v);
  const int64_t suf = block_incl_sum(hv, ws) - hv;  // sum over buckets > v
  bstart[v] = (int32_t)suf;
  gt[v] = suf;
  __syncthreads();
  const int mx = smx;
  const int64_t c = block_incl_sum(t >= 1 && t < FPX_HMAX - 1 ? gt[t] : 0, ws);
  if (t < 2) cum[t] = 0;
  if (t >= 1 && t < FPX_HMAX - 1) cum[t + 1] = c;
  if (t == 0) {
    *maxnp = mx;
    if (mx <= 1) *npairs = 0;
  }
  if (mx >= 2 && t + 1 == mx) *npairs = c;
}

static __global__ void k_rest_scatter(const int64_t* __restrict__ nun_dev, const int32_t* __restrict__ nps,
                               const int32_t* __restrict__ bstart, int32_t* bcur, int32_t* perm) {
  const int64_t nun = *nun_dev;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < nun;
       u += (int64_t)gridDim.x * blockDim.x) {
    const int v = nps[u] < FPX_HMAX - 1 ? nps[u] : FPX_HMAX - 1;
    // warp-aggregated: one atomic per distinct bucket in the warp (a handful
    // of buckets hold all the rest points; per-point atomics serialised)
    const unsigned act = __activemask();
    const unsigned peers = __match_any_sync(act, v);
    const int lane = threadIdx.x % FPX_WARP;
    const int leader = __ffs(peers) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(&bcur[v], __popc(peers));
    base = __shfl_sync(peers, base, leader);
    perm[bstart[v] + base + __popc(peers & ((1u << lane) - 1u))] = (int32_t)u;
  }
}

// Rank-major pair list: pair g = cum[r] + (position of u in perm) for every
// rest point u and rank 1 <= r < npass(u): {point k, element (or -1 when
// beyond the ranked list), u, r}.
static __global__ void k_rest_pairlist(const int64_t* __restrict__ nun_dev,
                                       const int32_t* __restrict__ upts,
                                       const int32_t* __restrict__ perm,
                                       const int32_t* __restrict__ nps,
                                       const int32_t* __restrict__ clist,
                                       const int32_t* __restrict__ cnum,
                                       const int64_t* __restrict__ cum, int4* pairs,
                                       int64_t pair_cap) {
  const int64_t nun = *nun_dev;
  for (int64_t pp = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; pp < nun;
       pp += (int64_t)gridDim.x * blockDim.x) {
    const int u = perm[pp];
    const int np = nps[u] < FPX_HMAX - 1 ? nps[u] : FPX_HMAX - 1;
    const int cn = cnum[u];
    const int nl = cn < 0 ? -cn : cn;
    const int k = upts[u];
    for (int rr = 1; rr < np; ++rr) {
      const int64_t g = cum[rr] + pp;
      if (g >= pair_cap) break;  // the rest kernel rebuilds these itself
      pairs[g] = make_int4(k, rr < nl ? clist[(int64_t)u * FPX_RK + rr] : -1, u, rr);
    }
  }
}

// Rest kernel, L1 variant: the unit of work is one (point, candidate rank)
// pair, so a point with many candidates spreads over many lanes instead of
// serialising on one.  Pairs are enumerated rank-major (all rank-1 pairs,
// then all rank-2, ...); a pair whose point already has an INTERIOR result
// is skipped, which keeps the work close to the sequential early-exit order
// (SPEC.md:407).  Results are merged into the point's record under a
// per-point lock with the D6 rule.  The candidate's geometry is read in
// place (mesh.nodes_pad, 16-byte loads through L1/L2), so the number of
// pairs in flight is bounded by registers, not shared memory.
template <int D, int DR, int N>
__global__ void __launch_bounds__(128, 2)
    k_rest_l1(fpx_mesh_t m, const double* __restrict__ x, const int64_t* __restrict__ nun_dev,
              const int32_t* __restrict__ upts, const int32_t* __restrict__ clist,
              const int32_t* __restrict__ cnum,
              const int32_t* __restrict__ nps, const int32_t* __restrict__ perm,
              const int64_t* __restrict__ cum, const int32_t* __restrict__ maxnp_dev,
              const int32_t* __restrict__ best, const int4* __restrict__ pairs, int64_t pair_cap,
              const int64_t* __restrict__ npairs, int abortable, int4* redo, int64_t* nredo, int32_t* found, int32_t* lock,
              int32_t* code, int32_t* elem, double* r, double* dist, int32_t* iters,
              int64_t* counter, int64_t* stats) {
  using L = Lay<D, DR, N>;
  constexpr int ES = L::GEO;  // doubles per element in nodes_pad
  extern __shared__ __align__(16) double smem[];
  double* z = smem;
  double* scale = smem + N;
  const int warp = threadIdx.x / FPX_WARP, lane = threadIdx.x % FPX_WARP;
  double* sb = smem + 2 * ((N + 1) & ~1) + warp * Scratch<DR, N>::SLOTS * FPX_WARP + lane;
  double* stash = sb + Scratch<DR, N>::STASH * FPX_WARP;
  if (threadIdx.x < N) {
    z[threadIdx.x] = m.basis[FPX_BASIS_NODES(N, m.M) + threadIdx.x];
    scale[threadIdx.x] = m.basis[FPX_BASIS_SCALE(N, m.M) + threadIdx.x];
  }
  __syncthreads();
  const NewtonParams P = newton_of(m);
  (void)nun_dev;
  const int maxnp = maxnp_dev ? *maxnp_dev : 0;
  // all pairs of ranks 1 .. maxnp-1 (those beyond the list capacity are
  // rebuilt below from cum/perm), or the redo list (maxnp_dev == NULL;
  // clamped: its slots beyond the capacity were never used, those pairs ran
  // in full)
  const bool redo_pass = maxnp_dev == nullptr;
  const int64_t gmax = redo_pass && *npairs > pair_cap ? pair_cap : *npairs;
  int64_t s_newton = 0, s_iters = 0, nev = 0, nev2 = 0, nlev = 0;
  int64_t u = 0, k = 0;
  double xs[3] = {0.0, 0.0, 0.0};
  int phase = 0;  // 0 needs a pair, 1 needs its D7 seed, 3 iterating, 4 done
  int e = 0, it = 0;
  bool held_prev = false;
  // D7': pass 1 solves volume candidates from the affine seed (with R2);
  // d7 marks a solve from the nearest-node seed (redo pass, surfaces, or a
  // pass-1 pair restarted in place when the redo list is full)
  bool d7 = false;
  int4 cur = make_int4(0, 0, 0, 0);  // the pair being solved
  bool first = true;
  double rc[3] = {0.0, 0.0, 0.0}, rn[3] = {0.0, 0.0, 0.0};
  double alpha = 1.0, fcur = 0.0, pred = 0.0, smax = 0.0;
  NState st;
  while (true) {
    // (a) lanes without a pair claim the next ones (warp-aggregated) until
    // they find one still to do
    while (true) {
      const unsigned need = __ballot_sync(FPX_FULL, phase == 0);
      if (!need) break;
      int64_t base = 0;
      if (lane == __ffs(need) - 1)
        base = (int64_t)atomicAdd((unsigned long long*)counter, (unsigned long long)__popc(need));
      base = __shfl_sync(FPX_FULL, base, __ffs(need) - 1);
      if (phase != 0) continue;
      const int64_t g = base + __popc(need & ((1u << lane) - 1u));
      if (g >= gmax) {
        phase = 4;
        continue;
      }
      int4 pr;
      if (g < pair_cap) {
        pr = pairs[g];
      } else {  // beyond the pair-list capacity: locate (rank, point) directly
        int lo = 1, hi = maxnp;  // cum[lo] <= g < cum[hi]
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (cum[mid] <= g) lo = mid;
          else hi = mid;
        }
        const int uu = perm[g - cum[lo]];
        const int cn = cnum[uu];
        const int nl = cn < 0 ? -cn : cn;
        pr = make_int4(upts[uu], lo < nl ? clist[(int64_t)uu * FPX_RK + lo] : -1, uu, lo);
      }
      u = pr.z;
      if (*(volatile int32_t*)&found[u]) continue;  // an INTERIOR was found already
      k = pr.x;
      cur = pr;
      const int rank = pr.w;
#pragma unroll
      for (int c = 0; c < D; ++c) xs[c] = x[k * D + c];
      int en = pr.y;
      if (en < 0) {
        // beyond the ranked list: the (rank - nlist)-th passing candidate
        // ranked after the last listed one, in hash-list order (lists longer
        // than the ranking buffer, cn == -1: every passing candidate but the
        // round-1 one)
        const int cn = cnum[u];
        const int nlist = cn < 0 ? -cn : cn;
        const bool all = cn == -1;
        const int te = all ? best[k] : clist[u * FPX_RK + nlist - 1];
        double tv = -INFINITY;  // te < 0: a hinted point, nothing listed before
        if (te >= 0) tv = rest_rank_of<D>(m, te, xs);
        int ax[3];
        const int64_t cell = cell_of(D, m.grid, m.ncell, xs, ax);
        int want = rank - nlist;
        for (int q = m.offsets[cell]; q < m.offsets[cell + 1]; ++q) {
          const int ee = m.elems[q];
          if (ee == best[k]) continue;  // round 1's candidate (rank 0)
          double ve = 0.0;
          if (!frec_filter_rest<D>(m, ee, xs, &ve)) continue;
          if (!all && !bf_less(tv, te, ve, ee)) continue;
          if (want-- == 0) {
            en = ee;
            break;
          }
        }
      }
      if (en < 0) continue;
      e = en;
      cur.y = en;
      d7 = redo_pass || DR < D;
      if (!d7) {
        double fr[D + D * D];
        const double* gfr = m.frec + (int64_t)e * FPX_FREC + 3 * D + D * D;
#pragma unroll
        for (int t = 0; t < D + D * D; ++t) fr[t] = __ldg(gfr + t);
        affine_seed<D>(fr, xs, rc);
#pragma unroll
        for (int a = 0; a < 3; ++a) rn[a] = rc[a];
        first = true;
        held_prev = false;
        it = 0;
        alpha = P.alpha0;
        phase = 3;
        continue;
      }
      phase = 1;  // needs its D7 seed
    }
    // seeds (D7) of the lanes that just got a pair, 4 at a time: the warp
    // reads each candidate's nodes with coalesced loads
    for (unsigned sd = __ballot_sync(FPX_FULL, phase == 1); sd;) {
      int js[4], ej[4];
      double xj[4][3];
      int cnt = 0;
#pragma unroll
      for (int s2 = 0; s2 < 4; ++s2) {
        js[s2] = sd ? __ffs(sd) - 1 : 0;
        if (sd) {
          sd &= sd - 1;
          cnt = s2 + 1;
        }
        ej[s2] = __shfl_sync(FPX_FULL, e, js[s2]);
#pragma unroll
        for (int c = 0; c < D; ++c) xj[s2][c] = __shfl_sync(FPX_FULL, xs[c], js[s2]);
      }
      double bst[4];
      int bi[4];
#pragma unroll
      for (int s2 = 0; s2 < 4; ++s2) {
        bst[s2] = INFINITY;
        bi[s2] = 0x7fffffff;
      }
      for (int t = lane; t < L::K; t += FPX_WARP) {
        const int row = t / N, i = t - row * N;
        const int off = row * L::NP + i;
#pragma unroll
        for (int s2 = 0; s2 < 4; ++s2) {
          if (s2 < cnt) {
            const double* X = m.nodes_pad + (int64_t)ej[s2] * ES;
            double dd = 0.0;
#pragma unroll
            for (int c = 0; c < D; ++c) {
              const double tt = __dsub_rn(xj[s2][c], __ldg(X + c * L::CS + off));
              dd = __fma_rn(tt, tt, dd);
            }
            if (dd < bst[s2]) {
              bst[s2] = dd;
              bi[s2] = t;
            }
          }
        }
      }
#pragma unroll
      for (int s2 = 0; s2 < 4; ++s2) {
        if (s2 < cnt) bi[s2] = warp_argmin(bst[s2], bi[s2]);  // cnt is warp-uniform
      }
#pragma unroll
      for (int s2 = 0; s2 < 4; ++s2) {
        if (s2 < cnt && lane == js[s2]) {
          const int b = bi[s2];
          rc[0] = z[b % N];
          rc[1] = DR > 1 ? z[(b / N) % N] : 0.0;
          rc[2] = DR > 2 ? z[b / (N * N)] : 0.0;
#pragma unroll
          for (int a = 0; a < 3; ++a) rn[a] = rc[a];
          first = true;
          held_prev = false;
          it = 0;
          alpha = P.alpha0;
          phase = 3;
        }
      }
    }
    if (!__any_sync(FPX_FULL, phase != 4)) break;
    // (b) one map evaluation for every lane of the warp
    const bool w2 = __any_sync(FPX_FULL, phase == 3 && on_boundary<DR>(rn));
    ++nev;
    nev2 += w2 ? 1 : 0;
    nlev += phase == 3 ? 1 : 0;
    const double* X = m.nodes_pad + (int64_t)(phase == 3 ? e : 0) * ES;
    eval_state_rt<D, DR, N, 3>(X, z, scale, rn, xs, st, sb, w2);
    if (phase != 3) continue;
    // (c) trust-region Newton update (newton_warp, D8)
    bool done = false;
    if (first) {
      first = false;
    } else {
      const double decr = fcur - st.f;
      if (decr >= P.accept * pred) {
        if (decr >= P.keep * pred) alpha *= P.grow;
#pragma unroll
        for (int a = 0; a < DR; ++a) rc[a] = rn[a];
      } else {
        alpha *= P.shrink;
        unstash_state(stash, st);
        st.f = fcur;
      }
      if (smax < P.tol) done = true;
      else if (it >= P.max_iters) done = true;
    }
    if (!done && *(volatile int32_t*)&found[u]) {
      // another candidate of this point was INTERIOR meanwhile: its record
      // is final (an INTERIOR is unique up to shared faces), stop this one
      s_newton += 1;
      s_iters += it;
      phase = 0;
      continue;
    }
    if (!done && abortable && !d7 && it >= 1) {
      // held on a face (descent direction leaving it) for two consecutive
      // iterations (rule R2): this candidate is most likely not the owner.
      // Stop; under D7' the pair is redone from the D7 seed (redo pass) if
      // its point ends without an INTERIOR -- at once, in place, when the
      // redo list is full.
      const bool held = held_on_face<DR>(rc, st.J);
      if (held && held_prev) {
        const int64_t slot = (int64_t)atomicAdd((unsigned long long*)nredo, 1ull);
        s_newton += 1;
        s_iters += it;
        if (slot < pair_cap) {
          redo[slot] = cur;
          phase = 0;
        } else {
          d7 = true;
          phase = 1;
        }
        continue;
      }
      held_prev = held;
    }
    if (!done) {
      fcur = st.f;
      const bool go = propose_step<DR>(st, rc, it, alpha, xscale<D>(xs), P.tol, rn, pred, smax);
      ++it;
      if (!go) {
        done = true;
#pragma unroll
        for (int a = 0; a < DR; ++a) rc[a] = rn[a];
      } else {
        stash_state(stash, st);
      }
    }
    if (done) {
      const double dd = sqrt(st.f);
      s_newton += 1;
      s_iters += it;
      const double epsd = DR < D ? eps_d_of(m, e) : 0.0;
      const int cd = classify<D, DR>(rc, dd, epsd);
      if (!d7 && cd != kInterior) {
        // D7': a BORDER result from the affine seed is replaced by the
        // solve from the D7 seed (redo pass; in place when the list is full)
        const int64_t slot = (int64_t)atomicAdd((unsigned long long*)nredo, 1ull);
        if (slot < pair_cap) {
          redo[slot] = cur;
          phase = 0;
        } else {
          d7 = true;
          phase = 1;
        }
        continue;
      }
      // D6 merge into the point's record under its lock
      while (atomicCAS(&lock[u], 0, 1) != 0) {
      }
      __threadfence();
      const int bc = *(volatile int32_t*)&code[k], be = *(volatile int32_t*)&elem[k];
      const double bd = *(volatile double*)&dist[k];
      bool take;
      if (cd == kInterior) take = bc != kInterior || e < be;
      else  // (a hinted point's record starts as a NOT_FOUND placeholder)
        take = bc == kNotFound || (bc != kInterior && (dd < bd || (dd == bd && e < be)));
      if (take) {
        code[k] = cd;
        elem[k] = e;
        dist[k] = dd;
#pragma unroll
        for (int a = 0; a < DR; ++a) r[k * DR + a] = rc[a];
      }
      if (iters) iters[k] += it;
      if (cd == kInterior) found[u] = 1;
      __threadfence();
      atomicExch(&lock[u], 0);
      phase = 0;
    }
  }
  s_newton = warp_sum64(s_newton);
  s_iters = warp_sum64(s_iters);
  nlev = warp_sum64(nlev);
  if (lane == 0) {
    atomicAdd((unsigned long long*)&stats[FPX_STAT_NEWTON], (unsigned long long)s_newton);
    atomicAdd((unsigned long long*)&stats[FPX_STAT_ITERS], (unsigned long long)s_iters);
    atomicAdd((unsigned long long*)&stats[FPX_STAT_REST_WARP_EVALS], (unsigned long long)nev);
    atomicAdd((unsigned long long*)&stats[FPX_STAT_REST_W2_EVALS], (unsigned long long)nev2);
    atomicAdd((unsigned long long*)&stats[FPX_STAT_REST_LANE_EVALS], (unsigned long long)nlev);
  }
}

// Field values of the rest points (after k_rest_l1 settled their
// records): thread per point, NaN for NOT_FOUND (D12).
template <int DR, int N>
__global__ void k_rest_values(const double* __restrict__ fbasis, int M,
                              const int64_t* __restrict__ nun_dev,
                              const int32_t* __restrict__ upts, const int32_t* __restrict__ code,
                              const int32_t* __restrict__ elem, const double* __restrict__ r,
                              const double* __restrict__ field, int C, double* values,
                              int64_t* stats) {
  __shared__ double z[16], scale[16];
  if (threadIdx.x < N) {
    z[threadIdx.x] = fbasis[FPX_BASIS_NODES(N, M) + threadIdx.x];
    scale[threadIdx.x] = fbasis[FPX_BASIS_SCALE(N, M) + threadIdx.x];
  }
  __syncthreads();
  const int64_t nun = *nun_dev;
  int64_t s_evals = 0;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < nun;
       u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = upts[u];
    if (code[k] == kNotFound) {
      for (int c = 0; c < C; ++c) values[k * C + c] = NAN;
      continue;
    }
    double rr[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int a = 0; a < DR; ++a) rr[a] = r[k * DR + a];
    double v[DR][N];
    basis_values<DR, N>(z, scale, rr, v);
    const int64_t e = elem[k];
    for (int c = 0; c < C; ++c)
      values[k * C + c] = contract_gmem<DR, N>(field + (e * C + c) * Pow<DR, N>::K, v);
    ++s_evals;
  }
  for (int o = 16; o > 0; o >>= 1) s_evals += __shfl_xor_sync(FPX_FULL, s_evals, o);
  if ((threadIdx.x & 31) == 0 && s_evals)
    atomicAdd((unsigned long long*)&stats[FPX_STAT_EVALS], (unsigned long long)s_evals);
}

// ---------------------------------------------------------------- round 1, streamed
// Element-major round 1 without fixed work items.  The points are sorted by
// their best-first element; a warp consumes chunks (FPX_R1_CHUNK points,
// default 64: small enough that the last chunks balance across warps) of
// that stream through a
// ring of S shared-memory element slots (geometry + field block, loaded
// asynchronously ahead of use, completion on a per-slot mbarrier).  A lane
// takes the next point as soon as its own solve finishes, so a warp never
// waits for its slowest lane and never runs with lanes left empty by a
// small element; the lanes of one warp read at most S distinct slots per
// load, whose bank offsets differ (slot stride = 16 mod 128 bytes), so the
// loads stay single-wavefront broadcasts.  Seeds are warp-cooperative.
#ifndef FPX_CHUNK_DEFAULT
#define FPX_CHUNK_DEFAULT 64
#endif

// L1 prefetch of a claimed chunk's stream records (ux, umeta): the lanes
// that take its units later read them from L1 instead of a DRAM round trip.
// One line per lane, no loop (a chunk is <= FPX_CHUNK_DEFAULT = 64 units:
// <= 13 lines of ux, <= 9 of umeta): the loader sits in the hot loop, whose
// instruction footprint matters.
__device__ __forceinline__ void prefetch_chunk3(const void* p0, size_t b0, const void* p1,
                                                size_t b1, int lane) {
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(p0) & ~uintptr_t(127);
  const uintptr_t a1 = reinterpret_cast<uintptr_t>(p1) & ~uintptr_t(127);
  const int n0 = (int)((reinterpret_cast<uintptr_t>(p0) + b0 - a0 + 127) / 128);
  const uintptr_t q = lane < n0 ? a0 + (uintptr_t)lane * 128 : a1 + (uintptr_t)(lane - n0) * 128;
  if (q < (lane < n0 ? reinterpret_cast<uintptr_t>(p0) + b0 : reinterpret_cast<uintptr_t>(p1) + b1))
    asm volatile("prefetch.L1 [%0];\n" ::"l"(q));
}
template <int D>
__device__ __forceinline__ void prefetch_chunk(const double* ux, const int4* umeta, int64_t c0,
                                               int len, int lane) {
  prefetch_chunk3(ux + c0 * D, (size_t)len * D * sizeof(double), umeta + c0,
                  (size_t)len * sizeof(int4), lane);
}

// Round-1 per-lane scratch: the axis-1..d_r-1 basis values, plus the
// Newton-state stash below order 7.  From N = 8 on (16.5 KB element slots)
// a rejected step re-evaluates the current iterate instead, and the stash's
// 4 KB per warp buys resident warps (rejections are rare: at N = 5 both
// forms measured the same).
template <int DR, int N>
struct StreamScratch {
  static constexpr bool LEAN = N >= 8;
  static constexpr int SLOTS = (DR - 1) * 3 * N + (LEAN ? 0 : 16);
};

template <int S>
struct StreamMeta {
  uint64_t mbar[S];
  int elem[S], start[S], end[S], fsh[S];
  unsigned parity[S];
};

template <int D, int DR, int N, int S>
__global__ void __launch_bounds__(128, FPX_NEWTON_MINB)
    k_newton_stream(fpx_mesh_t m, const double* __restrict__ ux, const int4* __restrict__ umeta,
                    const uint64_t* __restrict__ packed_off, const int32_t* __restrict__ npass,
                    int32_t* code, int32_t* elem, double* r, double* dist, int32_t* iters,
                    const double* __restrict__ field, int C, double* values, int32_t* upts,
                    int64_t* nun_dev, int64_t* chunk_ctr, int slot_stride, int nslot,
                    int fstage, int chunk, int4* redo, int64_t* nredo, int64_t redo_cap,
                    int64_t* stats) {
  using L = Lay<D, DR, N>;
  constexpr int K = L::K;
  constexpr int SCR = StreamScratch<DR, N>::SLOTS;
  constexpr bool LEAN = StreamScratch<DR, N>::LEAN;
  constexpr int FRAME = DR == D ? D + D * D : 0;  // affine frame doubles per slot
  extern __shared__ __align__(16) double smem[];
  double* z = smem;
  double* scale = smem + N;
  const int warp = threadIdx.x / FPX_WARP, lane = threadIdx.x % FPX_WARP;
  // slot (nslot <= S of them per warp): geometry [D][ROWS][NP] (= the
  // mesh.nodes_pad block) | frame (x_c, J_c^-1) | field [C][K] from the
  // 16-byte boundary below the element's block (when fstage)
  constexpr int frame_off = L::GEO;
  constexpr int field_off = L::GEO + ((FRAME + 1) & ~1);
  double* slots =
      smem + 2 * ((N + 1) & ~1) + (size_t)warp * (nslot * slot_stride + SCR * FPX_WARP);
  double* sb = slots + nslot * slot_stride + lane;
  double* stash = sb + Scratch<DR, N>::STASH * FPX_WARP;  // (unused when LEAN)
  // ring metadata in static shared memory (shared-space loads, not generic)
  __shared__ StreamMeta<S> s_meta[4];
  StreamMeta<S>* meta = s_meta + warp;
  if (threadIdx.x < N) {
    z[threadIdx.x] = m.basis[FPX_BASIS_NODES(N, m.M) + threadIdx.x];
    scale[threadIdx.x] = m.basis[FPX_BASIS_SCALE(N, m.M) + threadIdx.x];
  }
  for (int t = lane; t < nslot * slot_stride; t += FPX_WARP) slots[t] = 0.0;
  if (lane < S) {
    mbar_init(&meta->mbar[lane], 1);
    meta->fsh[lane] = 0;
    meta->parity[lane] = 0;
    meta->start[lane] = meta->end[lane] = 0;
    meta->elem[lane] = -1;
  }
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  // the zero fill (generic proxy) before the bulk copies (async proxy)
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();
  const NewtonParams P = newton_of(m);
  const int64_t nu = (int64_t)(packed_off[m.E] & 0xffffffffull);
  // warp-local unit sequence = claimed chunk A then chunk B
  int64_t a0 = 0, b0 = 0;
  int alen = 0, blen = 0;
  bool exhausted = false, bclaimed = false;
  int q = 0, ld = 0, nord = 0;
  unsigned ready = 0;  // slots whose current load has landed
  // lane state: 0 idle, 1 needs seed, 2 iterating
  int phase = 0, myslot = 0, pt = 0, it = 0;
  bool first = true, held_prev = false;
  double xs[3] = {0.0, 0.0, 0.0}, rc[3] = {0.0, 0.0, 0.0}, rn[3] = {0.0, 0.0, 0.0};
  double alpha = 1.0, fcur = 0.0, pred = 0.0, smax = 0.0;
  NState st;
  int64_t s_newton = 0, s_iters = 0, s_evals = 0, nev = 0, nev2 = 0, s_chunks = 0, nlev = 0;
  bool reeval = false;  // LEAN: this evaluation recomputes the state at rc
  // first chunk
  {
    int64_t c = 0;
    if (lane == 0) c = (int64_t)atomicAdd((unsigned long long*)chunk_ctr, (unsigned long long)chunk);
    c = __shfl_sync(FPX_FULL, c, 0);
    if (c >= nu) exhausted = true;
    else {
      a0 = c;
      alen = (int)(nu - c < chunk ? nu - c : chunk);
      prefetch_chunk<D>(ux, umeta, a0, alen, lane);
      ++s_chunks;
    }
  }
  while (true) {
    // ---- loader: schedule the next element of the stream into the ring
    while (!exhausted || ld < alen + blen) {
      if (ld >= alen + blen) {  // need chunk B
        if (bclaimed) break;
        int64_t c = 0;
        if (lane == 0)
          c = (int64_t)atomicAdd((unsigned long long*)chunk_ctr, (unsigned long long)chunk);
        c = __shfl_sync(FPX_FULL, c, 0);
        if (c >= nu) {
          exhausted = true;
          break;
        }
        b0 = c;
        blen = (int)(nu - c < chunk ? nu - c : chunk);
        prefetch_chunk<D>(ux, umeta, b0, blen, lane);
        bclaimed = true;
        ++s_chunks;
      }
      const int s = nslot == 3 ? nord % 3 : nord & 1;
      const bool busy = __any_sync(FPX_FULL, phase != 0 && myslot == s);
      if (busy || meta->end[s] > q) break;  // slot still has lanes or unassigned units
      const int64_t g = ld < alen ? a0 + ld : b0 + (ld - alen);
      const int4 um = umeta[g];
      const int e = um.y;
      const int64_t gend = um.z;
      const int64_t cend = ld < alen ? a0 + alen : b0 + blen;
      const int lend = ld + (int)((gend < cend ? gend : cend) - g);
      __syncwarp();
      if (lane == 0) {
        // one elected lane stages the element with TMA bulk copies: the
        // padded geometry block, the affine frame (seeds), the field block
        double* sl = slots + s * slot_stride;
        const unsigned gb = L::GEO * 8, fb = FRAME * 8;
        uintptr_t ua = 0;
        unsigned ub = 0;
        if (fstage) {
          const uintptr_t u0 = reinterpret_cast<uintptr_t>(field + (int64_t)e * C * K);
          ua = u0 & ~uintptr_t(15);
          ub = (unsigned)(((u0 + (uintptr_t)C * K * 8 + 15) & ~uintptr_t(15)) - ua);
          meta->fsh[s] = (int)((u0 - ua) / 8);
        }
        uint64_t* mb = &meta->mbar[s];
        mbar_expect_tx(mb, gb + fb + ub);
        bulk_g2s(sl, m.nodes_pad + (int64_t)e * L::GEO, gb, mb);
        if (FRAME) bulk_g2s(sl + frame_off, m.frec + (int64_t)e * FPX_FREC + 3 * D + D * D, fb, mb);
        if (ub) bulk_g2s(sl + field_off, reinterpret_cast<const double*>(ua), ub, mb);
        meta->elem[s] = e;
        meta->start[s] = ld;
        meta->end[s] = lend;
      }
      __syncwarp();
      ready &= ~(1u << s);
      ++nord;
      ld = lend;
    }
    // ---- which pending slot loads have landed
    {
      bool ok = false;
      if (lane < S && !(ready & (1u << lane)) && meta->end[lane] > meta->start[lane])
        ok = mbar_test(&meta->mbar[lane], meta->parity[lane]);
      const unsigned landed = __ballot_sync(FPX_FULL, ok);
      // every lane acquires the completed phase itself (all lanes issued the
      // slot's copies): their reads of the slot, and its next refill, are
      // then ordered after the landing for each lane, not only for lane s
      for (unsigned l = landed; l; l &= l - 1) {
        const int s2 = __ffs(l) - 1;
        while (!mbar_test(&meta->mbar[s2], meta->parity[s2])) {
        }
      }
      __syncwarp();
      if (ok) meta->parity[lane] ^= 1u;
      ready |= landed;
      __syncwarp();
    }
    // ---- refill idle lanes with the next units whose slot is ready
    {
      const unsigned idle = __ballot_sync(FPX_FULL, phase == 0);
      int avail = 0;
      for (int o = 0; o < S && idle; ++o) {  // slots in stream order from q
        int sq = -1;
#pragma unroll
        for (int s2 = 0; s2 < S; ++s2)
          if (meta->start[s2] <= q + avail && q + avail < meta->end[s2]) sq = s2;
        if (sq < 0 || !(ready & (1u << sq))) break;
        avail = meta->end[sq] - q;
      }
      const int take = avail < __popc(idle) ? avail : __popc(idle);
      const int rk = __popc(idle & ((1u << lane) - 1u));
      if (phase == 0 && rk < take) {
        const int p = q + rk;
        const int64_t g = p < alen ? a0 + p : b0 + (p - alen);
        pt = umeta[g].x;
#pragma unroll
        for (int s2 = 0; s2 < S; ++s2)
          if (meta->start[s2] <= p && p < meta->end[s2]) myslot = s2;
#pragma unroll
        for (int c = 0; c < D; ++c) xs[c] = ux[g * D + c];
        if constexpr (DR == D) {
          // seed (decision D7'): the affine prediction of the element's
          // centre frame; an INTERIOR result is final (the unique zero of the
          // injective element map), a BORDER or aborted one is recomputed
          // from the D7 nearest-node seed by the redo pass.  On cfg-2 it
          // halves the owner's Newton iterations (3.0 -> 1.7).
          affine_seed<D>(slots + myslot * slot_stride + frame_off, xs, rc);
#pragma unroll
          for (int a = 0; a < 3; ++a) rn[a] = rc[a];
          first = true;
          held_prev = false;
          it = 0;
          alpha = P.alpha0;
          phase = 2;
        } else {
          phase = 1;
        }
      }
      q += take;
      if (q >= alen && bclaimed) {  // chunk A consumed: B becomes A
        const int sh = alen;
        a0 = b0;
        alen = blen;
        blen = 0;
        bclaimed = false;
        q -= sh;
        ld -= sh;
        if (lane < S) {
          meta->start[lane] -= sh;
          meta->end[lane] -= sh;
        }
        __syncwarp();
      }
    }
    // ---- cooperative seeds (D7) of the lanes that just got a point
    // (surfaces and lines; volume elements seed from their frame above)
    for (unsigned sd = DR < D ? __ballot_sync(FPX_FULL, phase == 1) : 0u; sd;) {
      unsigned js[4];
      const double* sj[4];
      double xj[4][3];
      int cnt = 0;
#pragma unroll
      for (int s2 = 0; s2 < 4; ++s2) {
        js[s2] = sd ? (unsigned)(__ffs(sd) - 1) : 0u;
        if (sd) {
          sd &= sd - 1;
          cnt = s2 + 1;
        }
        sj[s2] = slots + __shfl_sync(FPX_FULL, myslot, js[s2]) * slot_stride;
#pragma unroll
        for (int c = 0; c < D; ++c) xj[s2][c] = __shfl_sync(FPX_FULL, xs[c], js[s2]);
      }
      const int bi = seed_batch<D, DR, N, true>(js, cnt, sj, xj, lane);
      if (bi >= 0) {
        rc[0] = z[bi % N];
        rc[1] = DR > 1 ? z[(bi / N) % N] : 0.0;
        rc[2] = DR > 2 ? z[bi / (N * N)] : 0.0;
#pragma unroll
        for (int a = 0; a < 3; ++a) rn[a] = rc[a];
        first = true;
        held_prev = false;
        it = 0;
        alpha = P.alpha0;
        phase = 2;
      }
    }
    const bool any_iter = __any_sync(FPX_FULL, phase == 2);
    if (!any_iter) {
      if (exhausted && q >= alen + blen) break;  // stream done, all lanes idle
      continue;                                   // waiting for a slot load
    }
    // ---- one map evaluation for every lane of the warp (second derivatives
    // whenever any lane's trial point is on a face: deferring them to batched
    // passes measured slower, the waiting lanes cost more passes than the
    // batching saved)
    double* sX = slots + myslot * slot_stride;
    const bool w2 = __any_sync(FPX_FULL, phase == 2 && on_boundary<DR>(rn));
    ++nev;
    nev2 += w2 ? 1 : 0;
    nlev += phase == 2 ? 1 : 0;
    // two compile-time bodies: without second derivatives when no lane of
    // the warp is on a face (31% of the warp evaluations at cfg-2; the extra
    // code cost more than it saved until the loop's footprint was trimmed:
    // 0.711 vs 0.688 ms then, 0.578 vs 0.598 ms now)
    if (w2) eval_state_rt<D, DR, N, 0, 1>(sX, z, scale, rn, xs, st, sb, true);
    else eval_state_rt<D, DR, N, 0, 0>(sX, z, scale, rn, xs, st, sb, false);
    if (phase != 2) continue;
    // ---- this lane's trust-region Newton update (newton_warp, D8)
    bool done = false;
    if (first) {
      first = false;
    } else if (LEAN && reeval) {
      reeval = false;  // st is the state at rc again: on to the abort rule and the step
    } else {
      const double decr = fcur - st.f;
      bool rejected = false;
      if (decr >= P.accept * pred) {
        if (decr >= P.keep * pred) alpha *= P.grow;
#pragma unroll
        for (int a = 0; a < DR; ++a) rc[a] = rn[a];
      } else {
        alpha *= P.shrink;
        if constexpr (!LEAN) unstash_state(stash, st);
        st.f = fcur;
        rejected = true;
      }
      if (smax < P.tol) done = true;
      else if (it >= P.max_iters) done = true;
      if (LEAN && rejected && !done) {  // the state at rc is re-evaluated next
#pragma unroll
        for (int a = 0; a < DR; ++a) rn[a] = rc[a];
        reeval = true;
        continue;
      }
    }
    if (!done && redo && it >= 1) {
      // the abort rule of the rest kernel: held on a face for two
      // consecutive iterations -> stop, hand the point to the rest phase
      // (its other candidates) and this candidate to the redo pass, which
      // runs it in full only if no candidate turns out INTERIOR
      const bool held = held_on_face<DR>(rc, st.J);
      if (held && held_prev) {
        const int64_t rs = (int64_t)atomicAdd((unsigned long long*)nredo, 1ull);
        if (rs < redo_cap) {
          const int e = meta->elem[myslot];
          const int slot = (int)atomicAdd((unsigned long long*)nun_dev, 1ull);
          upts[slot] = pt;
          redo[rs] = make_int4(pt, e, slot, 0);
          code[pt] = kBorder;  // placeholder: any computed record replaces it
          elem[pt] = e;
          dist[pt] = INFINITY;
#pragma unroll
          for (int a = 0; a < DR; ++a) r[(int64_t)pt * DR + a] = rc[a];
          if (iters) iters[pt] = it;
          s_newton += 1;
          s_iters += it;
          phase = 0;
          continue;
        }
      }
      held_prev = held;
    }
    if (!done) {
      fcur = st.f;
      const bool go = propose_step<DR>(st, rc, it, alpha, xscale<D>(xs), P.tol, rn, pred, smax);
      ++it;
      if (!go) {
        done = true;
#pragma unroll
        for (int a = 0; a < DR; ++a) rc[a] = rn[a];
      } else {
        if constexpr (!LEAN) stash_state(stash, st);
      }
    }
    if (done) {
      const double dd = sqrt(st.f);
      const int e = meta->elem[myslot];
      s_newton += 1;
      s_iters += it;
      const double epsd = DR < D ? eps_d_of(m, e) : 0.0;
      const int cd = classify<D, DR>(rc, dd, epsd);
      if (DR == D && cd != kInterior && redo) {
        // a solve from the affine seed that ends BORDER is not final: like
        // an aborted one it goes to the redo pass, which recomputes it from
        // the D7 seed if the point finds no INTERIOR (at most one round-1
        // entry per point: the list cannot overflow)
        const int64_t rs = (int64_t)atomicAdd((unsigned long long*)nredo, 1ull);
        const int slot = (int)atomicAdd((unsigned long long*)nun_dev, 1ull);
        upts[slot] = pt;
        redo[rs] = make_int4(pt, e, slot, 0);
        code[pt] = kBorder;  // placeholder: any computed record replaces it
        elem[pt] = e;
        dist[pt] = INFINITY;
#pragma unroll
        for (int a = 0; a < DR; ++a) r[(int64_t)pt * DR + a] = rc[a];
        if (iters) iters[pt] = it;
        phase = 0;
        continue;
      }
      // npass < 0: a hinted find (fpx_set_find_hint) -- the hint is not
      // known to be a candidate, so only an INTERIOR result (inside the
      // element, hence passing its filter) is kept; otherwise the record is
      // a NOT_FOUND placeholder and the rest phase searches all candidates
      const int np = npass[pt];
      const bool final = cd == kInterior || (np >= 0 && np <= 1);
      const bool drop = !final && np < 0;
      code[pt] = drop ? kNotFound : cd;
      elem[pt] = drop ? -1 : e;
#pragma unroll
      for (int a = 0; a < DR; ++a) r[(int64_t)pt * DR + a] = drop ? NAN : rc[a];
      dist[pt] = drop ? NAN : dd;
      if (iters) iters[pt] = it;
      if (final) {
        if (field) {
          const double* fu = fstage ? sX + field_off + meta->fsh[myslot]
                                    : field + (int64_t)e * C * K;
          if constexpr (DR == 3) {
            // the lane's scratch is free once its solve is done: the three
            // axes' basis values from one rolled copy of the recursion
#pragma unroll 1
            for (int a = 0; a < 3; ++a) {
              double w[N], g[N], h[N];
              lagrange<N, false>(z, scale, a == 0 ? rc[0] : (a == 1 ? rc[1] : rc[2]), w, g, h);
#pragma unroll
              for (int k = 0; k < N; ++k) sb[(a * N + k) * FPX_WARP] = w[k];
            }
            double v0[N], v1[N];
#pragma unroll
            for (int k = 0; k < N; ++k) {
              v0[k] = sb[k * FPX_WARP];
              v1[k] = sb[(N + k) * FPX_WARP];
            }
            for (int c = 0; c < C; ++c)
              values[(int64_t)pt * C + c] =
                  contract_flat_k<N>(fu + c * K, v0, v1, sb + 2 * N * FPX_WARP);
          } else {
            double v[DR][N];
            basis_values<DR, N>(z, scale, rc, v);
            for (int c = 0; c < C; ++c)
              values[(int64_t)pt * C + c] = contract_flat<DR, N>(fu + c * K, v);
          }
          ++s_evals;
        }
      } else {
        const int slot = (int)atomicAdd((unsigned long long*)nun_dev, 1ull);
        upts[slot] = pt;
      }
      phase = 0;
    }
  }
  s_newton = warp_sum64(s_newton);
  s_iters = warp_sum64(s_iters);
  s_evals = warp_sum64(s_evals);
  nlev = warp_sum64(nlev);
  if (lane == 0) {
    atomicAdd((unsigned long long*)&stats[FPX_STAT_NEWTON], (unsigned long long)s_newton);
    atomicAdd((unsigned long long*)&stats[FPX_STAT_ITERS], (unsigned long long)s_iters);
    atomicAdd((unsigned long long*)&stats[FPX_STAT_EVALS], (unsigned long long)s_evals);
    atomicAdd((unsigned long long*)&stats[FPX_STAT_NEWTON_R1], (unsigned long long)s_newton);
    atomicAdd((unsigned long long*)&stats[FPX_STAT_ITERS_R1], (unsigned long long)s_iters);
    atomicAdd((unsigned long long*)&stats[FPX_STAT_EVALS_R1], (unsigned long long)s_evals);
    atomicAdd((unsigned long long*)&stats[FPX_STAT_R1_WARP_EVALS], (unsigned long long)nev);
    atomicAdd((unsigned long long*)&stats[FPX_STAT_R1_W2_EVALS], (unsigned long long)nev2);
    atomicAdd((unsigned long long*)&stats[FPX_STAT_R1_ITEMS], (unsigned long long)s_chunks);
    atomicAdd((unsigned long long*)&stats[FPX_STAT_R1_LANE_EVALS], (unsigned long long)nlev);
  }
}

// findpts_eval over element-grouped records: warp per item, field block in
// shared memory, one point per lane.
template <int DR, int N>
__global__ void __launch_bounds__(128)
    k_eval_items(const double* __restrict__ fbasis, int M, int C,
                 const double* __restrict__ field, const double* __restrict__ r,
                 const int32_t* __restrict__ sorted, const Item* __restrict__ items,
                 const int64_t* __restrict__ nitems_dev, double* values) {
  using L = Lay<1, DR, N>;
  extern __shared__ __align__(16) double smem[];
  double* z = smem;
  double* scale = smem + N;
  const int warp = threadIdx.x / FPX_WARP, lane = threadIdx.x % FPX_WARP;
  const int wpb = blockDim.x / FPX_WARP;
  double* sU = smem + 2 * ((N + 1) & ~1) + warp * (C * L::CS);
  if (threadIdx.x < N) {
    z[threadIdx.x] = fbasis[FPX_BASIS_NODES(N, M) + threadIdx.x];
    scale[threadIdx.x] = fbasis[FPX_BASIS_SCALE(N, M) + threadIdx.x];
  }
  __syncthreads();
  const int64_t nitems = *nitems_dev;
  for (int64_t w = (int64_t)blockIdx.x * wpb + warp; w < nitems; w += (int64_t)gridDim.x * wpb) {
    const Item itm = items[w];
    stage_block<DR, N>(sU, field + (int64_t)itm.elem * C * L::K, C, lane);
    cp_async_wait_all();
    __syncwarp();
    if (lane < itm.count) {
      const int pt = sorted[itm.start + lane];
      double rr[3] = {0, 0, 0};
#pragma unroll
      for (int a = 0; a < DR; ++a) rr[a] = r[(int64_t)pt * DR + a];
      double v[DR][N];
      basis_values<DR, N>(z, scale, rr, v);
      for (int c = 0; c < C; ++c)
        values[(int64_t)pt * C + c] = contract_smem<DR, N>(sU + c * L::CS, v);
    }
    __syncwarp();
  }
}

// forward_map at explicit (element, r): thread per query, geometry from
// global memory (API / test path, not the find hot loop).
template <int D, int DR, int N>
__global__ void k_forward_map(fpx_mesh_t m, int64_t n, const int32_t* __restrict__ elem,
                              const double* __restrict__ r, double* xo, double* Go, double* H2o) {
  __shared__ double z[16], scale[16];
  if (threadIdx.x < N) {
    z[threadIdx.x] = m.basis[FPX_BASIS_NODES(N, m.M) + threadIdx.x];
    scale[threadIdx.x] = m.basis[FPX_BASIS_SCALE(N, m.M) + threadIdx.x];
  }
  __syncthreads();
  constexpr int K = Pow<DR, N>::K;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const double* X = m.nodes + (int64_t)elem[q] * D * K;
    double v[DR][N], g[DR][N], h[DR][N];
    for (int a = 0; a < DR; ++a) lagrange<N, true>(z, scale, r[q * DR + a], v[a], g[a], h[a]);
    for (int c = 0; c < D; ++c) {
      double acc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
      for (int t = 0; t < K; ++t) {
        const int i = t % N, j = (t / N) % N, k = t / (N * N);
        const double xv = X[c * K + t];
        double fi[3] = {v[0][i], DR > 1 ? v[1][j] : 1.0, DR > 2 ? v[2][k] : 1.0};
        double di[3] = {g[0][i], DR > 1 ? g[1][j] : 0.0, DR > 2 ? g[2][k] : 0.0};
        double hi[3] = {h[0][i], DR > 1 ? h[1][j] : 0.0, DR > 2 ? h[2][k] : 0.0};
        acc[0] += xv * fi[0] * fi[1] * fi[2];
        acc[1] += xv * di[0] * fi[1] * fi[2];
        acc[2] += xv * fi[0] * di[1] * fi[2];
        acc[3] += xv * fi[0] * fi[1] * di[2];
        acc[4] += xv * hi[0] * fi[1] * fi[2];
        acc[5] += xv * fi[0] * hi[1] * fi[2];
        acc[6] += xv * fi[0] * fi[1] * hi[2];
        acc[7] += xv * di[0] * di[1] * fi[2];
        acc[8] += xv * di[0] * fi[1] * di[2];
        acc[9] += xv * fi[0] * di[1] * di[2];
      }
      xo[q * D + c] = acc[0];
      for (int a = 0; a < DR; ++a) Go[(q * D + c) * DR + a] = acc[1 + a];
      if (H2o)
        for (int t = 0; t < 6; ++t) H2o[(q * D + c) * 6 + t] = acc[4 + t];
    }
  }
}

inline unsigned persistent_blocks(const void* fn, int threads, size_t smem, int64_t work_warps) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem);
  if (per_sm < 1) per_sm = 1;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t cap = (int64_t)sms * per_sm;
  int64_t need = (work_warps + threads / FPX_WARP - 1) / (threads / FPX_WARP);
  if (need < 1) need = 1;
  return (unsigned)(need < cap ? need : cap);
}

inline size_t newton_smem(int geo, int fsz, int N, int wpb) {
  return (size_t)(2 * ((N + 1) & ~1) + wpb * (geo + fsz)) * sizeof(double);
}

template <int D, int DR, int N>
struct Stream {
  static constexpr int S = 3;
  static cudaError_t run(const fpx_mesh_t& m, const double* ux, const int4* umeta,
                         const uint64_t* packed_off, const int32_t* npass, int32_t* code,
                         int32_t* elem, double* r,
                         double* dist, int32_t* iters, const double* field, int C, double* values,
                         int32_t* upts, int64_t* nun_dev, int64_t* chunk_ctr, int64_t n_cap,
                         int4* redo, int64_t* nredo, int64_t redo_cap, int64_t* stats,
                         cudaStream_t st) {
    using L = Lay<D, DR, N>;
    constexpr int FRAME = DR == D ? D + D * D : 0;
    auto fn = k_newton_stream<D, DR, N, S>;
    // Slot configuration: the deepest ring (3 slots, field staged) that
    // still fits 8 resident warps per SM; at high order (p = 7: 16.5 KB per
    // slot) fewer slots and the field read from global memory at the final
    // evaluation instead, for more resident warps.
    int best_warps = -1, nslot = S, fstage = 0, ss = 0, wpb = 4;
    size_t smem = 0;
    for (int cfg = 0; cfg < 4; ++cfg) {
      const int ns = cfg < 2 ? 3 : 2;
      const int fs = (cfg % 2 == 0 && field) ? 1 : 0;
      if (cfg % 2 == 0 && !field) continue;
      int sst = L::GEO + ((FRAME + 1) & ~1) + (fs ? C * L::K + 2 : 0);
      sst = (sst + 13) / 16 * 16 + 2;  // slot stride = 16 bytes mod 128: distinct bank groups
      const size_t per_warp =
          (size_t)(ns * sst + StreamScratch<DR, N>::SLOTS * FPX_WARP) * 8 + sizeof(StreamMeta<S>);
      // (+ the metadata, static shared memory: one StreamMeta per warp)
      for (int w = 4; w >= 1; --w) {  // warps per CTA
        const size_t sm = (size_t)(2 * ((N + 1) & ~1)) * 8 + (size_t)w * per_warp;
        if (sm > 227 * 1024) continue;
        int warps_sm = (int)((228 * 1024) / (sm + 1024)) * w;
        if (warps_sm > 8) warps_sm = 8;  // 242 registers: at most 8 warps per SM
        if (warps_sm > best_warps) {
          best_warps = warps_sm;
          nslot = ns;
          fstage = fs;
          ss = sst;
          wpb = w;
          smem = sm;
        }
      }
    }
    if (best_warps < 0) return cudaErrorInvalidValue;
    const int threads = wpb * FPX_WARP;
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    // chunk: FPX_CHUNK_DEFAULT points, shrunk when the stream is too short to
    // give every resident warp a chunk (a sparse stream - about one point per
    // element - keeps at most S lanes of a warp busy, so its latency is the
    // per-warp point count, not the total)
    int chunk;
    {
      const int64_t warps = (int64_t)persistent_blocks((const void*)fn, threads, smem,
                                                       INT64_C(1) << 40) * wpb;
      const int64_t want = (n_cap + warps - 1) / (warps > 0 ? warps : 1);
      chunk = want < 1 ? 1 : want > FPX_CHUNK_DEFAULT ? FPX_CHUNK_DEFAULT : (int)want;
    }
    unsigned blocks = persistent_blocks((const void*)fn, threads, smem,
                                        (n_cap + chunk - 1) / chunk);
    fn<<<blocks, threads, smem, st>>>(m, ux, umeta, packed_off, npass, code, elem, r, dist,
                                      iters, field, C, values, upts, nun_dev, chunk_ctr, ss,
                                      nslot, fstage, chunk, redo, nredo, redo_cap, stats);
    return cudaGetLastError();
  }
};

template <int D, int DR, int N>
struct Pairs {
  static cudaError_t run(const fpx_mesh_t& m, const double* x, const int32_t* pair_pt,
                         const int32_t* sorted, const Item* items, const int64_t* nitems_dev,
                         int64_t items_cap, const double* r0, int32_t* pcode, double* pr,
                         double* pdist, int32_t* piters, int32_t* pconv, int64_t* stats,
                         cudaStream_t st) {
    using L = Lay<D, DR, N>;
    const int threads = 128;
    const size_t smem = newton_smem(L::GEO + Scratch<DR, N>::SLOTS * FPX_WARP, 0, N,
                                    threads / FPX_WARP);
    auto fn = k_newton_pairs<D, DR, N>;
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    unsigned blocks = persistent_blocks((const void*)fn, threads, smem, items_cap);
    fn<<<blocks, threads, smem, st>>>(m, x, pair_pt, sorted, items, nitems_dev, r0, pcode, pr,
                                      pdist, piters, pconv, stats);
    return cudaGetLastError();
  }
};

template <int D, int DR, int N>
struct Rest {
  static cudaError_t run(const fpx_mesh_t& m, const double* x, int64_t nun_cap,
                         const int64_t* nun_dev, const int32_t* upts, const int32_t* clist,
                         const int32_t* cnum, const int32_t* nps,
                         const int32_t* perm,
                         const int64_t* cum, const int32_t* maxnp, const int32_t* best,
                         const int4* pairs, const int64_t* npairs, int4* redo, int64_t* nredo,
                         int32_t* found, int32_t* lock, int32_t* code, int32_t* elem, double* r,
                         double* dist, int32_t* iters, const double* field, int C,
                         double* values, int64_t* counter, int64_t* stats, cudaStream_t st) {
    const int threads = 128;
    const size_t smem = (size_t)(2 * ((N + 1) & ~1) + 4 * Scratch<DR, N>::SLOTS * FPX_WARP) * 8;
    auto fn = k_rest_l1<D, DR, N>;
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    unsigned blocks = persistent_blocks((const void*)fn, threads, smem,
                                        (nun_cap + FPX_WARP - 1) / FPX_WARP);
    const int64_t cap = 2 * nun_cap + 1024;
    // Pass 1 stops candidates held on a face (descent direction leaving it)
    // for two consecutive iterations; pass 2 redoes every stopped candidate
    // (of round 1 and of pass 1) in full for points still without an
    // INTERIOR.  The records are those of the full solves either way.
    fn<<<blocks, threads, smem, st>>>(m, x, nun_dev, upts, clist, cnum, nps, perm, cum,
                                      maxnp, best, pairs, cap, npairs, 1, redo, nredo, found,
                                      lock, code, elem, r, dist, iters, counter, stats);
    fn<<<blocks, threads, smem, st>>>(m, x, nun_dev, upts, clist, cnum, nps, perm, cum,
                                      nullptr, best, redo, cap, nredo, 0, nullptr, nullptr,
                                      found, lock, code, elem, r, dist, iters, counter + 1, stats);
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess || !field) return err;
    int64_t b = (nun_cap + 127) / 128;
    if (b > 148 * 8) b = 148 * 8;
    if (b < 1) b = 1;
    k_rest_values<DR, N><<<(unsigned)b, 128, 0, st>>>(m.basis, m.M, nun_dev, upts, code, elem, r,
                                                      field, C, values, stats);
    return cudaGetLastError();
  }
  static cudaError_t lists(const fpx_mesh_t& m, const double* x, int64_t nun_cap,
                           const int64_t* nun_dev, const int32_t* upts, int32_t* best,
                           const int32_t* npass, int32_t* clist,
                           int32_t* cnum, int32_t* nps, int32_t* hist, int32_t* bstart,
                           int32_t* bcur, int32_t* perm, int64_t* cum, int32_t* maxnp,
                           int4* pairs, int64_t* npairs, cudaStream_t st) {
    int64_t b = (nun_cap + kRlGroups - 1) / kRlGroups;
    if (b > 148 * 16) b = 148 * 16;
    if (b < 1) b = 1;
    k_rest_lists<D><<<(unsigned)b, 128, 0, st>>>(m, x, nun_dev, upts, best, npass, clist, cnum,
                                                 nps, hist);
    k_rest_order<<<1, FPX_HMAX, 0, st>>>(hist, bstart, cum, maxnp, npairs);
    int64_t b2 = (nun_cap + 255) / 256;
    if (b2 > 148 * 8) b2 = 148 * 8;
    if (b2 < 1) b2 = 1;
    k_rest_scatter<<<(unsigned)b2, 256, 0, st>>>(nun_dev, nps, bstart, bcur, perm);
    k_rest_pairlist<<<(unsigned)b2, 256, 0, st>>>(nun_dev, upts, perm, nps, clist, cnum, cum, pairs,
                                                  2 * nun_cap + 1024);
    return cudaGetLastError();
  }
};

template <int D, int DR, int N>
struct FMap {
  static cudaError_t run(const fpx_mesh_t& m, int64_t n, const int32_t* elem, const double* r,
                         double* x, double* G, double* H2, cudaStream_t st) {
    int64_t b = (n + 127) / 128;
    if (b > 148 * 16) b = 148 * 16;
    if (b < 1) b = 1;
    k_forward_map<D, DR, N><<<(unsigned)b, 128, 0, st>>>(m, n, elem, r, x, G, H2);
    return cudaGetLastError();
  }
};

template <int DR, int N>
struct EvalRun {
  static cudaError_t run(const double* fbasis, int M, int C, const double* field,
                            const double* r, const int32_t* sorted, const Item* items,
                            const int64_t* nitems_dev, int64_t items_cap, double* values,
                            cudaStream_t st) {
  using L = Lay<1, DR, N>;
  const int threads = 128;
  const size_t smem = newton_smem(0, C * L::CS, N, threads / FPX_WARP);
  auto fn = k_eval_items<DR, N>;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  unsigned blocks = persistent_blocks((const void*)fn, threads, smem, items_cap);
  fn<<<blocks, threads, smem, st>>>(fbasis, M, C, field, r, sorted, items, nitems_dev, values);
  return cudaGetLastError();
}
};


}  // namespace fpx
