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

#include "fpx_common.cuh"
#include "fpx_kernels.cuh"

#ifndef FPX_NEWTON_MINB
#define FPX_NEWTON_MINB 2  // CTAs of 128 threads per SM the Newton kernels are built for
#endif

namespace fpx {

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
template <int D, int DR, int N, bool W2, bool GEO = false>
__device__ __forceinline__ void eval_state(const double* __restrict__ sX,
                                           const double* __restrict__ z,
                                           const double* __restrict__ scale, const double* r,
                                           const double* xs, NState& S, double* sb) {
  // GEO = false: geometry staged in shared memory, rows padded to NP;
  // GEO = true: geometry read in place from global memory ([d][N^dr]).
  using Lp = Lay<D, DR, N>;
  constexpr int GCS = GEO ? Lp::K : Lp::CS;
  constexpr int GNP = GEO ? N : Lp::NP;
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
#pragma unroll 1
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

__device__ __forceinline__ int symi(int a, int b) {
  return a == b ? a : (a + b == 1 ? 3 : (a + b == 2 ? 4 : 5));
}

// Cholesky solve on the active principal submatrix (oracle chol_solve):
// pivot must exceed 1e-14 |trace|.  A is symmetric-packed.
template <int DR>
__device__ __forceinline__ bool chol_solve(const double* A, const bool* act, const double* b,
                                           double* x) {
  double L[3][3], y[3], iL[3];
  double tr = 0.0;
#pragma unroll
  for (int k = 0; k < DR; ++k)
    if (act[k]) tr += A[k];
  const double thr = 1e-14 * fabs(tr);
#pragma unroll
  for (int k = 0; k < DR; ++k) {
    if (!act[k]) continue;
    double s = A[k];
#pragma unroll
    for (int m = 0; m < k; ++m)
      if (act[m]) s -= L[k][m] * L[k][m];
    if (!(s > thr)) return false;
    L[k][k] = sqrt(s);
    iL[k] = 1.0 / L[k][k];
#pragma unroll
    for (int i = k + 1; i < DR; ++i) {
      if (!act[i]) continue;
      double t = A[symi(i, k)];
#pragma unroll
      for (int m = 0; m < k; ++m)
        if (act[m]) t -= L[i][m] * L[k][m];
      L[i][k] = t * iL[k];
    }
  }
#pragma unroll
  for (int k = 0; k < DR; ++k) {
    if (!act[k]) continue;
    double t = b[k];
#pragma unroll
    for (int m = 0; m < k; ++m)
      if (act[m]) t -= L[k][m] * y[m];
    y[k] = t * iL[k];
  }
#pragma unroll
  for (int k = DR - 1; k >= 0; --k) {
    if (!act[k]) continue;
    double t = y[k];
#pragma unroll
    for (int m = k + 1; m < DR; ++m)
      if (act[m]) t -= L[m][k] * x[m];
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
      if (freem[a] && ((r[a] == 1.0 && y[a] > 0.0) || (r[a] == -1.0 && y[a] < 0.0))) {
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

template <int DR>
__device__ __forceinline__ bool on_boundary(const double* r) {
  bool b = false;
#pragma unroll
  for (int a = 0; a < DR; ++a) b |= (r[a] == -1.0) | (r[a] == 1.0);
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
template <int D, int DR, int N, bool GEO = false>
__device__ __forceinline__ NewtonOut newton_warp(const double* __restrict__ sX,
                                                 const double* __restrict__ z,
                                                 const double* __restrict__ scale,
                                                 const double* xs, bool active,
                                                 const NewtonParams& P, double* sb) {
  using L = Lay<D, DR, N>;
  double* stash = sb + Scratch<DR, N>::STASH * FPX_WARP;
  // seed: nearest GLL node, ties -> lowest lexicographic index (D7); the
  // distance is accumulated with fma exactly as the oracle does.
  double best = INFINITY;
  int bi = 0;
#pragma unroll 1
  for (int row = 0; row < L::ROWS; ++row) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double dd = 0.0;
#pragma unroll
      for (int c = 0; c < D; ++c) {
        const double xn = GEO ? __ldg(sX + c * L::K + row * N + i) : sX[c * L::CS + row * L::NP + i];
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
  // One evaluation site (the seed is evaluated as the first "trial") and one
  // constrained_step site (the Hessian fallbacks loop over it) keep the
  // kernel's code small: instruction fetch was the top stall when inlined.
  NState st;
  double rn[3] = {r[0], r[1], r[2]};
  double alpha = P.alpha0, fcur = 0.0, pred = 0.0, smax = 0.0;
  int it = 0;
  bool done = !active, conv = false, first = true, step = active;
  while (true) {
    if (__any_sync(FPX_FULL, step && on_boundary<DR>(rn)))
      eval_state<D, DR, N, true, GEO>(sX, z, scale, rn, xs, st, sb);
    else
      eval_state<D, DR, N, false, GEO>(sX, z, scale, rn, xs, st, sb);
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
        if ((r[a] == 1.0 && st.J[a] < 0.0) || (r[a] == -1.0 && st.J[a] > 0.0)) freem[a] = false;
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
      if (!(pred > 1e-15 * fcur)) {  // step below what |dx|^2 resolves
        conv = true;
        done = true;
      } else {
        step = true;
#pragma unroll
        for (int a = 0; a < DR; ++a) {
          double v = r[a] + s[a];
          if (hit & (1 << a)) v = s[a] > 0.0 ? 1.0 : -1.0;  // lands on the face
          v = v < -1.0 ? -1.0 : (v > 1.0 ? 1.0 : v);
          rn[a] = v;
        }
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
        const double* row = sU + (j + N * k) * NP;
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < N; ++i) s = fma(row[i], v[0][i], s);
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

// Round 1: every found point's best-first candidate.  Final for INTERIOR or
// single-candidate points (fused field evaluation); otherwise a tentative
// BORDER record and the point joins the exhaustive round 2.
template <int D, int DR, int N>
__global__ void __launch_bounds__(128, FPX_NEWTON_MINB)
    k_newton_round1(fpx_mesh_t m, const double* __restrict__ x, const int32_t* __restrict__ sorted,
                    const Item* __restrict__ items, const int64_t* __restrict__ nitems_dev,
                    const int32_t* __restrict__ npass, int32_t* code, int32_t* elem, double* r,
                    double* dist, int32_t* iters, const double* __restrict__ field, int C,
                    double* values, int32_t* upts, int64_t* upair_cnt, int64_t* nun_dev,
                    int64_t* stats) {
  using L = Lay<D, DR, N>;
  extern __shared__ __align__(16) double smem[];
  double* z = smem;
  double* scale = smem + N;
  const int warp = threadIdx.x / FPX_WARP, lane = threadIdx.x % FPX_WARP;
  const int wpb = blockDim.x / FPX_WARP;
  const int fsz = field ? C * L::CS : 0;
  constexpr int SCR = Scratch<DR, N>::SLOTS * FPX_WARP;
  double* sX = smem + 2 * ((N + 1) & ~1) + warp * (L::GEO + SCR + fsz);
  double* sb = sX + L::GEO + lane;
  double* sU = sX + L::GEO + SCR;
  if (threadIdx.x < N) {
    z[threadIdx.x] = m.basis[FPX_BASIS_NODES(N, m.M) + threadIdx.x];
    scale[threadIdx.x] = m.basis[FPX_BASIS_SCALE(N, m.M) + threadIdx.x];
  }
  __syncthreads();
  const NewtonParams P = newton_of(m);
  const int64_t nitems = *nitems_dev;
  int64_t s_newton = 0, s_iters = 0, s_evals = 0;
  for (int64_t w = (int64_t)blockIdx.x * wpb + warp; w < nitems; w += (int64_t)gridDim.x * wpb) {
    const Item itm = items[w];
    const int e = itm.elem;
    stage_block<DR, N>(sX, m.nodes + (int64_t)e * D * L::K, D, lane);
    if (field) stage_block<DR, N>(sU, field + (int64_t)e * C * L::K, C, lane);
    cp_async_wait_all();
    __syncwarp();
    const bool active = lane < itm.count;
    const int pt = active ? sorted[itm.start + lane] : 0;
    double xs[3] = {0.0, 0.0, 0.0};
    if (active)
#pragma unroll
      for (int c = 0; c < D; ++c) xs[c] = x[(int64_t)pt * D + c];
    NewtonOut o = newton_warp<D, DR, N>(sX, z, scale, xs, active, P, sb);
    if (active) {
      s_newton += 1;
      s_iters += o.iters;
      const double epsd = DR < D ? eps_d_of(m, e) : 0.0;
      const int cd = classify<D, DR>(o.r, o.dist, epsd);
      const bool final = cd == kInterior || npass[pt] <= 1;
      code[pt] = cd;
      elem[pt] = e;
#pragma unroll
      for (int a = 0; a < DR; ++a) r[(int64_t)pt * DR + a] = o.r[a];
      dist[pt] = o.dist;
      if (iters) iters[pt] = o.iters;
      if (final) {
        if (field) {
          double v[DR][N];
          basis_values<DR, N>(z, scale, o.r, v);
          for (int c = 0; c < C; ++c) values[(int64_t)pt * C + c] = contract_smem<DR, N>(sU + c * L::CS, v);
          ++s_evals;
        }
      } else {
        const int slot = (int)atomicAdd((unsigned long long*)nun_dev, 1ull);
        upts[slot] = pt;
        upair_cnt[slot] = npass[pt] - 1;
      }
    }
    __syncwarp();
  }
  s_newton = warp_sum64(s_newton);
  s_iters = warp_sum64(s_iters);
  s_evals = warp_sum64(s_evals);
  if (lane == 0) {
    atomicAdd((unsigned long long*)&stats[FPX_STAT_NEWTON], (unsigned long long)s_newton);
    atomicAdd((unsigned long long*)&stats[FPX_STAT_ITERS], (unsigned long long)s_iters);
    atomicAdd((unsigned long long*)&stats[FPX_STAT_EVALS], (unsigned long long)s_evals);
    atomicAdd((unsigned long long*)&stats[FPX_STAT_NEWTON_R1], (unsigned long long)s_newton);
    atomicAdd((unsigned long long*)&stats[FPX_STAT_ITERS_R1], (unsigned long long)s_iters);
    atomicAdd((unsigned long long*)&stats[FPX_STAT_EVALS_R1], (unsigned long long)s_evals);
  }
}

// Round 2 (and fpx_invert_pairs): Newton per explicit (point, element) pair.
template <int D, int DR, int N>
__global__ void __launch_bounds__(128, FPX_NEWTON_MINB)
    k_newton_pairs(fpx_mesh_t m, const double* __restrict__ x, const int32_t* __restrict__ pair_pt,
                   const int32_t* __restrict__ sorted, const Item* __restrict__ items,
                   const int64_t* __restrict__ nitems_dev, int32_t* pcode, double* pr,
                   double* pdist, int32_t* piters, int32_t* pconv, int64_t* stats) {
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
    double xs[3] = {0.0, 0.0, 0.0};
    if (active)
#pragma unroll
      for (int c = 0; c < D; ++c) xs[c] = x[(int64_t)pt * D + c];
    NewtonOut o = newton_warp<D, DR, N>(sX, z, scale, xs, active, P, sb);
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

// Sparse rounds (2 and 3): one (point, element) pair per lane, geometry read
// in place from global memory (L1/L2) -- no element grouping.  The rounds
// carry ~1 pair per element, where the element-major mapping would leave a
// warp with one active lane.
template <int D, int DR, int N>
__global__ void __launch_bounds__(128, FPX_NEWTON_MINB)
    k_newton_sparse(fpx_mesh_t m, const double* __restrict__ x,
                    const int32_t* __restrict__ pair_pt, const int32_t* __restrict__ pair_elem,
                    const int64_t* __restrict__ npairs_dev, int32_t* pcode, double* pr,
                    double* pdist, int32_t* piters, int64_t* stats) {
  using L = Lay<D, DR, N>;
  extern __shared__ __align__(16) double smem[];
  double* z = smem;
  double* scale = smem + N;
  const int warp = threadIdx.x / FPX_WARP, lane = threadIdx.x % FPX_WARP;
  const int wpb = blockDim.x / FPX_WARP;
  constexpr int SCR = Scratch<DR, N>::SLOTS * FPX_WARP;
  double* sb = smem + 2 * ((N + 1) & ~1) + warp * SCR + lane;
  if (threadIdx.x < N) {
    z[threadIdx.x] = m.basis[FPX_BASIS_NODES(N, m.M) + threadIdx.x];
    scale[threadIdx.x] = m.basis[FPX_BASIS_SCALE(N, m.M) + threadIdx.x];
  }
  __syncthreads();
  const NewtonParams P = newton_of(m);
  const int64_t npairs = *npairs_dev;
  int64_t s_newton = 0, s_iters = 0;
  // whole warps stride over the pairs so every lane reaches the shuffles
  for (int64_t base = ((int64_t)blockIdx.x * wpb + warp) * FPX_WARP; base < npairs;
       base += (int64_t)gridDim.x * wpb * FPX_WARP) {
    const int64_t p = base + lane;
    const int e = p < npairs ? pair_elem[p] : -1;
    const bool active = e >= 0;
    const int pt = active ? pair_pt[p] : 0;
    double xs[3] = {0.0, 0.0, 0.0};
    if (active)
#pragma unroll
      for (int c = 0; c < D; ++c) xs[c] = x[(int64_t)pt * D + c];
    const double* X = m.nodes + (int64_t)(active ? e : 0) * D * L::K;
    NewtonOut o = newton_warp<D, DR, N, true>(X, z, scale, xs, active, P, sb);
    if (active) {
      s_newton += 1;
      s_iters += o.iters;
      const double epsd = DR < D ? eps_d_of(m, e) : 0.0;
      pcode[p] = classify<D, DR>(o.r, o.dist, epsd);
#pragma unroll
      for (int a = 0; a < DR; ++a) pr[p * DR + a] = o.r[a];
      pdist[p] = o.dist;
      if (piters) piters[p] = o.iters;
    }
  }
  s_newton = warp_sum64(s_newton);
  s_iters = warp_sum64(s_iters);
  if (lane == 0) {
    atomicAdd((unsigned long long*)&stats[FPX_STAT_NEWTON], (unsigned long long)s_newton);
    atomicAdd((unsigned long long*)&stats[FPX_STAT_ITERS], (unsigned long long)s_iters);
  }
}

// Merge of a round's pairs into the points' records (winner rule D6 over the
// current record and the pairs: INTERIOR (lowest id) > min d* (ties lowest
// id)).  pair_off == NULL: one pair per point at index u (next-best round).
// Points still unresolved that have more than `min_pass` passing candidates
// go to the next round when next_upts != NULL; all others are final and get
// their field value.
template <int D, int DR, int N>
__global__ void k_round2_finalize(fpx_mesh_t m, const int64_t* __restrict__ nun_dev,
                                  const int32_t* __restrict__ upts,
                                  const int64_t* __restrict__ pair_off, int64_t pair_cap,
                                  const int32_t* __restrict__ pair_elem,
                                  const int32_t* __restrict__ pcode, const double* __restrict__ pr,
                                  const double* __restrict__ pdist,
                                  const int32_t* __restrict__ piters, int32_t* code, int32_t* elem,
                                  double* r, double* dist, int32_t* iters,
                                  const double* __restrict__ field, int C, double* values,
                                  const int32_t* __restrict__ npass, int min_pass,
                                  int32_t* next_upts, int64_t* next_cnt, int64_t* nnext,
                                  int64_t* stats) {
  __shared__ double z[16], scale[16];
  if (threadIdx.x < N) {
    z[threadIdx.x] = m.basis[FPX_BASIS_NODES(N, m.M) + threadIdx.x];
    scale[threadIdx.x] = m.basis[FPX_BASIS_SCALE(N, m.M) + threadIdx.x];
  }
  __syncthreads();
  const int64_t nun = *nun_dev;
  int64_t s_evals = 0;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < nun;
       u += (int64_t)gridDim.x * blockDim.x) {
    const int k = upts[u];
    int bc = code[k], be = elem[k];
    double bd = dist[k];
    double br[3] = {0, 0, 0};
    for (int a = 0; a < DR; ++a) br[a] = r[(int64_t)k * DR + a];
    int it = iters ? iters[k] : 0;
    const int64_t p0 = pair_off ? pair_off[u] : u, p1 = pair_off ? pair_off[u + 1] : u + 1;
    for (int64_t p = p0; p < p1 && p < pair_cap; ++p) {
      const int e = pair_elem[p];
      if (e < 0) continue;
      const int c = pcode[p];
      const double dd = pdist[p];
      if (piters) it += piters[p];
      bool take;
      if (c == kInterior) take = bc != kInterior || e < be;
      else take = bc != kInterior && (dd < bd || (dd == bd && e < be));
      if (take) {
        bc = c;
        be = e;
        bd = dd;
        for (int a = 0; a < DR; ++a) br[a] = pr[p * DR + a];
      }
    }
    code[k] = bc;
    elem[k] = be;
    dist[k] = bd;
    for (int a = 0; a < DR; ++a) r[(int64_t)k * DR + a] = br[a];
    if (iters) iters[k] = it;
    if (next_upts && bc != kInterior && npass[k] > min_pass) {
      const int slot = (int)atomicAdd((unsigned long long*)nnext, 1ull);
      next_upts[slot] = k;
      next_cnt[slot] = npass[k] - min_pass;
      continue;
    }
    if (field) {
      double v[DR][N];
      basis_values<DR, N>(z, scale, br, v);
      for (int c = 0; c < C; ++c)
        values[(int64_t)k * C + c] =
            contract_gmem<DR, N>(field + ((int64_t)be * C + c) * Pow<DR, N>::K, v);
      ++s_evals;
    }
  }
  if (field && s_evals)
    atomicAdd((unsigned long long*)&stats[FPX_STAT_EVALS], (unsigned long long)s_evals);
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
struct Round1 {
  static cudaError_t run(const fpx_mesh_t& m, const double* x, const int32_t* sorted,
                         const Item* items, const int64_t* nitems_dev, int64_t items_cap,
                         const int32_t* npass, int32_t* code, int32_t* elem, double* r,
                         double* dist, int32_t* iters, const double* field, int C, double* values,
                         int32_t* upts, int64_t* upair_cnt, int64_t* nun_dev, int64_t* stats,
                         cudaStream_t st) {
    using L = Lay<D, DR, N>;
    const int threads = 128;
    const size_t smem = newton_smem(L::GEO + Scratch<DR, N>::SLOTS * FPX_WARP,
                                    field ? C * L::CS : 0, N, threads / FPX_WARP);
    auto fn = k_newton_round1<D, DR, N>;
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    unsigned blocks = persistent_blocks((const void*)fn, threads, smem, items_cap);
    fn<<<blocks, threads, smem, st>>>(m, x, sorted, items, nitems_dev, npass, code, elem, r, dist,
                                      iters, field, C, values, upts, upair_cnt, nun_dev, stats);
    return cudaGetLastError();
  }
};

template <int D, int DR, int N>
struct Pairs {
  static cudaError_t run(const fpx_mesh_t& m, const double* x, const int32_t* pair_pt,
                         const int32_t* sorted, const Item* items, const int64_t* nitems_dev,
                         int64_t items_cap, int32_t* pcode, double* pr, double* pdist,
                         int32_t* piters, int32_t* pconv, int64_t* stats, cudaStream_t st) {
    using L = Lay<D, DR, N>;
    const int threads = 128;
    const size_t smem = newton_smem(L::GEO + Scratch<DR, N>::SLOTS * FPX_WARP, 0, N,
                                    threads / FPX_WARP);
    auto fn = k_newton_pairs<D, DR, N>;
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    unsigned blocks = persistent_blocks((const void*)fn, threads, smem, items_cap);
    fn<<<blocks, threads, smem, st>>>(m, x, pair_pt, sorted, items, nitems_dev, pcode, pr, pdist,
                                      piters, pconv, stats);
    return cudaGetLastError();
  }
};

template <int D, int DR, int N>
struct Sparse {
  static cudaError_t run(const fpx_mesh_t& m, const double* x, const int32_t* pair_pt,
                         const int32_t* pair_elem, const int64_t* npairs_dev, int64_t cap,
                         int32_t* pcode, double* pr, double* pdist, int32_t* piters,
                         int64_t* stats, cudaStream_t st) {
    const int threads = 128;
    const size_t smem = newton_smem(Scratch<DR, N>::SLOTS * FPX_WARP, 0, N, threads / FPX_WARP);
    auto fn = k_newton_sparse<D, DR, N>;
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    unsigned blocks = persistent_blocks((const void*)fn, threads, smem,
                                        (cap + FPX_WARP - 1) / FPX_WARP);
    fn<<<blocks, threads, smem, st>>>(m, x, pair_pt, pair_elem, npairs_dev, pcode, pr, pdist,
                                      piters, stats);
    return cudaGetLastError();
  }
};

template <int D, int DR, int N>
struct Finalize {
  static cudaError_t run(const fpx_mesh_t& m, int64_t nun_cap, const int64_t* nun_dev,
                         const int32_t* upts, const int64_t* pair_off, int64_t pair_cap,
                         const int32_t* pair_elem, const int32_t* pcode, const double* pr,
                         const double* pdist, const int32_t* piters, int32_t* code, int32_t* elem,
                         double* r, double* dist, int32_t* iters, const double* field, int C,
                         double* values, const int32_t* npass, int min_pass, int32_t* next_upts,
                         int64_t* next_cnt, int64_t* nnext, int64_t* stats, cudaStream_t st) {
    int64_t b = (nun_cap + 127) / 128;
    if (b > 148 * 16) b = 148 * 16;
    if (b < 1) b = 1;
    k_round2_finalize<D, DR, N><<<(unsigned)b, 128, 0, st>>>(
        m, nun_dev, upts, pair_off, pair_cap, pair_elem, pcode, pr, pdist, piters, code, elem, r,
        dist, iters, field, C, values, npass, min_pass, next_upts, next_cnt, nnext, stats);
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
