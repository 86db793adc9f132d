// fpx_exact.cu -- setup bounds, local hash map and the find prefilter.
//
// Compiled with --fmad=false: every multiply and add is rounded separately,
// as the numpy reference evaluates them, so the per-element AABB/OBB, the
// hash boxes, cell_of and the AABB/OBB membership tests are bit-identical to
// the oracle given identical basis constants.
#include <climits>
#include <math.h>

#include "fpx_common.cuh"
#include "fpx_kernels.cuh"
#include "fpx_boxes.cuh"

namespace fpx {

// ------------------------------------------------------------ basis views
struct BasisView {
  const double *z, *scale, *proj0, *proj1, *eta, *lo, *hi;
  int N, M;
  __device__ BasisView(const double* b, int N_, int M_) : N(N_), M(M_) {
    z = b + FPX_BASIS_NODES(N_, M_);
    scale = b + FPX_BASIS_SCALE(N_, M_);
    proj0 = b + FPX_BASIS_PROJ0(N_, M_);
    proj1 = b + FPX_BASIS_PROJ1(N_, M_);
    eta = b + FPX_BASIS_ETA(N_, M_);
    lo = b + FPX_BASIS_LO(N_, M_);
    hi = b + FPX_BASIS_HI(N_, M_);
  }
};

// Runtime-N Lagrange values and first derivatives (basis.py:138-198), used
// by the setup frame (r = 0) only.
__device__ void lagrange_rt(const BasisView& B, double r, double* v, double* g) {
  const int N = B.N;
  double pv[FPX_SETUP_MAXN + 1], pd[FPX_SETUP_MAXN + 1];
  double sv[FPX_SETUP_MAXN + 1], sd[FPX_SETUP_MAXN + 1];
  pv[0] = 1.0; pd[0] = 0.0; sv[N] = 1.0; sd[N] = 0.0;
  for (int k = 0; k < N; ++k) {
    double u = r - B.z[k];
    pd[k + 1] = pd[k] * u + pv[k];
    pv[k + 1] = pv[k] * u;
  }
  for (int k = N - 1; k >= 0; --k) {
    double u = r - B.z[k];
    sd[k] = sd[k + 1] * u + sv[k + 1];
    sv[k] = sv[k + 1] * u;
  }
  for (int i = 0; i < N; ++i) {
    v[i] = (pv[i] * sv[i + 1]) * B.scale[i];
    g[i] = (pd[i] * sv[i + 1] + pv[i] * sd[i + 1]) * B.scale[i];
  }
}

// Sequential contraction, axis 0 first (basis.py:285-303 order).
__device__ double contract_rt(const double* X, int N, int dr, const double* f0,
                              const double* f1, const double* f2) {
  if (dr == 1) {
    double s = 0.0;
    for (int i = 0; i < N; ++i) s += X[i] * f0[i];
    return s;
  }
  if (dr == 2) {
    double t = 0.0;
    for (int j = 0; j < N; ++j) {
      double s = 0.0;
      for (int i = 0; i < N; ++i) s += X[i + N * j] * f0[i];
      t += s * f1[j];
    }
    return t;
  }
  double q = 0.0;
  for (int k = 0; k < N; ++k) {
    double t = 0.0;
    for (int j = 0; j < N; ++j) {
      double s = 0.0;
      for (int i = 0; i < N; ++i) s += X[i + N * j + N * N * k] * f0[i];
      t += s * f1[j];
    }
    q += t * f2[k];
  }
  return q;
}

__device__ double det_n(int d, const double m[3][3]) {
  if (d == 2) return m[0][0] * m[1][1] - m[0][1] * m[1][0];
  return m[0][0] * (m[1][1] * m[2][2] - m[1][2] * m[2][1]) -
         m[0][1] * (m[1][0] * m[2][2] - m[1][2] * m[2][0]) +
         m[0][2] * (m[1][0] * m[2][1] - m[1][1] * m[2][0]);
}

__device__ void inv_n(int d, const double m[3][3], double o[3][3]) {
  double det = det_n(d, m);
  if (d == 2) {
    o[0][0] = m[1][1] / det; o[0][1] = -m[0][1] / det;
    o[1][0] = -m[1][0] / det; o[1][1] = m[0][0] / det;
    return;
  }
  o[0][0] = (m[1][1] * m[2][2] - m[1][2] * m[2][1]) / det;
  o[0][1] = (m[0][2] * m[2][1] - m[0][1] * m[2][2]) / det;
  o[0][2] = (m[0][1] * m[1][2] - m[0][2] * m[1][1]) / det;
  o[1][0] = (m[1][2] * m[2][0] - m[1][0] * m[2][2]) / det;
  o[1][1] = (m[0][0] * m[2][2] - m[0][2] * m[2][0]) / det;
  o[1][2] = (m[0][2] * m[1][0] - m[0][0] * m[1][2]) / det;
  o[2][0] = (m[1][0] * m[2][1] - m[1][1] * m[2][0]) / det;
  o[2][1] = (m[0][1] * m[2][0] - m[0][0] * m[2][1]) / det;
  o[2][2] = (m[0][0] * m[1][1] - m[0][1] * m[1][0]) / det;
}

__device__ void matmul_n(int d, const double a[3][3], const double b[3][3], double o[3][3]) {
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) {
      double s = 0.0;
      for (int k = 0; k < d; ++k) s += a[i][k] * b[k][j];
      o[i][j] = s;
    }
}

__device__ void rodrigues(const double k_in[3], double sk, double ck, double R[3][3]) {
  double k[3] = {k_in[0] / sk, k_in[1] / sk, k_in[2] / sk};
  double kx[3][3] = {{0, -k[2], k[1]}, {k[2], 0, -k[0]}, {-k[1], k[0], 0}};
  double kk[3][3];
  matmul_n(3, kx, kx, kk);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      R[i][j] = (i == j ? 1.0 : 0.0) + sk * kx[i][j] + (1.0 - ck) * kk[i][j];
}

// _rotation_to_x (bounds.py:300-323).
__device__ int rotation_to_x(int d, const double* tin, double R[3][3]) {
  double nt = 0.0;
  for (int c = 0; c < d; ++c) nt += tin[c] * tin[c];
  nt = sqrt(nt);
  if (nt == 0.0) return -1;
  double t[3] = {0, 0, 0};
  for (int c = 0; c < d; ++c) t[c] = tin[c] / nt;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) R[i][j] = 0.0;
  if (d == 2) {
    R[0][0] = t[0]; R[0][1] = t[1]; R[1][0] = -t[1]; R[1][1] = t[0];
    return 0;
  }
  double k[3] = {0.0, t[2], -t[1]};
  double sk = sqrt(k[0] * k[0] + k[1] * k[1] + k[2] * k[2]);
  double ck = t[0];
  if (sk < 1e-14) {
    if (ck > 0.0) { R[0][0] = R[1][1] = R[2][2] = 1.0; }
    else { R[0][0] = -1.0; R[1][1] = -1.0; R[2][2] = 1.0; }
    return 0;
  }
  rodrigues(k, sk, ck, R);
  return 0;
}

// _rotation_normal_to_z (bounds.py:326-338).
__device__ int rotation_normal_to_z(const double* nin, double R[3][3]) {
  double nn = sqrt(nin[0] * nin[0] + nin[1] * nin[1] + nin[2] * nin[2]);
  if (nn == 0.0) return -1;
  double n[3] = {nin[0] / nn, nin[1] / nn, nin[2] / nn};
  double k[3] = {n[1], -n[0], 0.0};
  double sk = sqrt(k[0] * k[0] + k[1] * k[1] + k[2] * k[2]);
  double ck = n[2];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) R[i][j] = 0.0;
  if (sk < 1e-14) {
    if (ck > 0.0) { R[0][0] = R[1][1] = R[2][2] = 1.0; }
    else { R[0][0] = 1.0; R[1][1] = -1.0; R[2][2] = -1.0; }
    return 0;
  }
  rodrigues(k, sk, ck, R);
  return 0;
}

// center_map_and_jacobian + _center_frame (bounds.py:97-107, 341-363):
// returns 0 and (x_c, M) or -1 (SingularTransformError).
__device__ int center_frame(const BasisView& B, int d, int dr, const double* X, double* xc,
                            double Mf[3][3]) {
  const int N = B.N;
  const int K = dr == 1 ? N : (dr == 2 ? N * N : N * N * N);
  double v0[FPX_SETUP_MAXN], d0[FPX_SETUP_MAXN];
  lagrange_rt(B, 0.0, v0, d0);
  double jac[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  for (int c = 0; c < d; ++c) {
    xc[c] = contract_rt(X + c * K, N, dr, v0, v0, v0);
    for (int a = 0; a < dr; ++a) {
      const double* f0 = a == 0 ? d0 : v0;
      const double* f1 = a == 1 ? d0 : v0;
      const double* f2 = a == 2 ? d0 : v0;
      jac[c][a] = contract_rt(X + c * K, N, dr, f0, f1, f2);
    }
  }
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) Mf[i][j] = 0.0;
  if (dr == d) {
    double det = det_n(d, jac);
    double scale = 1.0;
    for (int a = 0; a < d; ++a) {
      double s = 0.0;
      for (int c = 0; c < d; ++c) s += jac[c][a] * jac[c][a];
      scale *= sqrt(s);
    }
    if (fabs(det) < 1e-13 * (scale > 1e-300 ? scale : 1e-300)) return -1;
    for (int i = 0; i < d; ++i)
      for (int j = 0; j < d; ++j) Mf[i][j] = jac[i][j];
    return 0;
  }
  double rot[3][3];
  if (dr == 1) {
    double t[3] = {jac[0][0], jac[1][0], d == 3 ? jac[2][0] : 0.0};
    if (rotation_to_x(d, t, rot)) return -1;
    inv_n(d, rot, Mf);
    return 0;
  }
  double t1[3] = {jac[0][0], jac[1][0], jac[2][0]};
  double t2[3] = {jac[0][1], jac[1][1], jac[2][1]};
  double nv[3] = {t1[1] * t2[2] - t1[2] * t2[1], t1[2] * t2[0] - t1[0] * t2[2],
                  t1[0] * t2[1] - t1[1] * t2[0]};
  double r1[3][3];
  if (rotation_normal_to_z(nv, r1)) return -1;
  double a[3][3];
  for (int i = 0; i < 3; ++i) {
    a[i][0] = r1[i][0] * t1[0] + r1[i][1] * t1[1] + r1[i][2] * t1[2];
    a[i][1] = r1[i][0] * t2[0] + r1[i][1] * t2[1] + r1[i][2] * t2[2];
    a[i][2] = (i == 2) ? 1.0 : 0.0;
  }
  if (fabs(det_n(3, a)) < 1e-14) return -1;
  double ai[3][3];
  inv_n(3, a, ai);
  matmul_n(3, ai, r1, rot);
  inv_n(3, rot, Mf);
  return 0;
}

// _expand_box (bounds.py:236-250); -1 for a degenerate element.
__device__ int expand_box(int d, double* lo, double* hi, double factor) {
  double ext[3], pad[3];
  double mx = -INFINITY;
  for (int c = 0; c < d; ++c) {
    ext[c] = hi[c] - lo[c];
    if (ext[c] > mx) mx = ext[c];
  }
  if (mx <= 0.0) return -1;
  int anyflat = 0;
  double minlive = INFINITY;
  for (int c = 0; c < d; ++c) {
    pad[c] = factor * ext[c];
    if (ext[c] < FPX_ZERO_EXTENT_REL * mx) anyflat = 1;
    else if (ext[c] < minlive) minlive = ext[c];
  }
  if (anyflat)
    for (int c = 0; c < d; ++c)
      if (ext[c] < FPX_ZERO_EXTENT_REL * mx) pad[c] = factor * minlive;
  for (int c = 0; c < d; ++c) {
    lo[c] -= 0.5 * pad[c];
    hi[c] += 0.5 * pad[c];
  }
  return 0;
}

// Number of (face|edge|patch, coordinate) bound tasks and whether they are
// 2D tensor bounds (_coordinate_bounds, bounds.py:253-289).
__device__ __forceinline__ int n_faces(int d, int dr) {
  if (dr == 1) return 1;
  if (dr == 2) return d == 2 ? 4 : 1;
  return 6;
}
__device__ __forceinline__ bool faces_2d(int d, int dr) { return dr == 3 || (dr == 2 && d == 3); }

// Flat node index of the t-th entry (t = a + N*b for 2D faces) of face f.
__device__ __forceinline__ int face_node(int d, int dr, int N, int f, int t) {
  if (dr == 1) return t;
  if (dr == 2 && d == 2) {  // edges: j=0, j=N-1, i=0, i=N-1 (bounds.py:276-278)
    if (f == 0) return t;
    if (f == 1) return t + N * (N - 1);
    if (f == 2) return N * t;
    return N * t + N - 1;
  }
  if (dr == 2) return t;  // whole patch
  const int a = t % N, b = t / N;
  const int fix = (f & 1) ? N - 1 : 0;  // faces k=0,k=N-1,j=0,j=N-1,i=0,i=N-1
  if (f < 2) return a + N * b + N * N * fix;
  if (f < 4) return a + N * fix + N * N * b;
  return fix + N * a + N * N * b;
}

struct SetupSmemLayout {
  // per CTA: basis (FPX_BASIS_SIZE), per warp: X (d*K), u (N*N), alo/ahi (2*N*M)
  static __host__ __device__ size_t per_warp(int d, int K, int N, int M) {
    return (size_t)d * K + (size_t)N * N + 2 * (size_t)N * M + 16;
  }
};

// Accumulate lane-partial min/max of one bound function into (lo, hi).
// 1D: bound_function_1d (bounds.py:155-171); 2D: bound_function_2d
// (bounds.py:174-201).  u in shared memory (N or N*N values), a* scratch.
__device__ void bound_task(const BasisView& B, bool two_d, const double* u, double* alo,
                           double* ahi, int lane, double& lo, double& hi) {
  const int N = B.N, M = B.M;
  if (!two_d) {
    double a0 = 0.0, a1 = 0.0;
    for (int i = 0; i < N; ++i) { a0 += u[i] * B.proj0[i]; a1 += u[i] * B.proj1[i]; }
    for (int j = lane; j < M; j += FPX_WARP) {
      double slo = 0.0, shi = 0.0;
      for (int i = 0; i < N; ++i) {
        double w = u[i] - a0 - a1 * B.z[i];
        double tl = w * B.lo[i * M + j], th = w * B.hi[i * M + j];
        double mn = tl < th ? tl : th, mx = tl > th ? tl : th;
        if (i == 0) { slo = mn; shi = mx; } else { slo += mn; shi += mx; }
      }
      double lin = a0 + a1 * B.eta[j];
      double L = lin + slo, U = lin + shi;
      lo = L < lo ? L : lo;
      hi = U > hi ? U : hi;
    }
    return;
  }
  for (int t = lane; t < N * M; t += FPX_WARP) {
    const int j = t / M, k = t % M;
    double slo = 0.0, shi = 0.0;
    for (int i = 0; i < N; ++i) {
      double uij = u[i + N * j];
      double tl = uij * B.lo[i * M + k], th = uij * B.hi[i * M + k];
      double mn = tl < th ? tl : th, mx = tl > th ? tl : th;
      if (i == 0) { slo = mn; shi = mx; } else { slo += mn; shi += mx; }
    }
    alo[j * M + k] = slo;
    ahi[j * M + k] = shi;
  }
  __syncwarp();
  for (int t = lane; t < M * M; t += FPX_WARP) {
    const int k = t / M, l = t % M;
    double slo = 0.0, shi = 0.0;
    for (int j = 0; j < N; ++j) {
      double al = alo[j * M + k], ah = ahi[j * M + k];
      double vl = B.lo[j * M + l], vh = B.hi[j * M + l];
      double c0 = al * vl, c1 = al * vh, c2 = ah * vl, c3 = ah * vh;
      double mn = c0, mx = c0;
      mn = c1 < mn ? c1 : mn; mn = c2 < mn ? c2 : mn; mn = c3 < mn ? c3 : mn;
      mx = c1 > mx ? c1 : mx; mx = c2 > mx ? c2 : mx; mx = c3 > mx ? c3 : mx;
      if (j == 0) { slo = mn; shi = mx; } else { slo += mn; shi += mx; }
    }
    lo = slo < lo ? slo : lo;
    hi = shi > hi ? shi : hi;
  }
  __syncwarp();
}

__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double w = __shfl_xor_sync(FPX_FULL, v, o);
    v = w < v ? w : v;
  }
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double w = __shfl_xor_sync(FPX_FULL, v, o);
    v = w > v ? w : v;
  }
  return v;
}

// Raw (unexpanded) per-axis coordinate bounds of the element, or of its
// pull-back through (xc, Mi) when local != 0 (_coordinate_bounds).
__device__ void coordinate_bounds(const BasisView& B, int d, int dr, const double* X,
                                  bool local, const double* xc, const double Mi[3][3],
                                  double* u, double* alo, double* ahi, int lane, double* lo,
                                  double* hi) {
  const int N = B.N;
  const int K = dr == 1 ? N : (dr == 2 ? N * N : N * N * N);
  const bool two = faces_2d(d, dr);
  const int nf = n_faces(d, dr);
  const int fsize = two ? N * N : N;
  for (int c = 0; c < d; ++c) { lo[c] = INFINITY; hi[c] = -INFINITY; }
  for (int f = 0; f < nf; ++f)
    for (int c = 0; c < d; ++c) {
      for (int t = lane; t < fsize; t += FPX_WARP) {
        int n = face_node(d, dr, N, f, t);
        double val;
        if (!local) {
          val = X[c * K + n];
        } else {
          double s = 0.0;
          for (int b = 0; b < d; ++b) s += Mi[c][b] * (X[b * K + n] - xc[b]);
          val = s;
        }
        u[t] = val;
      }
      __syncwarp();
      bound_task(B, two, u, alo, ahi, lane, lo[c], hi[c]);
      __syncwarp();
    }
  for (int c = 0; c < d; ++c) {
    lo[c] = warp_min(lo[c]);
    hi[c] = warp_max(hi[c]);
  }
}

// One warp per element: AABB, OBB, hash box (D5) and centre frame.
__global__ void k_setup_bounds(int d, int dr, int N, int M, int64_t E,
                               const double* __restrict__ basis, const double* __restrict__ nodes,
                               double expansion, double* aabb, double* obb_c, double* obb_inv,
                               double* hbox, double* frame, uint8_t* obb_ok, int32_t* status) {
  extern __shared__ double smem[];
  const int K = dr == 1 ? N : (dr == 2 ? N * N : N * N * N);
  const int bsize = FPX_BASIS_SIZE(N, M);
  double* sB = smem;
  for (int t = threadIdx.x; t < bsize; t += blockDim.x) sB[t] = basis[t];
  __syncthreads();
  BasisView B(sB, N, M);
  const int warp = threadIdx.x / FPX_WARP, lane = threadIdx.x % FPX_WARP;
  const int wpb = blockDim.x / FPX_WARP;
  double* W = smem + bsize + warp * SetupSmemLayout::per_warp(d, K, N, M);
  double* X = W;
  double* u = X + d * K;
  double* alo = u + N * N;
  double* ahi = alo + N * M;
  for (int64_t e = (int64_t)blockIdx.x * wpb + warp; e < E; e += (int64_t)gridDim.x * wpb) {
    const double* src = nodes + e * d * K;
    for (int t = lane; t < d * K; t += FPX_WARP) X[t] = src[t];
    __syncwarp();
    double lo[3], hi[3];
    double dummy[3][3];
    coordinate_bounds(B, d, dr, X, false, nullptr, dummy, u, alo, ahi, lane, lo, hi);
    int st = expand_box(d, lo, hi, expansion) ? 1 : 0;
    // centre frame: every lane computes it redundantly (bitwise identical).
    double xc[3] = {0, 0, 0}, Mf[3][3], Mi[3][3];
    int ok = center_frame(B, d, dr, X, xc, Mf) == 0;
    double olo[3], ohi[3];
    if (ok) {
      inv_n(d, Mf, Mi);
      coordinate_bounds(B, d, dr, X, true, xc, Mi, u, alo, ahi, lane, olo, ohi);
      if (expand_box(d, olo, ohi, expansion)) ok = 0;
    }
    if (lane == 0) {
      for (int c = 0; c < d; ++c) {
        aabb[e * 2 * d + c] = lo[c];
        aabb[e * 2 * d + d + c] = hi[c];
      }
      if (ok) {
        double half[3], bc[3];
        for (int c = 0; c < d; ++c) {
          half[c] = 0.5 * (ohi[c] - olo[c]);
          bc[c] = 0.5 * (ohi[c] + olo[c]);
        }
        double cen[3];
        for (int c = 0; c < d; ++c) {
          double s = 0.0;
          for (int b = 0; b < d; ++b) s += Mf[c][b] * bc[b];
          cen[c] = xc[c] + s;
          obb_c[e * d + c] = cen[c];
          for (int b = 0; b < d; ++b) obb_inv[(e * d + c) * d + b] = Mi[c][b] / half[c];
        }
        for (int c = 0; c < d; ++c) {
          double h = 0.0;
          for (int b = 0; b < d; ++b) h += fabs(Mf[c][b] * half[b]);
          h = h * (1.0 + 1e-9) + 4.0 * 2.220446049250313e-16 * fabs(cen[c]);
          double l = cen[c] - h, uu = cen[c] + h;
          hbox[e * 2 * d + c] = l > lo[c] ? l : lo[c];
          hbox[e * 2 * d + d + c] = uu < hi[c] ? uu : hi[c];
        }
        obb_ok[e] = 1;
      } else {
        for (int c = 0; c < d; ++c) {
          obb_c[e * d + c] = NAN;
          for (int b = 0; b < d; ++b) obb_inv[(e * d + c) * d + b] = NAN;
          hbox[e * 2 * d + c] = lo[c];
          hbox[e * 2 * d + d + c] = hi[c];
        }
        obb_ok[e] = 0;
        if (st == 0) st = 2;
      }
      // centre frame for the best-first candidate order: x_c, M^{-1}
      double* fr = frame + e * (d + d * d);
      for (int c = 0; c < d; ++c) fr[c] = xc[c];
      for (int c = 0; c < d; ++c)
        for (int b = 0; b < d; ++b) fr[d + c * d + b] = ok ? Mi[c][b] : 0.0;
      status[e] = st;
    }
    __syncwarp();
  }
}

// Batched bound_function_1d / 2d: one warp per function.
__global__ void k_bound_function(int dr, int N, int M, int64_t nf, const double* __restrict__ basis,
                                 const double* __restrict__ values, double* lower, double* upper) {
  extern __shared__ double smem[];
  const int bsize = FPX_BASIS_SIZE(N, M);
  double* sB = smem;
  for (int t = threadIdx.x; t < bsize; t += blockDim.x) sB[t] = basis[t];
  __syncthreads();
  BasisView B(sB, N, M);
  const int warp = threadIdx.x / FPX_WARP, lane = threadIdx.x % FPX_WARP;
  const int wpb = blockDim.x / FPX_WARP;
  const int K = dr == 1 ? N : N * N;
  double* W = smem + bsize + warp * ((size_t)K + 2 * N * M + 2);
  double* u = W;
  double* alo = u + K;
  double* ahi = alo + N * M;
  for (int64_t f = (int64_t)blockIdx.x * wpb + warp; f < nf; f += (int64_t)gridDim.x * wpb) {
    for (int t = lane; t < K; t += FPX_WARP) u[t] = values[f * K + t];
    __syncwarp();
    if (dr == 1) {
      double a0 = 0.0, a1 = 0.0;
      for (int i = 0; i < N; ++i) { a0 += u[i] * B.proj0[i]; a1 += u[i] * B.proj1[i]; }
      for (int j = lane; j < M; j += FPX_WARP) {
        double slo = 0.0, shi = 0.0;
        for (int i = 0; i < N; ++i) {
          double w = u[i] - a0 - a1 * B.z[i];
          double tl = w * B.lo[i * M + j], th = w * B.hi[i * M + j];
          double mn = tl < th ? tl : th, mx = tl > th ? tl : th;
          if (i == 0) { slo = mn; shi = mx; } else { slo += mn; shi += mx; }
        }
        double lin = a0 + a1 * B.eta[j];
        lower[f * M + j] = lin + slo;
        upper[f * M + j] = lin + shi;
      }
    } else {
      for (int t = lane; t < N * M; t += FPX_WARP) {
        const int j = t / M, k = t % M;
        double slo = 0.0, shi = 0.0;
        for (int i = 0; i < N; ++i) {
          double uij = u[i + N * j];
          double tl = uij * B.lo[i * M + k], th = uij * B.hi[i * M + k];
          double mn = tl < th ? tl : th, mx = tl > th ? tl : th;
          if (i == 0) { slo = mn; shi = mx; } else { slo += mn; shi += mx; }
        }
        alo[j * M + k] = slo;
        ahi[j * M + k] = shi;
      }
      __syncwarp();
      for (int t = lane; t < M * M; t += FPX_WARP) {
        const int k = t / M, l = t % M;
        double slo = 0.0, shi = 0.0;
        for (int j = 0; j < N; ++j) {
          double al = alo[j * M + k], ah = ahi[j * M + k];
          double vl = B.lo[j * M + l], vh = B.hi[j * M + l];
          double c0 = al * vl, c1 = al * vh, c2 = ah * vl, c3 = ah * vh;
          double mn = c0, mx = c0;
          mn = c1 < mn ? c1 : mn; mn = c2 < mn ? c2 : mn; mn = c3 < mn ? c3 : mn;
          mx = c1 > mx ? c1 : mx; mx = c2 > mx ? c2 : mx; mx = c3 > mx ? c3 : mx;
          if (j == 0) { slo = mn; shi = mx; } else { slo += mn; shi += mx; }
        }
        lower[f * M * M + t] = slo;
        upper[f * M * M + t] = shi;
      }
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------ hash map
// Union of boxes per axis: one block, grid = lo, hi, h.
__global__ void k_hash_grid(int d, int64_t E, const double* __restrict__ box, int ncell,
                            double* grid) {
  __shared__ double slo[3][32], shi[3][32];
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t e = threadIdx.x; e < E; e += blockDim.x)
    for (int c = 0; c < d; ++c) {
      double l = box[e * 2 * d + c], h = box[e * 2 * d + d + c];
      lo[c] = l < lo[c] ? l : lo[c];
      hi[c] = h > hi[c] ? h : hi[c];
    }
  const int lane = threadIdx.x % 32, warp = threadIdx.x / 32;
  for (int c = 0; c < 3; ++c) {
    double a = warp_min(lo[c]), b = warp_max(hi[c]);
    if (lane == 0) { slo[c][warp] = a; shi[c][warp] = b; }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int nw = blockDim.x / 32;
    for (int c = 0; c < 3; ++c) {
      double a = INFINITY, b = -INFINITY;
      for (int w = 0; w < nw; ++w) {
        a = slo[c][w] < a ? slo[c][w] : a;
        b = shi[c][w] > b ? shi[c][w] : b;
      }
      if (c < d) {
        grid[c] = a;
        grid[3 + c] = b;
        grid[6 + c] = (b - a) / ncell;
      } else {
        grid[c] = 0.0;
        grid[3 + c] = 0.0;
        grid[6 + c] = 1.0;
      }
    }
  }
}

__device__ void box_cells(int d, const double* grid, int n, const double* b, int* a0, int* a1) {
  a0[0] = a0[1] = a0[2] = 0;
  a1[0] = a1[1] = a1[2] = 0;
  cell_of(d, grid, n, b, a0);
  cell_of(d, grid, n, b + d, a1);
}

// Conservative cell-vs-OBB overlap (oracle cell_meets_obb, decision D5b):
// the cell centre in the OBB frame lies within the unit cube grown by the
// cell's half-extent in that frame (1e-9 relative margin).
__device__ __forceinline__ bool cell_meets_obb(int d, const double* grid, int i, int j, int k,
                                               const double* __restrict__ cen,
                                               const double* __restrict__ inv) {
  const int q[3] = {i, j, k};
  double dx[3];
  for (int b = 0; b < d; ++b) {
    const double cc = grid[b] + ((double)q[b] + 0.5) * grid[6 + b];
    dx[b] = cc - cen[b];
  }
  for (int a = 0; a < d; ++a) {
    double y = 0.0, ee = 0.0;
    for (int b = 0; b < d; ++b) {
      y += inv[a * d + b] * dx[b];
      ee += fabs(inv[a * d + b]) * (0.5 * grid[6 + b]);
    }
    if (!(fabs(y) <= (1.0 + ee) * (1.0 + 1e-9))) return false;
  }
  return true;
}

// Warp per element, lanes over the flattened cell range of its hash box
// (SPEC.md:230-238 build_local_map; D5b culling): at cfg-2 a box spans ~170
// cells of the refined grid, so a thread-per-element loop ran one wave of
// long serial trips (7 ms); here every lane tests ~5 cells.
// fill == nullptr: count pass (cnt[cell] += 1); else fill pass.
__global__ void __launch_bounds__(256)
    k_hash_cells(int d, int64_t E, const double* __restrict__ box,
                 const double* __restrict__ obb_c, const double* __restrict__ obb_inv,
                 const uint8_t* __restrict__ obb_ok, const double* __restrict__ grid, int n,
                 int32_t* cnt, const int32_t* __restrict__ offsets, int32_t* elems) {
  const int lane = threadIdx.x % 32;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32;
  const int64_t nw = (int64_t)gridDim.x * blockDim.x / 32;
  for (int64_t e = w0; e < E; e += nw) {
    int a[3], b[3];
    box_cells(d, grid, n, box + e * 2 * d, a, b);
    const int ni = b[0] - a[0] + 1, nj = b[1] - a[1] + 1, nk = b[2] - a[2] + 1;
    const int tot = ni * nj * nk;
    const bool cull = obb_ok && obb_ok[e];
    for (int t = lane; t < tot; t += 32) {
      const int i = a[0] + t % ni, j = a[1] + (t / ni) % nj, k = a[2] + t / (ni * nj);
      if (cull && !cell_meets_obb(d, grid, i, j, k, obb_c + e * d, obb_inv + e * d * d))
        continue;
      const int64_t cell = i + (int64_t)n * (j + (int64_t)n * k);
      const int slot = atomicAdd(&cnt[cell], 1);
      if (elems) elems[offsets[cell] + slot] = (int32_t)e;
    }
  }
}

// Ascending element ids per cell: insertion sort per list.
__global__ void k_hash_sort(int64_t ncells, const int32_t* __restrict__ offsets, int32_t* elems,
                            int32_t* max_list) {
  int local_max = 0;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ncells;
       c += (int64_t)gridDim.x * blockDim.x) {
    const int s = offsets[c], t = offsets[c + 1];
    local_max = (t - s) > local_max ? (t - s) : local_max;
    for (int i = s + 1; i < t; ++i) {
      int v = elems[i];
      int j = i - 1;
      while (j >= s && elems[j] > v) {
        elems[j + 1] = elems[j];
        --j;
      }
      elems[j + 1] = v;
    }
  }
  atomicMax(max_list, local_max);
}

__global__ void k_cell_of(int d, const double* __restrict__ grid, int n, int64_t npts,
                          const double* __restrict__ x, int64_t* cell) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < npts;
       k += (int64_t)gridDim.x * blockDim.x) {
    int ax[3];
    double xx[3] = {0, 0, 0};
    for (int c = 0; c < d; ++c) xx[c] = x[k * d + c];
    cell[k] = cell_of(d, grid, n, xx, ax);
  }
}

// ------------------------------------------------------------ find prefilter
// Point ordering by hash cell (counting sort): adjacent lanes of the
// prefilter then walk the same candidate lists and read the same element
// records.  Points outside the grid go to the extra bucket `ncells`.
__global__ void k_point_cells(fpx_mesh_t m, int64_t n, const double* __restrict__ x,
                              int32_t* cellid, int32_t* cell_count) {
  const int d = m.d;
  int64_t nc = 1;
  for (int c = 0; c < d; ++c) nc *= m.ncell;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    double xx[3] = {0, 0, 0};
    for (int c = 0; c < d; ++c) xx[c] = x[k * d + c];
    int ax[3];
    int64_t cell = cell_of(d, m.grid, m.ncell, xx, ax);
    if (cell < 0) cell = nc;
    cellid[k] = (int32_t)cell;
    atomicAdd(&cell_count[cell], 1);
  }
}

// Counting-sort scatter of the points by hash cell; also writes the
// cell-ordered copies the prefilter reads (coordinates, cell id), so its
// per-point start is one load instead of order -> cellid -> x.
__global__ void k_point_scatter(int64_t n, int64_t base, int d, const double* __restrict__ x,
                                const int32_t* __restrict__ cellid,
                                const int32_t* __restrict__ cell_off, int32_t* cursor,
                                int32_t* order, double* xo, const int32_t* __restrict__ offsets,
                                int64_t nc, int2* lr) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int c = cellid[k];
    const int64_t pos = cell_off[c] + atomicAdd(&cursor[c], 1);
    order[pos] = (int32_t)(base + k);
    // the cell's hash-list range (empty outside the grid): one load in the
    // prefilter's chain of dependent loads instead of cell -> offsets
    lr[pos] = c < nc ? make_int2(offsets[c], offsets[c + 1]) : make_int2(0, 0);
    for (int a = 0; a < d; ++a) xo[pos * d + a] = x[k * d + a];
  }
}

// Records of a point with no passing candidate: final NOT_FOUND (D10).
__device__ __forceinline__ void write_not_found(int64_t k, int dr, int32_t* code, int32_t* elem,
                                                double* r, double* dist, int32_t* iters,
                                                double* values, int C) {
  code[k] = kNotFound;
  elem[k] = -1;
  for (int a = 0; a < dr; ++a) r[k * dr + a] = NAN;
  dist[k] = NAN;
  if (iters) iters[k] = 0;
  if (values)
    for (int c = 0; c < C; ++c) values[k * C + c] = NAN;
}

// Candidate loop of engine.find Phase A up to the Newton solve (SPEC.md:
// 404-413): the hash list of the point's cell through the AABB then OBB
// filter.  Per point: npass (candidates that passed) and best, the
// best-first candidate (smallest |J_c^{-1}(x - x_c)|_inf, ties -> lower id;
// DESIGN.md §3 "Candidate order").  Points with none are final NOT_FOUND.
// The rest kernel re-derives the further best-first candidates of the ~5%
// of points round 1 leaves unresolved, so nothing else is stored.

//
// kPfLanes lanes per point, points in hash-cell order: lane j of a point
// tests list entries j, j + kPfLanes, ...; the lanes' (count, best) are
// combined with a shuffle.  Consecutive points share one or two cells'
// lists, so the records a warp reads at one time are few (L1 broadcast).
// Per entry: the element's 80-byte float row (box + OBB pre-tests, one
// round trip; the double record only in the ~1e-7 undecided band), then
// the double affine frame only if it passes (best-first value).  At cfg-2
// 99% of listed candidates pass the AABB and 30% the OBB.
// Measured variants (cfg-2, ncu, us).  Double records, 256-byte rows:
// thread per point 330-343; lanes x trip (entries in flight per lane) 1x2
// ~310, 2x2 300-310, 2x4 ~310, 4x2 ~320; 48 or 64 resident warps per SM
// (register caps, spills at 64) 300 / 360; lane per (point, entry) with a
// segmented warp reduction 447 (32 different records per load);
// element-major (warp per element over its hash-box cell rows, atomics per
// point) 872 (3x the tests without the D5b cull); cell-major (warp per hash
// cell, lanes = list entries holding their records, ballot + shuffle
// reduction per point) 760 (cells hold ~1.1 points: the per-cell chain of
// dependent loads is paid per point); a float hash box per list entry
// (184 MB beside the lists) as a pre-test before the record 409 (six
// scalar loads per entry and the extra DRAM traffic cost more than the
// record loads they saved).  Float pre-tests (ABI 7): separate box and OBB
// rows, double OBB arithmetic 232 (L1 wavefronts 82% -> 58% of peak; the
// kernel turns latency bound); + registers capped at 48 (5 blocks/SM) 208
// (64: 232, 40 with spills: 225); one 80-byte row 195 (2x2 lanes x trip:
// 243, 4x1 216, 1x1 231); float OBB arithmetic 187; next entry's id loaded
// ahead 181; warp-uniform loop bounds (spills 40 -> 8 bytes) 174 (kept;
// register caps 62: 181, 40: 200, 32: 246).  Points in input order (no
// cell sort, uniform points): prefilter 256 + scatter 18 against 177 + 55.
// 256-bit loads (LDG.E.ENL2.256) of 96-byte rows and a 32-byte aligned
// frame: 176 against 176 (the load instruction count is not the bound).
// Both lanes of a point on the same entry, each reading half of every row
// and frame (3 + 3 loads instead of 5 + 6, outcomes exchanged by a
// pair-masked shuffle): 375 (the per-point chain of entries doubles).
// The next point's header loaded ahead: 190 (spills at 48 registers); the
// next entry's row loaded ahead: 290 (48 registers) / 225 (64).
constexpr int kPfLanes = 2;  // lanes per point

template <int D>
__global__ void __launch_bounds__(256, 5)  // 48 registers: 40 warps per SM
    k_prefilter_points(fpx_mesh_t m, int64_t n, const double* __restrict__ xo,
                       const int32_t* __restrict__ order, const int2* __restrict__ lr,
                       int32_t* best, int32_t* npass, int32_t* code, int32_t* elem, double* r,
                       double* dist, int32_t* iters, double* values, int C, int32_t* elem_count,
                       int64_t* stats) {
  int64_t boxtests = 0;
  const bool vol = m.dr == D;
  const int sub = threadIdx.x % kPfLanes;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x / kPfLanes;
  // whole warps iterate together (the shuffles below need every lane): the
  // loop runs on the warp's first point, the same in all its lanes
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31)) / kPfLanes;
  const int lp = (threadIdx.x & 31) / kPfLanes;
  for (int64_t tw = w0; tw < n; tw += stride) {
    const int64_t t = tw + lp;
    const bool valid = t < n;
    const int64_t k = valid ? order[t] : 0;
    const int2 rng = valid ? lr[t] : make_int2(0, 0);
    double xx[D];
#pragma unroll
    for (int c = 0; c < D; ++c) xx[c] = valid ? xo[t * D + c] : 0.0;
    int cnt = 0, bst = INT_MAX;
    double bval = INFINITY;
    {
      const int s = rng.x, e1 = rng.y;
      if (sub == 0) boxtests += e1 - s;
      // entries q, q + kPfLanes, ...; the next entry's id is loaded before
      // this one's row, so the list -> row chain overlaps across entries
      int en = s + sub < e1 ? m.elems[s + sub] : -1;
      for (int q = s + sub; q < e1; q += kPfLanes) {
        const int e = en;
        en = q + kPfLanes < e1 ? m.elems[q + kPfLanes] : -1;
        float B[FPX_FROW];
        frow_load<D>(m.fbox, e, B);
        float yn = 0.0f;
        if (!frow_passes<D>(m, e, B, xx, &yn)) continue;
        double R[FPX_FREC];
        frec_range<D, 3 * D + D * D, 4 * D + 2 * D * D>(m.frec, e, R);
        ++cnt;
        // round 1's candidate: the smallest affine best-first value plus, for
        // volume meshes, the OBB norm (cfg-2 sample: 4.3% of the points
        // left for the rest phase against 5.1% with the affine value alone;
        // tests/rank_study.py)
        const double v = bestfirst_value(D, R + 3 * D + D * D, xx) + (vol ? (double)yn : 0.0);
        if (v < bval) {  // strict: ties keep the lower (earlier) id
          bval = v;
          bst = e;
        }
      }
    }
    // (v, e)-lexicographic minimum over the point's lanes == the first
    // minimum in list order (lists ascend in element id)
#pragma unroll
    for (int o = 1; o < kPfLanes; o <<= 1) {
      const int co = __shfl_xor_sync(FPX_FULL, cnt, o);
      const double vo = __shfl_xor_sync(FPX_FULL, bval, o);
      const int eo = __shfl_xor_sync(FPX_FULL, bst, o);
      cnt += co;
      if (bf_less(vo, eo, bval, bst)) {
        bval = vo;
        bst = eo;
      }
    }
    if (valid && sub == 0) {
      if (cnt == 0) bst = -1;
      best[k] = bst;
      npass[k] = cnt;
      if (bst < 0) write_not_found(k, m.dr, code, elem, r, dist, iters, values, C);
      else atomicAdd(&elem_count[bst], 1);
    }
  }
  for (int o = 16; o > 0; o >>= 1) boxtests += __shfl_xor_sync(FPX_FULL, boxtests, o);
  if ((threadIdx.x & 31) == 0 && boxtests)
    atomicAdd((unsigned long long*)&stats[FPX_STAT_BOXTESTS], (unsigned long long)boxtests);
}


// Packed candidate-filter records (include/fpx.h, FPX_FREC): one 256-byte
// row per element so the prefilter fetches a candidate in one round trip.
// Also the float pre-test rows (include/fpx.h, fbox): the box rounded
// outwards, the OBB rounded to nearest where float keeps 24 bits of every
// value (fpx_boxes.cuh, fbox_aabb / fobb_in).
__device__ __forceinline__ bool float_exact_range(double v) {
  const double a = fabs(v);
  return a == 0.0 || (a >= 0x1p-100 && a <= 0x1p100);
}

__global__ void k_filter_records(int d, int64_t E, const double* __restrict__ aabb,
                                 const double* __restrict__ obb_c,
                                 const double* __restrict__ obb_inv,
                                 const uint8_t* __restrict__ obb_ok,
                                 const double* __restrict__ frame, double* frec, float* fbox) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x) {
    double* R = frec + e * FPX_FREC;
    int o = 0;
    for (int t = 0; t < 2 * d; ++t) R[o++] = aabb[e * 2 * d + t];
    for (int t = 0; t < d; ++t) R[o++] = obb_c[e * d + t];
    for (int t = 0; t < d * d; ++t) R[o++] = obb_inv[e * d * d + t];
    for (int t = 0; t < d + d * d; ++t) R[o++] = frame[e * (d + d * d) + t];
    while (o < FPX_FREC - 1) R[o++] = 0.0;
    R[FPX_FREC - 1] = obb_ok[e] ? 1.0 : 0.0;
    float* B = fbox + e * FPX_FROW;
    float* O = B + kFrowObb;
    for (int t = 0; t < FPX_FROW; ++t) B[t] = 0.0f;
    for (int c = 0; c < d; ++c) {
      B[c] = __double2float_rd(aabb[e * 2 * d + c]);
      B[d + c] = __double2float_ru(aabb[e * 2 * d + d + c]);
    }
    bool fl = true;
    for (int t = 0; t < d; ++t) {
      O[t] = __double2float_rn(obb_c[e * d + t]);
      fl = fl && float_exact_range(obb_c[e * d + t]);
    }
    for (int t = 0; t < d * d; ++t) {
      O[d + t] = __double2float_rn(obb_inv[e * d * d + t]);
      fl = fl && float_exact_range(obb_inv[e * d * d + t]);
    }
    B[kFboxMode] = !obb_ok[e] ? 0.0f : (fl ? 1.0f : 2.0f);
  }
}

// ------------------------------------------------------------ host launchers
static int setup_warps(size_t per_warp_bytes, size_t base_bytes) {
  int w = 4;
  while (w > 1 && base_bytes + w * per_warp_bytes > 96 * 1024) --w;
  return w;
}

cudaError_t launch_setup_bounds(int d, int dr, int N, int M, int64_t E, const double* basis,
                                const double* nodes, double expansion, double* aabb, double* obb_c,
                                double* obb_inv, double* hbox, double* frame, uint8_t* obb_ok,
                                int32_t* status, cudaStream_t st) {
  const int K = dr == 1 ? N : (dr == 2 ? N * N : N * N * N);
  size_t pw = SetupSmemLayout::per_warp(d, K, N, M) * sizeof(double);
  size_t base = FPX_BASIS_SIZE(N, M) * sizeof(double);
  int w = setup_warps(pw, base);
  size_t smem = base + w * pw;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_setup_bounds, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int64_t blocks = (E + w - 1) / w;
  if (blocks > 148 * 64) blocks = 148 * 64;
  if (blocks < 1) blocks = 1;
  k_setup_bounds<<<(unsigned)blocks, w * FPX_WARP, smem, st>>>(d, dr, N, M, E, basis, nodes,
                                                               expansion, aabb, obb_c, obb_inv,
                                                               hbox, frame, obb_ok, status);
  return cudaGetLastError();
}

cudaError_t launch_bound_function(int dr, int N, int M, int64_t nf, const double* basis,
                                  const double* values, double* lower, double* upper,
                                  cudaStream_t st) {
  const int K = dr == 1 ? N : N * N;
  size_t pw = ((size_t)K + 2 * N * M + 2) * sizeof(double);
  size_t base = FPX_BASIS_SIZE(N, M) * sizeof(double);
  int w = setup_warps(pw, base);
  size_t smem = base + w * pw;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_bound_function, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int64_t blocks = (nf + w - 1) / w;
  if (blocks > 148 * 64) blocks = 148 * 64;
  if (blocks < 1) blocks = 1;
  k_bound_function<<<(unsigned)blocks, w * FPX_WARP, smem, st>>>(dr, N, M, nf, basis, values,
                                                                 lower, upper);
  return cudaGetLastError();
}

static unsigned grid_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  if (b > 148 * 32) b = 148 * 32;
  if (b < 1) b = 1;
  return (unsigned)b;
}

// nodes [E][d][K] -> [E][d][K/N][NP] (NP = N rounded up to even; pad = 0).
__global__ void k_pad_nodes(int d, int N, int K, int64_t E, const double* __restrict__ nodes,
                            double* pad) {
  const int NP = N + (N & 1), R = K / N;
  const int64_t tot = E * d * R * NP;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(t % NP);
    const int64_t rowg = t / NP;  // (e, c, row)
    pad[t] = i < N ? nodes[rowg * N + i] : 0.0;
  }
}
cudaError_t launch_pad_nodes(int d, int dr, int N, int64_t E, const double* nodes, double* pad,
                             cudaStream_t st) {
  const int K = dr == 1 ? N : (dr == 2 ? N * N : N * N * N);
  const int64_t tot = E * d * (K / N) * (N + (N & 1));
  k_pad_nodes<<<grid_for(tot, 256), 256, 0, st>>>(d, N, K, E, nodes, pad);
  return cudaGetLastError();
}
cudaError_t launch_filter_records(int d, int64_t E, const double* aabb, const double* obb_c,
                                  const double* obb_inv, const uint8_t* obb_ok,
                                  const double* frame, double* frec, float* fbox,
                                  cudaStream_t st) {
  k_filter_records<<<grid_for(E, 256), 256, 0, st>>>(d, E, aabb, obb_c, obb_inv, obb_ok, frame,
                                                     frec, fbox);
  return cudaGetLastError();
}
cudaError_t launch_hash_grid(int d, int64_t E, const double* box, int ncell, double* grid,
                             cudaStream_t st) {
  k_hash_grid<<<1, 1024, 0, st>>>(d, E, box, ncell, grid);
  return cudaGetLastError();
}
cudaError_t launch_hash_count(int d, int64_t E, const double* box, const double* obb_c,
                              const double* obb_inv, const uint8_t* obb_ok, const double* grid,
                              int n, int32_t* cnt, cudaStream_t st) {
  k_hash_cells<<<grid_for(E * 32, 256), 256, 0, st>>>(d, E, box, obb_c, obb_inv, obb_ok, grid,
                                                      n, cnt, nullptr, nullptr);
  return cudaGetLastError();
}
cudaError_t launch_hash_fill(int d, int64_t E, const double* box, const double* obb_c,
                             const double* obb_inv, const uint8_t* obb_ok, const double* grid,
                             int n, const int32_t* offsets, int32_t* cursor, int32_t* elems,
                             cudaStream_t st) {
  k_hash_cells<<<grid_for(E * 32, 256), 256, 0, st>>>(d, E, box, obb_c, obb_inv, obb_ok, grid,
                                                      n, cursor, offsets, elems);
  return cudaGetLastError();
}
cudaError_t launch_hash_sort(int64_t ncells, const int32_t* offsets, int32_t* elems,
                             int32_t* max_list, cudaStream_t st) {
  k_hash_sort<<<grid_for(ncells, 256), 256, 0, st>>>(ncells, offsets, elems, max_list);
  return cudaGetLastError();
}
cudaError_t launch_cell_of(int d, const double* grid, int n, int64_t npts, const double* x,
                           int64_t* cell, cudaStream_t st) {
  k_cell_of<<<grid_for(npts, 256), 256, 0, st>>>(d, grid, n, npts, x, cell);
  return cudaGetLastError();
}
cudaError_t launch_prefilter(const fpx_mesh_t& m, int64_t n, const double* xo,
                             const int32_t* order, const int2* co, int32_t* best,
                             int32_t* npass, int32_t* code, int32_t* elem, double* r,
                             double* dist, int32_t* iters, double* values, int C,
                             int32_t* elem_count, int64_t* stats, cudaStream_t st) {
  auto fn = m.d == 3 ? k_prefilter_points<3> : k_prefilter_points<2>;
  fn<<<grid_for(n * kPfLanes, 256), 256, 0, st>>>(m, n, xo, order, co, best, npass, code, elem,
                                                   r, dist, iters, values, C, elem_count, stats);
  return cudaGetLastError();
}
cudaError_t launch_point_cells(const fpx_mesh_t& m, int64_t n, const double* x, int32_t* cellid,
                               int32_t* cell_count, cudaStream_t st) {
  k_point_cells<<<grid_for(n, 256), 256, 0, st>>>(m, n, x, cellid, cell_count);
  return cudaGetLastError();
}
cudaError_t launch_point_scatter(int64_t n, int64_t base, int d, const double* x,
                                 const int32_t* cellid, const int32_t* cell_off, int32_t* cursor,
                                 int32_t* order, double* xo, const int32_t* offsets, int64_t nc,
                                 int2* lr, cudaStream_t st) {
  k_point_scatter<<<grid_for(n, 256), 256, 0, st>>>(n, base, d, x, cellid, cell_off, cursor,
                                                    order, xo, offsets, nc, lr);
  return cudaGetLastError();
}
}  // namespace fpx
