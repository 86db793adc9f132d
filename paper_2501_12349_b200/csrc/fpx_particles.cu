// fpx_particles.cu -- the particle update of the Lagrangian tracking loop
// (Algorithm 1: ParticleRHS + Integrate + ParticleBC).
//
// One fused, HBM-bound pass per step: Stokes drag a = (u - v) / tau, second
// order Adams-Bashforth for (x, v) (forward Euler on the first step), then
// the periodic wrap of the box.  Thread per particle, SoA-free [n][d] rows.
#include "fpx_common.cuh"
#include "fpx_kernels.cuh"

namespace fpx {

__global__ void k_particles_advance(int d, int64_t n, double* __restrict__ x,
                                    double* __restrict__ v, const double* __restrict__ u,
                                    double* __restrict__ v_prev, double* __restrict__ a_prev,
                                    double tau, double dt, int first, double lo0, double lo1,
                                    double lo2, double hi0, double hi1, double hi2, int periodic) {
  const double lo[3] = {lo0, lo1, lo2}, hi[3] = {hi0, hi1, hi2};
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    for (int c = 0; c < d; ++c) {
      const int64_t i = p * d + c;
      const double vn = v[i];
      const double an = (u[i] - vn) / tau;  // Stokes drag (§6.7)
      double xn = x[i];
      double vn1;
      if (first) {  // AB1 start
        xn = xn + dt * vn;
        vn1 = vn + dt * an;
      } else {      // AB2: y+ = y + dt (3/2 f_n - 1/2 f_{n-1})
        xn = xn + dt * (1.5 * vn - 0.5 * v_prev[i]);
        vn1 = vn + dt * (1.5 * an - 0.5 * a_prev[i]);
      }
      if ((periodic >> c) & 1) {  // periodic box (ParticleBC)
        const double L = hi[c] - lo[c];
        xn = lo[c] + (xn - lo[c]) - L * floor((xn - lo[c]) / L);
      }
      x[i] = xn;
      v_prev[i] = vn;
      a_prev[i] = an;
      v[i] = vn1;
    }
  }
}

cudaError_t launch_particles_advance(int d, int64_t n, double* x, double* v, const double* u,
                                     double* v_prev, double* a_prev, double tau, double dt,
                                     int first, const double* box, int periodic,
                                     cudaStream_t st) {
  int64_t b = (n + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  if (b < 1) b = 1;
  double lo[3] = {0, 0, 0}, hi[3] = {1, 1, 1};
  for (int c = 0; c < d; ++c) {
    lo[c] = box[c];
    hi[c] = box[d + c];
  }
  k_particles_advance<<<(unsigned)b, 256, 0, st>>>(d, n, x, v, u, v_prev, a_prev, tau, dt, first,
                                                   lo[0], lo[1], lo[2], hi[0], hi[1], hi[2],
                                                   periodic);
  return cudaGetLastError();
}

}  // namespace fpx
