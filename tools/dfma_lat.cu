// DFMA latency / issue microbenchmark (sm_100a): cycles per dependent DFMA
// with C independent chains per thread, W warps in one CTA on one SM.
#include <cstdio>
#include <cuda_runtime.h>
template <int C>
__global__ void k(double* out, long long* cyc, int iters, double a, double b) {
  double x[C];
#pragma unroll
  for (int c = 0; c < C; ++c) x[c] = threadIdx.x * 1e-9 + c;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < C; ++c) x[c] = fma(x[c], a, b);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) s += x[c];
  if (s == 1.2345) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int C>
void run(int warps) {
  double* o; long long* c; cudaMalloc(&o, 8); cudaMalloc(&c, 8);
  int iters = 4096;
  k<C><<<1, 32 * warps>>>(o, c, iters, 0.999999, 1e-7);
  k<C><<<1, 32 * warps>>>(o, c, iters, 0.999999, 1e-7);
  long long h; cudaDeviceSynchronize(); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  double per = (double)h / (iters * (double)C);
  printf("chains %d warps/SM %2d (per SMSP %.1f): %.2f cycles per DFMA per warp, SM rate %.2f warp-DFMA/clk\n",
         C, warps, warps / 4.0, per, warps / per);
  cudaFree(o); cudaFree(c);
}
int main() {
  for (int w : {1, 4, 8, 16}) { run<1>(w); run<2>(w); run<4>(w); run<6>(w); run<8>(w); }
  return 0;
}
