// FP64 DFMA-chain microbenchmark: measures the FP64 vector peak used as the
// roofline denominator for the findpts Newton kernel (tensor cores unused).
#include <cstdio>
#include <cuda_runtime.h>
template <int CHAINS>
__global__ void __launch_bounds__(256) dfma_chain(double* out, int iters, double a, double b) {
  double x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}
int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  double* out; cudaMalloc(&out, 8);
  const int iters = 20000; const int blocks = p.multiProcessorCount * 8; const int threads = 256;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 6; ++rep) {
    cudaEventRecord(e0);
    dfma_chain<8><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (rep > 0 && ms < best) best = ms;
  }
  double flops = 2.0 * 8 * (double)iters * blocks * threads;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"fp64_tflops\": %.3f, \"ms\": %.3f}\n", p.name, p.multiProcessorCount, flops / (best * 1e-3) / 1e12, best);
  return 0;
}
