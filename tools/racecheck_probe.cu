// Minimal cp.async + mbarrier ring (the k_newton_stream slot protocol) for
// compute-sanitizer racecheck: every lane issues its copies, arrives on the
// slot's mbarrier (noinc), every lane waits on the phase, reads the slot,
// __syncwarp, and the slot is refilled.  Any hazard racecheck reports here is
// a limitation of its cp.async/mbarrier model, not of the protocol.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o racecheck_probe racecheck_probe.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ void cp_async8(void* sdst, const void* gsrc) {
  unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t* mb, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(mb);
  unsigned ok;
  asm volatile("{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
               " selp.u32 %0, 1, 0, p;\n}\n" : "=r"(ok) : "r"(a), "r"(parity) : "memory");
  return ok != 0;
}

__global__ void probe(const double* g, double* out, int rounds) {
  __shared__ __align__(16) double slot[64];
  __shared__ uint64_t mb;
  const int lane = threadIdx.x;
  if (lane == 0) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(&mb);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(32) : "memory");
  }
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  double acc = 0.0;
  unsigned parity = 0;
  for (int k = 0; k < rounds; ++k) {
    __syncwarp();
    for (int t = lane; t < 64; t += 32) cp_async8(slot + t, g + k * 64 + t);
    const unsigned a = (unsigned)__cvta_generic_to_shared(&mb);
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(a) : "memory");
    while (!mbar_test(&mb, parity)) {
    }
    __syncwarp();
    parity ^= 1u;
    for (int t = 0; t < 64; ++t) acc += slot[(t + lane) & 63];
    __syncwarp();
  }
  out[lane] = acc;
}

int main() {
  double *g, *o;
  cudaMalloc(&g, 64 * 8 * sizeof(double));
  cudaMalloc(&o, 32 * sizeof(double));
  cudaMemset(g, 0, 64 * 8 * sizeof(double));
  probe<<<1, 32>>>(g, o, 8);
  cudaError_t e = cudaDeviceSynchronize();
  printf("probe %s\n", cudaGetErrorString(e));
  return e != cudaSuccess;
}
