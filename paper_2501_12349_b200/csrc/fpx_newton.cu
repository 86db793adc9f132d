// fpx_newton.cu -- dispatch of the Newton / eval kernels over (d, dr, N).
// The template instantiations live in generated per-order TUs
// (build.py writes build_obj/gen/fpx_inst_<d><dr>_<N>.cu) so they compile in
// parallel; `extern template` keeps them out of this TU.
#include "fpx_newton.cuh"
#include "fpx_inst.h"

namespace fpx {

// Marks records for eval grouping: unit_elem = elem (or -1) and NaN for
// NOT_FOUND (D12); counts per element.
__global__ void k_eval_mark(int64_t n, int C, const int32_t* __restrict__ code,
                            const int32_t* __restrict__ elem, double* values, int32_t* unit_elem,
                            int32_t* count) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int e = elem[k];
    if (code[k] == kNotFound || e < 0) {
      unit_elem[k] = -1;
      for (int c = 0; c < C; ++c) values[k * C + c] = NAN;
    } else {
      unit_elem[k] = e;
      atomicAdd(&count[e], 1);
    }
  }
}

// Compiled (d, dr, N) combinations come from the generated fpx_inst.h
// (FPX_INST_LIST(X) expands X(d, dr, N) for every instantiated order).
bool newton_supported(int d, int dr, int N) {
#define FPX_SUP(D_, DR_, N_) \
  if (d == D_ && dr == DR_ && N == N_) return true;
  FPX_INST_LIST(FPX_SUP)
#undef FPX_SUP
  return false;
}

template <template <int, int, int> class F, typename... A>
static cudaError_t dispatch(int d, int dr, int N, A... args) {
#define FPX_CASE(D_, DR_, N_) \
  if (d == D_ && dr == DR_ && N == N_) return F<D_, DR_, N_>::run(args...);
  FPX_INST_LIST(FPX_CASE)
#undef FPX_CASE
  return cudaErrorInvalidValue;
}

cudaError_t launch_newton_stream(const fpx_mesh_t& m, int64_t n, const double* ux,
                                 const int4* umeta, const uint64_t* packed_off,
                                 const int32_t* npass, int32_t* code, int32_t* elem, double* r,
                                 double* dist, int32_t* iters, const double* field, int C,
                                 double* values, int32_t* upts, int64_t* nun_dev,
                                 int64_t* chunk_ctr, int4* redo, int64_t* nredo, int64_t redo_cap,
                                 int64_t* stats, cudaStream_t st) {
  return dispatch<Stream>(m.d, m.dr, m.N, m, ux, umeta, packed_off, npass, code, elem, r, dist,
                          iters, field, C, values, upts, nun_dev, chunk_ctr, n, redo, nredo,
                          redo_cap, stats, st);
}

template <int D, int DR, int N>
struct RestLists {
  template <typename... A>
  static cudaError_t run(A... a) { return Rest<D, DR, N>::lists(a...); }
};

cudaError_t launch_rest_lists(const fpx_mesh_t& m, const double* x, int64_t nun_cap,
                              const int64_t* nun_dev, const int32_t* upts, int32_t* best,
                              const int32_t* npass, int32_t* clist,
                              int32_t* cnum, int32_t* nps, int32_t* hist, int32_t* bstart,
                              int32_t* bcur, int32_t* perm, int64_t* cum, int32_t* maxnp,
                              int4* pairs, int64_t* npairs, cudaStream_t st) {
  return dispatch<RestLists>(m.d, m.dr, m.N, m, x, nun_cap, nun_dev, upts, best, npass, clist,
                             cnum,
                             nps, hist,
                             bstart, bcur, perm, cum, maxnp, pairs, npairs, st);
}

cudaError_t launch_find_rest(const fpx_mesh_t& m, const double* x, int64_t nun_cap,
                             const int64_t* nun_dev, const int32_t* upts, const int32_t* clist,
                             const int32_t* cnum, const int32_t* nps, const int32_t* perm,
                             const int64_t* cum, const int32_t* maxnp, const int32_t* best,
                             const int4* pairs, const int64_t* npairs, int4* redo,
                             int64_t* nredo, int32_t* found,
                             int32_t* lock, int32_t* code, int32_t* elem, double* r, double* dist,
                             int32_t* iters, const double* field, int C, double* values,
                             int64_t* counter, int64_t* stats, cudaStream_t st) {
  return dispatch<Rest>(m.d, m.dr, m.N, m, x, nun_cap, nun_dev, upts, clist, cnum, nps, perm, cum,
                        maxnp, best, pairs, npairs, redo, nredo, found, lock, code, elem, r, dist,
                        iters, field, C,
                        values,
                        counter,
                        stats, st);
}

cudaError_t launch_forward_map(const fpx_mesh_t& m, int64_t n, const int32_t* elem,
                               const double* r, double* x, double* G, double* H2,
                               cudaStream_t st) {
  return dispatch<FMap>(m.d, m.dr, m.N, m, n, elem, r, x, G, H2, st);
}

// Explicit (point, element) pairs: grouping is done by the caller (ABI) with
// the same item machinery; here the pair id is the point id.
cudaError_t launch_invert_pairs_grouped(const fpx_mesh_t& m, const double* x,
                                        const int32_t* sorted, const Item* items,
                                        const int64_t* nitems_dev, int64_t items_cap,
                                        const double* r0, double* r, double* dist,
                                        int32_t* iters, int32_t* conv, cudaStream_t st) {
  return dispatch<Pairs>(m.d, m.dr, m.N, m, x, (const int32_t*)nullptr, sorted, items,
                         nitems_dev, items_cap, r0, (int32_t*)nullptr, r, dist, iters, conv,
                         (int64_t*)nullptr, st);
}

cudaError_t launch_eval_items(int dr, int Nf, const double* fbasis, int C, const double* field,
                              const double* r, const int32_t* sorted, const Item* items,
                              const int64_t* nitems_dev, int64_t items_cap, double* values,
                              cudaStream_t st) {
  // only the nodes and scales (offsets independent of M) are read
  const int M = 2 * Nf;
#define FPX_E(DR_, N_) \
  if (dr == DR_ && Nf == N_)  \
    return EvalRun<DR_, N_>::run(fbasis, M, C, field, r, sorted, items, nitems_dev, items_cap, values, st);
  FPX_EVAL_LIST(FPX_E)
#undef FPX_E
  return cudaErrorInvalidValue;
}

cudaError_t launch_eval_mark(int64_t n, int C, const int32_t* code, const int32_t* elem,
                             double* values, int32_t* unit_elem, int32_t* count,
                             cudaStream_t st) {
  int64_t b = (n + 255) / 256;
  if (b > 148 * 32) b = 148 * 32;
  if (b < 1) b = 1;
  k_eval_mark<<<(unsigned)b, 256, 0, st>>>(n, C, code, elem, values, unit_elem, count);
  return cudaGetLastError();
}

}  // namespace fpx

