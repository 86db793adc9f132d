// fpx_kernels.cuh -- host launchers shared between the kernel TUs and the ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/fpx.h"

#define FPX_SETUP_MAXN 16  // setup kernels: nodes per axis <= 16 (p <= 15)
#define FPX_ITEM 32        // (point|pair) slots per warp work item
#define FPX_RK 16          // best-first ranked candidates listed per rest point
#define FPX_HMAX 1024      // rest kernel: candidate-count histogram bins

namespace fpx {

// Work item of the element-major kernels: one warp, one element, <= 32 units.
struct Item {
  int32_t elem;
  int32_t start;  // offset into the element-sorted unit array
  int32_t count;
};

cudaError_t launch_setup_bounds(int d, int dr, int N, int M, int64_t E, const double* basis,
                                const double* nodes, double expansion, double* aabb, double* obb_c,
                                double* obb_inv, double* hbox, double* frame, uint8_t* obb_ok,
                                int32_t* status, cudaStream_t st);
cudaError_t launch_bound_function(int dr, int N, int M, int64_t nf, const double* basis,
                                  const double* values, double* lower, double* upper,
                                  cudaStream_t st);
cudaError_t launch_pad_nodes(int d, int dr, int N, int64_t E, const double* nodes, double* pad,
                             cudaStream_t st);
cudaError_t launch_filter_records(int d, int64_t E, const double* aabb, const double* obb_c,
                                  const double* obb_inv, const uint8_t* obb_ok,
                                  const double* frame, double* frec, float* fbox,
                                  cudaStream_t st);
cudaError_t launch_hash_grid(int d, int64_t E, const double* box, int ncell, double* grid,
                             cudaStream_t st);
cudaError_t launch_hash_count(int d, int64_t E, const double* box, const double* obb_c,
                              const double* obb_inv, const uint8_t* obb_ok, const double* grid,
                              int n, int32_t* cnt, cudaStream_t st);
cudaError_t launch_hash_fill(int d, int64_t E, const double* box, const double* obb_c,
                             const double* obb_inv, const uint8_t* obb_ok, const double* grid,
                             int n, const int32_t* offsets, int32_t* cursor, int32_t* elems,
                             cudaStream_t st);
cudaError_t launch_hash_sort(int64_t ncells, const int32_t* offsets, int32_t* elems,
                             int32_t* max_list, cudaStream_t st);
cudaError_t launch_cell_of(int d, const double* grid, int n, int64_t npts, const double* x,
                           int64_t* cell, cudaStream_t st);
// thread per point in hash-cell order (k_prefilter_points)
cudaError_t launch_prefilter(const fpx_mesh_t& m, int64_t n, const double* xo,
                             const int32_t* order, const int2* co, int32_t* best,
                             int32_t* npass, int32_t* code, int32_t* elem, double* r,
                             double* dist, int32_t* iters, double* values, int C,
                             int32_t* elem_count, int64_t* stats, cudaStream_t st);
cudaError_t launch_point_cells(const fpx_mesh_t& m, int64_t n, const double* x, int32_t* cellid,
                               int32_t* cell_count, cudaStream_t st);
cudaError_t launch_point_scatter(int64_t n, int64_t base, int d, const double* x,
                                 const int32_t* cellid, const int32_t* cell_off, int32_t* cursor,
                                 int32_t* order, double* xo, const int32_t* offsets, int64_t nc,
                                 int2* lr, cudaStream_t st);
// Element grouping (fpx_group.cu): count -> packed scan -> items + scatter.
cudaError_t launch_make_items(int64_t E, const int32_t* count, const uint64_t* packed_off,
                              Item* items, int64_t* nitems_dev, cudaStream_t st);
// Zero-copy patch of the rest points' records into mapped host arrays.
cudaError_t launch_rest_flag(int64_t n, const int64_t* nun_dev, const int32_t* upts,
                             int32_t* flag, cudaStream_t st);
cudaError_t launch_rest_patch_host(int dr, int C, int64_t k0, int64_t k1, int32_t* flag,
                                   const int32_t* code, const int32_t* elem, const double* r,
                                   const double* dist, const double* values, int32_t* hcode,
                                   int32_t* helem, double* hr, double* hdist, double* hvalues,
                                   cudaStream_t st);
cudaError_t launch_pack_counts(int64_t E, const int32_t* count, uint64_t* packed,
                               cudaStream_t st);
cudaError_t launch_scatter_units(int64_t nunits_cap, const int64_t* nunits_dev,
                                 const int32_t* unit_elem, const int32_t* unit_ids,
                                 const uint64_t* packed_off, int32_t* cursor, int32_t* sorted,
                                 cudaStream_t st);

// Newton / eval (fpx_newton.cu, FMA allowed).
bool newton_supported(int d, int dr, int N);
// Stream-ordered unit records (x and (point, element, group end)) of round 1.
cudaError_t launch_stream_units(int64_t n, int64_t E, const int32_t* best, const int32_t* count,
                                uint64_t* packed, uint64_t* packed_off, void* scan_temp,
                                size_t scan_bytes, int32_t* cursor, const double* x, int d,
                                const int32_t* order, double* ux, int4* umeta, cudaStream_t st);
// Round 1 streamed (k_newton_stream): points in best-first element order as
// stream records (ux / umeta from launch_stream_units; packed_off[E] = count).
cudaError_t launch_newton_stream(const fpx_mesh_t& m, int64_t n, const double* ux,
                                 const int4* umeta, const uint64_t* packed_off,
                                 const int32_t* npass, int32_t* code, int32_t* elem, double* r,
                                 double* dist, int32_t* iters, const double* field, int C,
                                 double* values, int32_t* upts, int64_t* nun_dev,
                                 int64_t* chunk_ctr, int4* redo, int64_t* nredo, int64_t redo_cap,
                                 int64_t* stats, cudaStream_t st);
// Remaining candidates of the points round 1 left unresolved: their
// best-first candidate lists (k_rest_lists), then the lane-per-point Newton
// (k_rest_lanes).
cudaError_t launch_rest_lists(const fpx_mesh_t& m, const double* x, int64_t nun_cap,
                              const int64_t* nun_dev, const int32_t* upts, int32_t* best,
                              const int32_t* npass, int32_t* clist,
                              int32_t* cnum, int32_t* nps, int32_t* hist, int32_t* bstart,
                              int32_t* bcur, int32_t* perm, int64_t* cum, int32_t* maxnp,
                              int4* pairs, int64_t* npairs, cudaStream_t st);
cudaError_t launch_find_rest(const fpx_mesh_t& m, const double* x, int64_t nun_cap,
                             const int64_t* nun_dev, const int32_t* upts, const int32_t* clist,
                             const int32_t* cnum, const int32_t* nps, const int32_t* perm,
                             const int64_t* cum, const int32_t* maxnp, const int32_t* best,
                             const int4* pairs, const int64_t* npairs, int4* redo,
                             int64_t* nredo, int32_t* found,
                             int32_t* lock, int32_t* code, int32_t* elem, double* r, double* dist,
                             int32_t* iters, const double* field, int C, double* values,
                             int64_t* counter, int64_t* stats, cudaStream_t st);
cudaError_t launch_eval_items(int dr, int Nf, const double* fbasis, int C, const double* field,
                              const double* r, const int32_t* sorted_pts, const Item* items,
                              const int64_t* nitems_dev, int64_t items_cap, double* values,
                              cudaStream_t st);
cudaError_t launch_eval_mark(int64_t n, int C, const int32_t* code, const int32_t* elem,
                             double* values, int32_t* unit_elem, int32_t* count,
                             cudaStream_t st);
cudaError_t launch_invert_pairs(const fpx_mesh_t& m, int64_t npairs, const double* x,
                                const int32_t* elem, double* r, double* dist, int32_t* iters,
                                int32_t* conv, cudaStream_t st);
cudaError_t launch_forward_map(const fpx_mesh_t& m, int64_t n, const int32_t* elem,
                               const double* r, double* x, double* G, double* H2,
                               cudaStream_t st);

// Particle update (fpx_particles.cu): Stokes RHS + AB2 + periodic wrap.
cudaError_t launch_particles_advance(int d, int64_t n, double* x, double* v, const double* u,
                                     double* v_prev, double* a_prev, double tau, double dt,
                                     int first, const double* box, int periodic,
                                     cudaStream_t st);

}  // namespace fpx
