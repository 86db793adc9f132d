// fpx_group.cu -- element grouping of find/eval work units.
//
// Units (points or (point, element) pairs) keyed by element id are bucketed
// with a counting sort: per-element counts, one exclusive scan of the packed
// (items << 32 | count) words, then a scatter.  A work item is one element
// and up to FPX_ITEM units; one warp processes one item.  Order within an
// element is irrelevant: every unit's result depends only on its own inputs.
#include <cub/device/device_scan.cuh>

#include "fpx_common.cuh"
#include "fpx_kernels.cuh"

namespace fpx {

static unsigned grid_of(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  if (b > 148 * 32) b = 148 * 32;
  if (b < 1) b = 1;
  return (unsigned)b;
}

__global__ void k_pack_counts(int64_t E, const int32_t* __restrict__ count, uint64_t* packed) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t c = (uint32_t)count[e];
    const uint64_t it = (c + FPX_ITEM - 1) / FPX_ITEM;
    packed[e] = (it << 32) | c;
  }
}

// packed_off = exclusive scan of packed (E + 1 entries: last = totals).
__global__ void k_make_items(int64_t E, const int32_t* __restrict__ count,
                             const uint64_t* __restrict__ packed_off, Item* items,
                             int64_t* nitems_dev) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int c = count[e];
    const uint64_t o = packed_off[e];
    const int64_t item0 = (int64_t)(o >> 32);
    const int64_t unit0 = (int64_t)(o & 0xffffffffull);
    for (int q = 0; q * FPX_ITEM < c; ++q) {
      Item it;
      it.elem = (int32_t)e;
      it.start = (int32_t)(unit0 + q * FPX_ITEM);
      it.count = c - q * FPX_ITEM < FPX_ITEM ? c - q * FPX_ITEM : FPX_ITEM;
      items[item0 + q] = it;
    }
    if (e == E - 1) *nitems_dev = (int64_t)(packed_off[E] >> 32);
  }
}

__global__ void k_scatter_units(int64_t cap, const int64_t* __restrict__ n_dev,
                                const int32_t* __restrict__ unit_elem,
                                const int32_t* __restrict__ unit_ids,
                                const uint64_t* __restrict__ packed_off, int32_t* cursor,
                                int32_t* sorted) {
  const int64_t n = n_dev ? *n_dev : cap;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n;
       u += (int64_t)gridDim.x * blockDim.x) {
    const int e = unit_elem[u];
    if (e < 0) continue;
    const int slot = atomicAdd(&cursor[e], 1);
    sorted[(int64_t)(packed_off[e] & 0xffffffffull) + slot] = unit_ids ? unit_ids[u] : (int32_t)u;
  }
}

// Stream-ordered unit records of round 1 (k_newton_stream), scattered
// straight from the points: point k with best-first element e gets a slot
// in e's group (packed_off = exclusive scan of the per-element counts) and
// writes its coordinates ux[g] and umeta[g] = (point, element, end of the
// element's group).  The round-1 loader and lane refill then read one
// record each; no intermediate sorted-index array, no work items.
__global__ void k_stream_scatter(int64_t n, const int32_t* __restrict__ best,
                                 const uint64_t* __restrict__ packed_off,
                                 const int32_t* __restrict__ ecount, const double* __restrict__ x,
                                 int d, const int32_t* __restrict__ order, int32_t* cursor,
                                 double* ux, int4* umeta) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    // points in hash-cell order (the prefilter's): neighbouring lanes mostly
    // share a best element, so their records land in consecutive slots
    const int64_t k = order ? order[t] : t;
    const int e = best[k];
    if (e < 0) continue;
    const unsigned act = __activemask();
    const unsigned peers = __match_any_sync(act, e);
    const int lane = threadIdx.x % 32;
    const int leader = __ffs(peers) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(&cursor[e], __popc(peers));
    base = __shfl_sync(peers, base, leader);
    const int64_t g0 = (int64_t)(packed_off[e] & 0xffffffffull);
    const int64_t g = g0 + base + __popc(peers & ((1u << lane) - 1u));
    for (int c = 0; c < d; ++c) ux[g * d + c] = x[k * d + c];
    umeta[g] = make_int4((int)k, e, (int)(g0 + ecount[e]), 0);
  }
}

cudaError_t launch_stream_units(int64_t n, int64_t E, const int32_t* best, const int32_t* count,
                                uint64_t* packed, uint64_t* packed_off, void* scan_temp,
                                size_t scan_bytes, int32_t* cursor, const double* x, int d,
                                const int32_t* order, double* ux, int4* umeta, cudaStream_t st) {
  cudaError_t e;
  k_pack_counts<<<grid_of(E, 256), 256, 0, st>>>(E, count, packed);
  if ((e = cudaMemsetAsync(packed + E, 0, sizeof(uint64_t), st)) != cudaSuccess) return e;
  size_t tb = scan_bytes;
  if ((e = cub::DeviceScan::ExclusiveSum(scan_temp, tb, packed, packed_off, (int)(E + 1), st)) !=
      cudaSuccess)
    return e;
  if ((e = cudaMemsetAsync(cursor, 0, sizeof(int32_t) * E, st)) != cudaSuccess) return e;
  k_stream_scatter<<<grid_of(n, 256), 256, 0, st>>>(n, best, packed_off, count, x, d, order,
                                                    cursor, ux, umeta);
  return cudaGetLastError();
}

// Zero-copy patch of host records: the rest points' records written straight
// into mapped pinned host arrays over PCIe, after the bulk download of the
// round-1 records (engine.find_and_interpolate_host).  No host thread touches
// those arrays, so the next download into them never snoops a CPU cache.
// dst[0..len) = src[0..len) with 16-byte stores where dst allows: each store
// is one PCIe write, and the write count bounds k_rest_patch_host
__device__ __forceinline__ void store_row(double* dst, const double* src, int len) {
  int a = 0;
  if (len >= 2 && (reinterpret_cast<uintptr_t>(dst) & 15)) {
    dst[0] = src[0];
    a = 1;
  }
  for (; a + 1 < len; a += 2)
    *reinterpret_cast<double2*>(dst + a) = make_double2(src[a], src[a + 1]);
  if (a < len) dst[a] = src[a];
}

// flag[k] marks the rest points (k_rest_flag); the patch threads walk the
// points in order, so the PCIe writes in flight land on neighbouring host
// pages (IOMMU / DRAM locality), and clear the flags behind them.
__global__ void k_rest_flag(const int64_t* __restrict__ nun_dev, const int32_t* __restrict__ upts,
                            int32_t* flag) {
  const int64_t nun = *nun_dev;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < nun;
       u += (int64_t)gridDim.x * blockDim.x)
    flag[upts[u]] = 1;
}

__global__ void k_rest_patch_host(int dr, int C, int64_t k0, int64_t k1, int32_t* flag,
                                  const int32_t* __restrict__ code,
                                  const int32_t* __restrict__ elem, const double* __restrict__ r,
                                  const double* __restrict__ dist,
                                  const double* __restrict__ values, int32_t* hcode,
                                  int32_t* helem, double* hr, double* hdist, double* hvalues) {
  for (int64_t k = k0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < k1;
       k += (int64_t)gridDim.x * blockDim.x) {
    if (!flag[k]) continue;
    flag[k] = 0;
    hcode[k] = code[k];
    helem[k] = elem[k];
    store_row(hr + k * dr, r + k * dr, dr);
    hdist[k] = dist[k];
    if (values) store_row(hvalues + k * C, values + k * C, C);
  }
}

cudaError_t launch_rest_flag(int64_t n, const int64_t* nun_dev, const int32_t* upts,
                             int32_t* flag, cudaStream_t st) {
  k_rest_flag<<<grid_of(n, 256), 256, 0, st>>>(nun_dev, upts, flag);
  return cudaGetLastError();
}

cudaError_t launch_rest_patch_host(int dr, int C, int64_t k0, int64_t k1, int32_t* flag,
                                   const int32_t* code, const int32_t* elem, const double* r,
                                   const double* dist, const double* values, int32_t* hcode,
                                   int32_t* helem, double* hr, double* hdist, double* hvalues,
                                   cudaStream_t st) {
  int64_t b = (k1 - k0 + 255) / 256;
  if (b > 148 * 8) b = 148 * 8;
  if (b < 1) b = 1;
  k_rest_patch_host<<<(unsigned)b, 256, 0, st>>>(dr, C, k0, k1, flag, code, elem, r, dist,
                                                 values, hcode, helem, hr, hdist, hvalues);
  return cudaGetLastError();
}

cudaError_t launch_pack_counts(int64_t E, const int32_t* count, uint64_t* packed,
                               cudaStream_t st) {
  k_pack_counts<<<grid_of(E, 256), 256, 0, st>>>(E, count, packed);
  return cudaGetLastError();
}

cudaError_t launch_make_items(int64_t E, const int32_t* count, const uint64_t* packed_off,
                              Item* items, int64_t* nitems_dev, cudaStream_t st) {
  k_make_items<<<grid_of(E, 256), 256, 0, st>>>(E, count, packed_off, items, nitems_dev);
  return cudaGetLastError();
}

cudaError_t launch_scatter_units(int64_t nunits_cap, const int64_t* nunits_dev,
                                 const int32_t* unit_elem, const int32_t* unit_ids,
                                 const uint64_t* packed_off, int32_t* cursor, int32_t* sorted,
                                 cudaStream_t st) {
  k_scatter_units<<<grid_of(nunits_cap, 256), 256, 0, st>>>(nunits_cap, nunits_dev, unit_elem,
                                                            unit_ids, packed_off, cursor, sorted);
  return cudaGetLastError();
}

}  // namespace fpx
