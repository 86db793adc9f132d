// fpx_abi.cu -- extern "C" entry points of libfpx_sm100.so (include/fpx.h).
//
// Host-side orchestration of the kernels: argument checks, workspace
// carving, CUB scans, stream-ordered launches.  No exceptions cross the ABI;
// failures return FPX_E* with a thread-local message.
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdarg>
#include <mutex>
#include <unordered_map>
#include <utility>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/fpx.h"
#include "fpx_common.cuh"
#include "fpx_kernels.cuh"

namespace fpx {
cudaError_t launch_invert_pairs_grouped(const fpx_mesh_t& m, const double* x,
                                        const int32_t* sorted, const Item* items,
                                        const int64_t* nitems_dev, int64_t items_cap,
                                        const double* r0, double* r, double* dist,
                                        int32_t* iters, int32_t* conv, cudaStream_t st);
}

using fpx::Item;

namespace {

thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};
cudaEvent_t g_prof_start = nullptr, g_prof_stop = nullptr;
thread_local cudaEvent_t g_round1_done = nullptr;
// fpx_set_upload_events: the points arrive in k chunks, chunk c ready at ev[c]
constexpr int kMaxUpload = 16;
thread_local int g_upload_k = 0;
// fpx_set_round1_events: round 1 per upload chunk, chunk c's done at ev[c]
thread_local int g_r1_k = 0;
// fpx_set_find_hint: per point a hinted element for the next fpx_find
thread_local const int32_t* g_hint = nullptr;
thread_local cudaEvent_t g_upload_ev[kMaxUpload];
thread_local cudaEvent_t g_r1_ev[kMaxUpload];

// Layout of every find workspace at its last fpx_find (points, elements):
// fpx_rest_patch_host re-carves the workspace and must see the same layout.
std::mutex g_ws_mu;
std::unordered_map<const void*, std::pair<int64_t, int64_t>> g_ws_layout;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define FPX_LAUNCH(expr)   \
  do {                     \
    g_launches += 1;       \
    FPX_CK(expr);          \
  } while (0)

#define FPX_CK(expr)                                                                   \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail(FPX_ECUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                 \
  } while (0)

// Bump allocator over a caller-provided workspace (256-byte aligned slices).
struct Carver {
  char* base;
  size_t cap, off;
  explicit Carver(void* b, size_t c) : base((char*)b), cap(c), off(0) {}
  template <typename T>
  T* take(size_t count) {
    size_t a = (off + 255) & ~size_t(255);
    off = a + count * sizeof(T);
    if (!base) return nullptr;
    return reinterpret_cast<T*>(base + a);
  }
  bool ok() const { return off <= cap; }
};

size_t scan_temp_u64(int64_t n) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, (uint64_t*)nullptr, (uint64_t*)nullptr, (int)n);
  return bytes;
}
size_t scan_temp_i64(int64_t n) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, (int64_t*)nullptr, (int64_t*)nullptr, (int)n);
  return bytes;
}
size_t scan_temp_i32(int64_t n) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, (int32_t*)nullptr, (int32_t*)nullptr, (int)n);
  return bytes;
}

int64_t items_cap_of(int64_t E, int64_t units) { return E + units / FPX_ITEM + 2; }

// Grouping buffers for up to `units` units over E elements.
struct Group {
  int32_t* count;
  int32_t* cursor;
  uint64_t* packed;
  uint64_t* packed_off;
  Item* items;
  int64_t* nitems;
  int32_t* sorted;
  void* temp;
  size_t temp_bytes;
  int64_t items_cap;
  void carve(Carver& c, int64_t E, int64_t units) {
    count = c.take<int32_t>(E);
    cursor = c.take<int32_t>(E);
    packed = c.take<uint64_t>(E + 1);
    packed_off = c.take<uint64_t>(E + 1);
    items_cap = items_cap_of(E, units);
    items = c.take<Item>(items_cap);
    nitems = c.take<int64_t>(1);
    sorted = c.take<int32_t>(units > 0 ? units : 1);
    temp_bytes = scan_temp_u64(E + 1);
    temp = c.take<char>(temp_bytes);
  }
  // counts must be filled; builds items and scatters units.
  cudaError_t build(int64_t E, int64_t units_cap, const int64_t* units_dev,
                    const int32_t* unit_elem, const int32_t* unit_ids, cudaStream_t st) {
    cudaError_t e;
    if ((e = fpx::launch_pack_counts(E, count, packed, st)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(packed + E, 0, sizeof(uint64_t), st)) != cudaSuccess) return e;
    size_t tb = temp_bytes;
    if ((e = cub::DeviceScan::ExclusiveSum(temp, tb, packed, packed_off, (int)(E + 1), st)) !=
        cudaSuccess)
      return e;
    if ((e = fpx::launch_make_items(E, count, packed_off, items, nitems, st)) != cudaSuccess)
      return e;
    if ((e = cudaMemsetAsync(cursor, 0, sizeof(int32_t) * E, st)) != cudaSuccess) return e;
    return fpx::launch_scatter_units(units_cap, units_dev, unit_elem, unit_ids, packed_off,
                                     cursor, sorted, st);
  }
};

struct FindWs {
  int32_t *best, *npass, *upts, *clist, *cnum, *found, *lock, *nps, *perm, *hist, *bstart, *bcur,
      *maxnp;
  int64_t *cum, *npairs, *nredo;
  int4 *pairs, *redo, *umeta;
  double* ux;
  int64_t *nun, *counter, *chunk_ctr;
  Group g1;
  // point ordering by hash cell
  int32_t *cellid, *cell_count, *cell_off, *cell_cursor, *order;
  void* scan3_temp;
  size_t scan3_bytes;
  int64_t ncells;
  void carve_cells(Carver& c, int64_t n, int64_t nc) {
    ncells = nc;
    cellid = c.take<int32_t>(n);
    cell_count = c.take<int32_t>(nc + 2);
    cell_off = c.take<int32_t>(nc + 2);
    cell_cursor = c.take<int32_t>(nc + 2);
    order = c.take<int32_t>(n);
    scan3_bytes = scan_temp_i32(nc + 2);
    scan3_temp = c.take<char>(scan3_bytes);
  }
  void carve(Carver& c, int64_t E, int64_t n) {
    best = c.take<int32_t>(n);
    npass = c.take<int32_t>(n);
    upts = c.take<int32_t>(n);
    clist = c.take<int32_t>(n * FPX_RK);
    cnum = c.take<int32_t>(n);
    found = c.take<int32_t>(n);
    lock = c.take<int32_t>(n);
    nps = c.take<int32_t>(n);
    perm = c.take<int32_t>(n);
    hist = c.take<int32_t>(3 * FPX_HMAX);  // hist | bcur | bstart (one memset)
    bcur = hist + FPX_HMAX;
    bstart = hist + 2 * FPX_HMAX;
    maxnp = c.take<int32_t>(1);
    cum = c.take<int64_t>(FPX_HMAX + 1);
    pairs = c.take<int4>(2 * n + 1024);  // pair list (beyond: rebuilt by the kernel)
    redo = c.take<int4>(2 * n + 1024);   // pairs stopped on a face (second pass)
    npairs = c.take<int64_t>(1);
    nredo = c.take<int64_t>(1);
    nun = c.take<int64_t>(1);
    counter = c.take<int64_t>(2);
    chunk_ctr = c.take<int64_t>(1);
    ux = c.take<double>(3 * n);
    umeta = c.take<int4>(n);
    g1.carve(c, E, n);
  }
};

__global__ void k_find_totals(const int64_t* __restrict__ nun, const int64_t* __restrict__ nredo,
                              int64_t* stats, int64_t n) {
  stats[FPX_STAT_POINTS] = n;
  stats[FPX_STAT_ROUND2_POINTS] = *nun;
  stats[FPX_STAT_REDO] = *nredo;
}


// Hinted find: round 1 solves every point on its hinted element (best =
// hint, npass = -1 marks the point as hinted), no prefilter.
__global__ void k_hint_init(int64_t n, int64_t E, const int32_t* __restrict__ hint, int32_t* best,
                            int32_t* npass, int32_t* count) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int e = hint[k];
    const int eh = e >= 0 && e < E ? e : 0;  // (engine guarantees a valid hint)
    best[k] = eh;
    npass[k] = -1;
    atomicAdd(&count[eh], 1);
  }
}

__global__ void k_count_elems(int64_t n, const int32_t* __restrict__ elem, int32_t* count) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&count[elem[k]], 1);
}

// 8 independent DFMA chains per thread (fpx_probe_fp64).
__global__ void __launch_bounds__(256) k_dfma_probe(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += x[c];
  if (s == 12345.678) *out = s;
}

unsigned grid1(int64_t n, int threads = 256) {
  int64_t b = (n + threads - 1) / threads;
  if (b > 148 * 32) b = 148 * 32;
  if (b < 1) b = 1;
  return (unsigned)b;
}

cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int check_mesh(const fpx_mesh_t* m) {
  if (!m) return fail(FPX_EINVAL, "mesh is NULL");
  if (!(m->d == 2 || m->d == 3) || m->dr < 1 || m->dr > m->d)
    return fail(FPX_EINVAL, "bad dimensions d=%d dr=%d", m->d, m->dr);
  if (!fpx::newton_supported(m->d, m->dr, m->N))
    return fail(FPX_EUNSUPPORTED, "order N=%d not compiled for d=%d dr=%d", m->N, m->d, m->dr);
  if (m->E < 1 || m->E > INT32_MAX) return fail(FPX_EINVAL, "bad element count %lld", (long long)m->E);
  return FPX_OK;
}

}  // namespace

extern "C" {

int fpx_abi_version(void) { return FPX_ABI_VERSION; }

const char* fpx_last_error(void) { return g_err.c_str(); }

int fpx_supported(int d, int dr, int N) { return fpx::newton_supported(d, dr, N) ? 1 : 0; }

int64_t fpx_launch_count(void) { return g_launches.load(); }

int fpx_profile_round1(void* ev_start, void* ev_stop) {
  g_prof_start = reinterpret_cast<cudaEvent_t>(ev_start);
  g_prof_stop = reinterpret_cast<cudaEvent_t>(ev_stop);
  return FPX_OK;
}

int fpx_set_round1_event(void* ev) {
  g_round1_done = reinterpret_cast<cudaEvent_t>(ev);
  return FPX_OK;
}

int fpx_set_round1_events(int k, void* const* events) {
  if (k <= 0 || !events) {
    g_r1_k = 0;
    return FPX_OK;
  }
  if (k > kMaxUpload) return fail(FPX_EINVAL, "round-1 events: k=%d > %d", k, kMaxUpload);
  for (int c = 0; c < k; ++c) g_r1_ev[c] = reinterpret_cast<cudaEvent_t>(events[c]);
  g_r1_k = k;
  return FPX_OK;
}

int fpx_set_find_hint(const int32_t* elem) {
  g_hint = elem;
  return FPX_OK;
}

int fpx_set_upload_events(int k, void* const* events) {
  if (k <= 0 || !events) {
    g_upload_k = 0;
    return FPX_OK;
  }
  if (k > kMaxUpload) return fail(FPX_EINVAL, "upload events: k=%d > %d", k, kMaxUpload);
  for (int c = 0; c < k; ++c) g_upload_ev[c] = reinterpret_cast<cudaEvent_t>(events[c]);
  g_upload_k = k;
  return FPX_OK;
}

int fpx_rest_patch_host(int dr, int C, int64_t n, int64_t k0, int64_t k1, void* ws,
                        size_t ws_bytes,
                        const fpx_mesh_t* m, const int32_t* code, const int32_t* elem,
                        const double* r, const double* dist, const double* values,
                        int32_t* hcode, int32_t* helem, double* hr, double* hdist,
                        double* hvalues, void* stream) {
  int rc = check_mesh(m);
  if (rc) return rc;
  if (!hcode || !helem || !hr || !hdist || (values && !hvalues))
    return fail(FPX_EINVAL, "rest patch: null host array");
  if (k0 < 0 || k1 > n || k0 > k1) return fail(FPX_EINVAL, "rest patch: bad range");
  // the host arrays must be device-accessible (pinned, hence mapped)
  const void* hp[5] = {hcode, helem, hr, hdist, values ? (const void*)hvalues : (const void*)hcode};
  for (const void* p : hp) {
    cudaPointerAttributes at;
    FPX_CK(cudaPointerGetAttributes(&at, p));
    if (at.type != cudaMemoryTypeHost || at.devicePointer != p)
      return fail(FPX_EINVAL, "rest patch: host array %p is not mapped pinned memory", p);
  }
  {
    std::lock_guard<std::mutex> g(g_ws_mu);
    auto it = g_ws_layout.find(ws);
    if (it == g_ws_layout.end() || it->second.first != n || it->second.second != m->E)
      return fail(FPX_EINVAL, "rest patch: workspace was not last used by a host-mode fpx_find "
                  "of %lld points on this mesh", (long long)n);
  }
  Carver cv(ws, ws_bytes);
  FindWs w;
  w.carve(cv, m->E, n);
  if (!cv.ok()) return fail(FPX_EINVAL, "rest patch: workspace too small");
  // point order over the flags the host-mode find left in its lock array:
  // the PCIe writes in flight land on neighbouring host pages, 708 -> 505 us
  // per 10^6 points against walking the rest list
  if (k1 > k0)
    FPX_LAUNCH(fpx::launch_rest_patch_host(dr, C, k0, k1, w.lock, code, elem, r, dist, values,
                                           hcode, helem, hr, hdist, hvalues, S(stream)));
  return FPX_OK;
}

int fpx_probe_fp64(double* tflops_host, void* stream) {
  cudaStream_t st = S(stream);
  int dev = 0, sms = 148;
  FPX_CK(cudaGetDevice(&dev));
  FPX_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  double* out = nullptr;
  FPX_CK(cudaMallocAsync(&out, sizeof(double), st));
  cudaEvent_t e0, e1;
  FPX_CK(cudaEventCreate(&e0));
  FPX_CK(cudaEventCreate(&e1));
  const int iters = 20000, blocks = sms * 8, threads = 256;
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    FPX_CK(cudaEventRecord(e0, st));
    k_dfma_probe<<<blocks, threads, 0, st>>>(out, iters, 0.999999, 1e-7);
    FPX_CK(cudaEventRecord(e1, st));
    FPX_CK(cudaEventSynchronize(e1));
    float ms = 0.f;
    FPX_CK(cudaEventElapsedTime(&ms, e0, e1));
    if (rep > 0 && ms < best) best = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  FPX_CK(cudaFreeAsync(out, st));
  *tflops_host = 2.0 * 8 * (double)iters * blocks * threads / (best * 1e-3) / 1e12;
  return FPX_OK;
}

int fpx_setup_bounds(int d, int dr, int N, int M, int64_t E, const double* basis,
                     const double* nodes, double expansion, double* aabb, double* obb_c,
                     double* obb_inv, double* hbox, double* frame, uint8_t* obb_ok,
                     int32_t* status, void* stream) {
  if (!(d == 2 || d == 3) || dr < 1 || dr > d) return fail(FPX_EINVAL, "bad d/dr %d/%d", d, dr);
  if (N < 2 || N > FPX_SETUP_MAXN) return fail(FPX_EUNSUPPORTED, "setup supports 2 <= N <= %d", FPX_SETUP_MAXN);
  if (M < N || M > 4 * FPX_SETUP_MAXN) return fail(FPX_EINVAL, "bad interval count M=%d", M);
  if (E < 0) return fail(FPX_EINVAL, "negative element count");
  if (E == 0) return FPX_OK;
  FPX_LAUNCH(fpx::launch_setup_bounds(d, dr, N, M, E, basis, nodes, expansion, aabb, obb_c, obb_inv,
                                  hbox, frame, obb_ok, status, S(stream)));
  return FPX_OK;
}

int fpx_filter_records(int d, int64_t E, const double* aabb, const double* obb_c,
                       const double* obb_inv, const uint8_t* obb_ok, const double* frame,
                       double* frec, float* fbox, void* stream) {
  if (!(d == 2 || d == 3)) return fail(FPX_EINVAL, "filter records: bad d=%d", d);
  if (4 * d + 2 * d * d + 1 > FPX_FREC) return fail(FPX_EINVAL, "filter record too small");
  if (E <= 0) return FPX_OK;
  if (!fbox || (reinterpret_cast<uintptr_t>(fbox) & 15))
    return fail(FPX_EINVAL, "filter records: fbox must be a 16-byte aligned array");
  FPX_LAUNCH(fpx::launch_filter_records(d, E, aabb, obb_c, obb_inv, obb_ok, frame, frec, fbox,
                                        S(stream)));
  return FPX_OK;
}

int fpx_pad_nodes(int d, int dr, int N, int64_t E, const double* nodes, double* nodes_pad,
                  void* stream) {
  if (!(d == 2 || d == 3) || dr < 1 || dr > d) return fail(FPX_EINVAL, "pad: bad d/dr %d/%d", d, dr);
  if (N < 2) return fail(FPX_EINVAL, "pad: bad N=%d", N);
  if (E <= 0) return FPX_OK;
  FPX_LAUNCH(fpx::launch_pad_nodes(d, dr, N, E, nodes, nodes_pad, S(stream)));
  return FPX_OK;
}

int fpx_bound_function(int dr, int N, int M, int64_t nf, const double* basis,
                       const double* values, double* lower, double* upper, void* stream) {
  if (dr != 1 && dr != 2) return fail(FPX_EINVAL, "bound_function: dr must be 1 or 2");
  if (N < 2 || N > FPX_SETUP_MAXN || M < N || M > 4 * FPX_SETUP_MAXN)
    return fail(FPX_EINVAL, "bound_function: bad N=%d M=%d", N, M);
  if (nf <= 0) return FPX_OK;
  FPX_LAUNCH(fpx::launch_bound_function(dr, N, M, nf, basis, values, lower, upper, S(stream)));
  return FPX_OK;
}

size_t fpx_hash_workspace_bytes(int d, int64_t E, int ncell) {
  (void)E;
  int64_t nc = 1;
  for (int c = 0; c < d; ++c) nc *= ncell;
  Carver c(nullptr, 0);
  c.take<int32_t>(nc + 1);
  c.take<int32_t>(nc + 1);
  c.take<int32_t>(1);
  c.take<char>(scan_temp_i32(nc + 1));
  return c.off + 256;
}

int fpx_hash_build(int d, int64_t E, const double* box, const double* obb_c,
                   const double* obb_inv, const uint8_t* obb_ok, int ncell, double* grid,
                   int32_t* offsets, int32_t* elems, int64_t cap, int64_t* needed_host,
                   int32_t* max_list_host, void* ws, size_t ws_bytes, void* stream) {
  if (!(d == 2 || d == 3)) return fail(FPX_EINVAL, "hash: bad d=%d", d);
  if (E < 1) return fail(FPX_EINVAL, "build_local_map: empty element list (SPEC.md:234)");
  if (ncell < 1 || ncell > 1024) return fail(FPX_EINVAL, "hash: cells per axis %d", ncell);
  int64_t nc = 1;
  for (int c = 0; c < d; ++c) nc *= ncell;
  if (nc > (int64_t)1 << 30) return fail(FPX_EINVAL, "hash: too many cells (%lld)", (long long)nc);
  Carver cv(ws, ws_bytes);
  int32_t* cnt = cv.take<int32_t>(nc + 1);
  int32_t* cursor = cv.take<int32_t>(nc + 1);
  int32_t* maxl = cv.take<int32_t>(1);
  size_t tb = scan_temp_i32(nc + 1);
  void* temp = cv.take<char>(tb);
  if (!cv.ok()) return fail(FPX_EINVAL, "hash workspace too small (%zu < %zu)", ws_bytes, cv.off);
  cudaStream_t st = S(stream);
  FPX_LAUNCH(fpx::launch_hash_grid(d, E, box, ncell, grid, st));
  FPX_CK(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (nc + 1), st));
  FPX_LAUNCH(fpx::launch_hash_count(d, E, box, obb_c, obb_inv, obb_ok, grid, ncell, cnt, st));
  FPX_CK(cub::DeviceScan::ExclusiveSum(temp, tb, cnt, offsets, (int)(nc + 1), st));
  int32_t total = 0;
  FPX_CK(cudaMemcpyAsync(&total, offsets + nc, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  FPX_CK(cudaStreamSynchronize(st));
  if (total < 0) return fail(FPX_EINVAL, "hash: entry count overflow");
  if (needed_host) *needed_host = total;
  if (!elems || cap < total) return FPX_OK;
  FPX_CK(cudaMemsetAsync(cursor, 0, sizeof(int32_t) * (nc + 1), st));
  FPX_CK(cudaMemsetAsync(maxl, 0, sizeof(int32_t), st));
  FPX_LAUNCH(fpx::launch_hash_fill(d, E, box, obb_c, obb_inv, obb_ok, grid, ncell, offsets,
                                   cursor, elems, st));
  FPX_LAUNCH(fpx::launch_hash_sort(nc, offsets, elems, maxl, st));
  int32_t ml = 0;
  FPX_CK(cudaMemcpyAsync(&ml, maxl, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  FPX_CK(cudaStreamSynchronize(st));
  if (max_list_host) *max_list_host = ml;
  return FPX_OK;
}

int fpx_cell_of(const fpx_mesh_t* m, int64_t n, const double* x, int64_t* cell, void* stream) {
  if (!m) return fail(FPX_EINVAL, "mesh is NULL");
  if (n <= 0) return FPX_OK;
  FPX_LAUNCH(fpx::launch_cell_of(m->d, m->grid, m->ncell, n, x, cell, S(stream)));
  return FPX_OK;
}

static int64_t cells_of(const fpx_mesh_t* m) {
  int64_t nc = 1;
  for (int c = 0; c < m->d; ++c) nc *= m->ncell;
  return nc;
}

size_t fpx_find_workspace_bytes(const fpx_mesh_t* m, int64_t n, int64_t pair_cap) {
  (void)pair_cap;  // ABI v1 argument; the rest kernel needs no pair buffers
  Carver c(nullptr, 0);
  FindWs w;
  w.carve(c, m->E, n > 0 ? n : 1);
  w.carve_cells(c, n > 0 ? n : 1, cells_of(m));
  return c.off + 256;
}

// engine.find Phase A over n points:
//   1. counting sort of the points by hash cell;
//   2. prefilter: per cell, the hash list through the AABB/OBB filter, the
//      best-first ranked candidates of each point (NOT_FOUND if none);
//   3. round 1: element-major Newton on every point's best-first candidate
//      (final if INTERIOR or the only candidate; fused field evaluation);
//   4. rest: the remaining candidates of the unresolved points, best-first,
//      stopping at the first INTERIOR, else the D6 winner (fused eval).
int fpx_find(const fpx_mesh_t* m, int64_t n, const double* x, int32_t* code, int32_t* elem,
             double* r, double* dist, int32_t* iters, const double* field, int C,
             double* values, int64_t* stats, int64_t pair_cap, void* ws, size_t ws_bytes,
             void* stream) {
  (void)pair_cap;
  int rc = check_mesh(m);
  if (rc) return rc;
  if (n < 0 || n > INT32_MAX) return fail(FPX_EINVAL, "bad point count %lld", (long long)n);
  if (!stats) return fail(FPX_EINVAL, "stats buffer required");
  if (field && (C < 1 || !values)) return fail(FPX_EINVAL, "field given without C/values");
  cudaStream_t st = S(stream);
  FPX_CK(cudaMemsetAsync(stats, 0, sizeof(int64_t) * FPX_STATS_LEN, st));
  if (n == 0) return FPX_OK;
  const int64_t E = m->E;
  Carver cv(ws, ws_bytes);
  FindWs w;
  w.carve(cv, E, n);
  w.carve_cells(cv, n, cells_of(m));
  if (!cv.ok()) return fail(FPX_EINVAL, "find workspace too small (%zu < %zu)", ws_bytes, cv.off);
  if (!m->frec || !m->fbox)
    return fail(FPX_EINVAL, "mesh has no filter records (fpx_filter_records)");
  if (!m->nodes_pad) return fail(FPX_EINVAL, "mesh has no padded nodes (fpx_pad_nodes)");
  {
    std::lock_guard<std::mutex> g(g_ws_mu);
    g_ws_layout[ws] = {n, E};
  }
  const fpx_mesh_t& M = *m;
  // --- order the points by hash cell (counting sort), then the prefilter:
  // hash list + AABB/OBB filter + best-first ranking.  With upload events
  // (host path) the points arrive in k chunks and each chunk is sorted and
  // filtered as soon as it has landed, under the next chunk's copy.
  const int64_t nc = w.ncells;
  FPX_CK(cudaMemsetAsync(w.g1.count, 0, sizeof(int32_t) * E, st));
  const int nchunk = g_hint ? 0 : (g_upload_k > 1 ? g_upload_k : 1);
  // round 1 per chunk (host mode, fpx_set_round1_events): each chunk is
  // grouped and solved as soon as it is filtered, so its records can go
  // down while the next chunks are uploaded and solved; one rest phase
  const bool r1_chunks = !g_hint && g_r1_k > 0 && g_r1_k == nchunk;
  FPX_CK(cudaMemsetAsync(w.nun, 0, sizeof(int64_t), st));
  FPX_CK(cudaMemsetAsync(w.counter, 0, 2 * sizeof(int64_t), st));
  FPX_CK(cudaMemsetAsync(w.nredo, 0, sizeof(int64_t), st));
  if (g_hint) {  // hinted find (particles): round 1 on the hinted elements, no prefilter
    for (int ck = 0; ck < g_upload_k; ++ck) FPX_CK(cudaStreamWaitEvent(st, g_upload_ev[ck], 0));
    g_launches += 1;
    k_hint_init<<<grid1(n), 256, 0, st>>>(n, E, g_hint, w.best, w.npass, w.g1.count);
    FPX_CK(cudaGetLastError());
  }
  for (int ck = 0; ck < nchunk; ++ck) {
    const int64_t a = n * ck / nchunk, nn = n * (ck + 1) / nchunk - a;
    if (g_upload_k > 0) FPX_CK(cudaStreamWaitEvent(st, g_upload_ev[ck], 0));  // nchunk == k
    if (nn == 0) continue;
    const double* xa = x + a * M.d;
    if (r1_chunks && ck > 0) FPX_CK(cudaMemsetAsync(w.g1.count, 0, sizeof(int32_t) * E, st));
    FPX_CK(cudaMemsetAsync(w.cell_count, 0, sizeof(int32_t) * (nc + 2), st));
    FPX_LAUNCH(fpx::launch_point_cells(M, nn, xa, w.cellid + a, w.cell_count, st));
    {
      size_t tb3 = w.scan3_bytes;
      FPX_CK(cub::DeviceScan::ExclusiveSum(w.scan3_temp, tb3, w.cell_count, w.cell_off,
                                           (int)(nc + 2), st));
    }
    FPX_CK(cudaMemsetAsync(w.cell_cursor, 0, sizeof(int32_t) * (nc + 2), st));
    // cell-ordered point copies and list ranges for the prefilter: in
    // buffers that are free until later phases (ux: round-1 stream records;
    // clist: rest lists)
    FPX_LAUNCH(fpx::launch_point_scatter(nn, a, M.d, xa, w.cellid + a, w.cell_off,
                                         w.cell_cursor, w.order + a, w.ux + a * M.d, M.offsets,
                                         nc, reinterpret_cast<int2*>(w.clist) + a, st));
    FPX_LAUNCH(fpx::launch_prefilter(M, nn, w.ux + a * M.d, w.order + a,
                                     reinterpret_cast<const int2*>(w.clist) + a, w.best,
                                     w.npass, code, elem, r, dist, iters,
                                     field ? values : nullptr, C, w.g1.count, stats, st));
    if (r1_chunks) {  // the chunk's round 1: its stream records in its own range
      g_launches += 1;
      FPX_LAUNCH(fpx::launch_stream_units(nn, E, w.best, w.g1.count, w.g1.packed,
                                          w.g1.packed_off, w.g1.temp, w.g1.temp_bytes,
                                          w.g1.cursor, x, M.d, w.order + a, w.ux + a * M.d,
                                          w.umeta + a, st));
      FPX_CK(cudaMemsetAsync(w.chunk_ctr, 0, sizeof(int64_t), st));
      FPX_LAUNCH(fpx::launch_newton_stream(M, nn, w.ux + a * M.d, w.umeta + a, w.g1.packed_off,
                                           w.npass, code, elem, r, dist, iters, field, C, values,
                                           w.upts, w.nun, w.chunk_ctr, w.redo, w.nredo,
                                           2 * n + 1024, stats, st));
      FPX_CK(cudaEventRecord(g_r1_ev[ck], st));
    }
  }
  if (!r1_chunks) {
    // --- round 1: group by best-first element, Newton, fused eval
    g_launches += 1;  // k_pack_counts (k_stream_scatter counted by FPX_LAUNCH)
    // in the prefilter's hash-cell order (no sort in hinted mode)
    FPX_LAUNCH(fpx::launch_stream_units(n, E, w.best, w.g1.count, w.g1.packed, w.g1.packed_off,
                                        w.g1.temp, w.g1.temp_bytes, w.g1.cursor, x, M.d,
                                        g_hint ? nullptr : w.order, w.ux, w.umeta, st));
    if (g_prof_start) FPX_CK(cudaEventRecord(g_prof_start, st));
    FPX_CK(cudaMemsetAsync(w.chunk_ctr, 0, sizeof(int64_t), st));
    // candidates held on a face twice in a row stop early and are redone in
    // full only if their point ends without an INTERIOR (see k_rest_l1)
    // (hinted: no abort rule / redo entries in round 1 -- the hinted element
    // may not be a candidate; non-INTERIOR points go to the rest phase whole)
    FPX_LAUNCH(fpx::launch_newton_stream(M, n, w.ux, w.umeta, w.g1.packed_off, w.npass, code,
                                         elem, r, dist, iters, field, C, values, w.upts, w.nun,
                                         w.chunk_ctr, g_hint ? nullptr : w.redo, w.nredo,
                                         2 * n + 1024, stats, st));
    if (g_prof_stop) FPX_CK(cudaEventRecord(g_prof_stop, st));
  }
  // external record: also a real event node when captured into a CUDA graph
  if (g_round1_done) FPX_CK(cudaEventRecord(g_round1_done, st));
  // --- rest: remaining candidates of the unresolved points
  FPX_CK(cudaMemsetAsync(w.hist, 0, sizeof(int32_t) * 2 * FPX_HMAX, st));
  g_launches += 3;  // k_rest_lists, k_rest_order, k_rest_scatter, k_rest_pairlist
  FPX_LAUNCH(fpx::launch_rest_lists(M, x, n, w.nun, w.upts, w.best, w.npass, w.clist, w.cnum,
                                    w.nps,
                                    w.hist,
                                    w.bstart, w.bcur, w.perm, w.cum, w.maxnp, w.pairs, w.npairs,
                                    st));
  FPX_CK(cudaMemsetAsync(w.found, 0, sizeof(int32_t) * n, st));
  FPX_CK(cudaMemsetAsync(w.lock, 0, sizeof(int32_t) * n, st));
  FPX_LAUNCH(fpx::launch_find_rest(M, x, n, w.nun, w.upts, w.clist, w.cnum, w.nps, w.perm,
                                   w.cum, w.maxnp, w.best, w.pairs, w.npairs, w.redo, w.nredo,
                                   w.found, w.lock, code, elem,
                                   r, dist,
                                   iters,
                                   field, C, values, w.counter, stats, st));
  g_launches += field ? 2 : 1;  // k_rest_l1 pass 1 + redo pass (+ k_rest_values)
  if (g_round1_done) {  // host mode: flag the rest points for fpx_rest_patch_host
    FPX_LAUNCH(fpx::launch_rest_flag(n, w.nun, w.upts, w.lock, st));
  }
  g_launches += 1;
  k_find_totals<<<1, 1, 0, st>>>(w.nun, w.nredo, stats, n);
  FPX_CK(cudaGetLastError());
  return FPX_OK;
}

size_t fpx_eval_workspace_bytes(int64_t E, int64_t n) {
  Carver c(nullptr, 0);
  c.take<int32_t>(n > 0 ? n : 1);
  Group g;
  g.carve(c, E, n > 0 ? n : 1);
  return c.off + 256;
}

int fpx_findpts_eval(int dr, int Nf, const double* fbasis, int C, int64_t E,
                     const double* field, int64_t n, const int32_t* code, const int32_t* elem,
                     const double* r, double* values, void* ws, size_t ws_bytes, void* stream) {
  if (dr < 1 || dr > 3) return fail(FPX_EINVAL, "eval: bad dr=%d", dr);
  if (!fpx::newton_supported(dr == 3 ? 3 : (dr == 2 ? 2 : 2), dr, Nf))
    return fail(FPX_EUNSUPPORTED, "eval: field order N=%d not compiled for dr=%d", Nf, dr);
  if (C < 1) return fail(FPX_EINVAL, "eval: components must be >= 1");
  if (E < 1 || n < 0) return fail(FPX_EINVAL, "eval: bad sizes");
  if (n == 0) return FPX_OK;
  cudaStream_t st = S(stream);
  Carver cv(ws, ws_bytes);
  int32_t* unit_elem = cv.take<int32_t>(n);
  Group g;
  g.carve(cv, E, n);
  if (!cv.ok()) return fail(FPX_EINVAL, "eval workspace too small (%zu < %zu)", ws_bytes, cv.off);
  FPX_CK(cudaMemsetAsync(g.count, 0, sizeof(int32_t) * E, st));
  FPX_LAUNCH(fpx::launch_eval_mark(n, C, code, elem, values, unit_elem, g.count, st));
  g_launches += 3;
  FPX_CK(g.build(E, n, nullptr, unit_elem, nullptr, st));
  FPX_LAUNCH(fpx::launch_eval_items(dr, Nf, fbasis, C, field, r, g.sorted, g.items, g.nitems,
                                g.items_cap, values, st));
  return FPX_OK;
}

int fpx_invert_pairs(const fpx_mesh_t* m, int64_t npairs, const double* x, const int32_t* elem,
                     const double* r0, double* r, double* dist, int32_t* iters,
                     int32_t* converged, void* stream) {
  int rc = check_mesh(m);
  if (rc) return rc;
  if (npairs <= 0) return FPX_OK;
  cudaStream_t st = S(stream);
  Carver probe(nullptr, 0);
  Group g;
  g.carve(probe, m->E, npairs);
  void* ws = nullptr;
  FPX_CK(cudaMallocAsync(&ws, probe.off + 256, st));
  Carver cv(ws, probe.off + 256);
  g.carve(cv, m->E, npairs);
  FPX_CK(cudaMemsetAsync(g.count, 0, sizeof(int32_t) * m->E, st));
  g_launches += 1;
  k_count_elems<<<grid1(npairs), 256, 0, st>>>(npairs, elem, g.count);
  FPX_CK(cudaGetLastError());
  g_launches += 3;
  FPX_CK(g.build(m->E, npairs, nullptr, elem, nullptr, st));
  FPX_LAUNCH(fpx::launch_invert_pairs_grouped(*m, x, g.sorted, g.items, g.nitems, g.items_cap, r0, r, dist,
                                          iters, converged, st));
  FPX_CK(cudaFreeAsync(ws, st));
  return FPX_OK;
}

int fpx_forward_map(const fpx_mesh_t* m, int64_t n, const int32_t* elem, const double* r,
                    double* x, double* G, double* H2, void* stream) {
  int rc = check_mesh(m);
  if (rc) return rc;
  if (n <= 0) return FPX_OK;
  FPX_LAUNCH(fpx::launch_forward_map(*m, n, elem, r, x, G, H2, S(stream)));
  return FPX_OK;
}

int fpx_particles_advance(int d, int64_t n, double* x, double* v, const double* u,
                          double* v_prev, double* a_prev, double tau, double dt, int first,
                          const double* box, int periodic, void* stream) {
  if (d < 1 || d > 3) return fail(FPX_EINVAL, "particles: bad d=%d", d);
  if (!(tau > 0.0) || !(dt > 0.0)) return fail(FPX_EINVAL, "particles: need tau > 0, dt > 0");
  if (periodic && !box) return fail(FPX_EINVAL, "particles: periodic axes need a box");
  if (n <= 0) return FPX_OK;
  const double unit[6] = {0, 0, 0, 1, 1, 1};
  FPX_LAUNCH(fpx::launch_particles_advance(d, n, x, v, u, v_prev, a_prev, tau, dt, first,
                                           box ? box : unit, periodic, S(stream)));
  return FPX_OK;
}

}  // extern "C"
