/* fpx.h -- C ABI of libfpx_sm100.so, the B200 (sm_100a) findpts hot path.
 *
 * Drop-in boundary for the reference package `fpx` (arXiv 2501.12349).  The
 * reference ships only Python (basis.py, bounds.py) and specifies the rest in
 * SPEC.md; each entry point below names the reference interface it replaces.
 * A host binding (ctypes, see paper_2501_12349_b200/_C.py and INTEGRATION.md)
 * passes plain device pointers and sizes; no torch types cross this ABI.
 *
 * Conventions
 *   - every pointer argument is a caller-owned DEVICE pointer unless the name
 *     ends in _host;
 *   - every call takes a cudaStream_t (as void*) and is stream-ordered and
 *     asynchronous unless documented as synchronising;
 *   - return 0 on success, a negative FPX_E* code otherwise; the message is in
 *     the thread-local fpx_last_error().  Per-point outcomes are codes in the
 *     outputs, never errors;
 *   - all coordinates are FP64, element / point indices int32 (int64 counts).
 *
 * Layouts (bounds.py:58-94)
 *   basis     packed per-order constants, see FPX_BASIS_* offsets
 *   nodes     [E][d][N^dr]   lexicographic, first reference axis fastest
 *   aabb      [E][2][d]      lo, hi (expanded)
 *   obb_c     [E][d]         OBB centre
 *   obb_inv   [E][d][d]      OBB inverse transform (unit cube frame)
 *   frame     [E][d + d*d]   element centre x_c and J_c^{-1} (best-first order)
 *   hbox      [E][2][d]      hash box = AABB  intersect  OBB enclosure (D5)
 *   grid      [9]            lo[3], hi[3], h[3] of the local hash grid
 *   x         [n][d]         query points
 *   r         [n][dr]        reference coordinates
 *   field     [E][C][Nf^dr]  nodal field blocks
 */
#ifndef FPX_H
#define FPX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FPX_ABI_VERSION 7

/* error codes */
#define FPX_OK 0
#define FPX_EINVAL -1     /* bad argument */
#define FPX_ECUDA -2      /* CUDA runtime error */
#define FPX_ECAPACITY -3  /* output capacity too small; *needed set */
#define FPX_EUNSUPPORTED -4 /* order / dimension not compiled in */

/* record codes (decision D10: gslib convention) */
#define FPX_INTERIOR 0
#define FPX_BORDER 1
#define FPX_NOT_FOUND 2

/* packed basis constants: offsets in doubles for order p, N = p+1, M */
#define FPX_BASIS_NODES(N, M) 0
#define FPX_BASIS_SCALE(N, M) (N)
#define FPX_BASIS_PROJ0(N, M) (2 * (N))
#define FPX_BASIS_PROJ1(N, M) (3 * (N))
#define FPX_BASIS_ETA(N, M) (4 * (N))
#define FPX_BASIS_LO(N, M) (4 * (N) + (M))
#define FPX_BASIS_HI(N, M) (4 * (N) + (M) + (N) * (M))
#define FPX_BASIS_SIZE(N, M) (4 * (N) + (M) + 2 * (N) * (M))

/* Device-resident setup of one rank's mesh (engine.EngineSetup).
 * POD of device pointers owned by the caller (torch tensors in EngineSetup). */
typedef struct fpx_mesh_t {
  int32_t d, dr, N, M;          /* phys dim, ref dim, nodes/axis, interval pts */
  int64_t E;                    /* elements on this rank */
  const double* basis;          /* packed constants (FPX_BASIS_*) */
  const double* nodes;
  const double* aabb;
  const double* obb_c;
  const double* obb_inv;
  const uint8_t* obb_ok;
  const double* frame;
  const double* grid;
  int32_t ncell;                /* cells per axis of the local map */
  int32_t max_list;             /* longest CSR list (capacity planning) */
  const int32_t* offsets;       /* [ncell^d + 1] */
  const int32_t* elems;         /* CSR element ids, ascending per cell */
  /* Newton settings (invmap.NewtonSettings) */
  int32_t max_iters;
  double tol, grow, keep, accept, shrink, alpha0;
  /* surface classification eps_d: abs >= 0 wins, else rel*diag */
  double eps_d_abs, eps_d_rel;
  /* (ABI 2) per-element candidate filter record, FPX_FREC doubles each:
   * aabb lo,hi [2d] | obb_c [d] | obb_inv [d*d] | frame x_c,J_c^-1 [d+d*d] |
   * ... | obb_ok as 0.0/1.0 at index FPX_FREC-1 (fpx_filter_records). */
  const double* frec;
  /* (ABI 2) nodes with rows padded to an even length NP (N rounded up):
   * [E][d][N^(dr-1)][NP], 16-byte aligned rows (fpx_pad_nodes). */
  const double* nodes_pad;
  /* (ABI 7) float pre-test rows of the candidate filter (fpx_filter_records),
   * [E][FPX_FROW] floats: aabb lo rounded down [d] at 0, hi rounded up [d] at
   * d, the OBB mode at 6 (0 no OBB test, 1 float pre-test, 2 double only),
   * obb_c [d] at 8 and obb_inv [d*d] at 8+d rounded to nearest (mode 1 only
   * when every value is 0 or of magnitude in [2^-100, 2^100]).  Each
   * pre-test decides pass / fail exactly where it can and leaves the rest
   * (points within ~1e-7 relative of a face) to the double record, so the
   * filter outcome is that of aabb_contains / obb_contains. */
  const float* fbox;
} fpx_mesh_t;

#define FPX_FREC 32
#define FPX_FROW 20

/* Diagnostic counters written by fpx_find (device int64[FPX_STATS_LEN]). */
#define FPX_STAT_POINTS 0        /* points processed */
#define FPX_STAT_BOXTESTS 1      /* candidate box tests (hash-list entries) */
#define FPX_STAT_NEWTON 2        /* Newton-ed (point, element) candidates */
#define FPX_STAT_ITERS 3         /* Newton iterations over all candidates */
#define FPX_STAT_ROUND2_POINTS 4 /* points unresolved after round 1 (rest kernel) */
#define FPX_STAT_R1_WARP_EVALS 5 /* round-1 map evaluations issued per warp (all lanes) */
#define FPX_STAT_R1_W2_EVALS 6   /* ... of which with second derivatives */
#define FPX_STAT_EVALS 7         /* fused field evaluations */
#define FPX_STAT_NEWTON_R1 8     /* Newton solves in the round-1 (best-first) kernel */
#define FPX_STAT_ITERS_R1 9      /* their iterations */
#define FPX_STAT_EVALS_R1 10     /* field evaluations fused into the round-1 kernel */
#define FPX_STAT_R1_ITEMS 11     /* round-1 warp work items */
#define FPX_STAT_REST_WARP_EVALS 12 /* rest kernel: map evaluations issued per warp */
#define FPX_STAT_REST_W2_EVALS 13   /* ... of which with second derivatives */
#define FPX_STAT_REST_LANE_EVALS 14 /* ... summed over the lanes that were iterating */
#define FPX_STAT_REDO 15            /* candidates handed to the redo pass (R2 abort or D7') */
#define FPX_STAT_R1_LANE_EVALS 16   /* round-1 map evaluations summed over iterating lanes */
#define FPX_STATS_LEN 17

int fpx_abi_version(void);
const char* fpx_last_error(void);
/* Number of kernels this library has launched in the process (its own
 * kernels, not CUB's or memsets): the bench's gpu_launches evidence. */
int64_t fpx_launch_count(void);
/* Record (start, stop) CUDA events (cudaEvent_t as void*) around the round-1
 * Newton kernel of the next fpx_find calls on the same stream; NULL clears.
 * Used by bench.py to time the dominant kernel live. */
int fpx_profile_round1(void* ev_start, void* ev_stop);
/* The next fpx_find calls on this thread record `ev` (a cudaEvent_t) on their
 * stream once round 1 is done: from then on only the records of the rest
 * points (fpx_rest_patch_host) still change.  NULL clears it. */
int fpx_set_round1_event(void* ev);

/* (ABI 6) The next fpx_find calls on this thread start every point i on the
 * element hint[i] (device int32 [n], local ids, all valid), e.g. a
 * particle's element of the previous step: round 1 solves it there without
 * the hash-list prefilter, keeps the result if it is INTERIOR (then it is
 * the point's record: the unique zero of the injective element map), and
 * otherwise searches the point's candidates in the rest phase as a find
 * without hint would.  The records are those of fpx_find without hint
 * (either owner on a shared face).  NULL clears it.
 * Replaces: the per-step re-location of PAPER.md Algorithm 1 (Find). */
int fpx_set_find_hint(const int32_t* elem);

/* (ABI 6) The next fpx_find calls on this thread take their n points in k
 * contiguous chunks [n*c/k, n*(c+1)/k): chunk c may be read once events[c]
 * (cudaEvent_t) has completed.  The find waits on each event on its stream
 * just before sorting and filtering that chunk, so the host-to-device copy
 * of chunk c+1 overlaps the prefilter of chunk c (k = 1: the find waits on
 * the one event before it starts).  k <= 0 or NULL clears. */
int fpx_set_upload_events(int k, void* const* events);

/* (ABI 7) With upload events for k chunks set, the next fpx_find calls on
 * this thread also group and solve round 1 per chunk, right after the
 * chunk is filtered, and record events[c] (cudaEvent_t) on their stream when
 * chunk c's round 1 is done: from then on the records of points
 * [n*c/k, n*(c+1)/k) are final except those of the rest points (revisited
 * after the last chunk; fpx_rest_patch_host).  k must equal the upload
 * chunk count to take effect; k <= 0 or NULL clears.  The records are
 * those of a find without it. */
int fpx_set_round1_events(int k, void* const* events);

/* After a host-mode fpx_find (fpx_set_round1_event set; same stream, same
 * workspace, same n): writes the records of the points in [k0, k1) that the
 * rest phase settled straight into host record arrays (pinned, mapped;
 * zero-copy over PCIe), in point order.  Enqueue it after any bulk download
 * of the same range into the same arrays; ranges may be patched as their
 * downloads land (ABI 6).  It clears the per-point flags the find left in
 * the lock array of `ws`.  FPX_EINVAL if `ws` was not last used by an
 * fpx_find of n points on `m`, or for a bad range.
 * Replaces: the record copy-back of engine.find_and_interpolate_host
 * (SPEC.md:423-426 find_and_interpolate, host arrays). */
int fpx_rest_patch_host(int dr, int C, int64_t n, int64_t k0, int64_t k1, void* ws,
                        size_t ws_bytes, const fpx_mesh_t* m, const int32_t* code,
                        const int32_t* elem, const double* r, const double* dist,
                        const double* values, int32_t* hcode, int32_t* helem, double* hr,
                        double* hdist, double* hvalues, void* stream);

/* FP64 FMA throughput probe (TFLOP/s): a DFMA-chain kernel over all SMs,
 * timed with CUDA events on `stream` (synchronising).  Roofline denominator. */
int fpx_probe_fp64(double* tflops_host, void* stream);
/* 1 if order N (nodes/axis) is compiled in for (d, dr) */
int fpx_supported(int d, int dr, int N);

/* Per-element bounds: element_aabb + element_obb batched over E elements
 * (replaces bounds.py:292-297 and bounds.py:366-384, built on
 * bound_function_1d/2d bounds.py:155-201), plus the D5 hash box and the
 * centre frame.  status[e]: 0 ok, 1 degenerate (bounds.py:244, setup error),
 * 2 OBB unusable (bounds.py:349,361 SingularTransformError -> AABB only,
 * SPEC.md:191).  Bit-identical to the oracle for identical basis constants
 * (no FMA contraction). */
int fpx_setup_bounds(int d, int dr, int N, int M, int64_t E, const double* basis,
                     const double* nodes, double expansion, double* aabb, double* obb_c,
                     double* obb_inv, double* hbox, double* frame, uint8_t* obb_ok,
                     int32_t* status, void* stream);

/* bound_function_1d (dr=1, values [nf][N] -> lower/upper [nf][M]) and
 * bound_function_2d (dr=2, values [nf][N*N] with i fastest -> [nf][M][M]),
 * replacing bounds.py:155-171 and bounds.py:174-201. */
/* Packs aabb/obb/frame/obb_ok into the per-element filter records (mesh.frec,
 * [E][FPX_FREC] doubles, 256-byte aligned rows) read by the find prefilter,
 * and (ABI 7) their float pre-test rows (mesh.fbox, [E][FPX_FROW] floats,
 * 16-byte aligned). */
int fpx_filter_records(int d, int64_t E, const double* aabb, const double* obb_c,
                       const double* obb_inv, const uint8_t* obb_ok, const double* frame,
                       double* frec, float* fbox, void* stream);

/* Copies nodes [E][d][N^dr] into the row-padded layout of mesh.nodes_pad. */
int fpx_pad_nodes(int d, int dr, int N, int64_t E, const double* nodes, double* nodes_pad,
                  void* stream);

int fpx_bound_function(int dr, int N, int M, int64_t nf, const double* basis,
                       const double* values, double* lower, double* upper, void* stream);

/* build_local_map over boxes [E][2][d]: grid over the union
 * of the boxes, CSR cell -> ascending element ids.  With OBBs
 * (obb_ok != NULL; obb_c/obb_inv as fpx_setup_bounds writes them), cells of
 * a box's range that cannot meet the element's OBB are culled (decision D5b,
 * result-preserving); NULL keeps the SPEC's full rectangular range.
 * Synchronising.  Pass elems == NULL (or cap too small) to get
 * offsets/grid and *needed_host; then call again with cap >= needed.
 * ws: FPX workspace of fpx_hash_workspace_bytes(). */
size_t fpx_hash_workspace_bytes(int d, int64_t E, int ncell);
int fpx_hash_build(int d, int64_t E, const double* box, const double* obb_c,
                   const double* obb_inv, const uint8_t* obb_ok, int ncell, double* grid,
                   int32_t* offsets, int32_t* elems, int64_t cap, int64_t* needed_host,
                   int32_t* max_list_host, void* ws, size_t ws_bytes, void* stream);

/* lookup_local's addressing: cell_of per point, -1 outside. */
int fpx_cell_of(const fpx_mesh_t* m, int64_t n, const double* x, int64_t* cell, void* stream);

/* engine.find Phase A on this rank:
 * hash lookup, AABB then OBB filter, trust-region Newton (invmap.invert_point
 * SPEC.md:298-307) per candidate, classify, winner rule D6.  Writes
 * code/elem/r/dist per point (NOT_FOUND: elem -1, r = dist = NaN).
 * If field != NULL, also evaluates the field at the winning (elem, r)
 * (engine.find_and_interpolate) into values [n][C]
 * (NaN for NOT_FOUND).  iters (optional) = Newton iterations per point.
 * stats: device int64[FPX_STATS_LEN] (zeroed by the call).
 * ws: fpx_find_workspace_bytes(m->E, n, pair_cap). */
size_t fpx_find_workspace_bytes(const fpx_mesh_t* m, int64_t n, int64_t pair_cap);
int fpx_find(const fpx_mesh_t* m, int64_t n, const double* x, int32_t* code, int32_t* elem,
             double* r, double* dist, int32_t* iters, const double* field, int C,
             double* values, int64_t* stats, int64_t pair_cap, void* ws, size_t ws_bytes,
             void* stream);

/* engine.interpolate local part (basis.py:285-303 contraction):
 * values [n][C] at records (code, elem, r); NOT_FOUND -> NaN (D12).
 * fbasis: packed constants of the field order (Nf may differ from N). */
size_t fpx_eval_workspace_bytes(int64_t E, int64_t n);
int fpx_findpts_eval(int dr, int Nf, const double* fbasis, int C, int64_t E,
                     const double* field, int64_t n, const int32_t* code, const int32_t* elem,
                     const double* r, double* values, void* ws, size_t ws_bytes, void* stream);

/* invmap.invert_point batched over explicit (point, element) pairs
 * (SPEC.md:298-307): r [npairs][dr], dist, iters, converged.  r0
 * [npairs][dr] is the initial guess (SPEC.md:298 r0), or NULL for the D7
 * seed (nearest GLL node). */
int fpx_invert_pairs(const fpx_mesh_t* m, int64_t npairs, const double* x, const int32_t* elem,
                     const double* r0, double* r, double* dist, int32_t* iters,
                     int32_t* converged, void* stream);

/* invmap.forward_map batched: x [n][d], G [n][d][dr],
 * H2 [n][d][6] (optional; symmetric order rr,ss,tt,rs,rt,st). */
int fpx_forward_map(const fpx_mesh_t* m, int64_t n, const int32_t* elem, const double* r,
                    double* x, double* G, double* H2, void* stream);

/* Lagrangian particle step (Algorithm 1, ParticleRHS + Integrate +
 * ParticleBC): a = (u - v)/tau, AB2 update of x and v (forward Euler when
 * `first`), periodic wrap of axis c of the box (lo[d], hi[d] in host memory)
 * when bit c of `periodic` is set.  x, v, u, v_prev, a_prev: device [n][d];
 * v_prev / a_prev receive this step's v and a for the next AB2 step. */
int fpx_particles_advance(int d, int64_t n, double* x, double* v, const double* u,
                          double* v_prev, double* a_prev, double tau, double dt, int first,
                          const double* box, int periodic, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FPX_H */
