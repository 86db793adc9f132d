/* fpx_oracle.h -- CPU ORACLE (test infrastructure only).
 *
 * Plain-C restatement of the reference algorithm for the findpts hot path.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library; the product never does.
 *
 * Parity status:
 *   basis/bounds   : pinned against golden vectors produced by the unmodified
 *                    reference (tests/golden/make_golden.py -> ref_*.npz).
 *   hash/Newton/find/eval : the reference ships no code for these
 *                    (SURVEY.md §0.2); restated from SPEC.md with the frozen
 *                    decisions D1-D12 and pinned against the
 *                    SPEC known-answer examples (tests/test_oracle_find.py).
 *                    Against gslib itself: parity unpinned (not vendored).
 */
#ifndef FPX_ORACLE_H
#define FPX_ORACLE_H
#include <stdint.h>

#define FPXO_MAXN 30
#define FPXO_MAXM 64

enum { FPXO_INTERIOR = 0, FPXO_BORDER = 1, FPXO_NOT_FOUND = 2 };

typedef struct {
  int p, N, M;
  double z[FPXO_MAXN];       /* GLL nodes                       basis.py:69-90  */
  double scale[FPXO_MAXN];   /* 1/prod_{j!=i}(z_i-z_j)          basis.py:124-125 */
  double proj0[FPXO_MAXN];   /* l=0 Legendre projector          basis.py:128-132 */
  double proj1[FPXO_MAXN];   /* l=1 Legendre projector                          */
  double eta[FPXO_MAXM];     /* Chebyshev interval points       basis.py:93-97  */
  double lo[FPXO_MAXN * FPXO_MAXM]; /* envelope lower [i*M+j]   basis.py:241-282 */
  double hi[FPXO_MAXN * FPXO_MAXM]; /* envelope upper                          */
} fpxo_basis;

typedef struct {
  int max_iters;    /* 50 */
  double tol;       /* 1e-10   */
  double grow;      /* 2.0     */
  double keep;      /* 0.9     */
  double accept;    /* 0.01    */
  double shrink;    /* 0.25    */
  double alpha0;    /* 1.0     */
} fpxo_newton;

typedef struct {
  int d, dr;
  int64_t E;
  const fpxo_basis* B;
  const double* nodes;          /* [E][d][N^dr] */
  const double* aabb;           /* [E][2][d]    */
  const double* obb_c;          /* [E][d]       */
  const double* obb_inv;        /* [E][d][d]    */
  const uint8_t* obb_ok;        /* [E]          */
  const double* grid;           /* lo[3] hi[3] h[3] */
  int ncell;                    /* cells per axis */
  const int32_t* offsets;       /* [ncell^d + 1] */
  const int32_t* elems;
  fpxo_newton newton;
  double eps_d_abs;             /* >= 0: absolute eps_d (surfaces) */
  double eps_d_rel;             /* used when eps_d_abs < 0: rel * AABB diagonal */
  const double* frame;          /* [E][d + d*d] centre frame (x_c, J_c^-1) or NULL (pure D7) */
} fpxo_mesh;

#endif
