"""ctypes front-end of the CPU ORACLE (oracle/fpx_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / `--impl reference` legs -- never by the product
package.  See fpx_oracle.h for what is pinned against the reference and what
is restated from SPEC.md.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liboracle.so")

MAXN = 30
MAXM = 64
INTERIOR, BORDER, NOT_FOUND = 0, 1, 2


class Basis(C.Structure):
    _fields_ = [
        ("p", C.c_int), ("N", C.c_int), ("M", C.c_int),
        ("z", C.c_double * MAXN), ("scale", C.c_double * MAXN),
        ("proj0", C.c_double * MAXN), ("proj1", C.c_double * MAXN),
        ("eta", C.c_double * MAXM),
        ("lo", C.c_double * (MAXN * MAXM)), ("hi", C.c_double * (MAXN * MAXM)),
    ]

    def arrays(self):
        N, M = self.N, self.M
        return dict(
            nodes=np.array(self.z[:N]), scale=np.array(self.scale[:N]),
            proj0=np.array(self.proj0[:N]), proj1=np.array(self.proj1[:N]),
            eta=np.array(self.eta[:M]),
            lo=np.array(self.lo[:N * M]).reshape(N, M),
            hi=np.array(self.hi[:N * M]).reshape(N, M))


class Newton(C.Structure):
    _fields_ = [("max_iters", C.c_int), ("tol", C.c_double), ("grow", C.c_double),
                ("keep", C.c_double), ("accept", C.c_double), ("shrink", C.c_double),
                ("alpha0", C.c_double)]


def default_newton():
    # SPEC.md:281
    return Newton(50, 1e-10, 2.0, 0.9, 0.01, 0.25, 1.0)


class Mesh(C.Structure):
    _fields_ = [
        ("d", C.c_int), ("dr", C.c_int), ("E", C.c_int64), ("B", C.POINTER(Basis)),
        ("nodes", C.c_void_p), ("aabb", C.c_void_p), ("obb_c", C.c_void_p),
        ("obb_inv", C.c_void_p), ("obb_ok", C.c_void_p), ("grid", C.c_void_p),
        ("ncell", C.c_int), ("offsets", C.c_void_p), ("elems", C.c_void_p),
        ("newton", Newton), ("eps_d_abs", C.c_double), ("eps_d_rel", C.c_double),
        ("frame", C.c_void_p),
    ]


_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        L.fpxo_basis_init.argtypes = [C.POINTER(Basis), C.c_int, C.c_int, C.c_int]
        L.fpxo_gll_nodes.argtypes = [C.c_int, P]
        L.fpxo_lagrange.argtypes = [C.POINTER(Basis), C.c_int64, P, P, P, P]
        L.fpxo_legendre_coeffs.argtypes = [C.POINTER(Basis), P, P, P]
        L.fpxo_bound1d.argtypes = [C.POINTER(Basis), P, P, P]
        L.fpxo_bound2d.argtypes = [C.POINTER(Basis), P, P, P]
        L.fpxo_envelope_violation.argtypes = [C.POINTER(Basis), C.c_int]
        L.fpxo_envelope_violation.restype = C.c_double
        L.fpxo_coord_bounds.argtypes = [C.POINTER(Basis), C.c_int, C.c_int, P, P, P]
        L.fpxo_element_boxes.argtypes = [C.POINTER(Basis), C.c_int, C.c_int, C.c_int64, P,
                                         C.c_double, P, P, P, P, P, P, P]
        L.fpxo_element_boxes.restype = C.c_int64
        L.fpxo_contains.argtypes = [C.c_int, C.c_int64, P, P, P, P, P, P]
        L.fpxo_hash_grid.argtypes = [C.c_int, C.c_int64, P, C.c_int, P]
        L.fpxo_cell_of.argtypes = [C.c_int, P, C.c_int, P]
        L.fpxo_cell_of.restype = C.c_int64
        L.fpxo_hash_build.argtypes = [C.c_int, C.c_int64, P, P, P, P, P, C.c_int, P, P]
        L.fpxo_hash_build.restype = C.c_int64
        L.fpxo_forward_map.argtypes = [C.POINTER(Basis), C.c_int, C.c_int, P, P, P, P, P]
        L.fpxo_invert.argtypes = [C.POINTER(Basis), C.c_int, C.c_int, P, P,
                                  C.POINTER(Newton), P, P, P, P]
        L.fpxo_invert_from.argtypes = [C.POINTER(Basis), C.c_int, C.c_int, P, P,
                                       C.POINTER(Newton), P, P, P, P, P]
        L.fpxo_find.argtypes = [C.POINTER(Mesh), C.c_int64, P, P, P, P, P, P, P, P, C.c_int]
        L.fpxo_eval.argtypes = [C.POINTER(Basis), C.c_int, C.c_int, P, C.c_int64, P, P, P, P,
                                C.c_int]
        L.fpxo_num_threads.restype = C.c_int
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class BasisError(ValueError):
    pass


def basis(p, M=None, validate=True):
    B = Basis()
    rc = lib().fpxo_basis_init(C.byref(B), int(p), int(M or 0), int(validate))
    if rc:
        raise BasisError(f"fpxo_basis_init(p={p}, M={M}) failed: {rc}")
    return B


def basis_from_arrays(nodes, scale, proj0, proj1, eta, lo, hi):
    """Build the oracle basis struct from externally computed constants (used
    to feed the oracle and the kernels identical constants)."""
    B = Basis()
    N, M = len(nodes), len(eta)
    B.p, B.N, B.M = N - 1, N, M
    B.z[:N] = list(nodes)
    B.scale[:N] = list(scale)
    B.proj0[:N] = list(proj0)
    B.proj1[:N] = list(proj1)
    B.eta[:M] = list(eta)
    B.lo[:N * M] = list(np.asarray(lo).reshape(-1))
    B.hi[:N * M] = list(np.asarray(hi).reshape(-1))
    return B


def gll_nodes(p):
    z = np.zeros(p + 1)
    if lib().fpxo_gll_nodes(int(p), _p(z)):
        raise BasisError(p)
    return z


def lagrange(B, r, second=True):
    r = _f64(np.atleast_1d(r))
    n = r.size
    v = np.zeros((n, B.N)); d1 = np.zeros((n, B.N)); d2 = np.zeros((n, B.N))
    lib().fpxo_lagrange(C.byref(B), n, _p(r), _p(v), _p(d1), _p(d2) if second else None)
    return v, d1, (d2 if second else None)


def legendre_coeffs(B, u):
    u = _f64(u)
    a0 = np.zeros(1); a1 = np.zeros(1)
    lib().fpxo_legendre_coeffs(C.byref(B), _p(u), _p(a0), _p(a1))
    return a0[0], a1[0]


def bound1d(B, u):
    u = _f64(u)
    lo = np.zeros(B.M); hi = np.zeros(B.M)
    lib().fpxo_bound1d(C.byref(B), _p(u), _p(lo), _p(hi))
    return lo, hi


def bound2d(B, u):
    """u[i, j] (i along r, j along s) as the reference bound_function_2d."""
    u = np.asarray(u, dtype=np.float64)
    flat = _f64(u.T.reshape(-1))   # flat[i + N*j] = u[i, j]
    lo = np.zeros(B.M * B.M); hi = np.zeros(B.M * B.M)
    lib().fpxo_bound2d(C.byref(B), _p(flat), _p(lo), _p(hi))
    return lo.reshape(B.M, B.M), hi.reshape(B.M, B.M)


def envelope_violation(B, samples=10000):
    return lib().fpxo_envelope_violation(C.byref(B), samples)


def coord_bounds(B, d, dr, X):
    X = _f64(X)
    lo = np.zeros(d); hi = np.zeros(d)
    lib().fpxo_coord_bounds(C.byref(B), d, dr, _p(X), _p(lo), _p(hi))
    return lo, hi


def element_boxes(B, d, dr, nodes, expansion=0.10):
    nodes = _f64(nodes)
    E = nodes.shape[0]
    out = dict(aabb=np.zeros((E, 2, d)), obb_c=np.zeros((E, d)), obb_inv=np.zeros((E, d, d)),
               hbox=np.zeros((E, 2, d)), obb_ok=np.zeros(E, np.uint8),
               status=np.zeros(E, np.int32), frame=np.zeros((E, d + d * d)))
    bad = lib().fpxo_element_boxes(C.byref(B), d, dr, E, _p(nodes), float(expansion),
                                   _p(out["aabb"]), _p(out["obb_c"]), _p(out["obb_inv"]),
                                   _p(out["hbox"]), _p(out["obb_ok"]), _p(out["status"]),
                                   _p(out["frame"]))
    out["degenerate"] = int(bad)
    return out


def contains(d, box, cen, inv, pts):
    pts = _f64(pts)
    n = pts.shape[0]
    a = np.zeros(n, np.uint8); o = np.zeros(n, np.uint8)
    lib().fpxo_contains(d, n, _p(_f64(box)), _p(_f64(cen)), _p(_f64(inv)), _p(pts), _p(a), _p(o))
    return a.astype(bool), o.astype(bool)


def n_cells(E, d):
    """Decision D5: smallest n >= 1 with n**d >= E, clamped to [1, 1024]
    (SPEC.md:262 N_L = ceil(E^(1/d)), computed in integers)."""
    n = max(1, int(round(E ** (1.0 / d))) - 1)
    while n ** d < E:
        n += 1
    while n > 1 and (n - 1) ** d >= E:
        n -= 1
    return int(min(max(n, 1), 1024))


def hash_build(d, box, ncell, obb_c=None, obb_inv=None, obb_ok=None):
    """Local map over boxes; with OBBs, cells that cannot meet an element's OBB
    are culled (D5b)."""
    box = _f64(box)
    E = box.shape[0]
    grid = np.zeros(9)
    L = lib()
    L.fpxo_hash_grid(d, E, _p(box), ncell, _p(grid))
    nc = ncell ** d
    offsets = np.zeros(nc + 1, np.int32)
    cull = obb_ok is not None
    oc = _f64(np.nan_to_num(obb_c)) if cull else None
    oi = _f64(np.nan_to_num(obb_inv)) if cull else None
    ok = np.ascontiguousarray(obb_ok, np.uint8) if cull else None
    args = (_p(oc), _p(oi), _p(ok)) if cull else (None, None, None)
    total = L.fpxo_hash_build(d, E, _p(box), *args, _p(grid), ncell, _p(offsets), None)
    elems = np.zeros(max(total, 1), np.int32)
    L.fpxo_hash_build(d, E, _p(box), *args, _p(grid), ncell, _p(offsets), _p(elems))
    # lists are filled in ascending element order already (outer loop over e)
    return grid, offsets, elems[:total]


def cell_of(d, grid, ncell, x):
    return lib().fpxo_cell_of(d, _p(_f64(grid)), ncell, _p(_f64(x)))


class OracleSetup:
    """Oracle counterpart of engine.setup: boxes, hash and the mesh struct."""

    def __init__(self, nodes, d, dr, p, expansion=0.10, B=None, ncell=None,
                 newton=None, eps_d_abs=-1.0, eps_d_rel=1e-10, nthreads=0, seeds="D7'"):
        """seeds: "D7'" (default; affine-frame seed first for volume
        elements, then the nearest node -- the kernels' rule) or "D7" (the
        SPEC's nearest-node seed only)."""
        self.nodes = _f64(nodes)
        self.d, self.dr, self.p = d, dr, p
        self.B = B if B is not None else basis(p)
        self.E = self.nodes.shape[0]
        bx = element_boxes(self.B, d, dr, self.nodes, expansion)
        if bx["degenerate"]:
            raise ValueError("degenerate element in oracle setup")
        self.boxes = bx
        self.ncell = ncell or 2 * n_cells(self.E, d)
        self.grid, self.offsets, self.elems = hash_build(d, bx["hbox"], self.ncell, bx["obb_c"],
                                                         bx["obb_inv"], bx["obb_ok"])
        self.obb_ok = bx["obb_ok"]
        self.mesh = Mesh()
        m = self.mesh
        m.d, m.dr, m.E = d, dr, self.E
        m.B = C.pointer(self.B)
        m.nodes = self.nodes.ctypes.data
        m.aabb = bx["aabb"].ctypes.data
        m.obb_c = bx["obb_c"].ctypes.data
        m.obb_inv = bx["obb_inv"].ctypes.data
        m.obb_ok = self.obb_ok.ctypes.data
        m.grid = self.grid.ctypes.data
        m.ncell = self.ncell
        m.offsets = self.offsets.ctypes.data
        self._elems = self.elems if self.elems.size else np.zeros(1, np.int32)
        m.elems = self._elems.ctypes.data
        m.newton = newton or default_newton()
        m.eps_d_abs = eps_d_abs
        m.eps_d_rel = eps_d_rel
        if seeds not in ("D7'", "D7"):
            raise ValueError(f"seeds must be D7' or D7, got {seeds!r}")
        m.frame = bx["frame"].ctypes.data if seeds == "D7'" else None
        self.nthreads = nthreads

    def find(self, x, nthreads=None):
        x = _f64(x).reshape(-1, self.d)
        n = x.shape[0]
        rec = dict(code=np.zeros(n, np.int32), elem=np.zeros(n, np.int32),
                   r=np.zeros((n, self.dr)), dist=np.zeros(n), iters=np.zeros(n, np.int32),
                   ncand=np.zeros(n, np.int32), nbox=np.zeros(n, np.int32))
        lib().fpxo_find(C.byref(self.mesh), n, _p(x), _p(rec["code"]), _p(rec["elem"]),
                        _p(rec["r"]), _p(rec["dist"]), _p(rec["iters"]), _p(rec["ncand"]),
                        _p(rec["nbox"]), int(self.nthreads if nthreads is None else nthreads))
        return rec


def evaluate(Bf, dr, field, code, elem, r, nthreads=0):
    field = _f64(field)
    E, Cc = field.shape[0], field.shape[1]
    n = len(code)
    out = np.zeros((n, Cc))
    lib().fpxo_eval(C.byref(Bf), dr, Cc, _p(field), n, _p(np.ascontiguousarray(code, np.int32)),
                    _p(np.ascontiguousarray(elem, np.int32)), _p(_f64(r).reshape(n, dr)),
                    _p(out), int(nthreads))
    return out


def invert(B, d, dr, X, xs, newton=None, r0=None):
    X = _f64(X); xs = _f64(xs)
    r = np.zeros(3); dist = np.zeros(1); it = np.zeros(1, np.int32); cv = np.zeros(1, np.int32)
    S = newton or default_newton()
    r0a = None if r0 is None else _f64(np.resize(np.asarray(r0, float), 3))
    lib().fpxo_invert_from(C.byref(B), d, dr, _p(X), _p(xs), C.byref(S),
                           _p(r0a) if r0a is not None else None, _p(r), _p(dist), _p(it), _p(cv))
    return r[:dr].copy(), float(dist[0]), int(it[0]), bool(cv[0])


def forward_map(B, d, dr, X, r, second=False):
    X = _f64(X); r = _f64(np.resize(np.asarray(r, float), 3))
    x = np.zeros(d); G = np.zeros(d * dr); H2 = np.zeros(d * 6)
    lib().fpxo_forward_map(C.byref(B), d, dr, _p(X), _p(r), _p(x), _p(G), _p(H2) if second else None)
    return x, G.reshape(d, dr), (H2.reshape(d, 6) if second else None)


def num_threads():
    return lib().fpxo_num_threads()
