"""Synthetic meshes, fields and query points (`toolkit`).

The reference ships no generators; the definitions here are
frozen so the oracle, the tests and bench.py all see identical inputs:

* ``kershaw``   -- CEED Kershaw map of [0,1]^3 with a
  quintic smoothstep, eps_y = eps_z = 0.3: the cfg-2/cfg-3 headline meshes.
* ``box``       -- "cartesian-deformed" box in 2D/3D: x_c + a*s_c*prod_b
  sin(2 pi x_b), s = (+1, -1, +1) (cfg-1 with a = 0.02).
* ``spiral``    -- one thick planar spiral element.
* ``sphere`` / ``torus`` -- quad surface meshes embedded in 3D (cfg-4).
* ``curve`` / ``helix`` -- line meshes (d_r = 1) in 2D and 3D.

Every mesh is a `MeshData`: nodes f64[E, d, N**dr], lexicographic node order
with the first reference axis fastest (bounds.py:58-94).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .basis import gll_nodes

__all__ = ["MeshData", "MeshSpec", "generate_mesh", "kershaw_mesh", "box_mesh",
           "spiral_mesh", "sphere_mesh", "torus_mesh", "curve_mesh", "helix_mesh",
           "analytic_field", "uniform_points", "surface_points", "curve_points",
           "partition_blocks"]


@dataclass
class MeshData:
    nodes: np.ndarray      # (E, d, N**dr)
    phys_dim: int
    ref_dim: int
    order: int

    @property
    def num_elements(self) -> int:
        return self.nodes.shape[0]


@dataclass
class MeshSpec:
    generator: str = "kershaw"
    dims: int = 3
    order: int = 4
    elements: int = 8          # per axis
    amplitude: float = 0.3     # kershaw eps / box deformation amplitude
    refinement: int = 0


def _ref_grid(p: int, dr: int) -> list[np.ndarray]:
    """Reference GLL coordinates of the N**dr element nodes, axis 0 fastest."""
    z = gll_nodes(p)
    axes = np.meshgrid(*([z] * dr), indexing="ij")
    return [a.transpose(tuple(range(dr))[::-1]).reshape(-1) for a in axes]


def _unit_cells(n: int, p: int, d: int) -> np.ndarray:
    """Nodes of an n^d Cartesian grid of [0,1]^d: (E, d, N^d), element index
    lexicographic (x fastest)."""
    ref = _ref_grid(p, d)
    idx = np.meshgrid(*([np.arange(n)] * d), indexing="ij")
    idx = [a.transpose(tuple(range(d))[::-1]).reshape(-1) for a in idx]
    E = n ** d
    out = np.empty((E, d, ref[0].size))
    for c in range(d):
        out[:, c, :] = (idx[c][:, None] + 0.5 * (ref[c][None, :] + 1.0)) / n
    return out


def _smoothstep(t):
    t = np.clip(t, 0.0, 1.0)
    return t * t * t * (t * (6.0 * t - 15.0) + 10.0)


def _right(e, x):
    return np.where(x <= 0.5, (2.0 - e) * x, 1.0 + e * (x - 1.0))


def _left(e, x):
    return 1.0 - _right(e, 1.0 - x)


def _kershaw_1d(x, y, e):
    layer = np.minimum(np.floor(6.0 * x), 5.0)
    lam = 6.0 * x - layer
    L, R = _left(e, y), _right(e, y)

    def step(a, b, t):
        return a + (b - a) * _smoothstep(t)

    out = np.select(
        [layer == 0, (layer == 1) | (layer == 4), layer == 2, layer == 3],
        [L, step(L, R, lam), step(R, L, lam / 2.0), step(R, L, (1.0 + lam) / 2.0)],
        default=R)
    return out


def kershaw_mesh(n: int, p: int, eps: float = 0.3) -> MeshData:
    """n^3 hexes of order p on [0,1]^3 under the Kershaw map (eps_y=eps_z)."""
    X = _unit_cells(n, p, 3)
    x, y, z = X[:, 0], X[:, 1], X[:, 2]
    out = np.stack([x, _kershaw_1d(x, y, eps), _kershaw_1d(x, z, eps)], axis=1)
    return MeshData(np.ascontiguousarray(out), 3, 3, p)


def box_mesh(d: int, n: int, p: int, amp: float = 0.02) -> MeshData:
    """Cartesian-deformed n^d box of [0,1]^d (cfg-1: d=2, n=16, p=3)."""
    X = _unit_cells(n, p, d)
    bump = np.prod(np.sin(2.0 * np.pi * X), axis=1)
    sgn = np.array([1.0, -1.0, 1.0])[:d]
    out = X + amp * sgn[None, :, None] * bump[:, None, :]
    return MeshData(np.ascontiguousarray(out), d, d, p)


def spiral_mesh(p: int = 9, turns: float = 0.75, r0: float = 0.5, r1: float = 1.5,
                thickness: float = 0.25) -> MeshData:
    """A single thick 2D spiral element of order p: reference
    r runs along the spiral arm, s across its thickness."""
    ref = _ref_grid(p, 2)
    r, s = ref
    t = 0.5 * (r + 1.0)
    theta = 2.0 * np.pi * turns * t
    rad = r0 + (r1 - r0) * t + 0.5 * thickness * s
    nodes = np.stack([rad * np.cos(theta), rad * np.sin(theta)])
    return MeshData(nodes[None].copy(), 2, 2, p)


def sphere_mesh(n: int, p: int, radius: float = 1.0) -> MeshData:
    """Cubed-sphere surface: 6 n^2 quads of order p (gnomonic face grid)."""
    ref = _ref_grid(p, 2)
    elems = []
    for face in range(6):
        for j in range(n):
            for i in range(n):
                a = np.pi / 4.0 * (-1.0 + 2.0 * (i + 0.5 * (ref[0] + 1.0)) / n)
                b = np.pi / 4.0 * (-1.0 + 2.0 * (j + 0.5 * (ref[1] + 1.0)) / n)
                u, v = np.tan(a), np.tan(b)
                one = np.ones_like(u)
                axis, sgn = face // 2, 1.0 if face % 2 == 0 else -1.0
                cube = [None, None, None]
                cube[axis] = sgn * one
                others = [k for k in range(3) if k != axis]
                cube[others[0]] = u * sgn
                cube[others[1]] = v
                P = np.stack(cube)
                P = radius * P / np.linalg.norm(P, axis=0, keepdims=True)
                elems.append(P)
    return MeshData(np.ascontiguousarray(np.stack(elems)), 3, 2, p)


def torus_mesh(n_major: int, n_minor: int, p: int, R: float = 1.0, r: float = 0.3) -> MeshData:
    """Torus surface (theta, phi) tensor grid of quads of order p."""
    ref = _ref_grid(p, 2)
    elems = []
    for j in range(n_minor):
        for i in range(n_major):
            th = 2.0 * np.pi * (i + 0.5 * (ref[0] + 1.0)) / n_major
            ph = 2.0 * np.pi * (j + 0.5 * (ref[1] + 1.0)) / n_minor
            rho = R + r * np.cos(ph)
            elems.append(np.stack([rho * np.cos(th), rho * np.sin(th), r * np.sin(ph)]))
    return MeshData(np.ascontiguousarray(np.stack(elems)), 3, 2, p)


def curve_mesh(n: int, p: int, R: float = 1.0, a: float = 0.15, lobes: int = 5) -> MeshData:
    """Closed planar curve of n line elements of order p (d = 2, d_r = 1):
    x(th) = (R + a cos(lobes th)) (cos th, sin th), th in [0, 2 pi)."""
    z = gll_nodes(p)
    elems = []
    for i in range(n):
        th = 2.0 * np.pi * (i + 0.5 * (z + 1.0)) / n
        rho = R + a * np.cos(lobes * th)
        elems.append(np.stack([rho * np.cos(th), rho * np.sin(th)]))
    return MeshData(np.ascontiguousarray(np.stack(elems)), 2, 1, p)


def helix_mesh(n: int, p: int, turns: float = 2.0, R: float = 0.5, pitch: float = 0.4) -> MeshData:
    """Helix of n line elements of order p in 3D (d = 3, d_r = 1)."""
    z = gll_nodes(p)
    elems = []
    for i in range(n):
        t = (i + 0.5 * (z + 1.0)) / n
        th = 2.0 * np.pi * turns * t
        elems.append(np.stack([R * np.cos(th), R * np.sin(th), pitch * turns * t]))
    return MeshData(np.ascontiguousarray(np.stack(elems)), 3, 1, p)


def curve_points(mesh: MeshData, n: int, seed: int = 1, offset_frac: float = 0.3,
                 max_offset: float = 1e-5):
    """Query points near a line mesh (d_r = 1): random (element, r) mapped to
    x(r); a fraction gets an offset |t| <= max_offset along a unit normal to
    the tangent (2D: the normal; 3D: a random perpendicular).  Returns
    (points, element, r, offset)."""
    from .basis import ReferenceBasis, lagrange_eval
    rng = np.random.default_rng(seed)
    rb = ReferenceBasis(mesh.order)
    d = mesh.phys_dim
    e = rng.integers(0, mesh.num_elements, size=n)
    r = rng.uniform(-1, 1, size=n)
    v, d1, _ = lagrange_eval(rb, r)
    Xe = mesh.nodes[e]                               # (n, d, N)
    x = np.einsum("nci,ni->nc", Xe, v)
    t = np.einsum("nci,ni->nc", Xe, d1)
    t /= np.linalg.norm(t, axis=1, keepdims=True)
    if d == 2:
        nrm = np.stack([-t[:, 1], t[:, 0]], axis=1)
    else:
        g = rng.normal(size=(n, 3))
        nrm = g - np.sum(g * t, axis=1, keepdims=True) * t
        nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    off = np.where(rng.uniform(size=n) < offset_frac,
                   rng.uniform(-max_offset, max_offset, size=n), 0.0)
    return x + off[:, None] * nrm, e, r, off


def generate_mesh(spec: MeshSpec) -> MeshData:
    """SPEC.md:464-467 `generate_mesh`; refinement is applied by increasing the
    per-axis element count 2**refinement (oct-refinement of a box)."""
    n = spec.elements * (2 ** spec.refinement)
    if spec.generator == "kershaw":
        return kershaw_mesh(n, spec.order, spec.amplitude)
    if spec.generator in ("box", "cartesian-deformed", "refined-box"):
        return box_mesh(spec.dims, n, spec.order, spec.amplitude)
    if spec.generator == "spiral":
        return spiral_mesh(spec.order)
    if spec.generator == "sphere":
        return sphere_mesh(n, spec.order)
    if spec.generator == "torus":
        return torus_mesh(2 * n, n, spec.order)
    if spec.generator == "curve":
        return curve_mesh(n, spec.order)
    if spec.generator == "helix":
        return helix_mesh(n, spec.order)
    raise ValueError(f"unknown generator {spec.generator!r}")


def analytic_field(name: str, mesh: MeshData, order: int | None = None, **kw) -> np.ndarray:
    """Nodal field f64[E, C, Nf**dr] by sampling at the mesh's own nodes
    (isoparametric: field order = geometry order)."""
    X = mesh.nodes
    if order is not None and order != mesh.order:
        raise ValueError("only isoparametric fields are generated here")
    d = mesh.phys_dim
    if name == "constant":
        return np.full((X.shape[0], 1, X.shape[2]), kw.get("value", 1.0))
    if name == "coordinates":
        return X.copy()
    if name == "polynomial":
        deg = kw.get("degree", mesh.order)
        # sum_c (c+1) x_c^deg (+ x0*x1 for deg >= 2): total degree <= deg;
        # reproduced exactly by interpolation only on affine elements
        s = sum((c + 1.0) * X[:, c] ** deg for c in range(d))
        if deg >= 2:
            s = s + X[:, 0] * X[:, 1]
        return s[:, None, :]
    if name == "smooth":
        x = X[:, 0]
        y = X[:, 1]
        z = X[:, 2] if d == 3 else 0.0
        return (np.sin(np.pi * x) * np.cos(np.pi * y) * np.exp(z))[:, None, :]
    if name == "wavefront":
        a = kw.get("alpha", 200.0)
        xc, yc, r = kw.get("xc", -0.05), kw.get("yc", -0.05), kw.get("r", 0.7)
        rr = np.sqrt((X[:, 0] - xc) ** 2 + (X[:, 1] - yc) ** 2)
        return np.arctan(a * (rr - r))[:, None, :]
    if name == "uniform_velocity":  # constant vector field (particle demo)
        val = np.asarray(kw.get("value", (1.0,) + (0.0,) * (d - 1)), dtype=float)
        return np.broadcast_to(val[None, :, None], (X.shape[0], d, X.shape[2])).copy()
    if name == "taylor_green":  # periodic, divergence-free in the x-y plane
        x, y = 2 * np.pi * X[:, 0], 2 * np.pi * X[:, 1]
        u = np.zeros((X.shape[0], d, X.shape[2]))
        u[:, 0] = np.sin(x) * np.cos(y)
        u[:, 1] = -np.cos(x) * np.sin(y)
        return u
    raise ValueError(f"unknown field {name!r}")


def uniform_points(n: int, d: int, seed: int = 1, lo=0.0, hi=1.0) -> np.ndarray:
    """n uniform points in [lo, hi]^d (seeded numpy Generator)."""
    rng = np.random.default_rng(seed)
    return rng.uniform(lo, hi, size=(n, d))


def surface_points(mesh: MeshData, n: int, seed: int = 1, offset_frac: float = 0.3,
                   max_offset: float = 1e-5):
    """cfg-4 query points: random (element, r) mapped to x(r); a fraction
    gets a normal offset |t| <= max_offset.  Returns
    (points, element, r, offset)."""
    from .basis import ReferenceBasis, lagrange_eval
    rng = np.random.default_rng(seed)
    rb = ReferenceBasis(mesh.order)
    E = mesh.num_elements
    e = rng.integers(0, E, size=n)
    r = rng.uniform(-1, 1, size=(n, 2))
    vr, dr_, _ = lagrange_eval(rb, r[:, 0])
    vs, ds, _ = lagrange_eval(rb, r[:, 1])
    N = mesh.order + 1
    Xe = mesh.nodes[e].reshape(n, 3, N, N)          # (n, d, s, r)
    x = np.einsum("ncji,ni,nj->nc", Xe, vr, vs)
    tr = np.einsum("ncji,ni,nj->nc", Xe, dr_, vs)
    ts = np.einsum("ncji,ni,nj->nc", Xe, vr, ds)
    nrm = np.cross(tr, ts)
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    off = np.where(rng.uniform(size=n) < offset_frac,
                   rng.uniform(-max_offset, max_offset, size=n), 0.0)
    return x + off[:, None] * nrm, e, r, off


def partition_blocks(E: int, nranks: int) -> list[tuple[int, int]]:
    """Contiguous block partition of element ids over ranks."""
    base, extra = divmod(E, nranks)
    out, start = [], 0
    for k in range(nranks):
        cnt = base + (1 if k < extra else 0)
        out.append((start, start + cnt))
        start += cnt
    return out


# ---------------------------------------------------------------- file formats
# SPEC.md "DESIGN DECISIONS": mesh text / binary files, points and records CSV.
MESH_MAGIC = b"FPXMESH1"


def write_mesh(path: str, mesh: MeshData, binary: bool = False) -> None:
    """Text: header `fpx-mesh v1; d; d_r; p; N_E`, then per element N^dr
    lines of d floats (repr precision), lexicographic node order.  Binary:
    magic, int32 d, d_r, p, int64 N_E, then the nodes as little-endian f64
    [E][N^dr][d]."""
    X = np.ascontiguousarray(mesh.nodes)            # [E, d, K]
    E, d, K = X.shape
    rows = np.transpose(X, (0, 2, 1))               # [E, K, d]
    if binary:
        with open(path, "wb") as f:
            f.write(MESH_MAGIC)
            f.write(np.array([d, mesh.ref_dim, mesh.order], "<i4").tobytes())
            f.write(np.array([E], "<i8").tobytes())
            f.write(np.ascontiguousarray(rows, dtype="<f8").tobytes())
        return
    with open(path, "w") as f:
        f.write(f"fpx-mesh v1; {d}; {mesh.ref_dim}; {mesh.order}; {E}\n")
        for e in range(E):
            for k in range(K):
                f.write(" ".join(repr(float(v)) for v in rows[e, k]) + "\n")


def read_mesh(path: str) -> MeshData:
    with open(path, "rb") as f:
        head = f.read(len(MESH_MAGIC))
        if head == MESH_MAGIC:
            d, dr, p = (int(v) for v in np.frombuffer(f.read(12), "<i4"))
            E = int(np.frombuffer(f.read(8), "<i8")[0])
            K = (p + 1) ** dr
            rows = np.frombuffer(f.read(E * K * d * 8), "<f8").reshape(E, K, d)
            return MeshData(np.ascontiguousarray(np.transpose(rows, (0, 2, 1))), d, dr, p)
    with open(path) as f:
        hdr = [t.strip() for t in f.readline().split(";")]
        if hdr[0] != "fpx-mesh v1" or len(hdr) != 5:
            raise ValueError(f"{path}: not an fpx-mesh v1 file")
        d, dr, p, E = (int(t) for t in hdr[1:])
        K = (p + 1) ** dr
        rows = np.loadtxt(f, dtype=float, ndmin=2)
    if rows.shape != (E * K, d):
        raise ValueError(f"{path}: expected {E * K} rows of {d} values, got {rows.shape}")
    X = np.transpose(rows.reshape(E, K, d), (0, 2, 1))
    return MeshData(np.ascontiguousarray(X), d, dr, p)


def write_points(path: str, x) -> None:
    """Points CSV: one point per line, d columns."""
    np.savetxt(path, np.asarray(x, dtype=float), delimiter=",", fmt="%.17g")


def read_points(path: str) -> np.ndarray:
    return np.loadtxt(path, delimiter=",", dtype=float, ndmin=2)


def write_records(path: str, records) -> None:
    """Records CSV: `idx, code, rank, elem, r0..r{dr-1}, dist`."""
    code = np.asarray(records.code.cpu() if hasattr(records.code, "cpu") else records.code)
    rank = np.asarray(records.rank.cpu() if hasattr(records.rank, "cpu") else records.rank)
    elem = np.asarray(records.elem.cpu() if hasattr(records.elem, "cpu") else records.elem)
    r = np.asarray(records.r.cpu() if hasattr(records.r, "cpu") else records.r)
    dist = np.asarray(records.dist.cpu() if hasattr(records.dist, "cpu") else records.dist)
    dr = r.shape[1]
    with open(path, "w") as f:
        f.write("idx,code,rank,elem," + ",".join(f"r{a}" for a in range(dr)) + ",dist\n")
        for i in range(code.shape[0]):
            f.write(f"{i},{int(code[i])},{int(rank[i])},{int(elem[i])},"
                    + ",".join(repr(float(v)) for v in r[i]) + f",{float(dist[i])!r}\n")


def read_records(path: str) -> dict:
    """Inverse of write_records: dict of numpy arrays code, rank, elem, r, dist."""
    with open(path) as f:
        cols = f.readline().strip().split(",")
    a = np.loadtxt(path, delimiter=",", skiprows=1, ndmin=2)
    dr = sum(1 for c in cols if c.startswith("r") and c[1:].isdigit())
    return {"code": a[:, 1].astype(np.int32), "rank": a[:, 2].astype(np.int32),
            "elem": a[:, 3].astype(np.int32), "r": a[:, 4:4 + dr], "dist": a[:, 4 + dr]}
