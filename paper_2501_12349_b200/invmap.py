"""Per-element inverse map (drop-in for SPEC.md:275-339 `invmap`).

Constrained trust-region Newton minimisation of f(r) = 1/2 |x* - x(r)|^2
over [-1, 1]^dr with the mechanics frozen as decision D8
(DESIGN.md §3.4).  All solves run in the CUDA kernel `k_newton_pairs`
(csrc/fpx_newton.cuh) through the C-ABI `fpx_invert_pairs`; `forward_map`
uses `fpx_forward_map`.  The scalar functions below wrap a one-element mesh;
`invert_points` is the batched form over an engine setup.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _C

__all__ = ["NewtonSettings", "InverseMapResult", "forward_map", "invert_point", "classify",
           "invert_points", "INTERIOR", "BORDER", "NOT_FOUND"]

INTERIOR, BORDER, NOT_FOUND = _C.INTERIOR, _C.BORDER, _C.NOT_FOUND
INTERIOR_TOL = 1e-12


@dataclass(frozen=True)
class NewtonSettings:
    """SPEC.md:280-283 defaults."""

    max_iters: int = 50
    step_tol: float = 1e-10
    trust_grow: float = 2.0
    trust_keep: float = 0.9
    trust_accept: float = 0.01
    trust_shrink: float = 0.25
    alpha0: float = 1.0

    def __post_init__(self):
        if not (0 < self.trust_accept < self.trust_keep <= 1):
            raise ValueError("need 0 < accept < keep <= 1")
        if not (self.trust_shrink < 1 < self.trust_grow):
            raise ValueError("need shrink < 1 < grow")
        if self.max_iters < 1 or self.step_tol <= 0:
            raise ValueError("bad max_iters / step_tol")

    def apply(self, m: _C.MeshT) -> None:
        m.max_iters = self.max_iters
        m.tol = self.step_tol
        m.grow = self.trust_grow
        m.keep = self.trust_keep
        m.accept = self.trust_accept
        m.shrink = self.trust_shrink
        m.alpha0 = self.alpha0


@dataclass
class InverseMapResult:
    """SPEC.md:284-287."""

    r: np.ndarray
    dist: float
    iterations: int
    converged: bool
    boundary_flags: np.ndarray = field(default=None)

    def __post_init__(self):
        if self.boundary_flags is None:
            self.boundary_flags = np.where(self.r == -1.0, -1, np.where(self.r == 1.0, 1, 0))


def classify(result: InverseMapResult, ref_dim: int, phys_dim: int | None = None,
             eps_d: float | None = None) -> int:
    """INTERIOR iff every |r_a| < 1 - 1e-12 (and, for surfaces, d* < eps_d);
    else BORDER.  Never NOT_FOUND."""
    inside = bool(np.all(np.abs(np.asarray(result.r)[:ref_dim]) < 1.0 - INTERIOR_TOL))
    if phys_dim is not None and ref_dim < phys_dim:
        inside = inside and eps_d is not None and result.dist < eps_d
    return INTERIOR if inside else BORDER


def _one_element_mesh(geom, envelope=None, settings: NewtonSettings | None = None):
    from .basis import ReferenceBasis, build_basis_envelope
    from .bounds import device_basis
    dev = _C.require_cuda()
    env = envelope or build_basis_envelope(ReferenceBasis(geom.order))
    bd = device_basis(env, dev)
    nodes = torch.from_numpy(np.ascontiguousarray(geom.nodes)[None]).to(dev)
    m = _C.MeshT()
    m.d, m.dr, m.N, m.M, m.E = geom.phys_dim, geom.ref_dim, geom.order + 1, \
        env.interval_points.size, 1
    m.basis, m.nodes = bd.data_ptr(), nodes.data_ptr()
    (settings or NewtonSettings()).apply(m)
    m.eps_d_abs, m.eps_d_rel = -1.0, 1e-10
    return m, (bd, nodes)


def forward_map(geom, r, second: bool = False, envelope=None):
    """x(r), G = dx/dr and optionally the second derivatives (symmetric
    order rr, ss, tt, rs, rt, st) at one or more reference points r
    (SPEC.md:290-297).  r: (dr,) or (n, dr)."""
    m, keep = _one_element_mesh(geom, envelope)
    dev = keep[1].device
    rr = np.atleast_2d(np.asarray(r, dtype=float))
    n = rr.shape[0]
    rt = torch.from_numpy(np.ascontiguousarray(rr)).to(dev)
    el = torch.zeros(n, dtype=torch.int32, device=dev)
    d, dr = geom.phys_dim, geom.ref_dim
    x = torch.empty((n, d), dtype=torch.float64, device=dev)
    G = torch.empty((n, d, dr), dtype=torch.float64, device=dev)
    H2 = torch.empty((n, d, 6), dtype=torch.float64, device=dev) if second else None
    _C.check(_C.lib().fpx_forward_map(m, n, _C.ptr(el), _C.ptr(rt), _C.ptr(x), _C.ptr(G),
                                      _C.ptr(H2), _C.stream_handle()), "fpx_forward_map")
    out = (x.cpu().numpy(), G.cpu().numpy(), H2.cpu().numpy() if second else None)
    if np.ndim(r) == 1:
        out = tuple(None if o is None else o[0] for o in out)
    return out


def _r0_tensor(r0, n: int, dr: int, dev):
    if r0 is None:
        return None
    t = torch.as_tensor(r0, dtype=torch.float64).reshape(n, dr)
    if not torch.all((t >= -1.0) & (t <= 1.0)):
        raise ValueError("r0 must lie in [-1, 1]^dr (SPEC.md:298 pre)")
    return t.to(dev).contiguous()


def invert_point(geom, x_star, r0=None, settings: NewtonSettings | None = None,
                 envelope=None) -> InverseMapResult:
    """Closest point x(r*) to x* over the element.  The
    initial guess is r0 when given, else the nearest GLL node (decision D7,
    SPEC.md:327)."""
    m, keep = _one_element_mesh(geom, envelope, settings)
    dev = keep[1].device
    xs = torch.from_numpy(np.asarray(x_star, dtype=float).reshape(1, -1)).to(dev)
    el = torch.zeros(1, dtype=torch.int32, device=dev)
    dr = geom.ref_dim
    rt = _r0_tensor(r0, 1, dr, dev)
    r = torch.empty((1, dr), dtype=torch.float64, device=dev)
    dist = torch.empty(1, dtype=torch.float64, device=dev)
    it = torch.empty(1, dtype=torch.int32, device=dev)
    cv = torch.empty(1, dtype=torch.int32, device=dev)
    _C.check(_C.lib().fpx_invert_pairs(m, 1, _C.ptr(xs), _C.ptr(el), _C.ptr(rt), _C.ptr(r),
                                       _C.ptr(dist), _C.ptr(it), _C.ptr(cv), _C.stream_handle()),
             "fpx_invert_pairs")
    return InverseMapResult(r[0].cpu().numpy(), float(dist[0]), int(it[0]), bool(cv[0]))


def invert_points(setup, x: torch.Tensor, elem: torch.Tensor, r0=None):
    """Batched invert_point over explicit (point, local element) pairs of an
    engine setup (initial guesses r0 [n, dr] or the D7 seed).  Returns
    (r [n, dr], dist [n], iters [n], converged [n])."""
    dev = setup.device
    x = torch.as_tensor(x, dtype=torch.float64, device=dev).contiguous()
    elem = torch.as_tensor(elem, dtype=torch.int32, device=dev).contiguous()
    n = x.shape[0]
    rt = _r0_tensor(r0, n, setup.ref_dim, dev)
    r = torch.empty((n, setup.ref_dim), dtype=torch.float64, device=dev)
    dist = torch.empty(n, dtype=torch.float64, device=dev)
    it = torch.empty(n, dtype=torch.int32, device=dev)
    cv = torch.empty(n, dtype=torch.int32, device=dev)
    _C.check(_C.lib().fpx_invert_pairs(setup.mesh_t, n, _C.ptr(x), _C.ptr(elem), _C.ptr(rt),
                                       _C.ptr(r), _C.ptr(dist), _C.ptr(it), _C.ptr(cv),
                                       _C.stream_handle()), "fpx_invert_pairs")
    return r, dist, it, cv.bool()
