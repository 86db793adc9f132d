"""Per-element bounding structures (drop-in for the reference `fpx.bounds`).

Public names, arguments, return types and exceptions follow
/root/reference/pkg/src/fpx/bounds.py:23-55.  The computation is the batched
CUDA setup kernel (csrc/fpx_exact.cu `k_setup_bounds`, C-ABI
`fpx_setup_bounds` / `fpx_bound_function`); the per-element functions below
launch it for one element.  `element_boxes` is the batched entry engine.setup
uses for a whole mesh.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _C
from .basis import BasisConstants, BasisEnvelope, ReferenceBasis, eval_tensor_product, lagrange_eval

__all__ = [
    "GeometryError",
    "DegenerateElementError",
    "SingularTransformError",
    "ElementGeometry",
    "Aabb",
    "Obb",
    "FunctionBounds1D",
    "FunctionBounds2D",
    "bound_function_1d",
    "bound_function_2d",
    "center_map_and_jacobian",
    "element_aabb",
    "element_obb",
    "aabb_contains",
    "obb_contains",
]

DEFAULT_EXPANSION = 0.10   # bounds.py:40
ZERO_EXTENT_REL = 1e-12    # bounds.py:43


class GeometryError(ValueError):
    """Inconsistent element geometry."""


class DegenerateElementError(GeometryError):
    """Element with no spatial extent on any axis."""


class SingularTransformError(GeometryError):
    """Center Jacobian (or tangent frame) unusable for an OBB."""


@dataclass
class ElementGeometry:
    """Nodal matrix of one element: shape (phys_dim, N**ref_dim), first
    reference axis fastest (bounds.py:58-94)."""

    phys_dim: int
    ref_dim: int
    order: int
    nodes: np.ndarray

    def __post_init__(self):
        self.nodes = np.ascontiguousarray(self.nodes, dtype=float)
        if self.phys_dim not in (2, 3):
            raise GeometryError(f"phys_dim must be 2 or 3, got {self.phys_dim}")
        if not 1 <= self.ref_dim <= self.phys_dim:
            raise GeometryError(f"ref_dim {self.ref_dim} incompatible with phys_dim "
                                f"{self.phys_dim}")
        want = (self.phys_dim, (self.order + 1) ** self.ref_dim)
        if self.nodes.shape != want:
            raise GeometryError(f"nodes shape {self.nodes.shape}, expected {want}")
        if not np.isfinite(self.nodes).all():
            raise GeometryError("non-finite nodal coordinates")

    @property
    def node_count_1d(self) -> int:
        return self.order + 1

    def tensor(self) -> np.ndarray:
        """(phys_dim, N, ..., N) view, last axis fastest."""
        n = self.order + 1
        return self.nodes.reshape((self.phys_dim,) + (n,) * self.ref_dim)


def _interval_sample(eta, r):
    x = np.atleast_1d(np.asarray(r, dtype=float))
    seg = np.clip(np.searchsorted(eta, x, side="right") - 1, 0, eta.size - 2)
    w = (x - eta[seg]) / (eta[seg + 1] - eta[seg])
    return seg, w


@dataclass
class FunctionBounds1D:
    """Piecewise-linear bounds of a 1D nodal function at the interval points."""

    interval_points: np.ndarray
    lower: np.ndarray
    upper: np.ndarray

    def sample(self, r):
        seg, w = _interval_sample(self.interval_points, r)
        lo = self.lower[seg] * (1 - w) + self.lower[seg + 1] * w
        hi = self.upper[seg] * (1 - w) + self.upper[seg + 1] * w
        return lo, hi


@dataclass
class FunctionBounds2D:
    """Piecewise-bilinear bounds on the M x M interval grid; lower[k, l] has
    k along r and l along s."""

    interval_points: np.ndarray
    lower: np.ndarray
    upper: np.ndarray

    def sample(self, r, s):
        ir, tr = _interval_sample(self.interval_points, r)
        js, ts = _interval_sample(self.interval_points, s)

        def bilinear(g):
            return (g[ir, js] * (1 - tr) * (1 - ts) + g[ir + 1, js] * tr * (1 - ts)
                    + g[ir, js + 1] * (1 - tr) * ts + g[ir + 1, js + 1] * tr * ts)

        return bilinear(self.lower), bilinear(self.upper)


@dataclass
class Aabb:
    """Axis-aligned box (post-expansion)."""

    lo: np.ndarray
    hi: np.ndarray
    expansion_factor: float = DEFAULT_EXPANSION

    @property
    def extents(self) -> np.ndarray:
        return self.hi - self.lo

    @property
    def diagonal(self) -> float:
        return float(np.linalg.norm(self.extents))

    def measure(self) -> float:
        return float(np.prod(self.extents))


@dataclass
class Obb:
    """Oriented box: the unit cube through `inv_transform` about `center`."""

    center: np.ndarray
    inv_transform: np.ndarray

    def measure(self) -> float:
        return float(2.0 ** self.center.size / abs(np.linalg.det(self.inv_transform)))


# ------------------------------------------------------------- device side
_const_cache: dict = {}


def device_basis(envelope: BasisEnvelope, device=None) -> torch.Tensor:
    """Packed basis constants of `envelope` on the device (cached)."""
    device = device or _C.require_cuda()
    key = (id(envelope), str(device))
    hit = _const_cache.get(key)
    if hit is not None and hit[0] is envelope:
        return hit[1]
    bc = BasisConstants.of(envelope.basis, envelope)
    t = torch.from_numpy(_C.pack_basis(bc)).to(device)
    _const_cache[key] = (envelope, t)
    return t


def element_boxes(nodes: torch.Tensor, d: int, dr: int, envelope: BasisEnvelope,
                  expansion: float = DEFAULT_EXPANSION, basis_dev: torch.Tensor | None = None):
    """Batched element_aabb + element_obb + hash box + centre frame on the
    device.  nodes: f64[E, d, N**dr] CUDA tensor.  Returns a dict of tensors
    (aabb [E,2,d], obb_c [E,d], obb_inv [E,d,d], hbox [E,2,d],
    frame [E,d+d*d], obb_ok [E] u8, status [E] i32)."""
    dev = nodes.device
    E = nodes.shape[0]
    N, M = envelope.basis.node_count, envelope.interval_points.size
    bd = basis_dev if basis_dev is not None else device_basis(envelope, dev)
    f64 = dict(dtype=torch.float64, device=dev)
    out = dict(aabb=torch.empty((E, 2, d), **f64), obb_c=torch.empty((E, d), **f64),
               obb_inv=torch.empty((E, d, d), **f64), hbox=torch.empty((E, 2, d), **f64),
               frame=torch.empty((E, d + d * d), **f64),
               obb_ok=torch.empty(E, dtype=torch.uint8, device=dev),
               status=torch.empty(E, dtype=torch.int32, device=dev))
    nodes = nodes.contiguous()
    _C.check(_C.lib().fpx_setup_bounds(
        d, dr, N, M, E, _C.ptr(bd), _C.ptr(nodes), float(expansion), _C.ptr(out["aabb"]),
        _C.ptr(out["obb_c"]), _C.ptr(out["obb_inv"]), _C.ptr(out["hbox"]), _C.ptr(out["frame"]),
        _C.ptr(out["obb_ok"]), _C.ptr(out["status"]), _C.stream_handle()), "fpx_setup_bounds")
    return out


def _function_bounds(envelope: BasisEnvelope, values: np.ndarray, dr: int):
    dev = _C.require_cuda()
    N, M = envelope.basis.node_count, envelope.interval_points.size
    vals = torch.from_numpy(np.ascontiguousarray(values, dtype=float).reshape(1, -1)).to(dev)
    shape = (1, M) if dr == 1 else (1, M, M)
    lo = torch.empty(shape, dtype=torch.float64, device=dev)
    hi = torch.empty(shape, dtype=torch.float64, device=dev)
    _C.check(_C.lib().fpx_bound_function(dr, N, M, 1, _C.ptr(device_basis(envelope, dev)),
                                         _C.ptr(vals), _C.ptr(lo), _C.ptr(hi),
                                         _C.stream_handle()), "fpx_bound_function")
    return lo[0].cpu().numpy(), hi[0].cpu().numpy()


def bound_function_1d(envelope: BasisEnvelope, values) -> FunctionBounds1D:
    """Legendre-compacted 1D bound (bounds.py:155-171), on the device."""
    u = np.asarray(values, dtype=float)
    if u.shape != (envelope.basis.node_count,):
        raise GeometryError(f"expected ({envelope.basis.node_count},) values, got {u.shape}")
    lo, hi = _function_bounds(envelope, u, 1)
    return FunctionBounds1D(envelope.interval_points, lo, hi)


def bound_function_2d(envelope: BasisEnvelope, values) -> FunctionBounds2D:
    """Uncompacted two-sweep 2D bound (bounds.py:174-201), on the device.
    values[i, j]: i along r, j along s."""
    u = np.asarray(values, dtype=float)
    n = envelope.basis.node_count
    if u.shape != (n, n):
        raise GeometryError(f"expected ({n}, {n}) coefficients, got {u.shape}")
    lo, hi = _function_bounds(envelope, u.T.reshape(-1), 2)   # flat[i + N j] = u[i, j]
    return FunctionBounds2D(envelope.interval_points, lo, hi)


def center_map_and_jacobian(geom: ElementGeometry, basis: ReferenceBasis):
    """x(0) (d,) and the Jacobian dx/dr(0) (d, d_r) of the element map at the
    reference centre (bounds.py:97-107): the nodes contracted with the
    centre Lagrange values, with axis a's factor replaced by the first
    derivatives for column a.  Host-side scalar helper (numpy), like
    aabb_contains; the setup kernel forms the same frame for every element
    on the GPU (k_setup_bounds)."""
    v, g, _ = lagrange_eval(basis, 0.0, second=False)
    dr = geom.ref_dim
    val = v[None, :]
    x_c = eval_tensor_product(geom.nodes, [val] * dr)[0]
    jac = np.empty((geom.phys_dim, dr))
    for a in range(dr):
        f = [val] * dr
        f[a] = g[None, :]
        jac[:, a] = eval_tensor_product(geom.nodes, f)[0]
    return x_c, jac


def _single(geom: ElementGeometry, envelope: BasisEnvelope, expansion: float):
    dev = _C.require_cuda()
    nodes = torch.from_numpy(geom.nodes[None]).to(dev)
    return element_boxes(nodes, geom.phys_dim, geom.ref_dim, envelope, expansion)


def element_aabb(geom: ElementGeometry, envelope: BasisEnvelope,
                 expansion: float = DEFAULT_EXPANSION) -> Aabb:
    """Axis-aligned bounding box (bounds.py:292-297).  Runs the setup kernel
    on the GPU (FpxNativeError without a CUDA device: no CPU fallback)."""
    out = _single(geom, envelope, expansion)
    if int(out["status"][0]) == 1:
        raise DegenerateElementError("element has zero extent on every axis")
    box = out["aabb"][0].cpu().numpy()
    return Aabb(box[0].copy(), box[1].copy(), expansion)


def element_obb(geom: ElementGeometry, envelope: BasisEnvelope,
                expansion: float = DEFAULT_EXPANSION) -> Obb:
    """Oriented bounding box from the centre frame (bounds.py:366-384).  Runs
    the setup kernel on the GPU (FpxNativeError without a CUDA device)."""
    out = _single(geom, envelope, expansion)
    if int(out["status"][0]) == 1:
        raise DegenerateElementError("element has zero extent on every axis")
    if int(out["obb_ok"][0]) == 0:
        raise SingularTransformError("singular center Jacobian or tangent frame")
    return Obb(out["obb_c"][0].cpu().numpy(), out["obb_inv"][0].cpu().numpy())


def aabb_contains(box: Aabb, x) -> bool:
    """Inclusive product test on every axis (bounds.py:387-390).  Scalar API
    predicate; the batched device test is in k_find_prefilter."""
    x = np.asarray(x, dtype=float)
    return bool(np.all((x - box.lo) * (box.hi - x) >= 0.0))


def obb_contains(box: Obb, x) -> bool:
    """Unit-cube membership in the OBB frame (bounds.py:393-396)."""
    y = box.inv_transform @ (np.asarray(x, dtype=float) - box.center)
    return bool(np.all(np.abs(y) <= 1.0))
