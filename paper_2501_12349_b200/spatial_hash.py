"""Cartesian hash maps (drop-in for SPEC.md:204-273 `spatial_hash`).

Psi_L (process-local cell -> ascending element ids, CSR) is built on the
device by `fpx_hash_build` (csrc/fpx_exact.cu: grid reduction, per-element
cell-range count, CUB scan, fill, per-cell sort).  Psi_G (cell -> candidate
ranks) is built collectively in `build_global_map` over a transport group
(NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _C

__all__ = ["CartesianGrid", "LocalMap", "GlobalMapShard", "cell_of", "n_cells",
           "build_local_map", "lookup_local", "build_global_map", "lookup_global",
           "box_cell_range"]


def n_cells(count: int, d: int) -> int:
    """Cells per axis: ceil(count^(1/d)) clamped to [1, 1024],
    evaluated in integers (smallest n with n**d >= count)."""
    n = max(1, int(round(max(count, 1) ** (1.0 / d))) - 1)
    while n ** d < count:
        n += 1
    while n > 1 and (n - 1) ** d >= count:
        n -= 1
    return int(min(max(n, 1), 1024))


@dataclass
class CartesianGrid:
    """Implicit grid: lower/upper corners and cells per axis."""

    lower: np.ndarray
    upper: np.ndarray
    cells: int

    @property
    def cell_size(self) -> np.ndarray:
        return (np.asarray(self.upper) - np.asarray(self.lower)) / self.cells

    @property
    def dim(self) -> int:
        return len(self.lower)

    def packed(self) -> np.ndarray:
        """lo[3], hi[3], h[3] as the kernels read it."""
        g = np.zeros(9)
        g[6:9] = 1.0
        d = self.dim
        g[:d] = self.lower
        g[3:3 + d] = self.upper
        g[6:6 + d] = self.cell_size
        return g

    @staticmethod
    def from_packed(g, d: int, cells: int) -> "CartesianGrid":
        g = np.asarray(g, dtype=float)
        return CartesianGrid(g[:d].copy(), g[3:3 + d].copy(), cells)


def cell_of(grid: CartesianGrid, x) -> int:
    """Lexicographic cell index of x, or -1 outside: floor of
    (x - lower)/h, exact upper boundary -> last cell."""
    x = np.asarray(x, dtype=float)
    h = grid.cell_size
    idx, mul = 0, 1
    for c in range(grid.dim):
        if not (grid.lower[c] <= x[c] <= grid.upper[c]):
            return -1
        q = int(np.floor((x[c] - grid.lower[c]) / h[c]))
        q = min(max(q, 0), grid.cells - 1)
        idx += q * mul
        mul *= grid.cells
    return idx


def box_cell_range(grid: CartesianGrid, lo, hi):
    """Per-axis inclusive cell ranges covered by a box inside the grid."""
    h = grid.cell_size
    a, b = [], []
    for c in range(grid.dim):
        qa = int(np.floor((lo[c] - grid.lower[c]) / h[c]))
        qb = int(np.floor((hi[c] - grid.lower[c]) / h[c]))
        a.append(min(max(qa, 0), grid.cells - 1))
        b.append(min(max(qb, 0), grid.cells - 1))
    return a, b


@dataclass
class LocalMap:
    """Psi_L: CSR of cell -> ascending element ids (device tensors)."""

    grid: CartesianGrid
    offsets: torch.Tensor   # int32 [cells^d + 1]
    elems: torch.Tensor     # int32 [entries]
    max_list: int
    grid_dev: torch.Tensor  # f64[9] packed grid on the device

    @property
    def entries(self) -> int:
        return int(self.elems.numel())

    def lookup(self, x) -> np.ndarray:
        return lookup_local(self, x)


def build_local_map(boxes, cells_per_axis: int | None = None, obbs=None) -> LocalMap:
    """Psi_L over element boxes [E, 2, d]: grid spans the
    union of the boxes; each box maps to the rectangular cell range between
    its corner cells; lists ascending.  With `obbs` = (obb_c, obb_inv, obb_ok)
    device tensors, cells that cannot meet an element's OBB are dropped
    (decision D5b; the AABB-and-OBB filtered candidates are unchanged).  Runs
    on the device."""
    dev = _C.require_cuda()
    boxes = torch.as_tensor(boxes, dtype=torch.float64).to(dev).contiguous()
    if boxes.ndim != 3 or boxes.shape[1] != 2 or boxes.shape[0] < 1:
        raise ValueError("build_local_map: need boxes of shape [E>=1, 2, d]")
    E, _, d = boxes.shape
    n = cells_per_axis or n_cells(E, d)
    L = _C.lib()
    grid = torch.empty(9, dtype=torch.float64, device=dev)
    offsets = torch.empty(n ** d + 1, dtype=torch.int32, device=dev)
    wsb = L.fpx_hash_workspace_bytes(d, E, n)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    need = np.zeros(1, np.int64)
    maxl = np.zeros(1, np.int32)
    st = _C.stream_handle()
    oc, oi, ok = (None, None, None) if obbs is None else \
        tuple(t.to(dev).contiguous() for t in obbs)
    ob = (_C.ptr(oc), _C.ptr(oi), _C.ptr(ok))
    _C.check(L.fpx_hash_build(d, E, _C.ptr(boxes), *ob, n, _C.ptr(grid), _C.ptr(offsets), None,
                              0, need.ctypes.data, maxl.ctypes.data, _C.ptr(ws), wsb, st),
             "fpx_hash_build(count)")
    elems = torch.empty(max(int(need[0]), 1), dtype=torch.int32, device=dev)
    _C.check(L.fpx_hash_build(d, E, _C.ptr(boxes), *ob, n, _C.ptr(grid), _C.ptr(offsets),
                              _C.ptr(elems), elems.numel(), need.ctypes.data, maxl.ctypes.data,
                              _C.ptr(ws), wsb, st), "fpx_hash_build(fill)")
    g = CartesianGrid.from_packed(grid.cpu().numpy(), d, n)
    return LocalMap(g, offsets, elems[:int(need[0])], int(maxl[0]), grid)


def lookup_local(lmap: LocalMap, x) -> np.ndarray:
    """Candidate element ids of one point, ascending; empty outside
    (SPEC.md:239-242)."""
    c = cell_of(lmap.grid, x)
    if c < 0:
        return np.zeros(0, dtype=np.int32)
    o = lmap.offsets[c:c + 2].cpu().numpy()
    return lmap.elems[o[0]:o[1]].cpu().numpy()


@dataclass
class GlobalMapShard:
    """Psi_G: the global grid (identical on all ranks) and, for every cell,
    the sorted deduplicated candidate ranks.  The rank lists of the cells
    owned by rank m (cell % N_P == m) are built there and all-gathered, so
    every rank holds the full map (result-preserving: removes the owner hop
    of lookup_global)."""

    grid: CartesianGrid
    nranks: int
    rank_mask: torch.Tensor   # int32 [cells^d] bitmask of candidate ranks (N_P <= 32)
    grid_dev: torch.Tensor

    def ranks_of_cell(self, cell: int) -> list[int]:
        if cell < 0:
            return []
        m = int(self.rank_mask[cell])
        return [k for k in range(self.nranks) if (m >> k) & 1]


def build_global_map(group, boxes: torch.Tensor, domain_lo, domain_hi,
                     cells_per_axis: int) -> GlobalMapShard:
    """Collective Psi_G build: each rank
    enumerates the global cells its element boxes overlap, sends (cell, rank)
    to the owner rank cell % N_P (all-to-all), owners deduplicate, and the
    shards are all-gathered into a per-cell rank bitmask."""
    from . import transport
    d = boxes.shape[-1]
    n = cells_per_axis
    grid = CartesianGrid(np.asarray(domain_lo, float), np.asarray(domain_hi, float), n)
    P = group.size
    if P > 32:
        raise ValueError("global map bitmask supports up to 32 ranks")
    cells = _overlapped_cells(grid, boxes.detach())
    owner = cells % P
    order = torch.argsort(owner, stable=True)
    counts = torch.bincount(owner, minlength=P)
    got, rc = transport.exchange_packed(group, cells[order], counts)
    nc = n ** d
    local = torch.zeros(nc, dtype=torch.int32, device=cells.device)
    src = torch.repeat_interleave(torch.arange(P, device=cells.device),
                                  torch.as_tensor(rc, device=cells.device))
    # (cell, source) pairs are unique per source: adding the bits is an OR
    local.index_put_((got,), (1 << src).to(torch.int32), accumulate=True)
    mask = transport.allreduce_bitor(group, local)
    dev = boxes.device
    return GlobalMapShard(grid, P, mask.to(dev), torch.from_numpy(grid.packed()).to(dev))


def _overlapped_cells(grid: CartesianGrid, boxes: torch.Tensor) -> torch.Tensor:
    """Unique global cells overlapped by any of the boxes [E, 2, d], on the
    boxes' device: per-box cell ranges (the IEEE operations of
    box_cell_range), expanded into cell ids with one repeat_interleave."""
    n, d = grid.cells, grid.dim
    dev = boxes.device
    if boxes.shape[0] == 0:
        return torch.zeros(0, dtype=torch.int64, device=dev)
    lo = torch.as_tensor(np.asarray(grid.lower, float), device=dev)
    h = torch.as_tensor(np.asarray(grid.cell_size, float), device=dev)
    qa = torch.floor((boxes[:, 0, :d] - lo) / h).clamp_(0, n - 1).to(torch.int64)
    qb = torch.floor((boxes[:, 1, :d] - lo) / h).clamp_(0, n - 1).to(torch.int64)
    ext = qb - qa + 1
    cnt = ext.prod(dim=1)
    eidx = torch.repeat_interleave(torch.arange(boxes.shape[0], device=dev), cnt)
    start = torch.cumsum(cnt, 0) - cnt
    rem = torch.arange(eidx.numel(), device=dev) - start[eidx]
    idx = torch.zeros_like(rem)
    mul = 1
    for c in range(d):
        e_c = ext[eidx, c]
        idx += (qa[eidx, c] + rem % e_c) * mul
        rem = rem // e_c
        mul *= n
    return torch.unique(idx)


def lookup_global(gmap: GlobalMapShard, x) -> list[int]:
    """Candidate ranks of a point; empty outside."""
    return gmap.ranks_of_cell(cell_of(gmap.grid, x))
