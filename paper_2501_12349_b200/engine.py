"""Setup / Find / Interpolate (drop-in for SPEC.md:381-447 `engine`).

Everything per point runs in the CUDA kernels of libfpx_sm100.so:
setup -> `fpx_setup_bounds` + `fpx_hash_build`; find -> `fpx_find`
(prefilter, element-grouped Newton, round 2, fused eval); interpolate ->
`fpx_findpts_eval`.  Multi-rank Phase B routes points and
records between ranks with torch.distributed all-to-alls (NCCL over NVLink on
GPUs) around those kernels.

Batched SoA interface:
  setup(nodes f64[E, d, N**dr], order, ref_dim, options=..., group=...)
  find(S, x f64[n, d]) -> FindRecords(code, rank, elem, r, dist)
  interpolate(S, field f64[E, C, Nf**dr] | Field, records) -> f64[n, C]
  find_and_interpolate(S, field, x) -> (values, records)
"""
from __future__ import annotations

from dataclasses import dataclass, field as dfield

from collections.abc import Mapping
import ctypes
import numpy as np
import torch

from . import _C, transport
from .basis import ReferenceBasis, build_basis_envelope
from .bounds import DegenerateElementError, GeometryError, device_basis, element_boxes
from .invmap import BORDER, INTERIOR, NOT_FOUND, NewtonSettings
from .spatial_hash import CartesianGrid, GlobalMapShard, build_global_map, n_cells

__all__ = ["EngineOptions", "EngineSetup", "Field", "FindRecord", "FindRecords", "setup",
           "find", "interpolate", "find_and_interpolate", "INTERIOR", "BORDER", "NOT_FOUND"]


@dataclass
class EngineOptions:
    """Setup options."""

    expansion: float = 0.10
    interval_count: int | None = None
    cells_local: int | None = None
    cells_global: int | None = None
    newton: NewtonSettings = dfield(default_factory=NewtonSettings)
    eps_d: float | None = None        # absolute surface threshold; None -> relative
    eps_d_rel: float = 1e-10
    # host-buffer API: replay its device part as a CUDA graph
    graphs: bool = True
    # local cells per axis = hash_refine * SPEC rule (perf only; results do not depend on it)
    hash_refine: int = 3


@dataclass
class Field:
    """Per-element coefficient blocks u^e [E, C, Nf**dr] of order `order`
    (SPEC.md:394-397)."""

    blocks: torch.Tensor
    order: int

    @property
    def components(self) -> int:
        return int(self.blocks.shape[1])


@dataclass
class FindRecord:
    """q* = {m*, e*, r*, d*, c*} of one point."""

    code: int
    rank: int
    elem: int
    r: np.ndarray
    dist: float


@dataclass
class FindRecords:
    """Batched records (device tensors).  NOT_FOUND: rank = elem = -1,
    r = dist = NaN (decision D10)."""

    code: torch.Tensor
    rank: torch.Tensor
    elem: torch.Tensor
    r: torch.Tensor
    dist: torch.Tensor
    iters: torch.Tensor | None = None
    stats: dict | None = None

    def __len__(self) -> int:
        return int(self.code.shape[0])

    def __getitem__(self, i: int) -> FindRecord:
        return FindRecord(int(self.code[i]), int(self.rank[i]), int(self.elem[i]),
                          self.r[i].cpu().numpy(), float(self.dist[i]))

    def counts(self) -> dict:
        c = torch.bincount(self.code.long(), minlength=3).tolist()
        return {"INTERIOR": c[0], "BORDER": c[1], "NOT_FOUND": c[2]}


class EngineSetup:
    """Device-resident setup of this rank's mesh partition;
    immutable after construction."""

    def __init__(self):
        self.workspace = None
        self.stats_host = None

    @property
    def num_elements(self) -> int:
        return self.E

    def local_map_entries(self) -> int:
        return int(self.elems.numel())


def _as_device_nodes(nodes, dev) -> torch.Tensor:
    if hasattr(nodes, "nodes") and hasattr(nodes, "order"):   # toolkit.MeshData
        nodes = nodes.nodes
    t = torch.as_tensor(nodes, dtype=torch.float64)
    return t.to(dev).contiguous()


def _assemble(S: EngineSetup) -> None:
    """The device mesh struct and its derived arrays (filter records, padded
    nodes) from the setup arrays (shared by setup and load_setup)."""
    opt, d, dr, N, E, dev = S.options, S.phys_dim, S.ref_dim, S.order + 1, S.E, S.device
    m = _C.MeshT()
    m.d, m.dr, m.N, m.M, m.E = d, dr, N, S.envelope.interval_points.size, E
    m.basis, m.nodes = S.basis_dev.data_ptr(), S.nodes.data_ptr()
    m.aabb, m.obb_c, m.obb_inv = S.aabb.data_ptr(), S.obb_c.data_ptr(), S.obb_inv.data_ptr()
    m.obb_ok, m.frame, m.grid = S.obb_ok.data_ptr(), S.frame.data_ptr(), S.grid_dev.data_ptr()
    m.ncell, m.max_list = S.ncell, S.max_list
    m.offsets, m.elems = S.offsets.data_ptr(), S.elems.data_ptr()
    opt.newton.apply(m)
    m.eps_d_abs = -1.0 if opt.eps_d is None else float(opt.eps_d)
    m.eps_d_rel = float(opt.eps_d_rel)
    # packed candidate-filter records (one 256-byte row per element)
    # and their float pre-test rows
    S.frec = torch.empty((E, _C.FREC), dtype=torch.float64, device=dev)
    S.fbox = torch.empty((max(E, 1), _C.FROW), dtype=torch.float32, device=dev)
    _C.check(_C.lib().fpx_filter_records(
        d, E, _C.ptr(S.aabb), _C.ptr(S.obb_c), _C.ptr(S.obb_inv), _C.ptr(S.obb_ok),
        _C.ptr(S.frame), _C.ptr(S.frec), _C.ptr(S.fbox), _C.stream_handle()),
        "fpx_filter_records")
    m.frec, m.fbox = S.frec.data_ptr(), S.fbox.data_ptr()
    # rows padded to even length: 16-byte vector loads of the geometry
    NP = N + (N % 2)
    S.nodes_pad = torch.empty((E, d, (N ** dr) // N, NP), dtype=torch.float64, device=dev)
    _C.check(_C.lib().fpx_pad_nodes(d, dr, N, E, _C.ptr(S.nodes), _C.ptr(S.nodes_pad),
                                    _C.stream_handle()), "fpx_pad_nodes")
    m.nodes_pad = S.nodes_pad.data_ptr()
    S.mesh_t = m


SETUP_CACHE_VERSION = 1
_CACHE_ARRAYS = ("nodes", "aabb", "obb_c", "obb_inv", "obb_ok", "frame", "hbox", "grid_dev",
                 "offsets", "elems")


def save_setup(S: EngineSetup, path: str) -> None:
    """Serialised setup: a versioned header and the
    device arrays of this rank's setup, little-endian, in one .npz file.
    The global map of a multi-rank setup is rebuilt on load (collective)."""
    opt = S.options
    hdr = dict(version=SETUP_CACHE_VERSION, d=S.phys_dim, dr=S.ref_dim, order=S.order, E=S.E,
               ncell=S.ncell, max_list=S.max_list, elem_offset=S.elem_offset,
               expansion=opt.expansion, interval_count=opt.interval_count,
               cells_global=opt.cells_global, hash_refine=opt.hash_refine,
               eps_d=opt.eps_d, eps_d_rel=opt.eps_d_rel, newton=vars(opt.newton))
    import json
    arrs = {k: getattr(S, k).cpu().numpy() for k in _CACHE_ARRAYS}
    np.savez(path, header=np.frombuffer(json.dumps(hdr).encode(), dtype=np.uint8), **arrs)


def load_setup(path: str, *, group: transport.RankGroup | None = None) -> EngineSetup:
    """Inverse of save_setup: uploads the arrays and reassembles the device
    mesh without recomputing bounds or the local map."""
    import json
    from .invmap import NewtonSettings
    from .spatial_hash import CartesianGrid, LocalMap
    z = np.load(path if path.endswith(".npz") else path + ".npz")
    hdr = json.loads(bytes(z["header"]).decode())
    if hdr.get("version") != SETUP_CACHE_VERSION:
        raise ValueError(f"setup cache version {hdr.get('version')} != {SETUP_CACHE_VERSION}")
    dev = _C.require_cuda()
    opt = EngineOptions(expansion=hdr["expansion"], interval_count=hdr["interval_count"],
                        cells_global=hdr["cells_global"], hash_refine=hdr["hash_refine"],
                        eps_d=hdr["eps_d"], eps_d_rel=hdr["eps_d_rel"],
                        newton=NewtonSettings(**hdr["newton"]))
    S = EngineSetup()
    S.device, S.phys_dim, S.ref_dim, S.order, S.E = dev, hdr["d"], hdr["dr"], hdr["order"], hdr["E"]
    S.basis = ReferenceBasis(S.order, opt.interval_count)
    S.envelope = build_basis_envelope(S.basis)
    S.basis_dev, S.options = device_basis(S.envelope, dev), opt
    for k in _CACHE_ARRAYS:
        setattr(S, k, torch.from_numpy(z[k]).to(dev).contiguous())
    S.ncell, S.max_list = hdr["ncell"], hdr["max_list"]
    g = CartesianGrid.from_packed(z["grid_dev"], S.phys_dim, S.ncell)
    S.local_map = LocalMap(g, S.offsets, S.elems, S.max_list, S.grid_dev)
    _assemble(S)
    S.group = group or transport.RankGroup()
    S.elem_offset = hdr["elem_offset"]
    S.global_map = None
    if not S.group.single:
        lo = S.hbox[:, 0].amin(0).cpu()
        hi = S.hbox[:, 1].amax(0).cpu()
        glo, ghi = transport.reduce_domain_bbox(S.group, lo, hi)
        etot = sum(transport.allgather_counts(S.group, S.E))
        ng = opt.cells_global or n_cells(etot, S.phys_dim)
        S.global_map = build_global_map(S.group, S.hbox, glo.numpy(), ghi.numpy(), ng)
    return S


def setup(nodes, order: int | None = None, ref_dim: int | None = None, *,
          options: EngineOptions | None = None, group: transport.RankGroup | None = None,
          elem_offset: int = 0) -> EngineSetup:
    """Build envelopes, per-element AABB/OBB, the local map Psi_L and, for
    several ranks, the global map Psi_G.  `nodes` holds this
    rank's elements f64[E, d, N**dr] (or a toolkit.MeshData)."""
    opt = options or EngineOptions()
    dev = _C.require_cuda()
    if hasattr(nodes, "order") and order is None:
        order, ref_dim = nodes.order, nodes.ref_dim
    X = _as_device_nodes(nodes, dev)
    if X.ndim != 3:
        raise GeometryError(f"nodes must be [E, d, N**dr], got {tuple(X.shape)}")
    E, d, K = X.shape
    if order is None:
        raise GeometryError("order required")
    N = order + 1
    if ref_dim is None:
        ref_dim = {N: 1, N * N: 2, N * N * N: 3}.get(K)
    if ref_dim is None or N ** ref_dim != K or not (1 <= ref_dim <= d) or d not in (2, 3):
        raise GeometryError(f"nodes shape {tuple(X.shape)} inconsistent with order {order}")
    if E < 1:
        raise GeometryError("setup needs at least one element")
    if not bool(torch.isfinite(X).all()):
        raise GeometryError("non-finite nodal coordinates")
    if not _C.lib().fpx_supported(d, ref_dim, N):
        raise _C.FpxNativeError(f"order {order} (d={d}, dr={ref_dim}) not compiled in")
    basis = ReferenceBasis(order, opt.interval_count)
    env = build_basis_envelope(basis)
    bdev = device_basis(env, dev)
    bx = element_boxes(X, d, ref_dim, env, opt.expansion, bdev)
    status = bx["status"]
    if bool((status == 1).any()):
        bad = int(torch.nonzero(status == 1)[0, 0])
        raise DegenerateElementError(f"element {bad} has zero extent on every axis")
    S = EngineSetup()
    S.device, S.phys_dim, S.ref_dim, S.order, S.E = dev, d, ref_dim, order, E
    S.basis, S.envelope, S.basis_dev, S.options = basis, env, bdev, opt
    S.nodes = X
    S.aabb, S.obb_c, S.obb_inv = bx["aabb"], bx["obb_c"], bx["obb_inv"]
    S.obb_ok, S.frame, S.hbox = bx["obb_ok"], bx["frame"], bx["hbox"]
    # Psi_L over the hash boxes (decision D5)
    from .spatial_hash import build_local_map
    lmap = build_local_map(S.hbox, opt.cells_local or min(1024, opt.hash_refine * n_cells(E, d)),
                           obbs=(S.obb_c, S.obb_inv, S.obb_ok))
    S.local_map = lmap
    S.grid_dev, S.offsets, S.elems, S.ncell, S.max_list = \
        lmap.grid_dev, lmap.offsets, lmap.elems if lmap.entries else \
        torch.zeros(1, dtype=torch.int32, device=dev), lmap.grid.cells, lmap.max_list
    _assemble(S)
    # multi-rank: global map Psi_G over the union of all ranks' boxes
    S.group = group or transport.RankGroup()
    S.elem_offset = elem_offset
    S.global_map = None
    if not S.group.single:
        lo = S.hbox[:, 0].amin(0).cpu()
        hi = S.hbox[:, 1].amax(0).cpu()
        glo, ghi = transport.reduce_domain_bbox(S.group, lo, hi)
        etot = sum(transport.allgather_counts(S.group, E))
        ng = opt.cells_global or n_cells(etot, d)
        S.global_map = build_global_map(S.group, S.hbox, glo.numpy(), ghi.numpy(), ng)
    return S


# ---------------------------------------------------------------- find
def _workspace(S: EngineSetup, n: int, pair_cap: int, slot: int = 0) -> torch.Tensor:
    """Find workspace `slot` (one per concurrently running find)."""
    need = _C.lib().fpx_find_workspace_bytes(S.mesh_t, n, pair_cap)
    if S.workspace is None:
        S.workspace = {}
    w = S.workspace.get(slot)
    if w is None or w.numel() < need:
        w = S.workspace[slot] = torch.empty(need, dtype=torch.uint8, device=S.device)
    return w


def _stats_dict(st: np.ndarray) -> dict:
    return {k: int(v) for k, v in zip(_C.STAT_NAMES, st)}


class DeviceStats(Mapping):
    """The kernel counters of one find (int64[FPX_STATS_LEN] on the device),
    read back on first access so a find does not synchronise the stream."""

    def __init__(self, t: torch.Tensor):
        self._t, self._d = t, None

    def _load(self) -> dict:
        if self._d is None:
            self._d = _stats_dict(self._t.cpu().numpy())
        return self._d

    def __getitem__(self, k):
        return self._load()[k]

    def __iter__(self):
        return iter(self._load())

    def __len__(self) -> int:
        return _C.STATS_LEN

    def __repr__(self) -> str:
        return repr(self._load())


def _find_local(S: EngineSetup, x: torch.Tensor, field: Field | None = None,
                want_iters: bool = False, hint: torch.Tensor | None = None):
    """Phase A on this rank: the fpx_find kernel pipeline.  Returns a dict of
    device tensors (code, elem [local ids], r, dist, values?, iters?) and the
    kernel counters."""
    n = int(x.shape[0])
    dev = S.device
    dr = S.ref_dim
    out = dict(code=torch.empty(n, dtype=torch.int32, device=dev),
               elem=torch.empty(n, dtype=torch.int32, device=dev),
               r=torch.empty((n, dr), dtype=torch.float64, device=dev),
               dist=torch.empty(n, dtype=torch.float64, device=dev))
    out["iters"] = torch.empty(n, dtype=torch.int32, device=dev) if want_iters else None
    blocks, C = None, 0
    if field is not None:
        blocks = field.blocks
        C = int(blocks.shape[1])
        out["values"] = torch.empty((n, C), dtype=torch.float64, device=dev)
    if n == 0:
        return out, _stats_dict(np.zeros(_C.STATS_LEN, np.int64))
    x = x.contiguous()
    return out, _find_into(S, x, out, field, hint=hint)


def _find_into(S: EngineSetup, x: torch.Tensor, out: dict, field: Field | None,
               slot: int = 0, ws: torch.Tensor | None = None,
               hint: torch.Tensor | None = None) -> DeviceStats:
    """fpx_find on the current stream writing into caller-provided device
    slices (x contiguous); `slot` selects the shared workspace unless the
    caller owns one (`ws`, e.g. a captured graph's)."""
    n = int(x.shape[0])
    stats = torch.zeros(_C.STATS_LEN, dtype=torch.int64, device=S.device)
    if n == 0:
        return DeviceStats(stats)
    blocks, C = (field.blocks, int(field.blocks.shape[1])) if field is not None else (None, 0)
    if ws is None:
        ws = _workspace(S, n, n, slot)
    L = _C.lib()
    if hint is not None:
        hint = hint.to(device=S.device, dtype=torch.int32).contiguous()
        if hint.shape[0] != n:
            raise ValueError(f"hint has {hint.shape[0]} entries for {n} points")
        L.fpx_set_find_hint(_C.ptr(hint))
    try:
        _C.check(L.fpx_find(
            S.mesh_t, n, _C.ptr(x), _C.ptr(out["code"]), _C.ptr(out["elem"]), _C.ptr(out["r"]),
            _C.ptr(out["dist"]), _C.ptr(out.get("iters")), _C.ptr(blocks), C,
            _C.ptr(out.get("values")), _C.ptr(stats), n, _C.ptr(ws), ws.numel(),
            _C.stream_handle()), "fpx_find")
    finally:
        if hint is not None:
            L.fpx_set_find_hint(None)
    return DeviceStats(stats)


def _prep_points(S: EngineSetup, x) -> torch.Tensor:
    t = torch.as_tensor(x, dtype=torch.float64)
    if t.ndim != 2 or t.shape[1] != S.phys_dim:
        raise ValueError(f"points must be [n, {S.phys_dim}], got {tuple(t.shape)}")
    return t.to(S.device, non_blocking=True).contiguous()


def _field_of(S: EngineSetup, field) -> Field:
    if isinstance(field, Field):
        f = field
    else:
        f = Field(torch.as_tensor(field, dtype=torch.float64), S.order)
    b = f.blocks.to(S.device).contiguous()
    if b.ndim != 3 or b.shape[0] != S.E or b.shape[2] != (f.order + 1) ** S.ref_dim:
        raise ValueError(f"field blocks {tuple(b.shape)} do not match the mesh "
                         f"(E={S.E}, Nf**dr with order {f.order})")
    return Field(b, f.order)


def find(S: EngineSetup, x, *, want_iters: bool = False, hint=None) -> FindRecords:
    """Computational coordinates of every point.

    hint: optional element per point (global ids, e.g. the previous step's
    records of moving particles, all found).  Each point is solved on its
    hinted element first, without the hash-list prefilter; the records are
    those of a find without hint (fpx_set_find_hint).  Single rank only
    (ignored across ranks)."""
    xt = _prep_points(S, x)
    if not S.group.single:
        from .routing import find_routed
        return find_routed(S, xt, None, want_iters)
    h = None
    if hint is not None:  # (an invalid id is harmless: solved as element 0)
        h = torch.as_tensor(hint).to(S.device).to(torch.int32) - S.elem_offset
    loc, stats = _find_local(S, xt, None, want_iters, hint=h)
    return _records_single(S, loc, stats)


def _records_single(S: EngineSetup, loc, stats, values_key=False) -> FindRecords:
    code, elem = loc["code"], loc["elem"]
    found = code != NOT_FOUND
    rank = torch.where(found, torch.zeros_like(elem), torch.full_like(elem, -1))
    if S.elem_offset:
        elem = torch.where(found, elem + S.elem_offset, elem)
    return FindRecords(code, rank, elem, loc["r"], loc["dist"], loc.get("iters"), stats)


def interpolate(S: EngineSetup, field, records: FindRecords) -> torch.Tensor:
    """Field values at found points; NaN for NOT_FOUND."""
    f = _field_of(S, field)
    if S.group.single:
        return _eval_local(S, f, records.code, records.elem - S.elem_offset, records.r)
    from .routing import interpolate_routed
    return interpolate_routed(S, f, records)


def _eval_local(S: EngineSetup, f: Field, code, elem, r) -> torch.Tensor:
    n = int(code.shape[0])
    C = f.components
    out = torch.empty((n, C), dtype=torch.float64, device=S.device)
    if n == 0:
        return out
    if f.order == S.order:
        fb, Nf = S.basis_dev, S.order + 1
    else:
        fenv = build_basis_envelope(ReferenceBasis(f.order))
        fb, Nf = device_basis(fenv, S.device), f.order + 1
    L = _C.lib()
    wsb = L.fpx_eval_workspace_bytes(S.E, n)
    ws = torch.empty(wsb, dtype=torch.uint8, device=S.device)
    code = code.to(torch.int32).contiguous()
    elem = elem.to(torch.int32).contiguous()
    r = r.contiguous()
    _C.check(L.fpx_findpts_eval(S.ref_dim, Nf, _C.ptr(fb), C, S.E, _C.ptr(f.blocks), n,
                                _C.ptr(code), _C.ptr(elem), _C.ptr(r), _C.ptr(out), _C.ptr(ws),
                                wsb, _C.stream_handle()), "fpx_findpts_eval")
    return out


class _SummedStats(Mapping):
    """Kernel counters of a chunked find: the chunks' counters summed on
    first access."""

    def __init__(self, parts):
        self._parts, self._d = parts, None

    def _load(self) -> dict:
        if self._d is None:
            tot = np.zeros(_C.STATS_LEN, np.int64)
            for p in self._parts:
                tot += np.array([p[k] for k in _C.STAT_NAMES], np.int64)
            self._d = _stats_dict(tot)
        return self._d

    def __getitem__(self, k):
        return self._load()[k]

    def __iter__(self):
        return iter(self._load())

    def __len__(self) -> int:
        return _C.STATS_LEN


# host path (tools/e2e_knobs.py, profiles/e2e_knobs_r3.txt)
_UPLOAD_CHUNKS = 4     # points uploaded in chunks, each filtered as it lands
_DOWNLOAD_PIECES = 4   # records downloaded in point ranges ...
_EARLY_PIECES = 1      # ... the first ones under the rest kernels (then patched)
_R1_PER_CHUNK = False  # round 1 per upload chunk (fpx_set_round1_events): each
                       # chunk's records go down as soon as it is solved; off:
                       # a round 1 on a quarter of the points takes 0.33 ms
                       # against 0.59 for all of them (e2e 2.4-3.0 ms against 2.36)


def _host_overlapped(S: EngineSetup, f: Field, x: torch.Tensor, out: dict, ws: dict,
                     sync: bool) -> dict:
    """One find with its host copies overlapped (captured once per buffer set
    as a CUDA graph; a replay is one launch):
      * the points go up in _UPLOAD_CHUNKS chunks on a copy stream, and the
        find sorts and prefilters each chunk as soon as it has landed
        (fpx_set_upload_events), under the next chunk's copy;
      * after round 1 every record except the ~5% the rest phase revisits
        is final, so the first _EARLY_PIECES of _DOWNLOAD_PIECES point ranges
        of the records go down on a second copy stream under the rest
        kernels (about what the link moves in that time), then the rank
        column (final after round 1 as well), the other ranges once the find
        is complete;
      * the early ranges' revisited records are written straight into the
        (pinned, mapped) host arrays by a zero-copy kernel
        (fpx_rest_patch_host) while the late ranges download.
    No host thread writes the output arrays: a host-side scatter leaves
    their lines in the CPU caches, and the next call's download into them
    then snoops (measured +2 ms per call)."""
    comp = torch.cuda.current_stream(S.device)
    up, dn, rk = _streams(S, 3)
    n = int(x.shape[0])
    npieces = _UPLOAD_CHUNKS if _R1_PER_CHUNK else _DOWNLOAD_PIECES
    if ws.get("events") is None or len(ws["events"]["up"]) != _UPLOAD_CHUNKS or \
            len(ws["events"]["dn"]) != npieces or "r1c" not in ws["events"]:
        evs = {k: [torch.cuda.Event() for _ in range(m)] for k, m in
               (("r1", 1), ("start", 1), ("up", _UPLOAD_CHUNKS), ("dn", npieces),
                ("rank", 1), ("done", 1), ("r1c", _UPLOAD_CHUNKS))}
        for lst in evs.values():  # torch creates the CUDA event on first record
            for e in lst:
                e.record(comp)
        ws["events"] = evs
    gkey = (n, x.data_ptr(), f.blocks.data_ptr(), f.components, _UPLOAD_CHUNKS,
            _DOWNLOAD_PIECES, _EARLY_PIECES, _R1_PER_CHUNK) + \
        tuple(out[k].data_ptr() for k in _REC_KEYS) + \
        tuple(ws[k].data_ptr() for k in ("x", "values", "code", "elem", "r", "dist"))
    if S.options.graphs and ws.get("graph_key") != gkey:
        _host_device_part(S, f, x, out, ws, up, dn, rk)  # warm-up outside capture
        comp.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            st = _host_device_part(S, f, x, out, ws, up, dn, rk)
        ws.update(graph=g, graph_key=gkey, graph_stats=st)
    if S.options.graphs:
        ws["graph"].replay()
        # a snapshot per call: the graph rewrites its counter buffer each replay
        st = DeviceStats(ws["graph_stats"]._t.clone())
    else:
        st = _host_device_part(S, f, x, out, ws, up, dn, rk)
    if not sync:
        raise ValueError("the overlapped host path completes on the host (sync=True)")
    comp.synchronize()
    out["stats"] = st
    return out


_REC_KEYS = ("values", "code", "elem", "r", "dist", "rank")


def _host_device_part(S: EngineSetup, f: Field, x: torch.Tensor, out: dict, ws: dict, up, dn,
                      rk):
    """Device work of _host_overlapped (capturable; see there)."""
    L = _C.lib()
    comp = torch.cuda.current_stream(S.device)
    ev = ws["events"]
    n, dr, C = int(ws["x"].shape[0]), S.ref_dim, f.components
    loc = dict(code=ws["code"], elem=ws["elem"], r=ws["r"], dist=ws["dist"], iters=None,
               values=ws["values"])
    # the pipeline owns its find workspace: a captured graph keeps its
    # pointer, so it must not be the shared one other calls may reallocate
    need = L.fpx_find_workspace_bytes(S.mesh_t, n, n)
    if ws.get("find_ws") is None or ws["find_ws"].numel() < need:
        ws["find_ws"] = torch.empty(need, dtype=torch.uint8, device=S.device)
    wsf = ws["find_ws"]
    # chunked upload on `up`
    K = _UPLOAD_CHUNKS
    ev["start"][0].record(comp)
    up.wait_event(ev["start"][0])
    with torch.cuda.stream(up):
        for c in range(K):
            a, b = n * c // K, n * (c + 1) // K
            ws["x"][a:b].copy_(x[a:b], non_blocking=True)
            ev["up"][c].record(up)
    handles = (ctypes.c_void_p * K)(*[e.cuda_event for e in ev["up"]])
    L.fpx_set_upload_events(K, ctypes.cast(handles, ctypes.c_void_p))
    if _R1_PER_CHUNK:
        r1h = (ctypes.c_void_p * K)(*[e.cuda_event for e in ev["r1c"]])
        L.fpx_set_round1_events(K, ctypes.cast(r1h, ctypes.c_void_p))
    L.fpx_set_round1_event(ev["r1"][0].cuda_event)
    try:
        st = _find_into(S, ws["x"], loc, f, ws=wsf)
    finally:
        L.fpx_set_round1_event(None)
        L.fpx_set_round1_events(0, None)
        L.fpx_set_upload_events(0, None)
    if _R1_PER_CHUNK:
        _host_downloads_per_chunk(S, f, out, ws, wsf, n, K, comp, dn, rk)
        return st
    # after round 1 every record but the rest points' is final: download the
    # early ranges on `dn` (copies only: a kernel there would wait for an SM
    # behind the persistent rest kernels) while the rest runs, the late ones
    # (and the rank column) once the find is complete
    Pn, Pe = _DOWNLOAD_PIECES, min(_EARLY_PIECES, _DOWNLOAD_PIECES)
    rng = [(n * j // Pn, n * (j + 1) // Pn) for j in range(Pn)]
    # the rank column is final after round 1 too: a find without hint only
    # turns BORDER records into other found records after it, and NOT_FOUND
    # is the prefilter's (no candidate); its small kernel runs beside the
    # rest kernels (which may rewrite a rest point's code meanwhile: from one
    # found code to another, the same rank either way) and the column goes
    # down behind the early ranges
    rk.wait_event(ev["r1"][0])
    with torch.cuda.stream(rk):
        torch.where(ws["code"] != NOT_FOUND, torch.zeros_like(ws["elem"]),
                    torch.full_like(ws["elem"], -1), out=ws["rank"])
        ev["rank"][0].record(rk)
    dn.wait_event(ev["r1"][0])
    with torch.cuda.stream(dn):
        for j in range(Pe):
            a, b = rng[j]
            for k in ("values", "code", "elem", "r", "dist"):
                out[k][a:b].copy_(ws[k][a:b], non_blocking=True)
            ev["dn"][j].record(dn)
    dn.wait_event(ev["rank"][0])
    with torch.cuda.stream(dn):
        out["rank"].copy_(ws["rank"], non_blocking=True)
    ev["done"][0].record(comp)
    dn.wait_event(ev["done"][0])
    with torch.cuda.stream(dn):
        for j in range(Pe, Pn):
            a, b = rng[j]
            for k in ("values", "code", "elem", "r", "dist"):
                out[k][a:b].copy_(ws[k][a:b], non_blocking=True)
    # the early ranges' rest records, each as soon as its download has landed
    for j in range(Pe):
        a, b = rng[j]
        comp.wait_event(ev["dn"][j])
        _C.check(L.fpx_rest_patch_host(dr, C, n, a, b, _C.ptr(wsf), wsf.numel(), S.mesh_t,
                                       _C.ptr(ws["code"]), _C.ptr(ws["elem"]), _C.ptr(ws["r"]),
                                       _C.ptr(ws["dist"]), _C.ptr(ws["values"]),
                                       out["code"].data_ptr(), out["elem"].data_ptr(),
                                       out["r"].data_ptr(), out["dist"].data_ptr(),
                                       out["values"].data_ptr(), _C.stream_handle()),
                 "fpx_rest_patch_host")
    comp.wait_stream(dn)
    return st


def _host_downloads_per_chunk(S, f, out, ws, wsf, n, K, comp, dn, rk):
    """Downloads of the per-chunk pipeline (_R1_PER_CHUNK): chunk c's point
    range goes down as soon as its round 1 is done (under the next chunks'
    work), the rank column once every round 1 is, and each range's rest
    records are patched in (fpx_rest_patch_host) after the rest phase."""
    L = _C.lib()
    ev = ws["events"]
    dr, C = S.ref_dim, f.components
    rng = [(n * c // K, n * (c + 1) // K) for c in range(K)]
    for c in range(K):
        a, b = rng[c]
        dn.wait_event(ev["r1c"][c])
        with torch.cuda.stream(dn):
            for k in ("values", "code", "elem", "r", "dist"):
                out[k][a:b].copy_(ws[k][a:b], non_blocking=True)
            ev["dn"][c].record(dn)
    # the rank column is final after round 1 (see _host_device_part)
    rk.wait_event(ev["r1"][0])
    with torch.cuda.stream(rk):
        torch.where(ws["code"] != NOT_FOUND, torch.zeros_like(ws["elem"]),
                    torch.full_like(ws["elem"], -1), out=ws["rank"])
        ev["rank"][0].record(rk)
    dn.wait_event(ev["rank"][0])
    with torch.cuda.stream(dn):
        out["rank"].copy_(ws["rank"], non_blocking=True)
    for c in range(K):
        a, b = rng[c]
        comp.wait_event(ev["dn"][c])
        _C.check(L.fpx_rest_patch_host(dr, C, n, a, b, _C.ptr(wsf), wsf.numel(), S.mesh_t,
                                       _C.ptr(ws["code"]), _C.ptr(ws["elem"]), _C.ptr(ws["r"]),
                                       _C.ptr(ws["dist"]), _C.ptr(ws["values"]),
                                       out["code"].data_ptr(), out["elem"].data_ptr(),
                                       out["r"].data_ptr(), out["dist"].data_ptr(),
                                       out["values"].data_ptr(), _C.stream_handle()),
                 "fpx_rest_patch_host")
    comp.wait_stream(dn)


def _streams(S: EngineSetup, k: int) -> list:
    """k side streams of this setup (created once)."""
    st = S.__dict__.setdefault("_side_streams", [])
    while len(st) < k:
        st.append(torch.cuda.Stream(device=S.device))
    return st[:k]


def find_and_interpolate_host(S: EngineSetup, field, x: torch.Tensor, *, chunks: int = 1,
                              out: dict | None = None, sync: bool = True):
    """find_and_interpolate for points in (pinned) host memory, with the
    records and values returned to host memory.  The points are split into
    `chunks` slices; slice c is uploaded, found and downloaded on side stream
    c, so copies overlap kernels and one slice's kernel tails run under the
    next slice's bulk work.  Returns a dict of host tensors values [n, C],
    code, rank, elem, r [n, dr], dist, and `stats` (complete on return when
    `sync`; else once the current stream reaches this point)."""
    if not S.group.single:  # routed multi-rank find: no overlap
        vals, rec = find_and_interpolate(S, field, x)
        res = dict(values=vals.cpu(), code=rec.code.cpu(), rank=rec.rank.cpu(),
                   elem=rec.elem.cpu(), r=rec.r.cpu(), dist=rec.dist.cpu(), stats=rec.stats)
        return res
    f = _field_of(S, field)
    fused = f.order == S.order
    x = torch.as_tensor(x, dtype=torch.float64)
    if x.ndim != 2 or x.shape[1] != S.phys_dim:
        raise ValueError(f"points must be [n, {S.phys_dim}], got {tuple(x.shape)}")
    if x.is_cuda:
        raise ValueError("find_and_interpolate_host takes host points")
    if not x.is_pinned():
        x = x.pin_memory()
    n, dr, dev, C = int(x.shape[0]), S.ref_dim, S.device, f.components
    pin = dict(pin_memory=True)
    if out is None:
        out = dict(values=torch.empty((n, C), dtype=torch.float64, **pin),
                   code=torch.empty(n, dtype=torch.int32, **pin),
                   rank=torch.empty(n, dtype=torch.int32, **pin),
                   elem=torch.empty(n, dtype=torch.int32, **pin),
                   r=torch.empty((n, dr), dtype=torch.float64, **pin),
                   dist=torch.empty(n, dtype=torch.float64, **pin))
    ws = S.__dict__.setdefault("_host_pipe", {})
    if ws.get("n") != n or ws.get("C") != C:
        # zero-filled once: the bulk download reads the rest points' records
        # before the zero-copy patch replaces them (initcheck-clean)
        ws.clear()
        ws.update(n=n, C=C, x=torch.zeros((n, S.phys_dim), dtype=torch.float64, device=dev),
                  values=torch.zeros((n, C), dtype=torch.float64, device=dev),
                  code=torch.zeros(n, dtype=torch.int32, device=dev),
                  rank=torch.zeros(n, dtype=torch.int32, device=dev),
                  elem=torch.zeros(n, dtype=torch.int32, device=dev),
                  r=torch.zeros((n, dr), dtype=torch.float64, device=dev),
                  dist=torch.zeros(n, dtype=torch.float64, device=dev))
    comp = torch.cuda.current_stream(dev)
    chunks = max(1, min(chunks, n))
    bounds = [n * c // chunks for c in range(chunks + 1)]
    keys = ("values", "code", "rank", "elem", "r", "dist")
    if chunks == 1 and fused and all(out[k].is_pinned() for k in keys):
        return _host_overlapped(S, f, x, out, ws, sync)
    if chunks == 1:  # upload, find, download in order on the caller's stream
        ws["x"].copy_(x, non_blocking=True)
        loc = dict(code=ws["code"], elem=ws["elem"], r=ws["r"], dist=ws["dist"], iters=None)
        st = _find_into(S, ws["x"], loc, None)
        ws["values"].copy_(_eval_local(S, f, loc["code"], loc["elem"], loc["r"]))
        torch.where(loc["code"] != NOT_FOUND, torch.zeros_like(loc["elem"]),
                    torch.full_like(loc["elem"], -1), out=ws["rank"])
        for k in keys:
            out[k].copy_(ws[k], non_blocking=True)
        if sync:
            comp.synchronize()
        out["stats"] = st
        return out
    streams = _streams(S, chunks)
    parts = []
    start = torch.cuda.Event()
    start.record(comp)
    for c in range(chunks):
        a, b = bounds[c], bounds[c + 1]
        sc = streams[c]
        sc.wait_event(start)
        with torch.cuda.stream(sc):
            ws["x"][a:b].copy_(x[a:b], non_blocking=True)
            loc = dict(code=ws["code"][a:b], elem=ws["elem"][a:b], r=ws["r"][a:b],
                       dist=ws["dist"][a:b], iters=None)
            if fused:
                loc["values"] = ws["values"][a:b]
            parts.append(_find_into(S, ws["x"][a:b], loc, f if fused else None, slot=c))
            if not fused:
                ws["values"][a:b] = _eval_local(S, f, loc["code"], loc["elem"], loc["r"])
            torch.where(loc["code"] != NOT_FOUND, torch.zeros_like(loc["elem"]),
                        torch.full_like(loc["elem"], -1), out=ws["rank"][a:b])
            for k in keys:
                out[k][a:b].copy_(ws[k][a:b], non_blocking=True)
    for c in range(chunks):
        comp.wait_stream(streams[c])
    if sync:
        comp.synchronize()
    out["stats"] = _SummedStats(parts)
    return out


def find_and_interpolate(S: EngineSetup, field, x, *, want_iters: bool = False):
    """find + interpolate with one record set.  For an
    isoparametric field the evaluation is fused into the find kernels."""
    f = _field_of(S, field)
    xt = _prep_points(S, x)
    fused = f.order == S.order
    if S.group.single:
        loc, stats = _find_local(S, xt, f if fused else None, want_iters)
        rec = _records_single(S, loc, stats)
        vals = loc["values"] if fused else _eval_local(S, f, loc["code"], loc["elem"], loc["r"])
        return vals, rec
    from .routing import find_routed
    rec = find_routed(S, xt, f if fused else None, want_iters)
    if fused:
        return rec.values, rec
    return interpolate(S, f, rec), rec
