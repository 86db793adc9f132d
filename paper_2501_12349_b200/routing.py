"""Multi-rank Phase B of find / interpolate (PAPER.md:388-397,
409, 457).

Points whose local code is BORDER or NOT_FOUND are routed to the candidate
ranks of their global-map cell (origin excluded, D11), searched there with the
same local kernel pipeline, and the records come back to the origin, where
the winner rule D6 merges them: INTERIOR > BORDER > smaller d* > smaller
(rank, element); a local INTERIOR is never replaced.  For the fused
find_and_interpolate the remote rank also evaluates the field at its record
and returns the value with it (2 all-to-alls in total).

Everything stays on the device: the (point, destination) pairs are
enumerated destination-major with one nonzero over the candidate bitmasks,
each exchange is one counts all-to-all plus one payload all-to-all with a
single host read of the split sizes (transport.exchange_packed), and the D6
merge is one vectorised compare-and-replace pass per source rank (each
origin point has at most one reply per source), with no sorts.  The search
itself is engine._find_local (the fpx_find kernels).
"""
from __future__ import annotations

import torch

from . import engine as E
from . import transport
from .invmap import INTERIOR, NOT_FOUND


def global_cells(gmap, x: torch.Tensor) -> torch.Tensor:
    """cell_of on the global grid for many points (-1 outside); identical
    IEEE operations to spatial_hash.box_cell_range, hence sound."""
    g = gmap.grid
    d = g.dim
    lo = torch.as_tensor(g.lower, dtype=torch.float64, device=x.device)
    hi = torch.as_tensor(g.upper, dtype=torch.float64, device=x.device)
    h = torch.as_tensor(g.cell_size, dtype=torch.float64, device=x.device)
    inside = ((x >= lo) & (x <= hi)).all(dim=1)
    q = torch.floor((x - lo) / h).to(torch.int64).clamp_(0, g.cells - 1)
    mul = torch.tensor([g.cells ** c for c in range(d)], dtype=torch.int64, device=x.device)
    cell = (q * mul).sum(dim=1)
    return torch.where(inside, cell, torch.full_like(cell, -1))


def _global_masks(S, x: torch.Tensor) -> torch.Tensor:
    """Candidate-rank bitmask of every point (Psi_G lookup; 0 outside)."""
    cells = global_cells(S.global_map, x)
    mask = S.global_map.rank_mask.to(x.device)
    return torch.where(cells >= 0, mask[cells.clamp(min=0)].to(torch.int64),
                       torch.zeros_like(cells))


def _candidate_masks(S, x: torch.Tensor) -> torch.Tensor:
    return _global_masks(S, x) & ~(1 << S.group.rank)


def find_routed(S, x: torch.Tensor, field, want_iters: bool = False) -> "E.FindRecords":
    """Multi-rank find: Phase A only on the points this rank can own (its
    bit in the global map: a point outside every local hash box has no local
    candidate, so its local record is NOT_FOUND without a search -- at N
    ranks with uniform points that skips (N-1)/N of the local work), then
    Phase B routing of the BORDER / NOT_FOUND records."""
    n = x.shape[0]
    dev = x.device
    dr = S.ref_dim
    mine = torch.nonzero((_global_masks(S, x) >> S.group.rank) & 1).flatten()
    sub, stats = E._find_local(S, x[mine].contiguous(), field, want_iters)
    nan = float("nan")
    loc = dict(code=torch.full((n,), NOT_FOUND, dtype=torch.int32, device=dev),
               elem=torch.full((n,), -1, dtype=torch.int32, device=dev),
               r=torch.full((n, dr), nan, dtype=torch.float64, device=dev),
               dist=torch.full((n,), nan, dtype=torch.float64, device=dev),
               iters=torch.zeros(n, dtype=torch.int32, device=dev) if want_iters else None)
    if field is not None:
        loc["values"] = torch.full((n, field.components), nan, dtype=torch.float64, device=dev)
    for k, v in sub.items():
        if v is not None and loc.get(k) is not None:
            loc[k][mine] = v
    stats = {**stats, "local_points": int(mine.numel())}
    return phase_b(S, x, loc, stats, field)


def _pack_by_dest(masks: torch.Tensor, P: int):
    """(row, destination) pairs of a candidate-rank bitmask per row, in
    destination-major order: returns (rows, counts[P]) on the device."""
    bits = (masks[None, :] >> torch.arange(P, device=masks.device)[:, None]) & 1
    dst, rows = torch.nonzero(bits, as_tuple=True)
    return rows, torch.bincount(dst, minlength=P)


def d6_better(cc, cd, ck, ce, bc, bd, bk, be):
    """Candidate (code, dist, rank, elem) beats the current record under the
    winner rule D6 (lexicographic; NaN distances count as +inf)."""
    cd = torch.nan_to_num(cd, nan=float("inf"))
    bd = torch.nan_to_num(bd, nan=float("inf"))
    return (cc < bc) | ((cc == bc) & ((cd < bd) | ((cd == bd) & (
        (ck < bk) | ((ck == bk) & (ce < be))))))


def phase_b(S, x: torch.Tensor, loc: dict, stats: dict, field) -> "E.FindRecords":
    G = S.group
    P, me = G.size, G.rank
    dev = x.device
    d, dr = S.phys_dim, S.ref_dim
    n = x.shape[0]
    C = field.components if field is not None else 0
    code = loc["code"].clone()
    elem = torch.where(code != NOT_FOUND, loc["elem"] + S.elem_offset, loc["elem"])
    rank = torch.where(code != NOT_FOUND, torch.full_like(code, me), torch.full_like(code, -1))
    r = loc["r"].clone()
    dist = loc["dist"].clone()
    values = loc["values"].clone() if field is not None else None
    # --- route BORDER / NOT_FOUND points to their candidate ranks (D11)
    todo = torch.nonzero(code != INTERIOR).flatten()
    masks = _candidate_masks(S, x[todo]) if todo.numel() else \
        torch.zeros(0, dtype=torch.int64, device=dev)
    rows, counts = _pack_by_dest(masks, P)
    src_idx = todo[rows]
    payload = torch.cat([x[src_idx], src_idx.to(torch.float64)[:, None]], dim=1)
    xr, counts_in = transport.exchange_packed(G, payload, counts)
    # --- remote Phase A on the received points
    rloc, rstats = E._find_local(S, xr[:, :d].contiguous(), field)
    rcode = rloc["code"]
    relem = torch.where(rcode != NOT_FOUND, rloc["elem"] + S.elem_offset, rloc["elem"])
    cols = [rcode.to(torch.float64)[:, None], relem.to(torch.float64)[:, None], rloc["r"],
            rloc["dist"][:, None]]
    if field is not None:
        cols.append(rloc["values"])
    cols.append(xr[:, d:d + 1])
    reply = torch.cat(cols, dim=1)
    got, counts_back = transport.exchange_packed(G, reply, counts_in)
    # --- D6 merge at the origin: one pass per source rank, in rank order
    # (a point has at most one reply per source, so a pass is conflict-free)
    o = 0
    for k, cnt in enumerate(counts_back):
        g = got[o:o + cnt]
        o += cnt
        if cnt == 0:
            continue
        t = g[:, -1].to(torch.int64)
        gc = g[:, 0].to(torch.int32)
        ge = g[:, 1].to(torch.int32)
        gd = g[:, 2 + dr]
        gk = torch.full_like(gc, k)
        win = d6_better(gc, gd, gk, ge, code[t], dist[t], rank[t], elem[t]) & (gc != NOT_FOUND)
        t = t[win]
        code[t] = gc[win]
        rank[t] = gk[win]
        elem[t] = ge[win]
        r[t] = g[win][:, 2:2 + dr]
        dist[t] = gd[win]
        if field is not None:
            values[t] = g[win][:, 3 + dr:3 + dr + C]
    rec = E.FindRecords(code, rank, elem, r, dist, None,
                        {**stats, "remote_points": int(sum(counts_in)),
                         "remote_newton": rstats.get("newton", 0)})
    if field is not None:
        rec.values = values
    return rec


def interpolate_routed(S, field, records: "E.FindRecords") -> torch.Tensor:
    """Two-phase interpolation: local records in place,
    remote ones shipped (origin, e*, r*) to m*, evaluated there, returned."""
    G = S.group
    P, me = G.size, G.rank
    dev = records.code.device
    n = records.code.shape[0]
    dr = S.ref_dim
    C = field.components
    out = torch.full((n, C), float("nan"), dtype=torch.float64, device=dev)
    found = records.code != NOT_FOUND
    mine = torch.nonzero(found & (records.rank == me)).flatten()
    if mine.numel():
        out[mine] = E._eval_local(S, field, records.code[mine], records.elem[mine] - S.elem_offset,
                                  records.r[mine])
    remote = torch.nonzero(found & (records.rank != me)).flatten()
    dst = records.rank[remote].to(torch.int64)
    order = torch.argsort(dst, stable=True)
    sel = remote[order]
    counts = torch.bincount(dst, minlength=P)
    payload = torch.cat([sel.to(torch.float64)[:, None],
                         records.elem[sel].to(torch.float64)[:, None], records.r[sel]], 1)
    g, counts_in = transport.exchange_packed(G, payload, counts)
    if g.shape[0]:
        el = g[:, 1].to(torch.int32) - S.elem_offset
        cd = torch.zeros(g.shape[0], dtype=torch.int32, device=dev)
        v = E._eval_local(S, field, cd, el, g[:, 2:2 + dr].contiguous())
    else:
        v = torch.zeros((0, C), dtype=torch.float64, device=dev)
    back, _ = transport.exchange_packed(G, torch.cat([g[:, 0:1], v], 1), counts_in)
    if back.shape[0]:
        out[back[:, 0].to(torch.int64)] = back[:, 1:]
    return out
