"""Multi-rank Phase B of find / interpolate (PAPER.md:388-397,
409, 457).

Points whose local code is BORDER or NOT_FOUND are routed to the candidate
ranks of their global-map cell (origin excluded, D11), searched there with the
same local kernel pipeline, and the records come back to the origin, where
the winner rule D6 merges them: INTERIOR > BORDER > smaller d* > smaller
(rank, element); a local INTERIOR is never replaced.  For the fused
find_and_interpolate the remote rank also evaluates the field at its record
and returns the value with it (2 all-to-alls in total).

The data movement is torch device ops around NCCL all-to-alls; the search
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


def _candidate_masks(S, x: torch.Tensor) -> torch.Tensor:
    cells = global_cells(S.global_map, x)
    mask = S.global_map.rank_mask.to(x.device)
    m = torch.where(cells >= 0, mask[cells.clamp(min=0)].to(torch.int64),
                    torch.zeros_like(cells))
    return m & ~(1 << S.group.rank)


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
    # --- route BORDER / NOT_FOUND points to their candidate ranks
    todo = torch.nonzero(code != INTERIOR).flatten()
    masks = _candidate_masks(S, x[todo]) if todo.numel() else \
        torch.zeros(0, dtype=torch.int64, device=dev)
    sends, send_idx = [], []
    for k in range(P):
        sel = todo[((masks >> k) & 1).bool()] if k != me else todo[:0]
        send_idx.append(sel)
        payload = torch.cat([x[sel], sel.to(torch.float64)[:, None]], dim=1)
        sends.append(payload)
    recv = transport.exchange(G, sends)
    counts_in = [t.shape[0] for t in recv]
    xr = torch.cat(recv, dim=0) if sum(counts_in) else torch.zeros((0, d + 1), dtype=torch.float64,
                                                                    device=dev)
    # --- remote Phase A on the received points
    rloc, rstats = E._find_local(S, xr[:, :d].contiguous(), field)
    rcode = rloc["code"]
    relem = torch.where(rcode != NOT_FOUND, rloc["elem"] + S.elem_offset, rloc["elem"])
    cols = [rcode.to(torch.float64)[:, None], relem.to(torch.float64)[:, None], rloc["r"],
            rloc["dist"][:, None], xr[:, d:d + 1]]
    if field is not None:
        cols.insert(4, rloc["values"])
    reply = torch.cat(cols, dim=1)
    backs, o = [], 0
    for c in counts_in:
        backs.append(reply[o:o + c])
        o += c
    got = transport.exchange(G, backs)
    # --- merge at the origin (D6): candidates = local record + replies
    width = 4 + dr + C
    cand = [torch.cat([code.to(torch.float64)[:, None], rank.to(torch.float64)[:, None],
                       elem.to(torch.float64)[:, None], r, dist[:, None]]
                      + ([values] if field is not None else []), dim=1)]
    cand_pt = [torch.arange(n, device=dev)]
    for k, g in enumerate(got):
        if g.shape[0] == 0:
            continue
        keep = g[:, 0] != NOT_FOUND
        g = g[keep]
        rk = torch.full((g.shape[0], 1), float(k), dtype=torch.float64, device=dev)
        row = torch.cat([g[:, 0:1], rk, g[:, 1:2], g[:, 2:2 + dr], g[:, 2 + dr:3 + dr]]
                        + ([g[:, 3 + dr:3 + dr + C]] if field is not None else []), dim=1)
        cand.append(row)
        cand_pt.append(g[:, -1].to(torch.int64))
    allc = torch.cat(cand, dim=0)
    allp = torch.cat(cand_pt)
    assert allc.shape[1] == width
    # lexicographic (point, code, dist, rank, elem) via stable sorts, least
    # significant key first; NaN distances (NOT_FOUND) sort last.
    dkey = torch.nan_to_num(allc[:, 3 + dr], nan=float("inf"))
    order = torch.arange(allc.shape[0], device=dev)
    for key in (allc[:, 2], allc[:, 1], dkey, allc[:, 0], allp.to(torch.float64)):
        idx = torch.sort(key[order], stable=True).indices
        order = order[idx]
    first = torch.ones(order.numel(), dtype=torch.bool, device=dev)
    ps = allp[order]
    first[1:] = ps[1:] != ps[:-1]
    win = order[first]
    wp = allp[win]
    best = allc[win]
    out_code = torch.empty(n, dtype=torch.int32, device=dev)
    out_code[wp] = best[:, 0].to(torch.int32)
    out_rank = torch.empty(n, dtype=torch.int32, device=dev)
    out_rank[wp] = best[:, 1].to(torch.int32)
    out_elem = torch.empty(n, dtype=torch.int32, device=dev)
    out_elem[wp] = best[:, 2].to(torch.int32)
    out_r = torch.empty((n, dr), dtype=torch.float64, device=dev)
    out_r[wp] = best[:, 3:3 + dr]
    out_d = torch.empty(n, dtype=torch.float64, device=dev)
    out_d[wp] = best[:, 3 + dr]
    rec = E.FindRecords(out_code, out_rank, out_elem, out_r, out_d, None,
                        {**stats, "remote_points": int(sum(counts_in)),
                         "remote_newton": rstats.get("newton", 0)})
    if field is not None:
        vals = torch.empty((n, C), dtype=torch.float64, device=dev)
        vals[wp] = best[:, 4 + dr:4 + dr + C]
        rec.values = vals
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
    sends, idxs = [], []
    for k in range(P):
        sel = torch.nonzero(found & (records.rank == k)).flatten() if k != me else \
            torch.zeros(0, dtype=torch.int64, device=dev)
        idxs.append(sel)
        sends.append(torch.cat([sel.to(torch.float64)[:, None],
                                records.elem[sel].to(torch.float64)[:, None], records.r[sel]], 1))
    recv = transport.exchange(G, sends)
    backs = []
    for g in recv:
        if g.shape[0]:
            el = g[:, 1].to(torch.int32) - S.elem_offset
            cd = torch.zeros(g.shape[0], dtype=torch.int32, device=dev)
            v = E._eval_local(S, field, cd, el, g[:, 2:2 + dr].contiguous())
        else:
            v = torch.zeros((0, C), dtype=torch.float64, device=dev)
        backs.append(torch.cat([g[:, 0:1], v], 1))
    got = transport.exchange(G, backs)
    for g in got:
        if g.shape[0]:
            out[g[:, 0].to(torch.int64)] = g[:, 1:]
    return out
