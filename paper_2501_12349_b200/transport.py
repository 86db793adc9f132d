"""Rank transport (SPEC.md:341-379 `transport`) over torch.distributed.

The reference specifies an in-process simulated MPI; here the ranks are
real processes (one per GPU) and the exchanges are NCCL collectives over
NVLink/NVSwitch (gloo for the CPU tests).  `exchange` is a variable-size
all-to-all (counts first, then payload); `reduce_domain_bbox` is a min/max
all-reduce.  Messages between a (sender, receiver) pair keep their send
order, and receivers get them grouped by sender -- the canonical
(sender, sequence) order of SPEC.md:370.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

__all__ = ["RankGroup", "exchange", "reduce_domain_bbox", "allreduce_bitor", "allgather_counts"]


@dataclass
class RankGroup:
    """N_P ranks of one find/interpolate collective."""

    rank: int = 0
    size: int = 1
    pg: object = None
    device: torch.device = torch.device("cpu")   # where collective buffers live

    @staticmethod
    def from_torch(pg=None) -> "RankGroup":
        if not dist.is_available() or not dist.is_initialized():
            return RankGroup(0, 1, None)
        backend = dist.get_backend(pg)
        dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" \
            else torch.device("cpu")
        return RankGroup(dist.get_rank(pg), dist.get_world_size(pg), pg, dev)

    @property
    def single(self) -> bool:
        return self.size == 1


def _a2a(group: RankGroup, out: torch.Tensor, inp: torch.Tensor, out_splits, in_splits):
    dist.all_to_all_single(out, inp, list(out_splits), list(in_splits), group=group.pg)


def exchange(group: RankGroup, sends: list[torch.Tensor]) -> list[torch.Tensor]:
    """All-to-all of one tensor per destination (leading dim = messages, equal
    trailing shape and dtype).  Returns one tensor per source rank."""
    P = group.size
    if len(sends) != P:
        raise ValueError(f"exchange needs {P} per-destination tensors, got {len(sends)}")
    if P == 1:
        return [sends[0]]
    counts = [int(s.shape[0]) for s in sends]
    recv, rc = exchange_packed(group, torch.cat(sends, dim=0), counts)
    return list(torch.split(recv, rc, dim=0))


def exchange_packed(group: RankGroup, payload: torch.Tensor, counts):
    """All-to-all of a buffer already packed by destination (rows grouped in
    rank order, `counts[k]` rows for rank k; a list or a device tensor).
    One counts all-to-all, one host read of the send and receive counts
    together (NCCL needs the splits on the host: buffer sizing only), one
    payload all-to-all.  Returns (recv, recv_counts)."""
    P = group.size
    if P == 1:
        return payload, [int(c) for c in (counts.tolist() if torch.is_tensor(counts) else counts)]
    home = payload.device
    payload = payload.to(group.device)
    dev = payload.device
    tail = tuple(payload.shape[1:])
    w = int(np.prod(tail)) if tail else 1
    ct = torch.as_tensor(counts, dtype=torch.int64).to(dev)
    rct = torch.empty_like(ct)
    _a2a(group, rct, ct, [1] * P, [1] * P)
    both = torch.cat([ct, rct]).tolist()
    sc, rc = both[:P], both[P:]
    recv = torch.empty((sum(rc),) + tail, dtype=payload.dtype, device=dev)
    _a2a(group, recv.reshape(-1), payload.reshape(-1).contiguous(), [c * w for c in rc],
         [c * w for c in sc])
    return recv.to(home), rc


def reduce_domain_bbox(group: RankGroup, lo, hi):
    """Componentwise min/max all-reduce of the local bounding box
    (SPEC.md:360-363)."""
    lo_t = torch.as_tensor(lo, dtype=torch.float64).clone().to(group.device)
    hi_t = torch.as_tensor(hi, dtype=torch.float64).clone().to(group.device)
    if group.size > 1:
        dist.all_reduce(lo_t, op=dist.ReduceOp.MIN, group=group.pg)
        dist.all_reduce(hi_t, op=dist.ReduceOp.MAX, group=group.pg)
    return lo_t.cpu(), hi_t.cpu()


def allreduce_bitor(group: RankGroup, mask: torch.Tensor) -> torch.Tensor:
    """OR of per-rank bitmasks whose non-zero cells are disjoint across ranks
    (each global cell has exactly one owner): a SUM all-reduce, which NCCL
    supports (it has no bitwise reduction)."""
    m = mask.clone().to(group.device)
    if group.size > 1:
        dist.all_reduce(m, op=dist.ReduceOp.SUM, group=group.pg)
    return m.to(mask.device)


def allgather_counts(group: RankGroup, value: int) -> list[int]:
    if group.size == 1:
        return [int(value)]
    t = torch.tensor([value], dtype=torch.int64, device=group.device)
    out = [torch.zeros(1, dtype=torch.int64, device=group.device) for _ in range(group.size)]
    dist.all_gather(out, t, group=group.pg)
    return [int(o) for o in out]
