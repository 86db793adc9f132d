"""One rank of the CPU (gloo) test of multi-rank Phase B routing.

Launched by tests/test_routing_gloo.py with RANK/WORLD_SIZE/MASTER_* set.
The per-rank local search (engine._find_local, the CUDA kernels on a GPU)
is replaced by the oracle -- test infrastructure -- so the host routing,
global map and merge logic run on CPU tensors over gloo.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2501_12349_b200 import engine, routing, toolkit, transport  # noqa: E402
from paper_2501_12349_b200.spatial_hash import build_global_map, n_cells  # noqa: E402


class OracleRankSetup:
    """Just the fields routing.phase_b reads, with the oracle as the search."""

    def __init__(self, nodes, p, group, elem_offset, etot):
        self.oracle = O.OracleSetup(nodes, 3, 3, p)
        self.phys_dim, self.ref_dim, self.order = 3, 3, p
        self.group = group
        self.elem_offset = elem_offset
        self.E = nodes.shape[0]
        hbox = torch.from_numpy(self.oracle.boxes["hbox"])
        lo, hi = transport.reduce_domain_bbox(group, hbox[:, 0].amin(0), hbox[:, 1].amax(0))
        self.global_map = build_global_map(group, hbox, lo.numpy(), hi.numpy(), n_cells(etot, 3))


def oracle_find_local(S, x, field=None, want_iters=False):
    rec = S.oracle.find(x.numpy())
    out = {"code": torch.from_numpy(rec["code"]), "elem": torch.from_numpy(rec["elem"]),
           "r": torch.from_numpy(rec["r"]), "dist": torch.from_numpy(rec["dist"])}
    if field is not None:
        v = O.evaluate(S.oracle.B, 3, field.blocks.numpy(), rec["code"], rec["elem"], rec["r"])
        out["values"] = torch.from_numpy(v)
    return out, {"newton": int(rec["ncand"].sum())}


def oracle_eval_local(S, field, code, elem, r):
    v = O.evaluate(S.oracle.B, 3, field.blocks.numpy(), code.numpy().astype(np.int32),
                   elem.numpy().astype(np.int32), r.numpy())
    return torch.from_numpy(v)


def main():
    rank, size = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    out_path = sys.argv[1]
    dist.init_process_group("gloo", rank=rank, world_size=size)
    G = transport.RankGroup.from_torch()
    mesh = toolkit.kershaw_mesh(6, 3)
    blocks = toolkit.partition_blocks(mesh.num_elements, size)
    a, b = blocks[rank]
    S = OracleRankSetup(mesh.nodes[a:b], 3, G, a, mesh.num_elements)
    field = toolkit.analytic_field("smooth", mesh)
    engine._find_local = oracle_find_local
    engine._eval_local = oracle_eval_local
    x = toolkit.uniform_points(3000, 3, seed=100 + rank, lo=-0.02, hi=1.02)
    # local search only where this rank can own the point, then Phase B
    rec = routing.find_routed(S, torch.from_numpy(x), engine.Field(torch.from_numpy(field[a:b]), 3))
    vals = routing.interpolate_routed(S, engine.Field(torch.from_numpy(field[a:b]), 3), rec)
    np.savez(out_path, x=x, code=rec.code.numpy(), rank=rec.rank.numpy(), elem=rec.elem.numpy(),
             r=rec.r.numpy(), dist=rec.dist.numpy(), values=rec.values.numpy(),
             ivalues=vals.numpy(), gmap_cells=int((S.global_map.rank_mask != 0).sum()))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
