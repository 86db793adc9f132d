"""One rank of the single-GPU multi-rank test: the real engine (fpx_find
kernels) on a block partition of the mesh, with Phase-B routing over gloo
(two ranks share cuda:0; NCCL refuses two ranks on one device)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_2501_12349_b200 import engine, toolkit, transport  # noqa: E402


def mesh_of(name):
    if name == "refined":  # SPEC acceptance 7: refined box, 8^3 -> 16^3 = 4096 hexes
        return toolkit.generate_mesh(toolkit.MeshSpec("refined-box", 3, 4, 8, 0.02, 1))
    return toolkit.kershaw_mesh(8, 4)


def main():
    rank, size = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    out = sys.argv[1]
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=size)
    G = transport.RankGroup.from_torch()
    mesh = mesh_of(os.environ.get("FPX_TEST_MESH", "kershaw"))
    field = toolkit.analytic_field("smooth", mesh)
    a, b = toolkit.partition_blocks(mesh.num_elements, size)[rank]
    S = engine.setup(torch.from_numpy(mesh.nodes[a:b]).cuda(), 4, 3, group=G, elem_offset=a)
    npts = int(os.environ.get("FPX_TEST_NPTS", "20000"))
    x = toolkit.uniform_points(npts, 3, seed=50 + rank, lo=-0.03, hi=1.03)
    F = engine.Field(torch.from_numpy(field[a:b]).cuda(), 4)
    vals, rec = engine.find_and_interpolate(S, F, x)
    v2 = engine.interpolate(S, F, rec)
    np.savez(out, x=x, code=rec.code.cpu().numpy(), rank=rec.rank.cpu().numpy(),
             elem=rec.elem.cpu().numpy(), r=rec.r.cpu().numpy(), dist=rec.dist.cpu().numpy(),
             values=vals.cpu().numpy(), ivalues=v2.cpu().numpy())
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
