"""One rank of the 2-rank particle-migration GPU test (gloo plumbing, both
ranks on cuda:0): the mesh is split into two z-slabs, every particle starts
on rank 0, so half of them are non-local (> 0.1) and migrate."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_2501_12349_b200 import engine, particles, toolkit, transport  # noqa: E402

dist.init_process_group("gloo")
rank, size = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
G = transport.RankGroup.from_torch()
mesh = toolkit.box_mesh(3, 4, 2)
E = mesh.nodes.shape[0]
blocks = toolkit.partition_blocks(E, size)
a, b = blocks[rank]
S = engine.setup(mesh.nodes[a:b], 2, 3, group=G, elem_offset=a)
vel = toolkit.analytic_field("uniform_velocity", mesh, value=(0.0, 0.0, 0.1))[a:b]
x0 = toolkit.uniform_points(400, 3, seed=9, lo=0.05, hi=0.95) if rank == 0 else np.zeros((0, 3))
st = particles.init_particles(S, x0, tau=0.05)
frac0 = particles.nonlocal_fraction(S, st)
particles.advance(S, vel, st, 1e-3, box=((0, 0, 0), (1, 1, 1)))
frac1 = particles.nonlocal_fraction(S, st)
tot = transport.allgather_counts(G, len(st))
print(json.dumps({"rank": rank, "n": len(st), "total": sum(tot), "frac0": frac0,
                  "frac1": frac1, "migrations": st.migrations}), flush=True)
dist.destroy_process_group()
