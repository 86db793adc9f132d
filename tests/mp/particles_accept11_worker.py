"""One rank of SPEC acceptance 11 on one GPU (gloo plumbing,
both ranks on cuda:0): 10^4 particles in a z-periodic box split into two
z-slabs, advected 10^3 steps by a uniform z-flow; migration must fire
exactly at the steps whose global non-local fraction exceeds 0.1, and the
particle count is conserved."""
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
mesh = toolkit.box_mesh(3, 8, 3, amp=0.0)
E = mesh.nodes.shape[0]
a, b = toolkit.partition_blocks(E, size)[rank]
S = engine.setup(mesh.nodes[a:b], 3, 3, group=G, elem_offset=a)
w = 0.5
vel = toolkit.analytic_field("uniform_velocity", mesh, value=(0.0, 0.0, w))[a:b]
vel = engine.Field(torch.from_numpy(np.ascontiguousarray(vel)).cuda(), 3)
n_half = 5000
rng = np.random.default_rng(40 + rank)
x0 = rng.uniform(0.02, 0.98, size=(n_half, 3))
x0[:, 2] = rng.uniform(0.5 * rank + 0.01, 0.5 * rank + 0.49, size=n_half)  # own slab
tau, dt, steps = 1e-3, 1e-3, 1000
st = particles.init_particles(S, x0, v=np.tile([0.0, 0.0, w], (n_half, 1)), tau=tau)
for _ in range(steps):
    particles.advance(S, vel, st, dt, box=((0, 0, 0), (1, 1, 1)), periodic=0b100)
tot = transport.allgather_counts(G, len(st))
hist = [(float(f), bool(m)) for f, m in st.history]
print(json.dumps({"rank": rank, "n": len(st), "total": sum(tot), "removed": st.removed,
                  "migrations": st.migrations, "history": hist,
                  "zmin": float(st.x[:, 2].min()) if len(st) else 0.0}), flush=True)
dist.destroy_process_group()
