"""Dump GPU-vs-oracle find mismatches with per-candidate oracle Newton runs."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from oracle import oracle as O
from paper_2501_12349_b200 import engine, toolkit, invmap
from paper_2501_12349_b200.basis import BasisConstants

def run(m, x):
    S = engine.setup(m)
    bc = BasisConstants.of(S.basis, S.envelope)
    B = O.basis_from_arrays(bc.nodes, bc.scale, bc.proj0, bc.proj1, bc.eta, bc.lo, bc.hi)
    OS = O.OracleSetup(m.nodes, 3, 3, m.order, B=B, ncell=S.ncell)
    rec = engine.find(S, x, want_iters=True)
    orec = OS.find(x)
    code, elem = rec.code.cpu().numpy(), rec.elem.cpu().numpy()
    r, dist = rec.r.cpu().numpy(), rec.dist.cpu().numpy()
    bad = np.nonzero((code != orec["code"]) | (elem != orec["elem"]))[0]
    print("mismatches", bad.size, "of", len(x))
    for i in bad[:8]:
        print(f"x={x[i].tolist()}\n  gpu ({code[i]}, {elem[i]}, {r[i]}, {dist[i]:.3e})"
              f"\n  orc ({orec['code'][i]}, {orec['elem'][i]}, {orec['r'][i]}, {orec['dist'][i]:.3e})")
        cell = O.cell_of(3, OS.grid, OS.ncell, x[i])
        for e in OS.elems[OS.offsets[cell]:OS.offsets[cell + 1]]:
            rr, dd, it, cv = O.invert(B, 3, 3, m.nodes[e], x[i])
            xe = torch.tensor([x[i]], dtype=torch.float64, device="cuda")
            gr, gd, git, gcv = invmap.invert_points(S, xe, torch.tensor([e], dtype=torch.int32))
            print(f"    e={e}: oracle r={rr} d={dd:.3e} it={it} cv={cv} | gpu r={gr[0].cpu().numpy()} d={float(gd[0]):.3e} it={int(git[0])}")

run(toolkit.kershaw_mesh(8, 4), toolkit.uniform_points(20_000, 3, seed=84))
run(toolkit.kershaw_mesh(6, 4), toolkit.uniform_points(4096, 3, seed=11, lo=-0.05, hi=1.05))
