"""Dump GPU-vs-oracle record differences for a parity case (diagnostic).

    python tools/parity_dump.py CASE OUT.npz
CASE: cfg2ext | torus | sphere | kershaw8
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_2501_12349_b200 import engine, toolkit  # noqa: E402
from paper_2501_12349_b200.basis import BasisConstants  # noqa: E402


def case(name):
    if name == "cfg2ext":
        m = toolkit.kershaw_mesh(32, 4)
        return m, toolkit.uniform_points(200_000, 3, seed=17, lo=-0.05, hi=1.05)
    if name == "kershaw8":
        m = toolkit.kershaw_mesh(8, 4)
        return m, toolkit.uniform_points(20_000, 3, seed=84, lo=-0.1, hi=1.1)
    m = toolkit.sphere_mesh(6, 4) if name == "sphere" else toolkit.torus_mesh(16, 8, 4)
    return m, toolkit.surface_points(m, 20_000, seed=8, offset_frac=0.3, max_offset=1e-5)[0]


def main():
    name, out = sys.argv[1], sys.argv[2]
    m, x = case(name)
    S = engine.setup(m)
    bc = BasisConstants.of(S.basis, S.envelope)
    B = O.basis_from_arrays(bc.nodes, bc.scale, bc.proj0, bc.proj1, bc.eta, bc.lo, bc.hi)
    OS = O.OracleSetup(m.nodes, S.phys_dim, S.ref_dim, S.order, B=B, ncell=S.ncell)
    rec = engine.find(S, x)
    orec = OS.find(x)
    g = dict(code=rec.code.cpu().numpy(), elem=rec.elem.cpu().numpy(),
             r=rec.r.cpu().numpy(), dist=rec.dist.cpu().numpy())
    same = (g["code"] == orec["code"]) & (g["elem"] == orec["elem"]) & (g["code"] != 2)
    err = np.where(same[:, None], np.abs(g["r"] - orec["r"]), 0).max(axis=1)
    bad = np.nonzero(err >= 1e-12)[0]
    print(name, "found", same.sum(), "r>=1e-12:", bad.size, "max", err.max())
    np.savez(out, idx=bad, x=x[bad], **{"g_" + k: v[bad] for k, v in g.items()},
             **{"o_" + k: orec[k][bad] for k in ("code", "elem", "r", "dist", "iters")})


if __name__ == "__main__":
    main()
