"""Candidate-ranking study on a cfg-2 sample (CPU, oracle boxes and local
map): how often each ranking puts a point's owner first -- for round 1's
pick among all passing candidates, and for the rest phase's order among the
remaining ones.  Records do not depend on either order.

    python tests/rank_study.py [npoints] > profiles/rank_study_r3.txt

Test infrastructure (it runs the oracle); test_rank_study.py checks the
same facts on a smaller sample."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402  (test infrastructure: the checker's boxes)
from paper_2501_12349_b200 import toolkit  # noqa: E402


def study(npts=30000, n=32, p=4):
    m = toolkit.kershaw_mesh(n, p)
    OS = O.OracleSetup(m.nodes, 3, 3, 4)
    bx = OS.boxes
    x = toolkit.uniform_points(npts, 3, seed=1001)
    rec = OS.find(x)
    g, n = OS.grid, OS.ncell
    ax = np.floor((x - g[0:3]) / g[6:9]).astype(int).clip(0, n - 1)
    cid = ax[:, 0] + n * (ax[:, 1] + n * ax[:, 2])
    fr = bx["frame"]
    picks = {"affine": 0, "obb": 0, "affine+obb": 0}
    rest = {"affine": [], "obb": []}
    total = 0
    for k in range(len(x)):
        if rec["code"][k] != 0:
            continue
        owner = rec["elem"][k]
        es = OS.elems[OS.offsets[cid[k]]:OS.offsets[cid[k] + 1]]
        lo, hi = bx["aabb"][es, 0], bx["aabb"][es, 1]
        ea = es[np.all((x[k] >= lo) & (x[k] <= hi), axis=1)]
        y = np.einsum('eij,ej->ei', bx["obb_inv"][ea], x[k] - bx["obb_c"][ea])
        ok = np.all(np.abs(y) <= 1, axis=1) | (bx["obb_ok"][ea] == 0)
        c, vo = ea[ok], np.abs(y[ok]).max(1)
        if owner not in c:
            continue
        total += 1
        ya = np.einsum('eij,ej->ei', fr[c, 3:].reshape(-1, 3, 3), x[k] - fr[c, :3])
        va = np.abs(ya).max(1)
        for name, v in (("affine", va), ("obb", vo), ("affine+obb", va + vo)):
            if c[np.lexsort((c, v))[0]] != owner:
                picks[name] += 1
        e0 = c[np.lexsort((c, va + vo))[0]]  # round 1's pick (k_prefilter_points)
        if e0 == owner:
            continue
        keep = c != e0
        for name, v in (("affine", va[keep]), ("obb", vo[keep])):
            cc = c[keep][np.lexsort((c[keep], v))]
            rest[name].append(int(np.nonzero(cc == owner)[0][0]) + 1)
    return total, {k: v / total for k, v in picks.items()}, {k: np.array(v) for k, v in rest.items()}


def main():
    npts = int(sys.argv[1]) if len(sys.argv) > 1 else 30000
    total, picks, rest = study(npts)
    print(f"# cfg-2 sample: {total} INTERIOR points with their owner among the candidates")
    for name, frac in picks.items():
        print(f"round-1 pick by {name:11s}: points left for the rest phase {frac:.4f}")
    for name, r in rest.items():
        print(f"rest order by {name:7s}: owner first {np.mean(r == 1):.3f}, mean owner rank {r.mean():.3f}"
              f" ({r.size} rest points)")


if __name__ == "__main__":
    main()
