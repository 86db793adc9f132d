"""Generate golden vectors from the UNMODIFIED reference package (`fpx`).

Run in THIS container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It writes `tests/golden/ref_basis.npz` and `tests/golden/ref_bounds.npz`.
These pin the oracle (`oracle/`) and the product against the reference's
own `basis.py` / `bounds.py` on identical inputs.  Nothing here is product
code; the fixtures are committed together with this script.

Reference call sites used:
  basis.py:69-90   gll_nodes            basis.py:100-136 ReferenceBasis
  basis.py:183-198 lagrange_eval        basis.py:201-212 legendre_coeffs
  basis.py:241-282 build_basis_envelope basis.py:285-303 eval_tensor_product
  bounds.py:155-201 bound_function_1d/2d
  bounds.py:292-297 element_aabb        bounds.py:366-384 element_obb
  bounds.py:387-396 aabb_contains / obb_contains
"""
from __future__ import annotations

import os
import sys

import numpy as np

import fpx  # noqa: F401  (must be the reference package)
from fpx.basis import (ReferenceBasis, build_basis_envelope, eval_tensor_product,
                       lagrange_eval, legendre_coeffs, gll_nodes)
from fpx import bounds as B

HERE = os.path.dirname(os.path.abspath(__file__))
assert "/root/reference" in os.path.abspath(fpx.__file__), fpx.__file__


def basis_goldens():
    out = {}
    rng = np.random.default_rng(2025)
    rs = np.concatenate([[-1.0, -0.5, 0.0, 0.3, 1.0], rng.uniform(-1, 1, 27)])
    out["r_samples"] = rs
    for p in range(1, 16):
        rb = ReferenceBasis(p)
        env = build_basis_envelope(rb)
        out[f"p{p}_nodes"] = rb.nodes
        out[f"p{p}_scale"] = rb._scale
        out[f"p{p}_proj0"] = rb._proj0
        out[f"p{p}_proj1"] = rb._proj1
        out[f"p{p}_eta"] = rb.interval_points
        out[f"p{p}_envlo"] = env.lower
        out[f"p{p}_envhi"] = env.upper
        v, d1, d2 = lagrange_eval(rb, rs)
        out[f"p{p}_lag_v"] = v
        out[f"p{p}_lag_d1"] = d1
        out[f"p{p}_lag_d2"] = d2
        u = rng.normal(size=p + 1)
        out[f"p{p}_lc_u"] = u
        out[f"p{p}_lc_a"] = np.array(legendre_coeffs(rb, u))
    # interval counts other than 2N (footnote-table style)
    for (n, m) in [(4, 7), (5, 9), (8, 14), (4, 8), (5, 6 + 6)]:
        rb = ReferenceBasis(n - 1, interval_count=m)
        env = build_basis_envelope(rb)
        out[f"n{n}m{m}_envlo"] = env.lower
        out[f"n{n}m{m}_envhi"] = env.upper
    # tensor-product contraction (2D and 3D), several points and components
    for dr, p in [(2, 3), (3, 2), (3, 4)]:
        rb = ReferenceBasis(p)
        n = p + 1
        blocks = rng.normal(size=(9, 2, n ** dr))
        pts = rng.uniform(-1, 1, size=(9, dr))
        mats = [lagrange_eval(rb, pts[:, a], second=False)[0] for a in range(dr)]
        out[f"etp_d{dr}p{p}_blocks"] = blocks
        out[f"etp_d{dr}p{p}_pts"] = pts
        out[f"etp_d{dr}p{p}_out"] = eval_tensor_product(blocks, mats)
    return out


def _tensor_nodes(p, dr):
    z = gll_nodes(p)
    grids = np.meshgrid(*([z] * dr), indexing="ij")
    # lexicographic with the first reference axis fastest
    return [g.transpose(*range(dr)[::-1]).reshape(-1) for g in grids]


def random_element(rng, d, dr, p, amp, offset=0.0, scale=1.0):
    """A smooth random curved element: affine map of the reference cube plus
    a low-order polynomial bump, sampled at the GLL nodes."""
    ref = _tensor_nodes(p, dr)
    R = np.stack(ref)                     # (dr, K)
    A = rng.normal(size=(d, dr)) * 0.3
    A[:dr, :dr] += np.eye(dr)
    X = A @ R
    for c in range(d):
        coeff = rng.normal(size=(dr, dr)) * amp
        bump = sum(coeff[a, b] * R[a] * R[b] for a in range(dr) for b in range(dr))
        X[c] += bump + amp * np.sin(1.3 * R[0] + c)
    return scale * X + offset


def bounds_goldens():
    out = {}
    rng = np.random.default_rng(77)
    cases = [
        ("quad", 2, 2, [1, 3, 4]),
        ("hex", 3, 3, [1, 2, 3, 4, 7]),
        ("line2", 2, 1, [1, 3, 4]),
        ("line3", 3, 1, [2, 4]),
        ("surf3", 3, 2, [2, 4]),
    ]
    for name, d, dr, orders in cases:
        for p in orders:
            rb = ReferenceBasis(p)
            env = build_basis_envelope(rb)
            elems, aabbs, obbc, obbi, ok = [], [], [], [], []
            nel = 12 if d == 3 else 16
            for e in range(nel):
                amp = [0.0, 0.05, 0.15][e % 3]
                off = [0.0, 0.5, -3.0, 10.0][e % 4]
                sc = [1.0, 1.0 / 32, 0.2][e % 3]
                X = random_element(rng, d, dr, p, amp, off, sc)
                g = B.ElementGeometry(d, dr, p, X)
                a = B.element_aabb(g, env)
                elems.append(X)
                aabbs.append(np.stack([a.lo, a.hi]))
                try:
                    o = B.element_obb(g, env)
                    obbc.append(o.center)
                    obbi.append(o.inv_transform)
                    ok.append(1)
                except B.SingularTransformError:
                    obbc.append(np.full(d, np.nan))
                    obbi.append(np.full((d, d), np.nan))
                    ok.append(0)
            key = f"{name}_p{p}"
            out[key + "_nodes"] = np.stack(elems)
            out[key + "_aabb"] = np.stack(aabbs)
            out[key + "_obbc"] = np.stack(obbc)
            out[key + "_obbi"] = np.stack(obbi)
            out[key + "_obbok"] = np.array(ok, dtype=np.int8)
            # containment queries: random points around each element
            pts, ina, ino = [], [], []
            for e, X in enumerate(elems):
                lo, hi = aabbs[e]
                c = 0.5 * (lo + hi)
                w = hi - lo
                q = c + (rng.uniform(-0.8, 0.8, size=(40, d)) * w)
                q = np.concatenate([q, lo[None], hi[None]])   # exact corners
                a = B.Aabb(lo, hi)
                ina.append([B.aabb_contains(a, x) for x in q])
                if ok[e]:
                    o = B.Obb(obbc[e], obbi[e])
                    ino.append([B.obb_contains(o, x) for x in q])
                else:
                    ino.append([False] * len(q))
                pts.append(q)
            out[key + "_qpts"] = np.stack(pts)
            out[key + "_in_aabb"] = np.array(ina, dtype=np.int8)
            out[key + "_in_obb"] = np.array(ino, dtype=np.int8)
    # function bounds: 1D and 2D
    for p in [2, 3, 4, 7]:
        rb = ReferenceBasis(p)
        env = build_basis_envelope(rb)
        n = p + 1
        U1 = rng.normal(size=(10, n))
        lo1, hi1 = zip(*[(b.lower, b.upper) for b in
                         (B.bound_function_1d(env, u) for u in U1)])
        U2 = rng.normal(size=(10, n, n))
        lo2, hi2 = zip(*[(b.lower, b.upper) for b in
                         (B.bound_function_2d(env, u) for u in U2)])
        out[f"fb_p{p}_u1"] = U1
        out[f"fb_p{p}_lo1"] = np.stack(lo1)
        out[f"fb_p{p}_hi1"] = np.stack(hi1)
        out[f"fb_p{p}_u2"] = U2
        out[f"fb_p{p}_lo2"] = np.stack(lo2)
        out[f"fb_p{p}_hi2"] = np.stack(hi2)
    # identity hexes / quads (known answers quoted in SURVEY.md §8c)
    for p in [3, 4, 7]:
        rb = ReferenceBasis(p)
        env = build_basis_envelope(rb)
        X = np.stack(_tensor_nodes(p, 3))
        g = B.ElementGeometry(3, 3, p, X)
        lo, hi = B._coordinate_bounds(g, env)
        out[f"ident_hex_p{p}_raw"] = np.stack([lo, hi])
        o = B.element_obb(g, env)
        out[f"ident_hex_p{p}_obbi"] = o.inv_transform
    return out


def main():
    b = basis_goldens()
    np.savez_compressed(os.path.join(HERE, "ref_basis.npz"), **b)
    c = bounds_goldens()
    np.savez_compressed(os.path.join(HERE, "ref_bounds.npz"), **c)
    print("wrote", len(b), "+", len(c), "arrays", file=sys.stderr)


if __name__ == "__main__":
    main()
