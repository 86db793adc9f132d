"""Brute-force closest point on a line or surface mesh (SPEC.md:512,
acceptance 8): the test oracle for d* of exterior points.

Level 1 samples 10^6 points uniformly in reference space over the elements
nearest to x* (by node distance); levels 2-4 re-sample a shrinking window
around the best sample, so the returned distance is the true minimum to
~1e-10 (the level-1 spacing only has to find the right basin)."""
import numpy as np

from paper_2501_12349_b200.basis import ReferenceBasis, lagrange_eval


def _map(rb, X, rs):
    """x(r) for one element X (d, N**dr) at reference points rs (m, dr)."""
    dr = rs.shape[1]
    N = rb.nodes.size
    vals = [lagrange_eval(rb, rs[:, a])[0] for a in range(dr)]
    if dr == 1:
        return vals[0] @ X.T
    Xt = X.reshape(X.shape[0], N, N)                      # (d, s, r)
    return np.einsum("cji,mi,mj->mc", Xt, vals[0], vals[1])


def closest_point(mesh, x, samples=1_000_000, nearest=8):
    """min over the mesh of |x - x_e(r)| (returns distance, element, r)."""
    rb = ReferenceBasis(mesh.order)
    dr = mesh.ref_dim
    X = mesh.nodes
    dn = np.min(np.linalg.norm(X - x[None, :, None], axis=1), axis=1)
    cand = np.argsort(dn)[:nearest]
    per = samples // len(cand)
    k = int(round(per ** (1.0 / dr)))
    g = np.linspace(-1.0, 1.0, k)
    grid = np.stack(np.meshgrid(*([g] * dr), indexing="ij"), -1).reshape(-1, dr)
    best = (np.inf, -1, None)
    for e in cand:
        d = np.linalg.norm(_map(rb, X[e], grid) - x, axis=1)
        j = int(np.argmin(d))
        if d[j] < best[0]:
            best = (float(d[j]), int(e), grid[j].copy())
    h = 2.0 / (k - 1)
    for _ in range(4):
        e, r0 = best[1], best[2]
        g = np.linspace(-2 * h, 2 * h, 101)
        loc = np.stack(np.meshgrid(*([g] * dr), indexing="ij"), -1).reshape(-1, dr) + r0
        loc = np.clip(loc, -1.0, 1.0)
        d = np.linalg.norm(_map(rb, X[e], loc) - x, axis=1)
        j = int(np.argmin(d))
        if d[j] <= best[0]:
            best = (float(d[j]), e, loc[j].copy())
        h = 4 * h / 100
    return best


def exterior_points(mesh, n, seed, tmin, tmax):
    """Points at normal distance t in [tmin, tmax] (either side) from random
    surface/curve points of the mesh."""
    from paper_2501_12349_b200 import toolkit
    if mesh.ref_dim == 2:
        x, e, r, _ = toolkit.surface_points(mesh, n, seed=seed, offset_frac=0.0)
        x2, _, _, _ = toolkit.surface_points(mesh, n, seed=seed, offset_frac=1.0, max_offset=1.0)
    else:
        x, e, r, _ = toolkit.curve_points(mesh, n, seed=seed, offset_frac=0.0)
        x2, _, _, _ = toolkit.curve_points(mesh, n, seed=seed, offset_frac=1.0, max_offset=1.0)
    nrm = x2 - x
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    rng = np.random.default_rng(seed + 1)
    t = rng.uniform(tmin, tmax, n) * rng.choice([-1.0, 1.0], n)
    return x + t[:, None] * nrm
