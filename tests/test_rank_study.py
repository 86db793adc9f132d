"""The candidate orders the kernels use (DESIGN.md §3 "Candidate order") on
a Kershaw sample, against the oracle's owners: round 1 picks by the affine
best-first value plus the OBB norm (fewer points left for the rest phase
than either alone), and the rest phase ranks the remaining candidates by
the OBB norm (the owner first far more often than in best-first order).
Records do not depend on either order; this pins the work they save."""
import numpy as np

from rank_study import study


def test_candidate_orders_on_kershaw_sample():
    total, picks, rest = study(npts=6000, n=16, p=4)
    assert total > 5000
    assert picks["affine+obb"] < picks["affine"] and picks["affine+obb"] < picks["obb"]
    first = {k: float(np.mean(v == 1)) for k, v in rest.items()}
    assert first["obb"] > first["affine"] + 0.15, first
    assert rest["obb"].mean() < rest["affine"].mean()
