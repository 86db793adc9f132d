"""CPU: line meshes (d_r = 1 in 2D and 3D) and the closest-point acceptance
criterion (acceptance 8) on the oracle.  bounds.py:273-274
(the dr == 1 coordinate bound) and bounds.py:351-353 (the curve frame) are
the reference branches exercised."""
import numpy as np
import pytest

from closest_point import closest_point, exterior_points
from oracle import oracle as O
from paper_2501_12349_b200 import toolkit


@pytest.mark.parametrize("kind", ["curve", "helix"])
def test_line_mesh_find_on_and_off_curve(kind):
    m = toolkit.curve_mesh(24, 4) if kind == "curve" else toolkit.helix_mesh(32, 5)
    OS = O.OracleSetup(m.nodes, m.phys_dim, 1, m.order)
    x, e, r, off = toolkit.curve_points(m, 4000, seed=3, offset_frac=0.3, max_offset=1e-6)
    rec = OS.find(x)
    on = off == 0
    # on-curve points: INTERIOR (d* < eps_d) at their own element and r
    assert np.mean(rec["code"][on] == 0) > 0.99
    ok = on & (rec["code"] == 0) & (rec["elem"] == e)
    assert ok.sum() > 0.98 * on.sum()
    assert np.max(np.abs(rec["r"][ok, 0] - r[ok])) < 1e-9
    # off-curve points (|t| > 1e-8 >> eps_d): BORDER, d* = |t|
    offc = np.abs(off) > 1e-8
    assert np.all(rec["code"][offc] == 1)
    np.testing.assert_allclose(rec["dist"][offc], np.abs(off[offc]), rtol=1e-6, atol=1e-12)


@pytest.mark.parametrize("kind", ["sphere", "curve"])
def test_closest_point_acceptance_8(kind):
    """100 exterior points near a curved surface (and a curve):
    the oracle's d* is within 1e-6 of the brute-force closest point."""
    if kind == "sphere":
        m = toolkit.sphere_mesh(3, 4)
        x = exterior_points(m, 100, seed=21, tmin=1e-4, tmax=4e-3)
    else:
        m = toolkit.curve_mesh(16, 4)
        x = exterior_points(m, 100, seed=22, tmin=1e-4, tmax=4e-3)
    # the paper widens the boxes by 100% for closest-point use
    OS = O.OracleSetup(m.nodes, m.phys_dim, m.ref_dim, m.order, expansion=1.0)
    rec = OS.find(x)
    assert np.all(rec["code"] != 2)
    for k in range(len(x)):
        db, eb, rb = closest_point(m, x[k], samples=50_000, nearest=4)
        assert rec["dist"][k] <= db + 1e-6, (k, rec["dist"][k], db)
        assert abs(rec["dist"][k] - db) < 1e-6, (k, rec["dist"][k], db, rec["elem"][k], eb)
