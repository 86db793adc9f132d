"""CPU: pin the oracle (oracle/fpx_oracle.c) against the golden vectors the
unmodified reference produced (tests/golden/make_golden.py).

Bit-exact where the reference's own arithmetic is sequential (GLL nodes,
scales, Chebyshev points, envelopes, Lagrange values, 2D function bounds,
hex / 3D-surface AABBs); a few ulp where numpy calls BLAS/LAPACK (Legendre
projectors, 1D bounds through the projector dot, OBB through det/inv).
"""
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")
GB = np.load(os.path.join(GOLD, "ref_basis.npz"))
GD = np.load(os.path.join(GOLD, "ref_bounds.npz"))


@pytest.mark.parametrize("p", range(1, 16))
def test_basis_constants_match_reference(p):
    a = O.basis(p).arrays()
    for k, g in [("nodes", "nodes"), ("scale", "scale"), ("eta", "eta"), ("lo", "envlo"),
                 ("hi", "envhi")]:
        assert np.array_equal(a[k], GB[f"p{p}_{g}"]), k
    np.testing.assert_allclose(a["proj0"], GB[f"p{p}_proj0"], rtol=0, atol=2e-15)
    np.testing.assert_allclose(a["proj1"], GB[f"p{p}_proj1"], rtol=0, atol=4e-15)


@pytest.mark.parametrize("p", [1, 2, 4, 7, 11, 15])
def test_lagrange_bitexact(p):
    B = O.basis(p)
    v, d1, d2 = O.lagrange(B, GB["r_samples"])
    assert np.array_equal(v, GB[f"p{p}_lag_v"])
    assert np.array_equal(d1, GB[f"p{p}_lag_d1"])
    assert np.array_equal(d2, GB[f"p{p}_lag_d2"])


@pytest.mark.parametrize("p", range(1, 16))
def test_legendre_coeffs(p):
    a0, a1 = O.legendre_coeffs(O.basis(p), GB[f"p{p}_lc_u"])
    np.testing.assert_allclose([a0, a1], GB[f"p{p}_lc_a"], rtol=0, atol=1e-14)


@pytest.mark.parametrize("n,m", [(4, 7), (5, 9), (8, 14), (4, 8), (5, 12)])
def test_envelope_other_interval_counts(n, m):
    a = O.basis(n - 1, m).arrays()
    assert np.array_equal(a["lo"], GB[f"n{n}m{m}_envlo"])
    assert np.array_equal(a["hi"], GB[f"n{n}m{m}_envhi"])


def test_footnote_minimum_interval_counts():
    # footnote table: valid at M_min; N=11 marginal (X2)
    table = {2: 2, 3: 4, 4: 7, 5: 9, 6: 11, 7: 12, 8: 14, 9: 16, 10: 18, 11: 20, 12: 21}
    for n, m in table.items():
        O.basis(n - 1, m)
        if m - 1 >= n and n != 11:
            with pytest.raises(O.BasisError):
                O.basis(n - 1, m - 1)


@pytest.mark.parametrize("p", [2, 3, 4, 7])
def test_function_bounds(p):
    B = O.basis(p)
    for k in range(10):
        lo, hi = O.bound1d(B, GD[f"fb_p{p}_u1"][k])
        np.testing.assert_allclose(lo, GD[f"fb_p{p}_lo1"][k], rtol=0, atol=2e-14)
        np.testing.assert_allclose(hi, GD[f"fb_p{p}_hi1"][k], rtol=0, atol=2e-14)
        lo2, hi2 = O.bound2d(B, GD[f"fb_p{p}_u2"][k])
        assert np.array_equal(lo2, GD[f"fb_p{p}_lo2"][k])
        assert np.array_equal(hi2, GD[f"fb_p{p}_hi2"][k])


CASES = {"quad": (2, 2), "hex": (3, 3), "line2": (2, 1), "line3": (3, 1), "surf3": (3, 2)}
KEYS = sorted({k.rsplit("_", 1)[0] for k in GD.files if k.endswith("_nodes")})


@pytest.mark.parametrize("key", KEYS)
def test_element_boxes_match_reference(key):
    name, ps = key.rsplit("_p", 1)
    d, dr = CASES[name]
    B = O.basis(int(ps))
    bx = O.element_boxes(B, d, dr, GD[key + "_nodes"])
    ref = GD[key + "_aabb"]
    if dr >= 2 and d == 3:
        assert np.array_equal(bx["aabb"], ref)          # sequential sums -> bit-exact
    else:
        np.testing.assert_allclose(bx["aabb"], ref, rtol=1e-15, atol=4e-15)
    ok = GD[key + "_obbok"].astype(bool)
    assert np.array_equal(bx["obb_ok"].astype(bool), ok)
    sc = np.abs(GD[key + "_obbi"][ok]).max()
    np.testing.assert_allclose(bx["obb_c"][ok], GD[key + "_obbc"][ok], rtol=0, atol=1e-13)
    np.testing.assert_allclose(bx["obb_inv"][ok], GD[key + "_obbi"][ok], rtol=0, atol=5e-12 * sc)
    # the hash box (D5) is inside the AABB and contains the OBB corners
    hb = bx["hbox"]
    assert np.all(hb[:, 0] >= bx["aabb"][:, 0]) and np.all(hb[:, 1] <= bx["aabb"][:, 1])


@pytest.mark.parametrize("key", KEYS)
def test_containment_flags_match_reference(key):
    name, _ = key.rsplit("_p", 1)
    d, _dr = CASES[name]
    ok = GD[key + "_obbok"]
    for e in range(GD[key + "_nodes"].shape[0]):
        a, o = O.contains(d, GD[key + "_aabb"][e].reshape(-1), np.nan_to_num(GD[key + "_obbc"][e]),
                          np.nan_to_num(GD[key + "_obbi"][e]), GD[key + "_qpts"][e])
        assert np.array_equal(a, GD[key + "_in_aabb"][e].astype(bool))
        if ok[e]:
            assert np.array_equal(o, GD[key + "_in_obb"][e].astype(bool))


@pytest.mark.parametrize("p", [3, 4, 7])
def test_identity_hex_known_answers(p):
    B = O.basis(p)
    z = O.gll_nodes(p)
    K, N = (p + 1) ** 3, p + 1
    idx = np.arange(K)
    X = np.stack([z[idx % N], z[(idx // N) % N], z[idx // (N * N)]])
    lo, hi = O.coord_bounds(B, 3, 3, X)
    ref = GD[f"ident_hex_p{p}_raw"]
    assert np.array_equal(lo, ref[0]) and np.array_equal(hi, ref[1])
    bx = O.element_boxes(B, 3, 3, X[None])
    np.testing.assert_allclose(bx["obb_inv"][0], GD[f"ident_hex_p{p}_obbi"], rtol=1e-14, atol=1e-15)
