"""CPU: the oracle's find / Newton / eval / hash restatement against the SPEC's
known-answer examples
and the acceptance criteria that are properties.  The
reference ships no code for these, so these examples are
what pins them."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2501_12349_b200 import toolkit
from paper_2501_12349_b200.spatial_hash import CartesianGrid, cell_of, n_cells


def tensor_nodes(p, dr):
    z = O.gll_nodes(p)
    N = p + 1
    idx = np.arange(N ** dr)
    cols = [z[idx % N], z[(idx // N) % N], z[idx // (N * N)]]
    return np.stack(cols[:dr])


def test_identity_element_inverse():
    """identity quad, x* = (0.3, -0.2) -> r* = x* in <= 2 its."""
    B = O.basis(4)
    X = tensor_nodes(4, 2)
    r, d, it, cv = O.invert(B, 2, 2, X, np.array([0.3, -0.2]))
    assert np.max(np.abs(r - [0.3, -0.2])) < 1e-14 and d < 1e-12 and cv
    assert it <= 3


def test_affine_recovery():
    """affine element, x* = A r + b -> r* = r to 1e-10."""
    rng = np.random.default_rng(0)
    for p in (1, 3, 5):
        B = O.basis(p)
        R = tensor_nodes(p, 3)
        A = np.eye(3) + 0.3 * rng.normal(size=(3, 3))
        b = rng.normal(size=3)
        X = A @ R + b[:, None]
        for _ in range(20):
            rh = rng.uniform(-0.95, 0.95, 3)
            r, d, it, cv = O.invert(B, 3, 3, X, A @ rh + b)
            assert np.max(np.abs(r - rh)) < 1e-10 and d < 1e-12 and cv


def test_forward_map_identity_and_fd():
    B = O.basis(3)
    X = tensor_nodes(3, 3)
    x, G, H2 = O.forward_map(B, 3, 3, X, [0.1, -0.4, 0.7], second=True)
    np.testing.assert_allclose(x, [0.1, -0.4, 0.7], atol=1e-14)
    np.testing.assert_allclose(G, np.eye(3), atol=1e-13)
    np.testing.assert_allclose(H2, 0, atol=1e-12)
    m = toolkit.kershaw_mesh(3, 3)
    Xe = m.nodes[13]
    r0 = np.array([0.2, -0.3, 0.5])
    x0, G0, _ = O.forward_map(B, 3, 3, Xe, r0)
    h = 1e-6
    for a in range(3):
        e = np.zeros(3)
        e[a] = h
        fd = (O.forward_map(B, 3, 3, Xe, r0 + e)[0] - O.forward_map(B, 3, 3, Xe, r0 - e)[0]) / (2 * h)
        np.testing.assert_allclose(fd, G0[:, a], atol=1e-6)


def test_spiral_newton_efficiency():
    """Acceptance 6: p=9 spiral, 10^4 interior points, all
    converge within 50 iterations, mean <= 15 (paper ~5)."""
    m = toolkit.spiral_mesh(9)
    B = O.basis(9)
    X = m.nodes[0]
    rng = np.random.default_rng(6)
    its, errs = [], []
    for _ in range(2000):   # 2000 keeps the CPU suite fast; the GPU test runs 10^4
        rh = rng.uniform(-0.98, 0.98, 2)
        xs = O.forward_map(B, 2, 2, X, rh)[0]
        r, d, it, cv = O.invert(B, 2, 2, X, xs)
        assert cv and it <= 50
        its.append(it)
        errs.append(np.max(np.abs(r - rh)))
    assert np.mean(its) <= 15
    assert np.max(errs) < 1e-9


def test_exterior_closest_point():
    """x* outside the element but in its box -> r* on the face,
    d* at the brute-force boundary minimum within 1e-6."""
    m = toolkit.kershaw_mesh(3, 4)
    B = O.basis(4)
    X = m.nodes[4]
    rng = np.random.default_rng(1)
    g = np.linspace(-1, 1, 101)
    for _ in range(5):
        face_r = np.array([rng.uniform(-0.8, 0.8), rng.uniform(-0.8, 0.8), 1.0])
        xf, G, _ = O.forward_map(B, 3, 3, X, face_r)
        nrm = np.cross(G[:, 0], G[:, 1])
        nrm /= np.linalg.norm(nrm)
        xs = xf + 0.01 * nrm * np.sign(nrm @ G[:, 2])
        r, d, it, cv = O.invert(B, 3, 3, X, xs)
        assert abs(r[2]) == 1.0
        best = min(np.linalg.norm(O.forward_map(B, 3, 3, X, [a, b, r[2]])[0] - xs)
                   for a in g[::2] for b in g[::2])
        assert d <= best + 1e-6


def test_classify_examples():
    """SPEC.md:313-316 via oracle find on the identity element."""
    B = O.basis(2)
    X = tensor_nodes(2, 3)[None]
    S = O.OracleSetup(X, 3, 3, 2, B=B)
    rec = S.find(np.array([[0.0, 0.0, 0.0], [1.0, 0.5, 0.0], [3.0, 3.0, 3.0]]))
    assert list(rec["code"]) == [0, 1, 2]
    assert rec["elem"][2] == -1 and np.isnan(rec["dist"][2]) and np.isnan(rec["r"][2]).all()


def test_vertex_tie_and_out_of_hull():
    """a vertex shared by 8 hexes -> d* < 1e-10, winner is
    deterministic (smallest element id among the BORDER ties, or the unique
    INTERIOR); a point outside the hull -> NOT_FOUND."""
    m = toolkit.box_mesh(3, 4, 2, amp=0.0)
    S = O.OracleSetup(m.nodes, 3, 3, 2)
    rec = S.find(np.array([[0.5, 0.5, 0.5], [1.5, 0.5, 0.5]]))
    assert rec["code"][0] in (0, 1) and rec["dist"][0] < 1e-10
    assert rec["code"][1] == 2
    # the 8 elements sharing the vertex: lexicographic ids of cells (1|2)^3
    sharing = sorted(i + 4 * j + 16 * k for i in (1, 2) for j in (1, 2) for k in (1, 2))
    assert rec["elem"][0] == sharing[0] or rec["code"][0] == 0


def test_constant_and_coordinate_fields():
    """SPEC.md:420-421."""
    m = toolkit.kershaw_mesh(4, 3)
    S = O.OracleSetup(m.nodes, 3, 3, 3)
    x = toolkit.uniform_points(3000, 3, seed=9)
    rec = S.find(x)
    one = O.evaluate(S.B, 3, toolkit.analytic_field("constant", m), rec["code"], rec["elem"], rec["r"])
    np.testing.assert_allclose(one, 1.0, atol=1e-13)
    xc = O.evaluate(S.B, 3, toolkit.analytic_field("coordinates", m), rec["code"], rec["elem"],
                    rec["r"])
    inter = rec["code"] == 0
    assert np.max(np.abs(xc[inter] - x[inter])) < 1e-10


def test_polynomial_exact_on_affine_mesh():
    """Acceptance 5: degree <= p fields exact (affine mesh, 1e-10 rel)."""
    m = toolkit.box_mesh(3, 4, 4, amp=0.0)
    S = O.OracleSetup(m.nodes, 3, 3, 4)
    x = toolkit.uniform_points(2000, 3, seed=3)
    rec = S.find(x)
    f = toolkit.analytic_field("polynomial", m, degree=4)
    v = O.evaluate(S.B, 3, f, rec["code"], rec["elem"], rec["r"])[:, 0]
    exact = sum((c + 1.0) * x[:, c] ** 4 for c in range(3)) + x[:, 0] * x[:, 1]
    np.testing.assert_allclose(v, exact, rtol=1e-10, atol=1e-12)


def test_cell_of_examples():
    """SPEC.md:227-229."""
    g = CartesianGrid(np.array([0.0, 0.0]), np.array([1.0, 2.0]), 4)
    assert cell_of(g, [0.0, 0.0]) == 0
    assert cell_of(g, [1.0, 2.0]) == 15
    assert cell_of(g, [1.0 + 1e-12, 1.0]) == -1
    assert O.cell_of(2, g.packed(), 4, np.array([1.0, 2.0])) == 15
    assert O.cell_of(2, g.packed(), 4, np.array([-1e-300, 0.5])) == -1


def test_n_cells_rule():
    """SPEC.md:262 computed in integers (float cube roots round up 27 -> 4)."""
    assert n_cells(27, 3) == 3 and n_cells(28, 3) == 4 and n_cells(32768, 3) == 32
    assert n_cells(1, 2) == 1 and n_cells(10 ** 12, 2) == 1024
    assert O.n_cells(27, 3) == 3


def test_fig8_replica_local_map():
    """one box overlapping 8 cells of a 6x6 grid appears in
    exactly those cells; single element spanning the grid -> every cell."""
    boxes = np.array([[[0.0, 0.0], [6.0, 6.0]], [[1.5, 2.5], [4.5, 3.5]]])
    grid, off, el = O.hash_build(2, boxes, 6)
    cells_of_1 = [c for c in range(36) if 1 in el[off[c]:off[c + 1]]]
    assert len(cells_of_1) == 8
    assert all(0 in el[off[c]:off[c + 1]] for c in range(36))
    assert all(np.all(np.diff(el[off[c]:off[c + 1]]) > 0) for c in range(36))


def test_hash_soundness_dense_sampling():
    """every point inside element e has e in its cell's list."""
    m = toolkit.kershaw_mesh(4, 3)
    S = O.OracleSetup(m.nodes, 3, 3, 3)
    B = S.B
    rng = np.random.default_rng(2)
    for e in rng.integers(0, m.num_elements, 12):
        for _ in range(30):
            x = O.forward_map(B, 3, 3, m.nodes[e], rng.uniform(-1, 1, 3))[0]
            c = O.cell_of(3, S.grid, S.ncell, x)
            assert e in S.elems[S.offsets[c]:S.offsets[c + 1]]


@pytest.mark.parametrize("n", [4, 6])
def test_find_all_points_in_domain(n):
    m = toolkit.kershaw_mesh(n, 4)
    S = O.OracleSetup(m.nodes, 3, 3, 4)
    rec = S.find(toolkit.uniform_points(4000, 3, seed=n))
    assert np.all(rec["code"] != 2)
    assert np.mean(rec["code"] == 0) > 0.99
    assert np.all(rec["dist"][rec["code"] == 0] < 1e-10)


def test_surface_classification_oracle():
    """Acceptance 9: on-manifold points INTERIOR, points pushed
    off the sphere along the normal BORDER under eps_d (cfg-4 style)."""
    m = toolkit.sphere_mesh(4, 4)
    S = O.OracleSetup(m.nodes, 3, 2, 4)
    x, e, r, off = toolkit.surface_points(m, 2000, seed=4, offset_frac=0.3, max_offset=1e-5)
    rec = S.find(x)
    on = off == 0
    assert np.mean(rec["code"][on] == 0) > 0.99
    assert np.all(rec["code"][~on & (np.abs(off) > 1e-8)] == 1)
    # off-surface points: d* = |offset| (closest point projection), r interior
    sel = (~on) & (rec["code"] == 1)
    np.testing.assert_allclose(rec["dist"][sel], np.abs(off[sel]), rtol=1e-3, atol=1e-9)
