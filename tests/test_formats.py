"""File formats (SPEC.md DESIGN DECISIONS) and the setup cache."""
import numpy as np
import pytest
import torch

from paper_2501_12349_b200 import toolkit


@pytest.mark.parametrize("binary", [False, True])
def test_mesh_roundtrip_bitexact(tmp_path, binary):
    mesh = toolkit.kershaw_mesh(3, 3)
    p = str(tmp_path / ("m.bin" if binary else "m.txt"))
    toolkit.write_mesh(p, mesh, binary=binary)
    back = toolkit.read_mesh(p)
    assert (back.phys_dim, back.ref_dim, back.order) == (3, 3, 3)
    assert np.array_equal(back.nodes, mesh.nodes)   # repr / raw f64: bit-exact


def test_mesh_text_header(tmp_path):
    mesh = toolkit.box_mesh(2, 2, 1)
    p = str(tmp_path / "m.txt")
    toolkit.write_mesh(p, mesh)
    first = open(p).readline().strip()
    assert first == "fpx-mesh v1; 2; 2; 1; 4"
    assert sum(1 for _ in open(p)) == 1 + 4 * 4


def test_points_and_records_roundtrip(tmp_path):
    from paper_2501_12349_b200.engine import FindRecords
    x = toolkit.uniform_points(50, 3, seed=2)
    toolkit.write_points(str(tmp_path / "p.csv"), x)
    assert np.array_equal(toolkit.read_points(str(tmp_path / "p.csv")), x)
    rng = np.random.default_rng(0)
    rec = FindRecords(torch.from_numpy(rng.integers(0, 3, 50, dtype=np.int32)),
                      torch.zeros(50, dtype=torch.int32),
                      torch.from_numpy(rng.integers(0, 99, 50, dtype=np.int32)),
                      torch.from_numpy(rng.uniform(-1, 1, (50, 3))),
                      torch.from_numpy(rng.uniform(0, 1, 50)))
    toolkit.write_records(str(tmp_path / "r.csv"), rec)
    back = toolkit.read_records(str(tmp_path / "r.csv"))
    assert np.array_equal(back["code"], rec.code.numpy())
    assert np.array_equal(back["r"], rec.r.numpy())
    assert np.array_equal(back["dist"], rec.dist.numpy())


@pytest.mark.gpu
def test_setup_cache_reuse_equals_recompute(tmp_path):
    # SPEC.md:426 reuse = recompute, through a save/load of the setup
    from paper_2501_12349_b200 import engine
    mesh = toolkit.kershaw_mesh(6, 4)
    S = engine.setup(mesh)
    p = str(tmp_path / "setup.npz")
    engine.save_setup(S, p)
    S2 = engine.load_setup(p)
    field = toolkit.analytic_field("smooth", mesh)
    x = toolkit.uniform_points(5000, 3, seed=8, lo=-0.05, hi=1.05)
    v1, r1 = engine.find_and_interpolate(S, field, x)
    v2, r2 = engine.find_and_interpolate(S2, field, x)
    assert torch.equal(r1.code, r2.code) and torch.equal(r1.elem, r2.elem)
    nn = torch.nan_to_num   # NOT_FOUND records carry NaN r / dist
    assert torch.equal(nn(r1.r), nn(r2.r)) and torch.equal(nn(r1.dist), nn(r2.dist))
    assert torch.equal(torch.nan_to_num(v1), torch.nan_to_num(v2))
