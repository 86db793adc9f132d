"""Ad-hoc GPU bring-up check: kernels vs the oracle on small meshes.

    python tools/gpu_smoke.py
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as O  # noqa: E402
from paper_2501_12349_b200 import engine, toolkit  # noqa: E402
from paper_2501_12349_b200.basis import BasisConstants  # noqa: E402


def oracle_setup_like(S, m):
    bc = BasisConstants.of(S.basis, S.envelope)
    B = O.basis_from_arrays(bc.nodes, bc.scale, bc.proj0, bc.proj1, bc.eta, bc.lo, bc.hi)
    return O.OracleSetup(m.nodes, m.phys_dim, m.ref_dim, m.order, B=B, ncell=S.ncell)


def compare(name, m, npts, seed=1, lo=0.0, hi=1.0):
    t = time.time()
    S = engine.setup(m)
    torch.cuda.synchronize()
    ts = time.time() - t
    OS = oracle_setup_like(S, m)
    # setup parity
    for k in ("aabb", "obb_c", "obb_inv", "hbox"):
        a = getattr(S, k).cpu().numpy()
        b = OS.boxes[k]
        ok = OS.boxes["obb_ok"].astype(bool)
        if k in ("obb_c", "obb_inv"):
            a, b = a[ok], b[ok]
        print(f"  {k}: bit-mismatch {np.sum(a != b)} / {a.size}  maxdiff {np.max(np.abs(a - b)):.2e}")
    print("  hash entries", S.elems.numel(), OS.elems.size, "offsets equal",
          np.array_equal(S.offsets.cpu().numpy(), OS.offsets),
          "elems equal", np.array_equal(S.elems.cpu().numpy(), OS.elems))
    x = toolkit.uniform_points(npts, m.phys_dim, seed=seed, lo=lo, hi=hi)
    f = toolkit.analytic_field("smooth" if m.phys_dim == 3 else "coordinates", m)
    vals, rec = engine.find_and_interpolate(S, f, x, want_iters=True)
    torch.cuda.synchronize()
    t = time.time()
    vals, rec = engine.find_and_interpolate(S, f, x, want_iters=True)
    torch.cuda.synchronize()
    tg = time.time() - t
    orec = OS.find(x)
    ov = O.evaluate(OS.B, m.ref_dim, f, orec["code"], orec["elem"], orec["r"])
    code = rec.code.cpu().numpy()
    elem = rec.elem.cpu().numpy()
    r = rec.r.cpu().numpy()
    dist = rec.dist.cpu().numpy()
    v = vals.cpu().numpy()
    cm = code != orec["code"]
    em = (elem != orec["elem"]) & ~cm
    print(f"{name}: setup {ts*1e3:.1f} ms, find+eval {tg*1e3:.2f} ms ({npts/tg:.3e} pts/s)")
    print("  codes gpu", np.bincount(code, minlength=3), "oracle", np.bincount(orec["code"], minlength=3))
    print("  code mismatches", cm.sum(), " elem mismatches", em.sum())
    both = (code == 0) & (orec["code"] == 0) & ~em
    if both.any():
        print("  interior max |dr|", np.max(np.abs(r[both] - orec["r"][both])),
              " max |dval| rel", np.max(np.abs(v[both] - ov[both]) / np.maximum(1, np.abs(ov[both]))))
    bb = (code == 1) & (orec["code"] == 1) & ~em
    if bb.any():
        print("  border max |ddist|", np.max(np.abs(dist[bb] - orec["dist"][bb])),
              " max |dr|", np.max(np.abs(r[bb] - orec["r"][bb])))
    print("  stats", rec.stats)
    idx = np.nonzero(cm | em)[0][:5]
    for i in idx:
        print("   mismatch", i, x[i], "gpu", code[i], elem[i], r[i], dist[i], "| oracle",
              orec["code"][i], orec["elem"][i], orec["r"][i], orec["dist"][i])


if __name__ == "__main__":
    compare("box2d 16x16 p3", toolkit.box_mesh(2, 16, 3), 10000)
    compare("kershaw 8^3 p4", toolkit.kershaw_mesh(8, 4), 20000)
    compare("kershaw 8^3 p4 outside", toolkit.kershaw_mesh(8, 4), 20000, seed=3, lo=-0.1, hi=1.1)
    compare("kershaw 16^3 p4", toolkit.kershaw_mesh(16, 4), 100000)
    m = toolkit.kershaw_mesh(32, 4)
    S = engine.setup(m)
    f = toolkit.analytic_field("smooth", m)
    x = torch.from_numpy(toolkit.uniform_points(1_000_000, 3, seed=7)).cuda()
    fb = torch.from_numpy(f).cuda()
    for it in range(5):
        torch.cuda.synchronize()
        t = time.time()
        vals, rec = engine.find_and_interpolate(S, fb, x)
        torch.cuda.synchronize()
        dt = time.time() - t
        print(f"cfg2 32^3 p4 1M: {dt*1e3:.2f} ms  {1e6/dt:.3e} pts/s", rec.stats if it == 0 else "")
