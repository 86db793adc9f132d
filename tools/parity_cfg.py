"""Full-contract parity of a BASELINE config on the GPU against the oracle
(test infrastructure), on a sample of the bench's own points.

    python tools/parity_cfg.py cfg3 [--frac 0.05] [--out profiles/parity_cfg3_r2.json]

cfg3: Kershaw 64^3, p = 7 (E = 262,144, N = 8), the 10^7 uniform points of
bench.py --workload cfg3 (seed 1000); the GPU finds + interpolates all of
them, the oracle (C port, all host cores) the sample, and
tests/test_gpu_parity.check_records applies the parity contract to the
sample: codes bit-exact, elements bit-exact except on shared faces,
INTERIOR r*/d* to 1e-12, BORDER d* to 1e-12 relative and r* to 1e-12 or 8x
its conditioning bound, values to 1e-10 relative.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import bench  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2501_12349_b200 import engine  # noqa: E402
from paper_2501_12349_b200.basis import BasisConstants  # noqa: E402
from test_gpu_parity import check_records  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload", choices=sorted(bench.WORKLOADS))
    ap.add_argument("--frac", type=float, default=0.05)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    W = bench.WORKLOADS[a.workload]
    bench.W = W
    t0 = time.time()
    mesh, field, x = bench.build_inputs(0)
    S = engine.setup(torch.from_numpy(mesh.nodes).cuda(), W.order, W.dr)
    F = engine.Field(torch.from_numpy(field).cuda(), W.order)
    vals, rec = engine.find_and_interpolate(S, F, torch.from_numpy(x).cuda())
    torch.cuda.synchronize()
    t_gpu = time.time() - t0
    rng = np.random.default_rng(5)
    idx = np.sort(rng.choice(len(x), size=int(a.frac * len(x)), replace=False))
    bc = BasisConstants.of(S.basis, S.envelope)
    B = O.basis_from_arrays(bc.nodes, bc.scale, bc.proj0, bc.proj1, bc.eta, bc.lo, bc.hi)
    nth = len(os.sched_getaffinity(0))
    t1 = time.time()
    OS = O.OracleSetup(mesh.nodes, mesh.phys_dim, W.dr, W.order, B=B, ncell=S.ncell,
                       nthreads=nth)
    t_osetup = time.time() - t1
    xs = x[idx]
    t2 = time.time()
    orec = OS.find(xs)
    t_ofind = time.time() - t2
    code = rec.code.cpu().numpy()[idx]
    g = dict(code=code, elem=rec.elem.cpu().numpy()[idx], r=rec.r.cpu().numpy()[idx],
             dist=rec.dist.cpu().numpy()[idx], values=vals.cpu().numpy()[idx])
    result = "pass"
    try:
        orec2, report = check_records(OS, xs, g["code"], g["elem"], g["r"], g["dist"],
                                      g["values"], field, orec=orec)
    except AssertionError as ex:
        result = "FAIL"
        report = ex.args[0] if ex.args and isinstance(ex.args[0], dict) else {"error": str(ex)[:2000]}
        err = np.max(np.abs(g["r"] - orec["r"]), axis=1)
        bad = np.nonzero((g["code"] == orec["code"]) & (g["elem"] == orec["elem"])
                         & (err >= 1e-12))[0]
        np.savez(os.path.join(ROOT, "gpurun_out", f"parity_{a.workload}_bad.npz"), idx=idx[bad],
                 x=xs[bad], **{"g_" + k: v[bad] for k, v in g.items()},
                 **{"o_" + k: orec[k][bad] for k in ("code", "elem", "r", "dist", "iters")})
    st = rec.stats
    out = {"workload": W.config(1)["workload"], "points": len(x), "sample": len(idx),
           "sample_rule": "uniform without replacement, numpy default_rng(5)",
           "codes": {k: int((code == v).sum()) for k, v in (("INTERIOR", 0), ("BORDER", 1),
                                                              ("NOT_FOUND", 2))},
           "element_mismatch_on_shared_faces": int((rec.elem.cpu().numpy()[idx]
                                                     != orec["elem"]).sum()),
           "contract": "codes bit-exact; elements bit-exact except shared faces; INTERIOR "
                       "r*, d* <= 1e-12; BORDER d* 1e-12 rel, r* 1e-12 or 8 kappa; "
                       "values 1e-10 rel",
           "result": result, **report,
           "work_gpu_all_points": {k: int(st[k]) for k in ("box_tests", "newton", "iters")},
           "work_oracle_sample": {"box_tests": int(orec["nbox"].sum()),
                                  "newton": int(orec["ncand"].sum()),
                                  "iters": int(orec["iters"].sum())},
           "seconds": {"gpu_setup_find_eval": t_gpu, "oracle_setup": t_osetup,
                       "oracle_find_sample": t_ofind, "oracle_threads": nth}}
    print(json.dumps(out, indent=1))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
