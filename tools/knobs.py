"""cfg-2 device step time under EngineOptions variants (performance knobs
whose results do not depend on them, e.g. hash_refine).

    python tools/knobs.py hash_refine=2,3,4,5
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_12349_b200 import engine, toolkit  # noqa: E402


def main():
    key, vals = sys.argv[1].split("=")
    mesh = toolkit.kershaw_mesh(32, 4)
    field = toolkit.analytic_field("smooth", mesh)
    x = torch.from_numpy(toolkit.uniform_points(10 ** 6, 3, seed=1000)).cuda()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    for v in vals.split(","):
        opt = engine.EngineOptions(**{key: type(getattr(engine.EngineOptions(), key))(v)})
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        S = engine.setup(mesh, options=opt)
        torch.cuda.synchronize()
        setup_ms = (time.perf_counter() - t0) * 1e3
        F = engine._field_of(S, field)
        for _ in range(3):
            engine.find_and_interpolate(S, F, x)
        ts = []
        for k in range(8):
            flush.fill_(k)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            _, rec = engine.find_and_interpolate(S, F, x)
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b))
        st = rec.stats
        print(json.dumps({key: v, "step_ms": sorted(ts)[len(ts) // 2], "setup_ms": setup_ms,
                          "ncell": S.ncell, "csr": int(S.elems.numel()),
                          "box_tests_per_pt": st["box_tests"] / 1e6,
                          "rest_points": st["rest_points"]}), flush=True)


if __name__ == "__main__":
    main()
