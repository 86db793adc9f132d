import os, sys, time, torch
sys.path.insert(0, os.getcwd())
from paper_2501_12349_b200 import engine, toolkit
m = toolkit.kershaw_mesh(32, 4)
S = engine.setup(m)
F = engine._field_of(S, toolkit.analytic_field("smooth", m))
x = torch.from_numpy(toolkit.uniform_points(10 ** 6, 3, seed=1000)).pin_memory()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for ch in (1, 2, 3, 4, 6, 8, 1):
    out = None
    ts = []
    for k in range(13):
        flush.fill_(k); torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = engine.find_and_interpolate_host(S, F, x, chunks=ch, out=out)
        ts.append((time.perf_counter() - t0) * 1e3)
    ts = sorted(ts[3:])
    print("chunks", ch, "median %.3f ms" % ts[len(ts) // 2], flush=True)
