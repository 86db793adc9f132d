import os, sys, time, torch
sys.path.insert(0, os.getcwd())
from paper_2501_12349_b200 import engine, toolkit
m = toolkit.kershaw_mesh(32, 4)
S = engine.setup(m)
F = engine._field_of(S, toolkit.analytic_field("smooth", m))
for n in (1000, 10000):
    x = torch.from_numpy(toolkit.uniform_points(n, 3, seed=1000)).cuda()
    for _ in range(5):
        engine.find_and_interpolate(S, F, x)
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter(); a.record()
        engine.find_and_interpolate(S, F, x)
        b.record(); t1 = time.perf_counter(); b.synchronize()
        ts.append((a.elapsed_time(b), (t1 - t0) * 1e3))
    ts.sort()
    print(n, "gpu %.3f ms, host enqueue %.3f ms" % ts[len(ts) // 2], flush=True)
