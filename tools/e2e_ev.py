"""Host-path find: wall time vs device span (CUDA events around the call on
the current stream), graphs on/off."""
import sys, time, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_2501_12349_b200 import engine, toolkit
mesh = toolkit.kershaw_mesh(32, 4)
S = engine.setup(mesh)
F = engine._field_of(S, toolkit.analytic_field("smooth", mesh))
xp = torch.from_numpy(toolkit.uniform_points(1000000, 3, seed=1)).pin_memory()
o = engine.find_and_interpolate_host(S, F, xp)
for g in (True, False, True):
    S.options.graphs = g
    for _ in range(3): engine.find_and_interpolate_host(S, F, xp, out=o)
    wall, dev = [], []
    for k in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t = time.perf_counter()
        a.record()
        engine.find_and_interpolate_host(S, F, xp, out=o)
        b.record()
        b.synchronize()
        wall.append(1e3 * (time.perf_counter() - t))
        dev.append(a.elapsed_time(b))
    print("graphs", g, "wall median %.2f  device span median %.2f" % (np.median(wall), np.median(dev)))
xd = xp.cuda()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(3): engine.find_and_interpolate(S, F, xd)
a.record()
for _ in range(10): engine.find_and_interpolate(S, F, xd)
b.record(); b.synchronize()
print("device find ms %.2f" % (a.elapsed_time(b) / 10))
