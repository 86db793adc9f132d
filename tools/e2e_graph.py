import sys, time, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_2501_12349_b200 import engine, toolkit
mesh = toolkit.kershaw_mesh(32, 4)
S = engine.setup(mesh)
F = engine._field_of(S, toolkit.analytic_field("smooth", mesh))
xp = torch.from_numpy(toolkit.uniform_points(1000000, 3, seed=1)).pin_memory()
def wall(f, k=9):
    ts = []
    for _ in range(k):
        torch.cuda.synchronize(); a = time.perf_counter(); f(); ts.append(time.perf_counter() - a)
    return 1e3 * np.median(ts)
for g in (False, True):
    S.options.graphs = g
    o = engine.find_and_interpolate_host(S, F, xp)
    o = engine.find_and_interpolate_host(S, F, xp, out=o)
    print("graphs", g, "host path wall ms", wall(lambda: engine.find_and_interpolate_host(S, F, xp, out=o)))
xd = xp.cuda()
print("device find wall", wall(lambda: (engine.find_and_interpolate(S, F, xd), torch.cuda.synchronize())))
