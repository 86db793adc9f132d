import sys, time, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_2501_12349_b200 import engine, toolkit
mesh = toolkit.kershaw_mesh(32, 4)
S = engine.setup(mesh)
F = engine._field_of(S, toolkit.analytic_field("smooth", mesh))
x = toolkit.uniform_points(1000000, 3, seed=1)
xp = torch.from_numpy(x).pin_memory()
xd = xp.cuda()
for _ in range(3): engine.find_and_interpolate(S, F, xd)
out = None
def wall(f, k=7):
    ts = []
    for _ in range(k):
        torch.cuda.synchronize(); a = time.perf_counter(); f(); torch.cuda.synchronize(); ts.append(time.perf_counter() - a)
    return 1e3 * np.median(ts)
def ev(f, k=7):
    ts = []
    for _ in range(k):
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); s0.record(); f(); s1.record(); s1.synchronize(); ts.append(s0.elapsed_time(s1))
    return np.median(ts)
o = engine.find_and_interpolate_host(S, F, xp)
print("device find wall", wall(lambda: engine.find_and_interpolate(S, F, xd)), "events", ev(lambda: engine.find_and_interpolate(S, F, xd)))
print("host overlapped wall", wall(lambda: engine.find_and_interpolate_host(S, F, xp, out=o)), "events", ev(lambda: engine.find_and_interpolate_host(S, F, xp, out=o)))
from paper_2501_12349_b200 import engine as E
def plain():
    vals, rec = E.find_and_interpolate(S, F, xp)
    o["values"].copy_(vals, non_blocking=True)
    for k in ("code", "elem", "rank", "r", "dist"):
        o[k].copy_(getattr(rec, k), non_blocking=True)
    torch.cuda.current_stream().synchronize()
print("plain h2d+find+d2h wall", wall(plain), "events", ev(plain))
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(5): engine.find_and_interpolate_host(S, F, xp, out=o)
pr.disable(); pstats.Stats(pr).sort_stats("cumulative").print_stats(12)
S.options.graphs = False
print("host plain-path wall", wall(lambda: engine.find_and_interpolate_host(S, F, xp, out=o)))
S.options.graphs = True
print("host graph wall", wall(lambda: engine.find_and_interpolate_host(S, F, xp, out=o)))
