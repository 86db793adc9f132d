"""Orderings of H2D and the captured device part (wall, median of 15)."""
import sys, time, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_2501_12349_b200 import engine, toolkit
mesh = toolkit.kershaw_mesh(32, 4)
S = engine.setup(mesh)
F = engine._field_of(S, toolkit.analytic_field("smooth", mesh))
xp = torch.from_numpy(toolkit.uniform_points(1000000, 3, seed=1)).pin_memory()
o = engine.find_and_interpolate_host(S, F, xp)
for _ in range(3): engine.find_and_interpolate_host(S, F, xp, out=o)
ws = S._host_pipe
g = ws["graph"]
xd2 = torch.empty_like(ws["x"])
def wall(f, k=15):
    ts = []
    for _ in range(3): f()
    for _ in range(k):
        torch.cuda.synchronize(); t = time.perf_counter(); f(); torch.cuda.synchronize()
        ts.append(1e3 * (time.perf_counter() - t))
    return np.median(ts)
def a(): ws["x"].copy_(xp, non_blocking=True); g.replay()
def b(): g.replay(); ws["x"].copy_(xp, non_blocking=True)
def c(): ws["x"].copy_(xp, non_blocking=True); torch.cuda.synchronize(); g.replay()
def d(): xd2.copy_(xp, non_blocking=True); g.replay()
def e(): ws["x"].copy_(xd2); g.replay()
def f(): g.replay()
for name, fn in (("h2d;replay", a), ("replay;h2d", b), ("h2d;sync;replay", c),
                 ("h2d(other buf);replay", d), ("d2d x;replay", e), ("replay", f)):
    print("%-24s %.3f ms" % (name, wall(fn)))
