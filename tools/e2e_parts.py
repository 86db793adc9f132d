"""Wall time of the pieces of the host-path find (H2D alone, D2H alone,
graph replay alone, whole call; default vs side stream)."""
import sys, time, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_2501_12349_b200 import engine, toolkit
mesh = toolkit.kershaw_mesh(32, 4)
S = engine.setup(mesh)
F = engine._field_of(S, toolkit.analytic_field("smooth", mesh))
xp = torch.from_numpy(toolkit.uniform_points(1000000, 3, seed=1)).pin_memory()
o = engine.find_and_interpolate_host(S, F, xp)
ws = S._host_pipe
def wall(f, k=15):
    ts = []
    for _ in range(3): f()
    for _ in range(k):
        torch.cuda.synchronize(); t = time.perf_counter(); f(); torch.cuda.synchronize()
        ts.append(1e3 * (time.perf_counter() - t))
    return np.median(ts)
print("H2D x        %.3f ms" % wall(lambda: ws["x"].copy_(xp, non_blocking=True)))
def d2h():
    for k in ("values", "code", "elem", "r", "dist"):
        o[k].copy_(ws[k], non_blocking=True)
print("D2H records  %.3f ms" % wall(d2h))
print("graph replay %.3f ms" % wall(lambda: ws["graph"].replay()))
print("whole call   %.3f ms" % wall(lambda: engine.find_and_interpolate_host(S, F, xp, out=o)))
s2 = torch.cuda.Stream()
with torch.cuda.stream(s2):
    o2 = engine.find_and_interpolate_host(S, F, xp)
    print("whole call on a side stream %.3f ms" % wall(lambda: engine.find_and_interpolate_host(S, F, xp, out=o2)))
xd = xp.cuda()
print("device find  %.3f ms" % wall(lambda: engine.find_and_interpolate(S, F, xd)))
