import sys, time, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_2501_12349_b200 import engine, toolkit
mesh = toolkit.kershaw_mesh(32, 4)
S = engine.setup(mesh)
F = toolkit.analytic_field("smooth", mesh)
Fd = engine._field_of(S, F)
x = toolkit.uniform_points(1000000, 3, seed=1)
xp = torch.from_numpy(x).pin_memory()
xd = xp.cuda()
for _ in range(3): engine.find_and_interpolate(S, Fd, xd)
torch.cuda.synchronize()
def t(f, k=5):
    ts=[]
    for _ in range(k):
        torch.cuda.synchronize(); a=time.perf_counter(); f(); torch.cuda.synchronize(); ts.append(time.perf_counter()-a)
    return 1e3*np.median(ts)
print("device api (F numpy)", t(lambda: engine.find_and_interpolate(S, F, xd)))
print("device api (F field)", t(lambda: engine.find_and_interpolate(S, Fd, xd)))
print("h2d 24MB", t(lambda: xp.cuda()))
print("_field_of(numpy)", t(lambda: engine._field_of(S, F)))
for c in (1, 4):
    print("host api chunks", c, t(lambda: engine.find_and_interpolate_host(S, Fd, xp, chunks=c)))
    print("host api (numpy F) chunks", c, t(lambda: engine.find_and_interpolate_host(S, F, xp, chunks=c)))
