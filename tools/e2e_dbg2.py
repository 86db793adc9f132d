import sys, time, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_2501_12349_b200 import engine, toolkit
mesh = toolkit.kershaw_mesh(32, 4)
S = engine.setup(mesh)
F = engine._field_of(S, toolkit.analytic_field("smooth", mesh))
xp = torch.from_numpy(toolkit.uniform_points(1000000, 3, seed=1)).pin_memory()
xd = xp.cuda()
o = engine.find_and_interpolate_host(S, F, xp)
def wall(f, k=7):
    ts = []
    for _ in range(k):
        torch.cuda.synchronize(); a = time.perf_counter(); f(); torch.cuda.synchronize(); ts.append(time.perf_counter() - a)
    return 1e3 * np.median(ts)
ws = S._host_pipe
print("is_pinned", wall(lambda: xp.is_pinned()))
print("h2d into ws", wall(lambda: ws["x"].copy_(xp, non_blocking=True)))
print("h2d fresh", wall(lambda: xp.to("cuda", non_blocking=True)))
loc = dict(code=ws["code"], elem=ws["elem"], r=ws["r"], dist=ws["dist"], iters=None, values=ws["values"])
print("find_into ws", wall(lambda: engine._find_into(S, ws["x"], loc, F)))
print("find_into on xd", wall(lambda: engine._find_into(S, xd, loc, F)))
print("find device api", wall(lambda: engine.find_and_interpolate(S, F, xd)))
print("d2h", wall(lambda: [o[k].copy_(ws[k], non_blocking=True) for k in ("values", "code", "rank", "elem", "r", "dist")]))
print("graph replay", wall(lambda: ws["graph"].replay()) if "graph" in ws else "no graph")
