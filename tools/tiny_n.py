import sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from torch.profiler import profile, ProfilerActivity
from paper_2501_12349_b200 import engine, toolkit
mesh = toolkit.kershaw_mesh(32, 4)
S = engine.setup(mesh)
F = engine._field_of(S, toolkit.analytic_field("smooth", mesh))
xall = torch.from_numpy(toolkit.uniform_points(100000, 3, seed=1)).cuda()
for n in (1, 32, 256, 1000, 10000, 100000):
    x = xall[:n].contiguous()
    for _ in range(3): v, rec = engine.find_and_interpolate(S, F, x, want_iters=True)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        engine.find_and_interpolate(S, F, x); torch.cuda.synchronize()
    tot = {}
    for e in prof.events():
        if e.device_type.name == "CUDA":
            k = e.name.split("<")[0].split("(")[0].replace("void ", "").replace("fpx::", "")
            tot[k] = tot.get(k, 0) + (e.time_range.end - e.time_range.start)
    it = rec.iters.cpu().numpy()
    print(n, "maxit", it.max(), {k: round(v) for k, v in tot.items() if v > 20})
