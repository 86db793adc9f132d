import sys, time, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_2501_12349_b200 import engine, toolkit
from paper_2501_12349_b200.invmap import NewtonSettings
from torch.profiler import profile, ProfilerActivity
mesh = toolkit.kershaw_mesh(32, 4)
x = torch.from_numpy(toolkit.uniform_points(1000000, 3, seed=1)).cuda()
for mi in (50, 20, 12, 8):
    S = engine.setup(mesh, options=engine.EngineOptions(newton=NewtonSettings(max_iters=mi), split=1))
    F = engine._field_of(S, toolkit.analytic_field("smooth", mesh))
    for n in (1000000, 500000):
        xx = x[:n].contiguous()
        for _ in range(2): engine.find_and_interpolate(S, F, xx)
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            v, rec = engine.find_and_interpolate(S, F, xx); torch.cuda.synchronize()
        tot = {}
        for e in prof.events():
            if e.device_type.name == "CUDA":
                k = e.name.split("<")[0].split("(")[0].replace("void ", "")
                tot[k] = tot.get(k, 0) + (e.time_range.end - e.time_range.start)
        st = rec.stats
        print(mi, n, {k: round(v) for k, v in tot.items() if v > 30}, "iters", st["iters"], "rest", st["rest_points"])
