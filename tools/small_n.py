import sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from torch.profiler import profile, ProfilerActivity
from paper_2501_12349_b200 import engine, toolkit
mesh = toolkit.kershaw_mesh(32, 4)
S = engine.setup(mesh)
F = engine._field_of(S, toolkit.analytic_field("smooth", mesh))
x = torch.from_numpy(toolkit.uniform_points(1000, 3, seed=1)).cuda()
for _ in range(3): v, rec = engine.find_and_interpolate(S, F, x, want_iters=True)
torch.cuda.synchronize()
it = rec.iters.cpu().numpy(); print("iters max", it.max(), "mean", it.mean(), "rest", rec.stats["rest_points"])
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    engine.find_and_interpolate(S, F, x); torch.cuda.synchronize()
evs = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
for e in evs:
    print(f"{e.time_range.start - t0:9.1f} {e.time_range.end - e.time_range.start:8.1f}  {e.name[:70]}")
