import sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from torch.profiler import profile, ProfilerActivity
from paper_2501_12349_b200 import engine, toolkit
mesh = toolkit.kershaw_mesh(32, 4)
S = engine.setup(mesh)
F = engine._field_of(S, toolkit.analytic_field("smooth", mesh))
xp = torch.from_numpy(toolkit.uniform_points(1000000, 3, seed=1)).pin_memory()
o = engine.find_and_interpolate_host(S, F, xp)
for _ in range(2): engine.find_and_interpolate_host(S, F, xp, out=o)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    engine.find_and_interpolate_host(S, F, xp, out=o)
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
t0 = min(e.time_range.start for e in evs)
for e in sorted(evs, key=lambda e: e.time_range.start):
    d = e.time_range.end - e.time_range.start
    if d > 3:
        print(f"{(e.time_range.start - t0):9.1f} {d:8.1f}  {e.name[:60]}")
