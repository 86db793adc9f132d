import sys, time, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_2501_12349_b200 import engine, toolkit
mesh = toolkit.kershaw_mesh(32, 4)
S = engine.setup(mesh)
F = engine._field_of(S, toolkit.analytic_field("smooth", mesh))
x = torch.from_numpy(toolkit.uniform_points(1000000, 3, seed=1)).cuda()
S.options.split = 1
def t(f, k=5):
    ts = []
    for _ in range(k):
        torch.cuda.synchronize(); a = time.perf_counter(); f(); torch.cuda.synchronize(); ts.append(time.perf_counter() - a)
    return 1e3 * np.median(ts)
for _ in range(2): engine.find_and_interpolate(S, F, x)
print("1M one call", t(lambda: engine.find_and_interpolate(S, F, x)))
h = x[:500000].contiguous(); h2 = x[500000:].contiguous()
print("500K one call", t(lambda: engine.find_and_interpolate(S, F, h)))
print("2x500K same stream", t(lambda: (engine.find_and_interpolate(S, F, h), engine.find_and_interpolate(S, F, h2))))
print("250K one call", t(lambda: engine.find_and_interpolate(S, F, x[:250000].contiguous())))
print("100K one call", t(lambda: engine.find_and_interpolate(S, F, x[:100000].contiguous())))
S.options.split = 2
print("1M split2", t(lambda: engine.find_and_interpolate(S, F, x)))
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    engine.find_and_interpolate(S, F, x); torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
t0 = min(e.time_range.start for e in evs)
for e in sorted(evs, key=lambda e: e.time_range.start):
    print(f"{(e.time_range.start - t0):9.1f} {(e.time_range.end - e.time_range.start):8.1f}  {e.name[:70]}")
