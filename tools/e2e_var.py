"""Per-call wall times of the host-path find (e2e leg of bench.py), to see
the spread, plus a profiler timeline of one call."""
import sys, time, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from torch.profiler import profile, ProfilerActivity
from paper_2501_12349_b200 import engine, toolkit
mesh = toolkit.kershaw_mesh(32, 4)
S = engine.setup(mesh)
F = engine._field_of(S, toolkit.analytic_field("smooth", mesh))
xp = torch.from_numpy(toolkit.uniform_points(1000000, 3, seed=1)).pin_memory()
o = engine.find_and_interpolate_host(S, F, xp)
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
tsy = []
orig_sy = torch.cuda.Stream.synchronize
def sy(self):
    t = time.perf_counter(); r = orig_sy(self); tsy.append(1e3 * (time.perf_counter() - t)); return r
torch.cuda.Stream.synchronize = sy
ts = []
for k in range(30):
    flush.fill_(float(k))
    torch.cuda.synchronize()
    a = time.perf_counter()
    engine.find_and_interpolate_host(S, F, xp, out=o)
    ts.append(1e3 * (time.perf_counter() - a))
print("wall ms", " ".join("%.2f" % t for t in ts))
print("median %.2f mean %.2f min %.2f" % (np.median(ts), np.mean(ts), np.min(ts)))
print("sync ms median %.3f" % np.median(tsy))
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    engine.find_and_interpolate_host(S, F, xp, out=o)
evs = list(prof.events())
t0 = min(e.time_range.start for e in evs)
for e in sorted(evs, key=lambda e: e.time_range.start):
    d = e.time_range.end - e.time_range.start
    if d > 3:
        print(f"{e.device_type.name[:4]} {(e.time_range.start - t0):9.1f} {d:8.1f}  {e.name[:60]}")
