"""Step timers through a replica of engine._host_overlapped (graph path)."""
import sys, time, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_2501_12349_b200 import engine, toolkit, _C
mesh = toolkit.kershaw_mesh(32, 4)
S = engine.setup(mesh)
F = engine._field_of(S, toolkit.analytic_field("smooth", mesh))
xp = torch.from_numpy(toolkit.uniform_points(1000000, 3, seed=1)).pin_memory()
o = engine.find_and_interpolate_host(S, F, xp)
for _ in range(3): engine.find_and_interpolate_host(S, F, xp, out=o)
ws = S._host_pipe
g0 = ws["graph"]
L = _C.lib()
T = {}
def tick(k, t):
    now = time.perf_counter(); T.setdefault(k, []).append(1e3 * (now - t)); return now
for it in range(20):
    torch.cuda.synchronize()
    t = t00 = time.perf_counter()
    f = engine._field_of(S, F); t = tick("field_of", t)
    x = torch.as_tensor(xp, dtype=torch.float64); pin = x.is_pinned(); t = tick("as_tensor+is_pinned", t)
    comp = torch.cuda.current_stream(S.device); t = tick("current_stream", t)
    ws["x"].copy_(x, non_blocking=True); t = tick("h2d enqueue", t)
    ws["graph"].replay(); t = tick("replay enqueue", t)
    comp.synchronize(); t = tick("sync", t)
    ph = ws["packed_host"]; cap = ph.shape[0] - 1
    c = int(ph[0, 0]); t = tick("count", t)
    L.fpx_scatter_packed_host(3, 1, ph.data_ptr(), cap, o["code"].data_ptr(), o["elem"].data_ptr(),
                              o["r"].data_ptr(), o["dist"].data_ptr(), o["values"].data_ptr())
    t = tick("scatter", t)
    tick("total", t00)
    t = time.perf_counter()
    engine.find_and_interpolate_host(S, F, xp, out=o); torch.cuda.synchronize()
    tick("engine call", t)
for k, v in T.items():
    print("%-22s median %.3f ms" % (k, np.median(v)))
print("graph recaptured:", ws["graph"] is not g0)
