"""Rest-phase pair outcomes by candidate rank (development build with
-DFPX_DIAG, run with FPX_DIAG_LEN=80 FPX_LIB=<diag lib>)."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_2501_12349_b200 import engine, toolkit
mesh = toolkit.kershaw_mesh(32, 4)
S = engine.setup(mesh)
F = engine._field_of(S, toolkit.analytic_field("smooth", mesh))
x = torch.from_numpy(toolkit.uniform_points(1000000, 3, seed=1)).cuda()
vals, rec = engine.find_and_interpolate(S, F, x)
torch.cuda.synchronize()
d = rec.stats._t.cpu().numpy()[16:96]
names = ["stopped(found)", "INTERIOR", "other"]
for p, pn in ((0, "pass1"), (16, "redo")):
    print(pn)
    for kind in range(3):
        cnt = d[p + kind * 5: p + kind * 5 + 5]
        its = d[32 + p + kind * 5: 32 + p + kind * 5 + 5]
        print("  %-15s count by rank 0..4+: %s   iters: %s" % (names[kind], cnt.tolist(), its.tolist()))
print("aborted(R2) pass1 count by rank:", d[64:69].tolist(), "iters:", d[69:74].tolist())
print("rest_points", rec.stats["rest_points"], "redo", rec.stats["redo"], "rest_lane_evals", rec.stats["rest_lane_evals"])
