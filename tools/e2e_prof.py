"""cProfile of the host-path find: where the host time beyond the device
span goes."""
import sys, os, cProfile, pstats
sys.path.insert(0, os.getcwd())
import torch
from paper_2501_12349_b200 import engine, toolkit
mesh = toolkit.kershaw_mesh(32, 4)
S = engine.setup(mesh)
F = engine._field_of(S, toolkit.analytic_field("smooth", mesh))
xp = torch.from_numpy(toolkit.uniform_points(1000000, 3, seed=1)).pin_memory()
o = engine.find_and_interpolate_host(S, F, xp)
for _ in range(3): engine.find_and_interpolate_host(S, F, xp, out=o)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(20): engine.find_and_interpolate_host(S, F, xp, out=o)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
