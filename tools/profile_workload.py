"""One pass over every kernel of the hot path, for ncu (per-kernel table)
and compute-sanitizer.

    python tools/profile_workload.py [cfg2|small] [--range]

cfg2: setup of the cfg-2 mesh (Kershaw 32^3, p=4), find_and_interpolate of
10^6 points, interpolate with the records, the host-buffer path, and one
particle step.  small: the same on a 6^3 Kershaw mesh, a 2D quad mesh
(cfg-1 style) and a sphere surface with 2000 points each (sanitizers).
--range: warm everything up first and bracket one pass with
cudaProfilerStart/Stop (ncu --profile-from-start off).
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_12349_b200 import engine, particles, toolkit  # noqa: E402


def cases(kind):
    if kind == "cfg2":
        m = toolkit.kershaw_mesh(32, 4)
        yield "hex", m, toolkit.uniform_points(1_000_000, 3, seed=7)
    else:
        m = toolkit.kershaw_mesh(6, 4)
        yield "hex", m, toolkit.uniform_points(2000, 3, seed=3, lo=-0.05, hi=1.05)
        m = toolkit.box_mesh(2, 16, 3, amp=0.02)
        yield "quad", m, toolkit.uniform_points(2000, 2, seed=4, lo=-0.02, hi=1.02)
        m = toolkit.sphere_mesh(4, 4)
        yield "surface", m, toolkit.surface_points(m, 2000, seed=5)[0]


def one_pass(name, m, x):
    S = engine.setup(m)
    f = toolkit.analytic_field("smooth", m)
    xd = torch.from_numpy(x).cuda()
    vals, rec = engine.find_and_interpolate(S, f, xd)
    engine.interpolate(S, f, rec)
    engine.find_and_interpolate_host(S, f, torch.from_numpy(x), sync=True)
    if name == "hex":
        vel = np.ascontiguousarray(np.repeat(toolkit.analytic_field("smooth", m), 3, axis=1))
        particles.run_particles(S, vel, x[: min(len(x), 100_000)], steps=1,
                                box=([0.0] * 3, [1.0] * 3))
    torch.cuda.synchronize()


def main():
    kind = sys.argv[1] if len(sys.argv) > 1 else "small"
    rng = "--range" in sys.argv
    torch.cuda.set_device(0)
    data = list(cases(kind))
    if rng:
        for c in data:
            one_pass(*c)
        torch.cuda.profiler.start()
    for c in data:
        one_pass(*c)
    if rng:
        torch.cuda.profiler.stop()
    print("profile workload done:", kind)


if __name__ == "__main__":
    main()
