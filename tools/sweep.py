"""SPEC.md "bench" sweep (§8 f4) on one GPU -> one JSON line:
  * find-phase time for N_pt = 10^3 .. 10^6 on the fixed cfg-2 mesh and the
    ratio between decades (acceptance 10: within [5, 13]; O(N_pt));
  * spiral p=9 Newton efficiency (acceptance 6);
  * particle-step time (Algorithm 1, cfg-5 scaled to one GPU:
    p=5 box mesh, 10^6 particles);
  * with --cfg5: cfg-5 on one GPU at its full particle count (10^7 particles,
    100 steps, Taylor-Green flow in a p=5 box mesh 32^3).
    python tools/sweep.py [--cfg5]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_12349_b200 import engine, invmap, particles, toolkit  # noqa: E402


def dev_ms(fn, steps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / steps


def main():
    out = {}
    mesh = toolkit.kershaw_mesh(32, 4)
    S = engine.setup(mesh)
    F = engine._field_of(S, toolkit.analytic_field("smooth", mesh))
    xs = torch.from_numpy(toolkit.uniform_points(10 ** 6, 3, seed=1)).cuda()
    sweep = {}
    for e in (3, 4, 5, 6):
        x = xs[:10 ** e].contiguous()
        sweep[10 ** e] = dev_ms(lambda: engine.find_and_interpolate(S, F, x))
    ks = sorted(sweep)
    out["find_ms"] = sweep
    out["decade_ratios"] = [sweep[ks[i + 1]] / sweep[ks[i]] for i in range(len(ks) - 1)]
    # spiral p=9 (one 2D element)
    sp = toolkit.spiral_mesh(9)
    Ss = engine.setup(sp)
    rng = np.random.default_rng(6)
    rh = rng.uniform(-0.98, 0.98, (100000, 2))
    # map reference samples with the device forward map
    elem = torch.zeros(rh.shape[0], dtype=torch.int32, device="cuda")
    from paper_2501_12349_b200 import _C
    xd = torch.empty((rh.shape[0], 2), dtype=torch.float64, device="cuda")
    G = torch.empty((rh.shape[0], 2, 2), dtype=torch.float64, device="cuda")
    rd = torch.from_numpy(rh).cuda()
    _C.check(_C.lib().fpx_forward_map(Ss.mesh_t, rh.shape[0], _C.ptr(elem), _C.ptr(rd), _C.ptr(xd),
                                      _C.ptr(G), None, _C.stream_handle()), "fpx_forward_map")
    r, dist, it, cv = invmap.invert_points(Ss, xd, elem)
    itn = it.cpu().numpy()
    out["spiral_p9"] = {"points": int(rh.shape[0]), "mean_iters": float(itn.mean()),
                        "max_iters": int(itn.max()), "converged": float(cv.float().mean()),
                        "max_r_err": float((r - rd).abs().max()),
                        "invert_ms": dev_ms(lambda: invmap.invert_points(Ss, xd, elem))}
    # particles: cfg-5 scaled to one GPU
    pm = toolkit.box_mesh(3, 24, 5)
    Sp = engine.setup(pm)
    vel = engine._field_of(Sp, toolkit.analytic_field("taylor_green", pm))
    x0 = toolkit.uniform_points(10 ** 6, 3, seed=2, lo=0.01, hi=0.99)
    st = particles.init_particles(Sp, x0, tau=5.0)
    for _ in range(3):
        particles.advance(Sp, vel, st, 1e-3, box=((0, 0, 0), (1, 1, 1)))
    st.timings = {}
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    steps = 10
    for _ in range(steps):
        particles.advance(Sp, vel, st, 1e-3, box=((0, 0, 0), (1, 1, 1)))
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / steps * 1e3
    out["particles"] = {"mesh": "box 24^3 p=5", "particles": len(st), "removed": st.removed,
                        "step_ms_wall": wall,
                        "phase_ms_per_step": {k: v / steps for k, v in st.timings.items()},
                        "particle_steps_per_s": len(st) / (wall * 1e-3)}
    if "--cfg5" in sys.argv:
        out["cfg5_one_gpu"] = cfg5()
    print(json.dumps(out))


def cfg5(n=10 ** 7, steps=100, ne=32):
    """BASELINE.json configs[4] on one GPU: 10^7 particles, 100 steps."""
    pm = toolkit.box_mesh(3, ne, 5)
    Sp = engine.setup(pm)
    vel = engine._field_of(Sp, toolkit.analytic_field("taylor_green", pm))
    x0 = toolkit.uniform_points(n, 3, seed=5, lo=0.01, hi=0.99)
    st = particles.init_particles(Sp, x0, tau=5.0)
    for _ in range(2):
        particles.advance(Sp, vel, st, 1e-3, box=((0, 0, 0), (1, 1, 1)))
    st.timings = {}
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        particles.advance(Sp, vel, st, 1e-3, box=((0, 0, 0), (1, 1, 1)))
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    return {"mesh": f"box {ne}^3 p=5 (Taylor-Green)", "particles": len(st),
            "removed": st.removed, "steps": steps, "wall_s": wall,
            "step_ms_wall": wall / steps * 1e3,
            "phase_ms_per_step": {k: v / steps for k, v in st.timings.items()},
            "particle_steps_per_s": len(st) * steps / wall}


if __name__ == "__main__":
    main()
