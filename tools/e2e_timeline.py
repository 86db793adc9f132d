"""Device timeline of the overlapped host path at cfg-2 (graphs off, timing
events in place of the pipeline's own), plus the bare PCIe copy rates."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_12349_b200 import engine, toolkit  # noqa: E402


def main():
    mesh = toolkit.kershaw_mesh(32, 4)
    S = engine.setup(mesh)
    F = engine._field_of(S, toolkit.analytic_field("smooth", mesh))
    x = torch.from_numpy(toolkit.uniform_points(10 ** 6, 3, seed=1000)).pin_memory()
    n = x.shape[0]
    # bare copy rates
    d = torch.empty(n * 3, dtype=torch.float64, device="cuda")
    big = torch.empty(52 * 10 ** 6 // 8, dtype=torch.float64, device="cuda")
    hb = torch.empty_like(big, device="cpu").pin_memory()
    for name, fn, nbytes in (("H2D 24 MB", lambda: d.copy_(x.view(-1), non_blocking=True), 24e6),
                             ("D2H 52 MB", lambda: hb.copy_(big, non_blocking=True), 52e6)):
        ts = []
        for _ in range(6):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); fn(); b.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        t = sorted(ts)[len(ts) // 2]
        print(f"{name}: {t:.3f} ms = {nbytes / t / 1e6:.1f} GB/s")
    engine.find_and_interpolate_host(S, F, x)  # buffers
    ws = S.__dict__["_host_pipe"]
    comp = torch.cuda.current_stream()
    mk = lambda m: [torch.cuda.Event(enable_timing=True) for _ in range(m)]  # noqa: E731
    evs = {"r1": mk(1), "start": mk(1), "up": mk(engine._UPLOAD_CHUNKS),
           "dn": mk(engine._DOWNLOAD_PIECES), "rank": mk(1), "done": mk(1)}
    for lst in evs.values():
        for e in lst:
            e.record(comp)
    torch.cuda.synchronize()
    ws["events"] = evs
    S.options.graphs = False
    for it in range(4):
        end = torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        out = engine.find_and_interpolate_host(S, F, x, out=None if it == 0 else out)
        end.record(comp)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
        s = evs["start"][0]
        row = [f"up{c}={s.elapsed_time(e):.3f}" for c, e in enumerate(evs["up"])]
        row.append(f"r1={s.elapsed_time(evs['r1'][0]):.3f}")
        row += [f"dn{j}={s.elapsed_time(e):.3f}" for j, e in enumerate(evs["dn"][:engine._EARLY_PIECES])]
        row.append(f"rank={s.elapsed_time(evs['rank'][0]):.3f}")
        row.append(f"done={s.elapsed_time(evs['done'][0]):.3f}")
        row.append(f"end={s.elapsed_time(end):.3f}")
        print(f"wall {wall:.3f} ms | " + " ".join(row), flush=True)


if __name__ == "__main__":
    main()
