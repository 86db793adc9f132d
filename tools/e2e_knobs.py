"""cfg-2 end-to-end wall time (engine.find_and_interpolate_host) under the
host-path pipeline constants (upload chunks, early download pieces)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_12349_b200 import engine, toolkit  # noqa: E402


def main():
    mesh = toolkit.kershaw_mesh(32, 4)
    S = engine.setup(mesh)
    F = engine._field_of(S, toolkit.analytic_field("smooth", mesh))
    x = torch.from_numpy(toolkit.uniform_points(10 ** 6, 3, seed=1000)).pin_memory()
    n = x.shape[0]
    pin = dict(pin_memory=True)
    out = dict(values=torch.empty((n, 1), dtype=torch.float64, **pin),
               code=torch.empty(n, dtype=torch.int32, **pin),
               rank=torch.empty(n, dtype=torch.int32, **pin),
               elem=torch.empty(n, dtype=torch.int32, **pin),
               r=torch.empty((n, 3), dtype=torch.float64, **pin),
               dist=torch.empty(n, dtype=torch.float64, **pin))
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    for up, pieces, early in ((2, 4, 1), (3, 4, 1), (4, 4, 1), (2, 4, 1)):
        if True:
            engine._UPLOAD_CHUNKS, engine._EARLY_PIECES = up, early
            engine._DOWNLOAD_PIECES = pieces
            ts = []
            for k in range(13):
                flush.fill_(k)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                engine.find_and_interpolate_host(S, F, x, out=out, sync=True)
                ts.append((time.perf_counter() - t0) * 1e3)
            ts = sorted(ts[3:])
            print(f"upload_chunks {up} pieces {pieces} early {early}: median {ts[len(ts) // 2]:.3f} ms "
                  f"min {ts[0]:.3f}", flush=True)


if __name__ == "__main__":
    main()
