"""findpts+eval throughput benchmark (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1]): 3D Kershaw-deformed
hex mesh 32^3 elements, p=4 (eps_y = eps_z = 0.3), field sin(pi x)cos(pi y)e^z,
10^6 uniform random query points per GPU in [0,1]^3, find + interpolate.
A step = engine.find_and_interpolate over the 10^6 points of this rank.
For N > 1 (torchrun) the mesh is block-partitioned into z-slabs and every
rank issues its own 10^6 points (weak scaling): (N-1)/N of them are routed
to other ranks with NCCL all-to-alls.

JSON line (rank 0): value = total points / max-over-ranks device step time
(inputs resident in HBM; L2 flushed between timed steps); e2e = the same
through the public API with host points copied in and values + records
copied out inside the timed region; roofline of the dominant kernel
(k_newton_stream, FP64-bound); cpu_baseline = the oracle port on the host
cores over a bounded sample.
--impl reference: the reference's CPU path (the C oracle port; the reference
package itself has no find/eval code) on all host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_ELEM_AXIS = 32
ORDER = 4
PTS_PER_GPU = 1_000_000
METRIC = "findpts+eval points/sec (3D hex, p=4, 1M pts/GPU) at 1/2/4/8 B200"
UNIT = "points/s"

# Algorithmic FP64 work per unit (frozen; N = p+1, d = dr = 3).
def f_iter(N):   # one Newton iteration: 3 basis evals + x,G contraction + 3x3 solve
    return 3 * 13 * N + 2 * 3 * (2 * N ** 3 + 3 * N ** 2 + 4 * N) + 130


def f_seed(N):   # nearest-node seed over N^3 nodes
    return 8 * N ** 3


def f_eval(N, C=1):
    return 3 * 8 * N + 2 * C * (N ** 3 + N ** 2 + N)


F_SEED_AFFINE = 2 * 3 * 3 + 3   # D7' seed: J_c^-1 (x* - x_c) (3x3 mat-vec + 3 subtractions)


def round1_flops(st, N):
    """Algorithmic FP64 work of the round-1 kernel: every lane evaluation of
    the map (basis, x + G contraction, step algebra = F_iter), the affine
    seed of every solve, the fused field evaluation of every final point."""
    return st["r1_lane_evals"] * f_iter(N) + st["newton_r1"] * F_SEED_AFFINE \
        + st["evals_r1"] * f_eval(N)


def step_flops(st, N):
    """Whole find+eval step: round 1, the rest kernels' lane evaluations
    (each rest solve counted with a nearest-node seed, 8 N^3: an upper bound,
    pass-1 solves seed from the frame), 30 flops per box test, and the field
    evaluation of every found point."""
    rest_solves = st["newton"] - st["newton_r1"]
    return round1_flops(st, N) + st["rest_lane_evals"] * f_iter(N) \
        + rest_solves * f_seed(N) + 30 * st["box_tests"] \
        + (st["evals"] - st["evals_r1"]) * f_eval(N)


def workload_config(n_gpus):
    return {"workload": f"cfg-2: Kershaw hex {N_ELEM_AXIS}^3 p={ORDER}, "
                        f"{PTS_PER_GPU} uniform pts/GPU, find+eval (C=1)",
            "mesh": f"kershaw{N_ELEM_AXIS}^3", "order": ORDER, "elements": N_ELEM_AXIS ** 3,
            "points_per_gpu": PTS_PER_GPU, "components": 1,
            "partition": "contiguous z-slabs" if n_gpus > 1 else "single",
            "l2": "flushed (256 MiB write) between timed steps"}


def build_inputs(rank=0):
    from paper_2501_12349_b200 import toolkit
    mesh = toolkit.kershaw_mesh(N_ELEM_AXIS, ORDER)
    field = toolkit.analytic_field("smooth", mesh)
    x = toolkit.uniform_points(PTS_PER_GPU, 3, seed=1000 + rank)
    return mesh, field, x


# ----------------------------------------------------------------- CPU arm
def cpu_find_eval(sample=20000, threads=None, steps=1, warmup=0, rank=0):
    """The oracle port (oracle/fpx_oracle.c, OpenMP) on the host cores."""
    from oracle import oracle as O
    mesh, field, x = build_inputs(rank)
    nthreads = threads or len(os.sched_getaffinity(0))
    # the same local grid as engine.setup's default (hash_refine x SPEC rule)
    from paper_2501_12349_b200.engine import EngineOptions
    ncell = min(1024, EngineOptions().hash_refine * O.n_cells(mesh.num_elements, 3))
    OS = O.OracleSetup(mesh.nodes, 3, 3, ORDER, nthreads=nthreads, ncell=ncell)
    xs = x[:sample]
    times = []
    for k in range(warmup + steps):
        t = time.perf_counter()
        rec = OS.find(xs, nthreads=nthreads)
        O.evaluate(OS.B, 3, field, rec["code"], rec["elem"], rec["r"], nthreads=nthreads)
        if k >= warmup:
            times.append(time.perf_counter() - t)
    work = {"points": int(sample), "box_tests": int(rec["nbox"].sum()),
            "newton": int(rec["ncand"].sum()), "iters": int(rec["iters"].sum())}
    return sample / float(np.mean(times)), nthreads, float(np.mean(times)), work


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    sample = args.cpu_sample
    v, cores, t, _ = cpu_find_eval(sample=sample, steps=args.steps, warmup=args.warmup)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args.gpus),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"{sample} of the {PTS_PER_GPU} cfg-2 points per step "
                                       "(oracle C port, OpenMP over points, setup excluded)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU arm
class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region: the
    query loop runs every 10 ms, is live before the region starts (the
    first row is awaited and dropped), and only rows stamped inside the
    region are kept."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu = gpu
        self.p = None
        self.rows = []
        self.t0 = self.t1 = 0.0

    def _read(self):
        for line in self.p.stdout:
            self.rows.append((time.perf_counter(), line))

    def __enter__(self):
        import threading
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "10"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
            t = time.perf_counter()
            while not self.rows and time.perf_counter() - t < 10.0 and self.p.poll() is None:
                time.sleep(0.005)
        except Exception:
            self.p = None
        self.t0 = time.perf_counter()
        return self

    def __exit__(self, *a):
        self.t1 = time.perf_counter()
        time.sleep(0.02)  # the row being sampled at the end of the region
        if self.p is not None:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
                self.th.join(timeout=5)
            except Exception:
                pass
        self.out = "\n".join(l.strip() for t, l in self.rows if self.t0 <= t <= self.t1 + 0.02)

    def summary(self):
        rows = [r.split(", ") for r in (self.out or "").strip().splitlines() if r.strip()]
        rows = [r for r in rows if len(r) >= 9]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[1]) for r in rows]
        mx = float(rows[0][2])
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].strip() == "Active"})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows), "power_w_max": max(float(r[3]) for r in rows)}


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2501_12349_b200 import _C, engine, toolkit, transport

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        group = transport.RankGroup.from_torch()
    mesh, field, x_host = build_inputs(rank)
    E = mesh.num_elements
    a, b = toolkit.partition_blocks(E, world)[rank]
    nodes = mesh.nodes[a:b]
    fblk = torch.from_numpy(np.ascontiguousarray(field[a:b])).to(dev)
    t0 = time.perf_counter()
    S = engine.setup(torch.from_numpy(np.ascontiguousarray(nodes)).to(dev), ORDER, 3,
                     group=group, elem_offset=a)
    torch.cuda.synchronize()
    setup_ms = (time.perf_counter() - t0) * 1e3
    F = engine.Field(fblk, ORDER)
    x_dev = torch.from_numpy(x_host).to(dev)
    x_pin = torch.from_numpy(x_host).pin_memory()
    n = x_host.shape[0]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t)

    # warm-up (also JIT of occupancy queries, workspace allocation)
    for _ in range(max(args.warmup, 3)):
        vals, rec = engine.find_and_interpolate(S, F, x_dev)
    barrier()
    # --- device-resident timed steps (per-step events, L2 flush between)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    for a_, b_ in kev:      # torch creates events lazily: force creation
        a_.record(stream)
        b_.record(stream)
    L = _C.lib()
    launches0 = L.fpx_launch_count()
    stats = []
    with ClockSampler(local) as clk:
        barrier()
        for k in range(args.steps):
            flush.fill_(float(k))
            ev[k][0].record(stream)
            vals, rec = engine.find_and_interpolate(S, F, x_dev)
            ev[k][1].record(stream)
            stats.append(rec.stats)
        barrier()
    launches = L.fpx_launch_count() - launches0
    step_ms = float(np.mean([s.elapsed_time(e) for s, e in ev]))
    # round-1 kernel alone (roofline): the same steps again, CUDA events
    # around the launch on its stream
    for k in range(args.steps):
        flush.fill_(float(k))
        L.fpx_profile_round1(kev[k][0].cuda_event, kev[k][1].cuda_event)
        vals, rec1 = engine.find_and_interpolate(S, F, x_dev)
    L.fpx_profile_round1(None, None)
    torch.cuda.synchronize()
    kern_ms = float(np.mean([s.elapsed_time(e) for s, e in kev]))
    step1 = rec1.stats
    step_ms_max = max_over_ranks(step_ms)
    value = n * world / (step_ms_max * 1e-3)
    # --- end to end through the public API: host points in, records out
    outs = dict(values=torch.empty((n, 1), dtype=torch.float64).pin_memory(),
                code=torch.empty(n, dtype=torch.int32).pin_memory(),
                elem=torch.empty(n, dtype=torch.int32).pin_memory(),
                rank=torch.empty(n, dtype=torch.int32).pin_memory(),
                r=torch.empty((n, 3), dtype=torch.float64).pin_memory(),
                dist=torch.empty(n, dtype=torch.float64).pin_memory())
    e2e_ms = []
    for _ in range(max(args.warmup, 3)):  # warm-up: host-path buffers, streams
        engine.find_and_interpolate_host(S, F, x_pin, out=outs, sync=True)
    barrier()
    for k in range(args.steps):
        flush.fill_(float(k))
        torch.cuda.synchronize()
        t0 = time.perf_counter()  # wall clock: the call returns host records
        engine.find_and_interpolate_host(S, F, x_pin, out=outs, sync=True)
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2e_max = max_over_ranks(float(np.mean(e2e_ms)))
    h2d = n * 3 * 8
    d2h = n * (8 + 4 + 4 + 4 + 24 + 8)
    # --- roofline of the dominant kernel (round-1 Newton, FP64-bound)
    st = dict(stats[-1])
    N = ORDER + 1
    flops_r1 = round1_flops(step1, N)
    tf = np.zeros(1)
    _C.check(L.fpx_probe_fp64(tf.ctypes.data, _C.stream_handle()), "fpx_probe_fp64")
    achieved = flops_r1 / (kern_ms * 1e-3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "newton_stream_dram.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get("bytes_per_launch")
    flops_all = step_flops(st, N)
    if world > 1:
        dist.barrier()
    if rank == 0:
        cpu_v, cores, cpu_t, owork = cpu_find_eval(sample=args.cpu_sample, steps=1, warmup=0)
        # the kernels' own work counters on the same sample, beside the
        # oracle's (the oracle visits candidates in ascending id, the kernels
        # best-first, so newton/iters differ by design; box_tests agree)
        _, srec = engine.find_and_interpolate(S, F, x_dev[:args.cpu_sample])
        ss = srec.stats
        kwork = {"points": int(ss["points"]), "box_tests": int(ss["box_tests"]),
                 "newton": int(ss["newton"]), "iters": int(ss["iters"])}
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": step_ms_max,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Kershaw mesh + uniform points)",
            "config": workload_config(world),
            "e2e": {"value": n * world / (e2e_max * 1e-3), "unit": UNIT,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": e2e_max,
                    "api": "engine.find_and_interpolate_host (host points in, host records "
                           "out; wall clock; round-1 records downloaded under the rest phase)"},
            "work_vs_oracle": {"sample": f"first {args.cpu_sample} points of the step",
                               "kernels": kwork, "oracle": owork},
            "roofline": {"bound": "fp64", "kernel": "k_newton_stream<3,3,5,3> (round 1)",
                         "achieved": achieved, "peak": float(tf[0]), "unit": "TFLOP/s",
                         "frac": achieved / float(tf[0]), "traffic": traffic,
                         "peak_source": "fpx_probe_fp64 DFMA chains, measured in this run "
                                        "(FP64 is not in MEASURED_PEAKS.json)",
                         "kernel_ms": kern_ms, "kernel_share": kern_ms / step_ms,
                         "kernel_timing": "CUDA events around the round-1 launch on its stream",
                         "flops_per_launch": flops_r1},
            "cpu_baseline": {"value": cpu_v, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"{args.cpu_sample} of the cfg-2 points, oracle C port "
                                       "(OpenMP over points), setup excluded"},
            "clocks": clocks, "gpu_launches": int(launches),
            "work": {"setup_ms": setup_ms, "step_flops": flops_all,
                     "step_tflops": flops_all / (step_ms * 1e-3) / 1e12, **st},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample", type=int, default=50000)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
