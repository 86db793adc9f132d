"""findpts+eval throughput benchmark (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload cfg2|cfg3|cfg4]

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
--workload cfg3 (Kershaw 64^3, p=7, 10^7 points, mesh replicated on the GPU)
and cfg4 (cubed sphere 6*32^2 quads, p=4, 10^6 on/near-surface points) run the
same step on the other BASELINE configs; cfg2 stays the default.
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

METRIC = "findpts+eval points/sec (3D hex, p=4, 1M pts/GPU) at 1/2/4/8 B200"
UNIT = "points/s"


class Workload:
    """One benchmark configuration (BASELINE.json configs).
    cfg2 is the headline (BASELINE metric); cfg3/cfg4 are the other
    single-GPU-sized configs, run with --workload."""

    def __init__(self, key, gen, n_axis, order, pts, dr, metric, desc, points="uniform"):
        self.key, self.gen, self.n_axis, self.order = key, gen, n_axis, order
        self.pts, self.dr, self.metric, self.desc, self.points = pts, dr, metric, desc, points

    def mesh(self):
        from paper_2501_12349_b200 import toolkit
        if self.gen == "kershaw":
            return toolkit.kershaw_mesh(self.n_axis, self.order)
        return toolkit.sphere_mesh(self.n_axis, self.order)

    def field(self, mesh):
        from paper_2501_12349_b200 import toolkit
        return toolkit.analytic_field("smooth", mesh)

    def query(self, mesh, n, rank):
        from paper_2501_12349_b200 import toolkit
        if self.points == "uniform":
            return toolkit.uniform_points(n, 3, seed=1000 + rank)
        return toolkit.surface_points(mesh, n, seed=1000 + rank)[0]

    def config(self, n_gpus):
        E = self.n_axis ** 3 if self.gen == "kershaw" else 6 * self.n_axis ** 2
        return {"workload": f"{self.key}: {self.desc}, {self.pts} pts/GPU, find+eval (C=1)",
                "mesh": f"{self.gen}{self.n_axis}" + ("^3" if self.gen == "kershaw" else ""),
                "order": self.order, "elements": E, "points_per_gpu": self.pts,
                "components": 1,
                "partition": "contiguous z-slabs" if n_gpus > 1 else "single",
                "l2": "flushed (256 MiB write) between timed steps"}


WORKLOADS = {
    "cfg2": Workload("cfg-2", "kershaw", 32, 4, 1_000_000, 3, METRIC,
                     "Kershaw hex 32^3 p=4 (eps 0.3)"),
    "cfg3": Workload("cfg-3", "kershaw", 64, 7, 10_000_000, 3,
                     "findpts+eval points/sec (3D hex 64^3, p=7, 1e7 pts) on B200",
                     "Kershaw hex 64^3 p=7 (eps 0.3), replicated mesh"),
    "cfg4": Workload("cfg-4", "sphere", 32, 4, 1_000_000, 2,
                     "surface findpts+eval points/sec (cubed sphere, p=4, 1e6 pts) on B200",
                     "cubed-sphere quads 6*32^2 p=4 in 3D", points="surface"),
}
W = WORKLOADS["cfg2"]


# Algorithmic FP64 work per unit (frozen; N = p+1; the
# contraction term generalises 2N^3+3N^2+4N (d_r = 3) to d_r = 2 and 1).
def _contr(N, dr):
    return {3: 2 * N ** 3 + 3 * N ** 2 + 4 * N, 2: 2 * N ** 2 + 3 * N, 1: 2 * N}[dr]


def f_iter(N, d=3, dr=3):  # one Newton iteration: basis evals + x,G contraction + solve
    return dr * 13 * N + 2 * d * _contr(N, dr) + 130


def f_seed(N, dr=3):   # nearest-node seed over N^dr nodes
    return 8 * N ** dr


def f_eval(N, C=1, dr=3):
    return dr * 8 * N + 2 * C * sum(N ** k for k in range(1, dr + 1))


F_SEED_AFFINE = 2 * 3 * 3 + 3   # D7' seed: J_c^-1 (x* - x_c) (3x3 mat-vec + 3 subtractions)


def round1_flops(st, N, d=3, dr=3):
    """Algorithmic FP64 work of the round-1 kernel: every lane evaluation of
    the map (basis, x + G contraction, step algebra = F_iter), the seed of
    every solve (affine for volumes, nearest node for d_r < d), the fused
    field evaluation of every final point."""
    seed = F_SEED_AFFINE if dr == d else f_seed(N, dr)
    return st["r1_lane_evals"] * f_iter(N, d, dr) + st["newton_r1"] * seed \
        + st["evals_r1"] * f_eval(N, 1, dr)


def step_flops(st, N, d=3, dr=3):
    """Whole find+eval step: round 1, the rest kernels' lane evaluations
    (each rest solve counted with a nearest-node seed, 8 N^dr: an upper
    bound, pass-1 solves seed from the frame), 30 flops per box test, and the
    field evaluation of every found point."""
    rest_solves = st["newton"] - st["newton_r1"]
    return round1_flops(st, N, d, dr) + st["rest_lane_evals"] * f_iter(N, d, dr) \
        + rest_solves * f_seed(N, dr) + 30 * st["box_tests"] \
        + (st["evals"] - st["evals_r1"]) * f_eval(N, 1, dr)


def workload_config(n_gpus):
    return W.config(n_gpus)


def build_inputs(rank=0, n=None):
    mesh = W.mesh()
    field = W.field(mesh)
    x = W.query(mesh, n or W.pts, rank)
    return mesh, field, x


# ----------------------------------------------------------------- CPU arm
def cpu_find_eval(sample=20000, threads=None, steps=1, warmup=0, rank=0, inputs=None):
    """The oracle port (oracle/fpx_oracle.c, OpenMP) on the host cores."""
    from oracle import oracle as O
    mesh, field, x = inputs or build_inputs(rank, sample)
    nthreads = threads or len(os.sched_getaffinity(0))
    # the same local grid as engine.setup's default (hash_refine x SPEC rule)
    from paper_2501_12349_b200.engine import EngineOptions
    d = mesh.phys_dim
    ncell = min(1024, EngineOptions().hash_refine * O.n_cells(mesh.num_elements, d))
    OS = O.OracleSetup(mesh.nodes, d, W.dr, W.order, nthreads=nthreads, ncell=ncell)
    xs = x[:sample]
    times = []
    for k in range(warmup + steps):
        t = time.perf_counter()
        rec = OS.find(xs, nthreads=nthreads)
        O.evaluate(OS.B, W.dr, field, rec["code"], rec["elem"], rec["r"], nthreads=nthreads)
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
    line = {"impl": "reference", "metric": W.metric, "value": v, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args.gpus),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"{sample} of the {W.pts} {W.key} points per step "
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
    local = local % max(torch.cuda.device_count(), 1) if args.backend == "gloo" else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if world > 1 and args.backend == "gloo":
        dist.init_process_group("gloo")
    elif world > 1:
        dist.init_process_group("nccl", device_id=dev)
        group = transport.RankGroup.from_torch()
    mesh, field, x_host = build_inputs(rank)
    E = mesh.num_elements
    a, b = toolkit.partition_blocks(E, world)[rank]
    nodes = mesh.nodes[a:b]
    fblk = torch.from_numpy(np.ascontiguousarray(field[a:b])).to(dev)
    t0 = time.perf_counter()
    S = engine.setup(torch.from_numpy(np.ascontiguousarray(nodes)).to(dev), W.order, W.dr,
                     group=group, elem_offset=a)
    torch.cuda.synchronize()
    setup_ms = (time.perf_counter() - t0) * 1e3
    F = engine.Field(fblk, W.order)
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
        t = torch.tensor([v], dtype=torch.float64, device=dev if args.backend == "nccl" else "cpu")
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
                r=torch.empty((n, W.dr), dtype=torch.float64).pin_memory(),
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
    d = mesh.phys_dim
    h2d = n * d * 8
    d2h = n * (8 + 4 + 4 + 4 + 8 * W.dr + 8)
    # --- roofline of the dominant kernel (round-1 Newton, FP64-bound)
    st = dict(stats[-1])
    N = W.order + 1
    flops_r1 = round1_flops(step1, N, d, W.dr)
    tf = np.zeros(1)
    _C.check(L.fpx_probe_fp64(tf.ctypes.data, _C.stream_handle()), "fpx_probe_fp64")
    achieved = flops_r1 / (kern_ms * 1e-3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "newton_stream_dram.json")
    if os.path.exists(tpath):  # ncu dram bytes of the same launch, per workload
        traffic = json.load(open(tpath)).get(W.key, {}).get("bytes_per_launch")
    flops_all = step_flops(st, N, d, W.dr)
    if world > 1:
        dist.barrier()
    if rank == 0:
        cpu_v, cores, cpu_t, owork = cpu_find_eval(sample=args.cpu_sample, steps=1, warmup=0,
                                                   inputs=(mesh, field, x_host))
        # the kernels' own work counters on the same sample, beside the
        # oracle's (the oracle visits candidates in ascending id, the kernels
        # best-first, so newton/iters differ by design; box_tests agree)
        _, srec = engine.find_and_interpolate(S, F, x_dev[:args.cpu_sample])
        ss = srec.stats
        kwork = {"points": int(ss["points"]), "box_tests": int(ss["box_tests"]),
                 "newton": int(ss["newton"]), "iters": int(ss["iters"])}
        clocks = clk.summary()
        line = {
            "metric": W.metric, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": step_ms_max,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Kershaw mesh + uniform points)",
            "config": workload_config(world),
            "e2e": {"value": n * world / (e2e_max * 1e-3), "unit": UNIT,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": e2e_max,
                    "api": "engine.find_and_interpolate_host (host points in, host records "
                           "out; wall clock; points up in chunks under the prefilter, "
                           "records down in ranges from round 1 on, rest records patched "
                           "per range)"},
            "work_vs_oracle": {"sample": f"first {args.cpu_sample} points of the step",
                               "kernels": kwork, "oracle": owork},
            "roofline": {"bound": "fp64",
                         "kernel": f"k_newton_stream<{d},{W.dr},{N},S> (round 1)",
                         "achieved": achieved, "peak": float(tf[0]), "unit": "TFLOP/s",
                         "frac": achieved / float(tf[0]), "traffic": traffic,
                         "peak_source": "fpx_probe_fp64 DFMA chains, measured in this run "
                                        "(FP64 is not in MEASURED_PEAKS.json)",
                         "kernel_ms": kern_ms, "kernel_share": kern_ms / step_ms,
                         "kernel_timing": "CUDA events around the round-1 launch on its stream",
                         "flops_per_launch": flops_r1},
            "cpu_baseline": {"value": cpu_v, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"{args.cpu_sample} of the {W.key} points, oracle C port "
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
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process group for N > 1 (gloo: several ranks sharing one GPU, "
                         "a check of the multi-rank path, not a measurement)")
    ap.add_argument("--workload", default="cfg2", choices=sorted(WORKLOADS),
                    help="cfg2 = the BASELINE headline (default); cfg3 / cfg4 = the other "
                         "BASELINE configs that fit one GPU")
    args = ap.parse_args()
    global W
    W = WORKLOADS[args.workload]
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
