"""Per-kernel ncu table (north_star: FP64 FLOP/s and HBM GB/s against the
B200 peaks, occupancy, divergence) from a --metrics CSV of
tools/profile_workload.py.

    python tools/ncu_table.py gpurun_out/ncu_table.csv FP64_PEAK_TFLOPS > profiles/...md
"""
import collections
import csv
import json
import os
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rows = list(csv.reader(open(sys.argv[1])))
fp64_peak = float(sys.argv[2]) if len(sys.argv) > 2 else 34.1
hbm_peak = json.load(open(os.path.join(HERE, "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(HERE, "MEASURED_PEAKS.json")) else 6551.0
hdr = None
launches = collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r and "Metric Name" in r:
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    key = d["ID"]
    L = launches.setdefault(key, {"name": d["Kernel Name"]})
    try:
        L[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    except ValueError:
        L[d["Metric Name"]] = d["Metric Value"]

agg = collections.OrderedDict()
for L in launches.values():
    nm = L["name"].split("(")[0].replace("void ", "")
    if nm.startswith("at::") or "dfma_probe" in nm or "cub::" in nm or "DeviceScan" in nm \
            or "DeviceRadix" in nm:
        nm = "(library) " + nm[:40]
    a = agg.setdefault(nm, collections.Counter())
    a["n"] += 1
    a["ns"] += L.get("gpu__time_duration.sum", 0)
    a["flop"] += 2 * L.get("sm__sass_thread_inst_executed_op_dfma_pred_on.sum", 0) + \
        L.get("sm__sass_thread_inst_executed_op_dmul_pred_on.sum", 0) + \
        L.get("sm__sass_thread_inst_executed_op_dadd_pred_on.sum", 0)
    a["dram"] += L.get("dram__bytes_read.sum", 0) + L.get("dram__bytes_write.sum", 0)
    w = L.get("gpu__time_duration.sum", 0)
    a["warps_w"] += w * L.get("sm__warps_active.avg.pct_of_peak_sustained_active", 0)
    a["tpi_w"] += w * L.get("smsp__thread_inst_executed_per_inst_executed.ratio", 0)
    a["fp64pipe_w"] += w * L.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 0)
    a["regs"] = max(a["regs"], L.get("launch__registers_per_thread", 0))

print(f"FP64 peak {fp64_peak:.1f} TFLOP/s (fpx_probe_fp64, measured); HBM peak {hbm_peak:.0f} GB/s "
      "(MEASURED_PEAKS.json). ncu replays are serialised and cold-cache: compare shares.\n")
print("| kernel | launches | µs | FP64 TFLOP/s (executed) | % FP64 peak | FP64 pipe % | DRAM GB/s | % HBM peak | warps active % | threads/inst | regs |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for nm, a in sorted(agg.items(), key=lambda kv: -kv[1]["ns"]):
    ns = max(a["ns"], 1)
    tf = a["flop"] / ns / 1e3
    gbs = a["dram"] / ns
    print(f"| `{nm[:60]}` | {a['n']} | {ns / 1e3:.1f} | {tf:.2f} | {100 * tf / fp64_peak:.1f} | "
          f"{a['fp64pipe_w'] / ns:.1f} | {gbs:.0f} | {100 * gbs / hbm_peak:.1f} | "
          f"{a['warps_w'] / ns:.1f} | {a['tpi_w'] / ns:.1f} | {int(a['regs'])} |")
