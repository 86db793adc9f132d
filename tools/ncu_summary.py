"""Key counters + SASS opcode mix + hottest source lines of one ncu report."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[2]
want = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__inst_executed.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "l1tex__t_bytes.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__sass_inst_executed_op_local_ld.sum", "smsp__sass_inst_executed_op_local_st.sum"]
for i, n in enumerate(h):
    if n in want:
        print(f"{n:70s} {v[i]}")
stalls = [(float(v[i]), n) for i, n in enumerate(h)
          if n.startswith("smsp__average_warps_issue_stalled") and n.endswith("per_issue_active.ratio")
          and v[i] not in ("", "n/a")]
for val, n in sorted(stalls, reverse=True)[:6]:
    print(f"  stall {n.replace('smsp__average_warps_issue_stalled_', ''):55s} {val:.3f}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
ia, ie, iss = h.index("Source"), h.index("Instructions Executed"), h.index(
    "Warp Stall Sampling (All Samples)")
c, s = collections.Counter(), collections.Counter()
tot = 0
for r in rows[2:]:
    if len(r) <= ie:
        continue
    t = r[ia].split()
    if not t:
        continue
    op = (t[1] if t[0].startswith("@") and len(t) > 1 else t[0]).split(".")[0]
    n = int(r[ie] or 0)
    c[op] += n
    s[op] += int(r[iss] or 0)
    tot += n
print("warp instructions", tot)
for op, n in c.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 14):
    print(f"  {op:10s} {n:12d} {100 * n / max(tot, 1):5.1f}%  stall-samples {s[op]}")
