"""Per-CUDA-source-line totals (instructions executed, stall samples) of one
ncu report: ncu -i REP --page source --print-source cuda,sass."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
fname, agg = None, []
rows = list(csv.reader(io.StringIO(txt)))
cur = None
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:  # cuda line row
        try:
            cur = [fname, r[0], r[1].strip()[:70], int(r[7] or 0), int(r[4] or 0)]
        except ValueError:
            continue
        agg.append(cur)
tot_i = sum(a[3] for a in agg)
tot_s = sum(a[4] for a in agg)
print(f"total inst {tot_i}  stall samples {tot_s}")
for a in sorted(agg, key=lambda a: -a[4])[:top]:
    print(f"{a[4]*100/max(tot_s,1):5.1f}% st {a[3]*100/max(tot_i,1):5.1f}% in  {a[0]}:{a[1]:5s} {a[2]}")
