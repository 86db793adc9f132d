"""Summarise an ncu launch list (gpu__time_duration.sum CSV): the kernels of
the last bench step (from the last k_point_cells launch)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, out = None, []
for r in rows:
    if 'Kernel Name' in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get('Metric Name') == 'gpu__time_duration.sum':
            out.append((d['Kernel Name'], float(d['Metric Value'])))
start = [i for i, o in enumerate(out) if 'k_point_cells' in o[0]][-1]
tot = 0.0
for name, ns in out[start:]:
    if 'dfma_probe' in name or 'at::' in name:
        continue
    tot += ns
    print(f"{ns / 1000:9.1f} us  {name[:90]}")
print(f"{tot / 1000:9.1f} us  total")
