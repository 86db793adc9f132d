"""Summarise an ncu launch list (gpu__time_duration.sum CSV): the kernels of
the longest find of the run (a full bench step)."""
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
# the finds of the run start at k_point_cells; report the longest one (the
# full-size bench step, not the small work-counter sample that follows it)
starts = [i for i, o in enumerate(out) if 'k_point_cells' in o[0]] + [len(out)]
spans = [(sum(ns for _, ns in out[a:b]), a, b) for a, b in zip(starts, starts[1:])]
_, start, stop = max(spans)
tot = 0.0
for name, ns in out[start:stop]:
    if 'dfma_probe' in name or 'at::' in name:
        continue
    tot += ns
    print(f"{ns / 1000:9.1f} us  {name[:90]}")
print(f"{tot / 1000:9.1f} us  total")
