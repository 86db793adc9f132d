"""Summarise an ncu launch list (gpu__time_duration.sum CSV): the kernels of
the longest device-mode find of the run (a full bench step: one sort +
prefilter) and, if present, of the longest host-mode find (points uploaded
in chunks, each sorted + prefiltered; rest records patched into host
memory in ranges).  Launches are serialised under ncu: shares, not overlap."""
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
# a find = the first k_point_cells after the previous find's k_find_totals,
# through k_find_totals and any host-patch kernels that follow it
finds, cur, started = [], [], False
for name, ns in out:
    if 'k_point_cells' in name and not started:
        if cur:
            finds.append(cur)
        cur, started = [], True
    if started or 'k_rest_patch_host' in name:
        cur.append((name, ns))
    if 'k_find_totals' in name:
        started = False
if cur:
    finds.append(cur)


def show(title, f):
    print(f"== {title}")
    tot = 0.0
    for name, ns in f:
        if 'dfma_probe' in name or 'at::' in name:
            continue
        tot += ns
        print(f"{ns / 1000:9.1f} us  {name[:90]}")
    print(f"{tot / 1000:9.1f} us  total")


dev = [f for f in finds if sum('k_point_cells' in n for n, _ in f) == 1
       and not any('patch_host' in n for n, _ in f)]
host = [f for f in finds if any('patch_host' in n for n, _ in f)]
if dev:
    show("device find (bench step)", max(dev, key=lambda f: sum(ns for _, ns in f)))
if host:
    show("host-mode find (e2e)", max(host, key=lambda f: sum(ns for _, ns in f)))
