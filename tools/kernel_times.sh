#!/bin/bash
# Per-kernel gpu time (ncu, serialised) of one cfg-2 find for every library
# variant in ablib/ (A/B of kernel variants).  usage: bash tools/kernel_times.sh REGEX
RX=${1:-prefilter}
cat > /tmp/one_find.py <<'PY'
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2501_12349_b200 import engine, toolkit
m = toolkit.kershaw_mesh(32, 4)
S = engine.setup(m)
F = engine._field_of(S, toolkit.analytic_field("smooth", m))
x = torch.from_numpy(toolkit.uniform_points(10 ** 6, 3, seed=1000)).cuda()
for _ in range(4):
    engine.find_and_interpolate(S, F, x)
torch.cuda.synchronize()
PY
for lib in ablib/*/libfpx_sm100.so; do
  FPX_LIB=$PWD/$lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:$RX --csv python /tmp/one_find.py 2>/dev/null \
    | python -c "
import csv,sys
v=[float(r[-1]) for r in csv.reader(sys.stdin) if len(r)>3 and r[-3]=='gpu__time_duration.sum']
print('%-40s' % sys.argv[1], ' '.join('%.1f' % (x/1000) for x in v[-4:]), 'us')" $lib
done
