#!/bin/bash
# A/B of library variants on the cfg-2 bench (dev builds in ablib/<name>/,
# git-ignored; they travel to the GPU box with the snapshot).
for lib in ablib/*/libfpx_sm100.so; do
  echo "== $lib"
  FPX_LIB=$PWD/$lib timeout 300 python bench.py --steps 5 --warmup 3 --cpu-sample 2000 "$@" 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('value %.3e pts/s  step %.3f ms  e2e %.3f ms  r1 %.3f ms frac %.3f' % (d['value'], d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac']))
    else: print(l.rstrip()[-300:])
"
done
