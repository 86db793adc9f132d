#!/bin/bash
# A/B of library variants on the cfg-2 bench (dev builds in tools/ab/).
for lib in tools/ab/*.so; do
  echo "== $lib"
  FPX_LIB=$PWD/$lib timeout 300 python bench.py --steps 5 --warmup 3 --cpu-sample 2000 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('value %.3e pts/s  step %.2f ms  e2e %.3e  kernel %.2f ms frac %.3f  regs? launches %d' % (d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['gpu_launches'])); print(json.dumps(d['work'])); print(json.dumps(d['clocks']))
    else: print(l.rstrip()[-300:])
"
done
