#!/bin/bash
# A/B of runtime knobs on the cfg-2 bench: each argument is an env assignment
# list ("FPX_HASH_REFINE=1 FPX_PREFILTER=1"); "-" = defaults.  Writes the
# launch list of each variant to gpurun_out/launches_ab<i>.csv when NCU=1.
i=0
for cfg in "$@"; do
  i=$((i+1))
  [ "$cfg" = "-" ] && cfg=""
  echo "== [$i] $cfg"
  env $cfg timeout 300 python bench.py --steps 5 --warmup 3 --cpu-sample 1000 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('value %.3e pts/s  step %.3f ms  e2e %.3e  r1 %.3f ms frac %.3f  launches %d' % (d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['gpu_launches'])); print(json.dumps(d['work']))
"
  if [ "$NCU" = "1" ]; then
    env $cfg timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_ab$i.csv python bench.py --steps 1 --warmup 3 --cpu-sample 500 > /dev/null 2>&1
    python tools/launches.py gpurun_out/launches_ab$i.csv
  fi
done
