for l in base lean base lean; do
  FPX_LIB=$PWD/ablib/$l/libfpx_sm100.so timeout 600 python bench.py --steps 3 --warmup 3 --cpu-sample 2000 --workload cfg3 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$l', 'step %.2f ms r1 %.2f ms frac %.3f' % (d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac']))
"
done
