# quick iteration: gpu tests + bench kernel timings for the default kernel
timeout 900 python -m pytest tests -m gpu -x -q -k "not config4" 2>&1 | tail -3
for c in c2 c1 c5_all1 c5_all5; do timeout 300 python bench.py --config $c --steps 50 --warmup 5 --cpu-seconds 0 --preroll 0.2 2>&1 | python3 -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print(d['config']['workload'], 'Gint/s %.1f'%d['value'], 'kernel_us %.1f'%(1e3*r['kernel_ms_avg']), 'frac %.3f'%r['frac'])
    else: print(l.rstrip()[-200:])
"; done
