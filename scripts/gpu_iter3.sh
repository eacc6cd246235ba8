# quick iteration: full gpu tests + default bench line (c2) + optional configs
O=gpurun_out/iter3; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo pytest rc=$?; tail -3 $O/pytest.log
for c in ${CFGS:-c2}; do timeout 300 python bench.py --config $c --steps 50 --warmup 5 --cpu-seconds 0 --preroll 0.2 2>$O/bench_$c.err | tee $O/bench_$c.json | python3 -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print(d['config']['workload'], 'Gint/s %.1f'%d['value'], 'kernel_us %.1f'%(1e3*r['kernel_ms_avg']), 'frac %.3f'%r['frac'], 'e2e %.2f'%d['e2e']['value'])
"; done
