# c3 (batched lists) bench line of every build_variants/*.so (VARS to pick); bench.py checks the output
for v in ${VARS:-$(ls build_variants/*.so)}; do
  MVB_CUDA_LIB=$PWD/$v timeout 600 python bench.py --config c3 --steps ${STEPS:-10} --warmup 3 --cpu-seconds 0 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step']*1e3,1), 'us', round(d['value'],1), 'Gint/s', round(d['roofline']['frac'],3))"
done
