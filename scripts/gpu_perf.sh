#!/bin/bash
# Perf iteration: GPU decode tests, c2/c1/c4-ish bench lines (no profiler), then one ncu --set full of c2.
# usage: bash scripts/gpu_perf.sh <tag>
TAG=${1:-x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_decode_gpu.py -m gpu -x -q -k "not config4" > gpurun_out/pt_$TAG.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pt_$TAG.log
for c in c2 c1 c5_all1 c5_all5; do
  timeout 300 python bench.py --config $c --steps 100 --warmup 5 --cpu-seconds 0 > gpurun_out/b_${TAG}_$c.log 2>&1
  python - "$c" "gpurun_out/b_${TAG}_$c.log" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(sys.argv[1], "kernel_ms %.4f" % d["roofline"]["kernel_ms_avg"], "frac %.3f" % d["roofline"]["frac"], "step_ms %.4f" % d["ms_per_step"], d["clocks"]["sm_mhz"])
except Exception as e:
    print(sys.argv[1], "FAILED", e); print(open(sys.argv[2]).read()[-1500:])
PY
done
Q="python bench.py --steps 20 --warmup 3 --cpu-seconds 0 --preroll 0 --config c2"
$Q > gpurun_out/q.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:vbyte_decode -s 12 -c 1 -o gpurun_out/prof_$TAG $Q > gpurun_out/ncu_$TAG.log 2>&1; echo ncu rc=$?
