Q="python bench.py --steps 20 --warmup 3 --cpu-seconds 0 --preroll 0 --config ${1:-c2}"
$Q > gpurun_out/q.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:vbyte_decode -s 12 -c 1 -o gpurun_out/prof_${2:-x} $Q > gpurun_out/ncu.log 2>&1; echo ncu rc=$?; tail -3 gpurun_out/ncu.log
