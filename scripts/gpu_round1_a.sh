set -x
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo rc=$?
cat gpurun_out/bench_default.json
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err; echo rc=$?
cat gpurun_out/bench_ref.json
for c in c1 c5_all1 c5_all5 c5_p50_delta; do python bench.py --config $c --steps 100 --cpu-seconds 0 --preroll 0.5 2>&1 | tail -1; done
Q="python bench.py --steps 20 --warmup 3 --cpu-seconds 0 --preroll 0"
$Q > gpurun_out/q.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches_c2.csv $Q > gpurun_out/ncu1.log 2>&1; echo ncu1 rc=$?
$Q > gpurun_out/q2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:vbyte_decode -s 12 -c 2 -o gpurun_out/prof_c2 $Q > gpurun_out/ncu2.log 2>&1; echo ncu2 rc=$?
ls -la gpurun_out
