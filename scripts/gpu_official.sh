# Official round measurement: bench line (default config), reference arm,
# launch list and one full ncu capture of the decode kernel (c2).
set -x
mkdir -p gpurun_out/official
python bench.py > gpurun_out/official/bench.json 2> gpurun_out/official/bench.err; echo bench rc=$?
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/official/bench_ref.json 2> gpurun_out/official/bench_ref.err; echo ref rc=$?
for c in c1 c4 c5_all1 c5_all5 c5_p50 c5_p50_delta; do python bench.py --config $c --steps 50 --warmup 5 --cpu-seconds 0 --preroll 0.3 > gpurun_out/official/bench_$c.json 2>&1; done
Q="python bench.py --steps 20 --warmup 3 --cpu-seconds 0 --preroll 0"
$Q > gpurun_out/official/q.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/official/launches_c2.csv $Q > gpurun_out/official/ncu_launch.log 2>&1; echo ncu1 rc=$?
$Q > gpurun_out/official/q2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:vbyte_decode -s 12 -c 1 -o gpurun_out/official/prof_c2 $Q > gpurun_out/official/ncu_full.log 2>&1; echo ncu2 rc=$?
ls -la gpurun_out/official
