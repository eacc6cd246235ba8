# Official measurement (part 1): bench lines of every config, reference arm,
# launch list of the default bench command (one ncu pass).
set -x
O=gpurun_out/official${TAG:-3}
mkdir -p $O
python bench.py > $O/bench.json 2> $O/bench.err; echo bench rc=$?
python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo ref rc=$?
python bench.py --config c4 --steps 20 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err; echo c4 rc=$?
python bench.py --config c3 --steps 10 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err; echo c3 rc=$?
for c in c1 c5_all1 c5_all5 c5_p50 c5_p50_delta; do python bench.py --config $c --steps 50 --warmup 5 --cpu-seconds 0 --preroll 0.3 > $O/bench_$c.json 2>&1; done
Q="python bench.py --steps 20 --warmup 3 --cpu-seconds 0 --preroll 0"
$Q > $O/q.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file $O/launches_c2.csv $Q > $O/ncu_launch.log 2>&1; echo ncu1 rc=$?
ls -la $O
