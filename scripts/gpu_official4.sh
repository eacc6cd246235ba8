# Official measurement (session 3 of round 1): GPU parity suite + smoke, bench lines of every config,
# the reference arm, the launch list of the default bench command, one ncu --set full capture (c2) and one of c1.
set -x
O=gpurun_out/official${TAG:-4}
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?
python bench.py > $O/bench.json 2> $O/bench.err; echo bench rc=$?
python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo ref rc=$?
python bench.py --config c4 --steps 20 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err; echo c4 rc=$?
python bench.py --config c3 --steps 10 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err; echo c3 rc=$?
for c in c1 c5_all1 c5_all5 c5_p50 c5_p50_delta; do python bench.py --config $c --steps 50 --warmup 5 --cpu-seconds 0 --preroll 0.3 > $O/bench_$c.json 2>&1; done
Q="python bench.py --steps 20 --warmup 3 --cpu-seconds 0 --preroll 0"
$Q > $O/q.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file $O/launches_c2.csv $Q > $O/ncu_launch.log 2>&1; echo ncu1 rc=$?
$Q > $O/q2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:vbyte_seg -s 24 -c 2 -o $O/prof_c2 $Q > $O/ncu_full.log 2>&1; echo ncu2 rc=$?
Q1="python bench.py --config c1 --steps 20 --warmup 3 --cpu-seconds 0 --preroll 0"
$Q1 > $O/q3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:vbyte_seg -s 24 -c 2 -o $O/prof_c1 $Q1 > $O/ncu_full_c1.log 2>&1; echo ncu3 rc=$?
tail -2 $O/pytest_gpu.log
ls -la $O
