# usage: bash scripts/r2/gpu_round.sh TAG -- GPU tests, smoke, default bench (c4) + reference arm,
# bench lines for every config, c4 launch list and one ncu --set full capture of the fused kernel.
O=gpurun_out/r2_$1
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo bench rc=$?; cat $O/bench.json
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo ref rc=$?; cat $O/bench_ref.json
for c in c1 c2 c3 c5_all1 c5_all5 c5_p10 c5_p25 c5_p50 c5_p75 c5_p90 c5_all1_delta c5_all5_delta c5_p10_delta c5_p25_delta c5_p50_delta c5_p75_delta c5_p90_delta; do
  timeout 300 python bench.py --config $c --steps 50 --warmup 5 --cpu-seconds 3 >> $O/bench_lines.jsonl 2>> $O/bench_lines.err; echo "$c rc=$?"
done
Q4="python bench.py --config c4 --steps 3 --warmup 3 --cpu-seconds 0 --preroll 0"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file $O/launches_c4.csv $Q4 > $O/ncu_launch.log 2>&1; echo launch rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vbyte_fused -s 4 -c 1 -o $O/prof_c4 $Q4 > $O/ncu_c4.log 2>&1; echo full rc=$?
