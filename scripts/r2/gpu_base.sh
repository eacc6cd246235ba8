# Round-2 baseline on the round-1 build: HBM ceiling probe, c4 bench, c4 launch list, ncu --set full of c4's kernels.
set -x
O=gpurun_out/r2_base
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/smi.txt 2>&1
./scripts/r2/hbm_probe > $O/hbm_probe.txt 2>&1; echo probe rc=$?
python bench.py --config c4 --steps 20 --warmup 3 --cpu-seconds 0 --preroll 0.5 > $O/bench_c4.json 2> $O/bench_c4.err; echo c4 rc=$?
python bench.py --config c2 --steps 200 --warmup 10 --cpu-seconds 0 > $O/bench_c2.json 2> $O/bench_c2.err; echo c2 rc=$?
Q4="python bench.py --config c4 --steps 2 --warmup 3 --cpu-seconds 0 --preroll 0"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:vbyte_seg -c 12 --csv --log-file $O/launches_c4.csv $Q4 > $O/ncu_l4.log 2>&1; echo l4 rc=$?
ncu --set full --clock-control none --import-source on -k regex:vbyte_seg -s 4 -c 2 -o $O/prof_c4 $Q4 > $O/ncu_c4.log 2>&1; echo full rc=$?
ls -la $O
