# baseline of the session's HEAD: quick timings, GPU tests, ncu --set full reps (with source) of the main configs
O=gpurun_out/r2_s3base
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
for c in c4 c2 c1 c5_all1 c5_all5 c5_all5_delta c5_p50_delta c5_p50; do python scripts/r2/sweep_chunk.py $c 0:0; done > $O/sweep.txt 2>&1; cat $O/sweep.txt
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -2 $O/pytest_gpu.log
for c in c4 c2 c1 c5_all5_delta; do
Q="python bench.py --config $c --steps 2 --warmup 3 --cpu-seconds 0 --preroll 0"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:vbyte_fused -s 4 -c 1 -o $O/prof_$c $Q > $O/ncu_$c.log 2>&1; echo full $c rc=$?
done
Q="python bench.py --config c3 --steps 2 --warmup 3 --cpu-seconds 0 --preroll 0"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:vbyte_lists -s 4 -c 1 -o $O/prof_c3 $Q > $O/ncu_c3.log 2>&1; echo full c3 rc=$?
ls -la $O
