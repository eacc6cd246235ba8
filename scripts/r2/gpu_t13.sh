O=gpurun_out/r2_t13
mkdir -p $O
for c in c4 c2 c1 c5_all1 c5_all5 c5_p50_delta c5_p50; do python scripts/r2/sweep_chunk.py $c 0:0; done > $O/sweep.txt 2>&1; cat $O/sweep.txt
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -2 $O/pytest_gpu.log
Q4="python bench.py --config c4 --steps 2 --warmup 3 --cpu-seconds 0 --preroll 0"
ncu --set full --clock-control none --import-source on -k regex:vbyte_fused -s 4 -c 1 -o $O/prof_c4 $Q4 > $O/ncu_c4.log 2>&1; echo full rc=$?
