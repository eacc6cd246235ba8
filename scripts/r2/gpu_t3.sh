set -x
O=gpurun_out/r2_t3
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 $O/pytest_gpu.log
python scripts/r2/sweep_chunk.py c4 4096:100 4096:50 4096:200 2048:100 8192:100 8192:50 16384:50 > $O/sweep_c4.txt 2>&1
python scripts/r2/sweep_chunk.py c2 1024:100 2048:100 4096:100 4096:50 > $O/sweep_c2.txt 2>&1
cat $O/sweep_*.txt
Q4="python bench.py --config c4 --steps 2 --warmup 3 --cpu-seconds 0 --preroll 0"
ncu --set full --clock-control none --import-source on -k regex:vbyte_fused -s 4 -c 1 -o $O/prof_c4 $Q4 > $O/ncu_c4.log 2>&1; echo full rc=$?
