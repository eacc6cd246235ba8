set -x
O=gpurun_out/r2_t2
mkdir -p $O
python scripts/r2/sweep_chunk.py c4 2097152 4194304 8388608 16777216 33554432 67108864 > $O/sweep_c4.txt 2>&1
python scripts/r2/sweep_chunk.py c2 1048576 2097152 4194304 8388608 16777216 33554432 > $O/sweep_c2.txt 2>&1
cat $O/sweep_*.txt
Q4="python bench.py --config c4 --steps 2 --warmup 3 --cpu-seconds 0 --preroll 0"
ncu --set full --clock-control none --import-source on -k regex:vbyte_fused -s 4 -c 1 -o $O/prof_c4 $Q4 > $O/ncu_c4.log 2>&1; echo full rc=$?
