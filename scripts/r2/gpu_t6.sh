O=gpurun_out/r2_t6
mkdir -p $O
python scripts/r2/sweep_chunk.py c4 4096:100 16384:100 16384:200 32768:100 32768:50 65536:100 65536:50 > $O/sweep_c4.txt 2>&1
python scripts/r2/sweep_chunk.py c2 4096:100 8192:100 2048:200 4096:200 > $O/sweep_c2.txt 2>&1
cat $O/sweep_*.txt
Q4="python bench.py --config c4 --steps 2 --warmup 3 --cpu-seconds 0 --preroll 0"
ncu --set full --clock-control none --import-source on -k regex:vbyte_fused -s 4 -c 1 -o $O/prof_c4 $Q4 > $O/ncu_c4.log 2>&1; echo full rc=$?
MVB_F_SEG=32768 MVB_F_LAG=100 ncu --set full --clock-control none --import-source on -k regex:vbyte_fused -s 4 -c 1 -o $O/prof_c4_32k $Q4 > $O/ncu_c4b.log 2>&1; echo full rc=$?
