# Final-build profiles of c3 (batched lists: one --set full capture) and c4 (2^30 ints: launch list of A / B)
set -x
O=gpurun_out/prof_c3c4
mkdir -p $O
Q3="python bench.py --config c3 --steps 3 --warmup 3 --cpu-seconds 0 --preroll 0"
$Q3 > $O/q3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:vbyte_lists -s 2 -c 1 -o $O/prof_c3 $Q3 > $O/ncu_c3.log 2>&1; echo ncu_c3 rc=$?
$Q3 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:mvbk -c 12 --csv --log-file $O/launches_c3.csv $Q3 > $O/ncu_l3.log 2>&1; echo l3 rc=$?
Q4="python bench.py --config c4 --steps 3 --warmup 3 --cpu-seconds 0 --preroll 0"
$Q4 > $O/q4.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:vbyte_seg -c 16 --csv --log-file $O/launches_c4.csv $Q4 > $O/ncu_l4.log 2>&1; echo l4 rc=$?
ls -la $O
