# c2 launch list + one ncu --set full capture of both kernels, on the current build
set -x
O=gpurun_out/prof_c2_head
mkdir -p $O
Q="python bench.py --steps 20 --warmup 3 --cpu-seconds 0 --preroll 0"
$Q > $O/q.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file $O/launches_c2.csv $Q > $O/ncu_launch.log 2>&1; echo ncu1 rc=$?
$Q > $O/q2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:vbyte_seg -s 24 -c 2 -o $O/prof_c2 $Q > $O/ncu_full.log 2>&1; echo ncu2 rc=$?
