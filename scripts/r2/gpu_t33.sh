O=gpurun_out/r2_t33
mkdir -p $O
./tests/cpp/sharded_abi_test 400000 1 2 3 5 8 > $O/cpp.txt 2>&1; echo cpp rc=$?; tail -3 $O/cpp.txt
for W in 2 8; do python scripts/r2/shard_traffic.py $W 0; done > $O/traffic.txt 2>&1; cat $O/traffic.txt
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:vbyte_fused -s 6 -c 4 --csv --log-file $O/ncu_shard8.csv python scripts/r2/shard_traffic.py 8 0 > $O/ncu.log 2>&1; echo ncu rc=$?
