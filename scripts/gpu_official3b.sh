# Official measurement (part 2): one ncu --set full capture of both kernels of the default c2 decode.
set -x
O=gpurun_out/official${TAG:-3}
mkdir -p $O
Q="python bench.py --steps 20 --warmup 3 --cpu-seconds 0 --preroll 0"
$Q > $O/q2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:vbyte_seg -s 24 -c 2 -o $O/prof_c2 $Q > $O/ncu_full.log 2>&1; echo ncu2 rc=$?
