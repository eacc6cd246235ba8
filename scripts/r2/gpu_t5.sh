O=gpurun_out/r2_t5
mkdir -p $O
for z in 2 0 1; do echo "swz=$z"; MVB_F_SWZ=$z python scripts/r2/dbg_fused.py c4 4096:100 8192:100 4096:100; done > $O/dbg_c4.txt 2>&1
cat $O/dbg_c4.txt
