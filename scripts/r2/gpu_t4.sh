set -x
O=gpurun_out/r2_t4
mkdir -p $O
python scripts/r2/dbg_fused.py c4 4096:100 4096:200 8192:100 > $O/dbg_c4.txt 2>&1
python scripts/r2/dbg_fused.py c2 4096:100 1024:100 > $O/dbg_c2.txt 2>&1
cat $O/dbg_*.txt
python scripts/r2/sweep_chunk.py c4 4096:100 4096:200 8192:100 8192:200 16384:200 > $O/sweep_c4.txt 2>&1
cat $O/sweep_c4.txt
