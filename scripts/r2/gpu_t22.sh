O=gpurun_out/r2_t22
mkdir -p $O
for v in u3k5 u2k6 u3k4; do for c in c4 c2 c1; do MVB_CUDA_LIB=build_variants/libmvb_$v.so python scripts/r2/sweep_chunk.py $c $v:0; done; done > $O/sweep.txt 2>&1; cat $O/sweep.txt
