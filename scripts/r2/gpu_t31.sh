O=gpurun_out/r2_t32
mkdir -p $O
for r in 1 2; do
for c in c4 c2 c5_p50_delta; do python scripts/r2/sweep_chunk.py $c new:0; MVB_CUDA_LIB=build_variants/libmvb_prev.so python scripts/r2/sweep_chunk.py $c prev:0; done
done > $O/sweep.txt 2>&1; cat $O/sweep.txt
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -2 $O/pytest_gpu.log
