# usage: bash scripts/r2/gpu_ab.sh TAG "cfg1 cfg2 ..." "variant1 variant2 ..." [pytest]
# times the default library ("new") and build_variants/libmvb_<variant>.so on each config, twice, interleaved
O=gpurun_out/r2_$1
mkdir -p $O
for r in 1 2; do
for c in $2; do
  python scripts/r2/sweep_chunk.py $c new:0
  for v in $3; do MVB_CUDA_LIB=build_variants/libmvb_$v.so python scripts/r2/sweep_chunk.py $c $v:0; done
done
done > $O/sweep.txt 2>&1; cat $O/sweep.txt
if [ "$4" = "pytest" ]; then
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 $O/pytest_gpu.log
fi
