timeout 900 python -m pytest tests -m gpu -x -q -k "not config4" 2>&1 | tail -2
for v in lw0 lw7; do
  for c in c2 c1; do MVB_CUDA_LIB=build_variants/lib_$v.so python scripts/trace_tiles.py $c $v 2>&1 | tail -1; done
done
