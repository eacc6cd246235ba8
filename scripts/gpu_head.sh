# head slices on the 2-byte / fast paths: full GPU parity suite, c3 path stats and timings of both builds
set -x
O=gpurun_out/headf
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo pytest rc=$?
tail -3 $O/pytest.log
MVB_CUDA_LIB=$PWD/build_variants/headfstats.so timeout 600 python scripts/path_stats.py c3 c1 > $O/stats.log 2>&1; cat $O/stats.log
VARS="build_variants/headf.so build_variants/noheadf.so build_variants/headf.so build_variants/noheadf.so" bash scripts/gpu_c3variants.sh > $O/c3.log 2>&1; cat $O/c3.log
