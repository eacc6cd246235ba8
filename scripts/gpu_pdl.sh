# kernel A as a programmatic dependent of the previous kernel B: full GPU parity suite with it, then timings of both builds
set -x
O=gpurun_out/pdl
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo pytest rc=$?
tail -3 $O/pytest.log
CFGS="c2 c1 p50d c4s c2 p50" timeout 900 bash scripts/gpu_libvariants.sh > $O/variants.log 2>&1; echo var rc=$?
cat $O/variants.log | grep -v "^+"
timeout 600 python bench.py --cpu-seconds 0 > $O/bench.json 2> $O/bench.err; echo bench rc=$?
cat $O/bench.json | cut -c1-400
