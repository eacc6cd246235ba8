# fast5 check: lane-local parity tests + default-kernel timings of the fast5 / nofast5 builds
set -x
O=gpurun_out/fast5
mkdir -p $O
timeout 900 python -m pytest tests/test_lane_local.py tests/test_decode_gpu.py -m gpu -x -q > $O/pytest.log 2>&1; echo pytest rc=$?
tail -3 $O/pytest.log
CFGS="c1 all5 c2 p50 c4s" timeout 900 bash scripts/gpu_libvariants.sh > $O/variants.log 2>&1; echo var rc=$?
cat $O/variants.log | grep -v "^+"
