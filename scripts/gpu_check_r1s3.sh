# Session-3 re-entry check: GPU parity suite, smoke, default bench, c3/c4 bench lines.
set -x
O=gpurun_out/check_s3
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo bench rc=$?
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --cpu-seconds 0 > $O/bench_c3.json 2> $O/bench_c3.err; echo c3 rc=$?
timeout 900 python bench.py --config c4 --steps 20 --warmup 3 --cpu-seconds 0 > $O/bench_c4.json 2> $O/bench_c4.err; echo c4 rc=$?
tail -3 $O/pytest_gpu.log
