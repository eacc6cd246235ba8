set -x
O=gpurun_out/r2_t1
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -5 $O/pytest_gpu.log
python bench.py --config c4 --steps 20 --warmup 3 --cpu-seconds 0 --preroll 0.5 > $O/bench_c4.json 2> $O/bench_c4.err; echo c4 rc=$?
python bench.py --config c2 --steps 200 --warmup 10 --cpu-seconds 0 > $O/bench_c2.json 2> $O/bench_c2.err; echo c2 rc=$?
python bench.py --config c1 --steps 50 --warmup 10 --cpu-seconds 0 > $O/bench_c1.json 2> $O/bench_c1.err; echo c1 rc=$?
tail -c 600 $O/bench_c4.err
