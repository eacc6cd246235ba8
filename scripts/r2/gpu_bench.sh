O=gpurun_out/r2_$1
mkdir -p $O
python bench.py > $O/bench.json 2> $O/bench.err; echo bench rc=$?
python bench.py --impl reference --steps 5 --warmup 2 > $O/bench_ref.json 2> $O/bench_ref.err; echo ref rc=$?
tail -3 $O/bench.err $O/bench_ref.err
