# quick iteration: gpu tests, traces, kernel timings
timeout 900 python -m pytest tests -m gpu -x -q -k "not config4" 2>&1 | tail -2
for c in c2 c1 all1 all5; do python scripts/trace_tiles.py $c 2>&1 | tail -1; done
