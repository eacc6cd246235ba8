#!/bin/bash
mkdir -p gpurun_out
for c in c2 all5 all1; do MVB_KERNEL=3 timeout 300 python scripts/trace_tiles.py $c v3 2>&1 | tail -1; done
python scripts/analyze_trace3.py c2_v3 all5_v3 all1_v3
