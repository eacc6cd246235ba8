# usage: bash scripts/r2/gpu_s4_base.sh TAG -- gpu_round.sh plus one ncu --set full capture of the decode kernel
# for c1, c2, c3 and c5 all-5B (plain and delta)
bash scripts/r2/gpu_round.sh $1
O=gpurun_out/r2_$1
for c in c1 c2 c5_all5 c5_all5_delta; do
  Q="python bench.py --config $c --steps 3 --warmup 3 --cpu-seconds 0 --preroll 0"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:vbyte_fused -s 4 -c 1 -o $O/prof_$c $Q > $O/ncu_$c.log 2>&1; echo "full $c rc=$?"
done
Q="python bench.py --config c3 --steps 3 --warmup 3 --cpu-seconds 0 --preroll 0"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:vbyte_lists -s 4 -c 1 -o $O/prof_c3 $Q > $O/ncu_c3.log 2>&1; echo "full c3 rc=$?"
ls -la $O
