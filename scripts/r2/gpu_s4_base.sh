# usage: bash scripts/r2/gpu_s4_base.sh TAG -- gpu_round.sh plus one ncu --set full capture of the decode kernel
# for c1, c2, c3 and c5 all-5B delta; the reports are summarised on the box (gpurun copies back <= 64 MiB)
rm -rf gpurun_out/*
bash scripts/r2/gpu_round.sh $1
O=gpurun_out/r2_$1
python scripts/ncu_summary.py $O/prof_c4.ncu-rep > $O/ncu_full_c4_summary.txt 2>&1
for c in c1 c2 c5_all5_delta; do
  Q="python bench.py --config $c --steps 3 --warmup 3 --cpu-seconds 0 --preroll 0"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:vbyte_fused -s 4 -c 1 -o $O/prof_$c $Q > $O/ncu_$c.log 2>&1; echo "full $c rc=$?"
  python scripts/ncu_summary.py $O/prof_$c.ncu-rep > $O/ncu_full_${c}_summary.txt 2>&1; rm -f $O/prof_$c.ncu-rep
done
Q="python bench.py --config c3 --steps 3 --warmup 3 --cpu-seconds 0 --preroll 0"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:vbyte_lists -s 4 -c 1 -o $O/prof_c3 $Q > $O/ncu_c3.log 2>&1; echo "full c3 rc=$?"
python scripts/ncu_summary.py $O/prof_c3.ncu-rep > $O/ncu_full_c3_summary.txt 2>&1
du -sh gpurun_out
