# ncu evidence for the batched-lists (c3) and large-stream (c4, 2^27-int slice of its distribution) decodes:
# a launch list of a short bench run and one --set full capture of the dominant kernel each.
O=gpurun_out/prof_c3c4; mkdir -p $O
python bench.py --config c3 --steps 3 --warmup 3 --cpu-seconds 0 > $O/c3_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:vbyte -c 12 --csv \
    --log-file $O/launches_c3.csv python bench.py --config c3 --steps 3 --warmup 3 --cpu-seconds 0 > $O/ncu_c3_list.log 2>&1
echo c3 list rc=$?
ncu --set full --clock-control none --import-source on -k regex:vbyte_lists -s 2 -c 1 -o $O/prof_c3 \
    python bench.py --config c3 --steps 3 --warmup 3 --cpu-seconds 0 > $O/ncu_c3_full.log 2>&1; echo c3 full rc=$?
cat > /tmp/c4run.py <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_1503_07387_b200 import mvb, workload as W
w = W.config4(n=1 << 27)
dev = torch.device("cuda", 0)
src = torch.from_numpy(w.encoded).to(dev); out = torch.empty(w.count, dtype=torch.int32, device=dev)
d = mvb.Decoder(dev, w.encoded.size)
for it in range(4): d.decode_delta(src, w.count, w.prev, out)
torch.cuda.synchronize()
assert np.array_equal(out.cpu().numpy().view(np.uint32), w.expected())
print("ok", d.result())
PY
python /tmp/c4run.py > $O/c4_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"seg_decode|seg_totals" -s 4 -c 2 -o $O/prof_c4s python /tmp/c4run.py > $O/ncu_c4_full.log 2>&1; echo c4 full rc=$?
ls -la $O
