"""PCIe pacing probe: 25 MB H2D + 67 MB D2H as N pieces; (a) all H2D queued
up front, D2H piece k after H2D piece k; (b) H2D piece k+L also waits for
D2H piece k (H2D paced by the output drain)."""
import time, torch
dev = torch.device("cuda", 0)
IN, OUT = 25 << 20, 67 << 20
h_in = torch.empty(IN, dtype=torch.uint8).pin_memory(); d_in = torch.empty(IN, dtype=torch.uint8, device=dev)
h_out = torch.empty(OUT, dtype=torch.uint8).pin_memory(); d_out = torch.empty(OUT, dtype=torch.uint8, device=dev)
sh, sd = torch.cuda.Stream(), torch.cuda.Stream()
def run(n, lead):
    ci, co = IN // n, OUT // n
    eh = [torch.cuda.Event() for _ in range(n)]; ed = [torch.cuda.Event() for _ in range(n)]
    for k in range(n):
        with torch.cuda.stream(sh):
            if lead is not None and k - lead >= 0: sh.wait_event(ed[k - lead])
            d_in[k*ci:(k+1)*ci].copy_(h_in[k*ci:(k+1)*ci], non_blocking=True); eh[k].record(sh)
        with torch.cuda.stream(sd):
            sd.wait_event(eh[k]); h_out[k*co:(k+1)*co].copy_(d_out[k*co:(k+1)*co], non_blocking=True); ed[k].record(sd)
def timeit(fn, reps=10):
    fn(); torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t) / reps * 1e6
for n in (8, 16, 32):
    res = [f"upfront {timeit(lambda: run(n, None)):.0f}"]
    for lead in (1, 2, 4):
        res.append(f"lead{lead} {timeit(lambda: run(n, lead)):.0f}")
    print(f"pieces {n:3d}: " + "  ".join(res) + " us")
