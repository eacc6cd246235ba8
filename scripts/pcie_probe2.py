"""Chunked copy patterns without kernels: is the DMA itself slow when
H2D and D2H chunks interleave?"""
import time, torch
dev = torch.device("cuda", 0)
N_IN, N_OUT = 335 << 20, 268 << 20
h_in = torch.empty(N_IN, dtype=torch.uint8).pin_memory()
h_out = torch.empty(N_OUT, dtype=torch.uint8).pin_memory()
d_in = torch.empty(N_IN, dtype=torch.uint8, device=dev)
d_out = torch.empty(N_OUT, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timeit(fn, reps=5):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3
for C in (1, 8, 40, 160):
    ci, co = N_IN // C, N_OUT // C
    def h2d_only():
        with torch.cuda.stream(s1):
            for k in range(C): d_in[k*ci:(k+1)*ci].copy_(h_in[k*ci:(k+1)*ci], non_blocking=True)
    def d2h_only():
        with torch.cuda.stream(s2):
            for k in range(C): h_out[k*co:(k+1)*co].copy_(d_out[k*co:(k+1)*co], non_blocking=True)
    def piped():
        evs = []
        with torch.cuda.stream(s1):
            for k in range(C):
                d_in[k*ci:(k+1)*ci].copy_(h_in[k*ci:(k+1)*ci], non_blocking=True)
                e = torch.cuda.Event(); e.record(s1); evs.append(e)
        with torch.cuda.stream(s2):
            for k in range(C):
                s2.wait_event(evs[k])
                h_out[k*co:(k+1)*co].copy_(d_out[k*co:(k+1)*co], non_blocking=True)
    print(f"chunks {C:4d}: h2d {timeit(h2d_only):.2f} ms  d2h {timeit(d2h_only):.2f} ms  piped {timeit(piped):.2f} ms", flush=True)
