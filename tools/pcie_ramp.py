"""H2D bandwidth over time from an idle GPU: does the link ramp up under load?"""
import time, torch
n = 17 << 20
d = torch.empty(n, dtype=torch.uint8, device="cuda")
hs = [torch.empty(n, dtype=torch.uint8).pin_memory() for _ in range(2)]
s = torch.cuda.Stream()
torch.cuda.synchronize()
time.sleep(2.0)
t_start = time.perf_counter()
for b in range(40):
    t0 = time.perf_counter()
    for r in range(5):
        with torch.cuda.stream(s):
            d.copy_(hs[r % 2], non_blocking=True)
    s.synchronize()
    t1 = time.perf_counter()
    print("t=%7.1f ms  %.1f GB/s" % (1e3 * (t1 - t_start), 5 * n / (t1 - t0) / 1e9))
