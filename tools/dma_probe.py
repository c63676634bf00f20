"""Does a small D2H on one stream wait behind a large H2D on another (shared DMA engine)?"""
import time, torch
h = torch.empty(17 << 20, dtype=torch.uint8).pin_memory()
d = torch.empty(17 << 20, dtype=torch.uint8, device="cuda")
small_d = torch.zeros(4096, dtype=torch.uint8, device="cuda")
small_h = torch.empty(4096, dtype=torch.uint8).pin_memory()
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
for trial in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(sa):
        d.copy_(h, non_blocking=True)
    t1 = time.perf_counter()
    with torch.cuda.stream(sb):
        small_h.copy_(small_d, non_blocking=True)
    sb.synchronize()
    t2 = time.perf_counter()
    sa.synchronize()
    t3 = time.perf_counter()
    print(f"issue {1e3*(t1-t0):.3f} small D2H done after {1e3*(t2-t0):.3f} ms, big H2D done {1e3*(t3-t0):.3f} ms")
# kernel concurrency with H2D
x = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for trial in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    with torch.cuda.stream(sa):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(sb):
        for _ in range(10): x.mul_(1.0001)
    sb.synchronize(); t2 = time.perf_counter(); sa.synchronize(); t3 = time.perf_counter()
    print(f"kernels done {1e3*(t2-t0):.3f} ms, H2D done {1e3*(t3-t0):.3f}")
