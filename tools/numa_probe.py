"""H2D bandwidth of pinned host memory allocated before/after binding to the GPU's NUMA-local CPUs."""
import os, time, torch


def h2d_gbs(h, d, reps=20):
    s = torch.cuda.Stream()
    for _ in range(3):
        with torch.cuda.stream(s):
            d.copy_(h, non_blocking=True)
    s.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        with torch.cuda.stream(s):
            d.copy_(h, non_blocking=True)
    s.synchronize()
    return reps * h.numel() / (time.perf_counter() - t0) / 1e9


def gpu_cpus(dev=0):
    import pynvml
    pynvml.nvmlInit()
    hnd = pynvml.nvmlDeviceGetHandleByIndex(dev)
    words = pynvml.nvmlDeviceGetCpuAffinity(hnd, (os.cpu_count() + 63) // 64)
    return {w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1}


n = 17 << 20
d = torch.empty(n, dtype=torch.uint8, device="cuda")
print("cpus", os.cpu_count(), "affinity now", len(os.sched_getaffinity(0)))
h = torch.empty(n, dtype=torch.uint8).pin_memory()
print("before bind: %.1f GB/s" % h2d_gbs(h, d))
cpus = gpu_cpus()
print("gpu-local cpus:", len(cpus), min(cpus) if cpus else None, max(cpus) if cpus else None)
os.sched_setaffinity(0, cpus)
h2 = torch.empty(n, dtype=torch.uint8)
h2.fill_(1)
h2 = h2.pin_memory()
print("after bind (new buffer): %.1f GB/s" % h2d_gbs(h2, d))
print("after bind (old buffer): %.1f GB/s" % h2d_gbs(h, d))
