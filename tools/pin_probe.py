"""Per-buffer H2D bandwidth: torch pin_memory() buffers vs 2 MiB-aligned, MADV_HUGEPAGE, cudaHostRegister'ed ones."""
import ctypes, mmap, time, torch
import numpy as np

n = 17 << 20
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()


def gbs(h, reps=10):
    with torch.cuda.stream(s):
        d.copy_(h, non_blocking=True)
    s.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        with torch.cuda.stream(s):
            d.copy_(h, non_blocking=True)
    s.synchronize()
    return reps * n / (time.perf_counter() - t0) / 1e9


print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip(),
      open("/sys/kernel/mm/transparent_hugepage/defrag").read().strip())
for i in range(6):
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    print("pin_memory %d: %.1f GB/s" % (i, gbs(h)))
libc = ctypes.CDLL("libc.so.6", use_errno=True)
libc.madvise.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
cudart = ctypes.CDLL("libcudart.so.12") if False else None
keep = []
for i in range(6):
    size = (n + (2 << 20) - 1) // (2 << 20) * (2 << 20)
    m = mmap.mmap(-1, size + (2 << 20), flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    base = ctypes.addressof(ctypes.c_char.from_buffer(m))
    al = (base + (2 << 20) - 1) & ~((2 << 20) - 1)
    r = libc.madvise(ctypes.c_void_p(al), ctypes.c_size_t(size), 14)  # MADV_HUGEPAGE
    arr = np.frombuffer(m, dtype=np.uint8, count=size, offset=al - base)
    arr[:] = 1
    t = torch.from_numpy(arr)
    err = torch.cuda.cudart().cudaHostRegister(t.data_ptr(), size, 0)
    keep.append((m, arr, t))
    with open("/proc/self/smaps") as f:
        pass
    print("hugepage+register %d (madvise %d, reg %s): %.1f GB/s" % (i, r, err, gbs(t[:n])))
ah = [l for l in open("/proc/meminfo") if "AnonHuge" in l or "Hugepagesize" in l]
print("".join(ah))
