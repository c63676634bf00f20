// Dependent-chain latencies (cycles/op) of the warp primitives on the selection critical path.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(unsigned* out, long long* cyc, int n) {
  unsigned v = threadIdx.x * 2654435761u;
  __shared__ unsigned long long sh[64];
  sh[threadIdx.x & 63] = v;
  __syncwarp();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) v = __reduce_min_sync(0xffffffffu, v ^ i) + threadIdx.x;
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) v = __ballot_sync(0xffffffffu, (v >> (i & 31)) & 1) + threadIdx.x;
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) v = __shfl_sync(0xffffffffu, v, (v + i) & 31);
  long long t3 = clock64();
  unsigned long long w = v;
  for (int i = 0; i < n; ++i) w = sh[(w + i) & 63];
  long long t4 = clock64();
  for (int i = 0; i < n; ++i) {  // full argmin of a 64-bit key: 2 redux + ballot + ffs + shfl
    const unsigned hi = (unsigned)(w >> 32), lo = (unsigned)w;
    const unsigned mh = __reduce_min_sync(0xffffffffu, hi);
    const unsigned ml = __reduce_min_sync(0xffffffffu, hi == mh ? lo : 0xffffffffu);
    const unsigned m = __ballot_sync(0xffffffffu, hi == mh && lo == ml);
    const int src = __ffs(m) - 1;
    w = __shfl_sync(0xffffffffu, w, src) * 6364136223846793005ull + threadIdx.x + i;
  }
  long long t5 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
  }
  out[threadIdx.x] = v + (unsigned)w;
}
int main() {
  unsigned* o; long long* c; cudaMalloc(&o, 4 * 1024); cudaMallocManaged(&c, 8 * 8);
  const char* names[] = {"redux.min.u32", "ballot", "shfl.idx", "lds.u64 chain", "argmin64 (2 redux+ballot+ffs+shfl)"};
  for (int rep = 0; rep < 2; ++rep) { k<<<1, 32>>>(o, c, 1000); cudaDeviceSynchronize(); }
  for (int i = 0; i < 5; ++i) printf("%-40s %.1f cycles/op\n", names[i], c[i] / 1000.0);
  return 0;
}
