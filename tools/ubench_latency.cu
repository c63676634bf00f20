// Dependent-chain latency microbenchmark (cycles per op) for the ops on the selection
// critical path: DADD, DMUL, DDIV, DSETP+select, IADD64 compare+select, SHFL, LDS, bar.sync.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double x0, int n) {
  double x = x0 + threadIdx.x, y = 1.0000001;
  unsigned long long u = 12345 + threadIdx.x;
  __shared__ double sh[64];
  sh[threadIdx.x & 63] = x;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dadd_rn(x, y);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = __dmul_rn(x, y);
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) x = __ddiv_rn(x, y);
  long long t3 = clock64();
  for (int i = 0; i < n; ++i) x = (x < y) ? y : x - 1e-300;
  long long t4 = clock64();
  for (int i = 0; i < n; ++i) u = (u < 1000000ull) ? u + 3 : u - 7;
  long long t5 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1);
  long long t6 = clock64();
  int idx = threadIdx.x & 63;
  for (int i = 0; i < n; ++i) { x = sh[idx]; idx = ((int)x + i) & 63; }
  long long t7 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t8 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3;
    cyc[4] = t5 - t4; cyc[5] = t6 - t5; cyc[6] = t7 - t6; cyc[7] = t8 - t7;
  }
  out[threadIdx.x] = x + (double)u;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 1024); cudaMallocManaged(&c, 8 * 8);
  const char* names[] = {"dadd", "dmul", "ddiv", "dsetp+sel", "u64 cmp+sel", "shfl.f64", "lds.f64", "bar.sync(64thr)"};
  for (int rep = 0; rep < 2; ++rep) {
    k<<<1, 64>>>(o, c, 1.5, 1000);
    cudaDeviceSynchronize();
  }
  for (int i = 0; i < 8; ++i) printf("%-16s %.1f cycles/op\n", names[i], c[i] / 1000.0);
  return 0;
}
