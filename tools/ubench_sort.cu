// Standalone timing of the register bitonic sort used by the batch selector (2048 tuples, 256 threads).
#include <cstdio>
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>
struct BatchItem { uint64_t k, a; uint32_t o, meta; };
__device__ __forceinline__ bool item_better(const BatchItem& x, const BatchItem& y) {
  if (x.k != y.k) return x.k < y.k;
  if (x.a != y.a) return x.a < y.a;
  if (x.o != y.o) return x.o < y.o;
  return (x.meta & 0xffffffu) < (y.meta & 0xffffffu);
}
__device__ __forceinline__ BatchItem shfl_item(const BatchItem& x, int m) {
  BatchItem y;
  y.k = __shfl_xor_sync(0xffffffffu, x.k, m); y.a = __shfl_xor_sync(0xffffffffu, x.a, m);
  y.o = __shfl_xor_sync(0xffffffffu, x.o, m); y.meta = __shfl_xor_sync(0xffffffffu, x.meta, m);
  return y;
}
template <int P>
__device__ __noinline__ void sortr(BatchItem* items, int Tn) {
  const int tid = threadIdx.x;
  BatchItem x[P];
#pragma unroll
  for (int p = 0; p < P; ++p) x[p] = items[tid * P + p];
  for (int k = 2; k <= Tn; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j < P) {
        auto cx = [&](auto J) {
          constexpr int jj = decltype(J)::value;
#pragma unroll
          for (int p = 0; p < P; ++p) {
            const int q = p ^ jj;
            if (q > p) {
              const int i = tid * P + p; const bool up = (i & k) == 0;
              if (up ? item_better(x[q], x[p]) : item_better(x[p], x[q])) { BatchItem t = x[p]; x[p] = x[q]; x[q] = t; }
            }
          }
        };
        if (j == 1) cx(std::integral_constant<int, 1>{});
        if constexpr (P > 2) if (j == 2) cx(std::integral_constant<int, 2>{});
        if constexpr (P > 4) if (j == 4) cx(std::integral_constant<int, 4>{});
      } else if (j < 32 * P) {
        const int m = j / P; const bool lower = ((tid & 31) & m) == 0;
#pragma unroll
        for (int p = 0; p < P; ++p) {
          const BatchItem y = shfl_item(x[p], m);
          const int i = tid * P + p; const bool up = (i & k) == 0;
          const bool want_min = lower == up;
          if (want_min ? item_better(y, x[p]) : item_better(x[p], y)) x[p] = y;
        }
      } else {
        __syncthreads();
#pragma unroll
        for (int p = 0; p < P; ++p) items[tid * P + p] = x[p];
        __syncthreads();
#pragma unroll
        for (int p = 0; p < P; ++p) {
          const int i = tid * P + p, ixj = i ^ j; const BatchItem y = items[ixj];
          const bool up = (i & k) == 0; const bool want_min = (i < ixj) == up;
          if (want_min ? item_better(y, x[p]) : item_better(x[p], y)) x[p] = y;
        }
      }
    }
  __syncthreads();
#pragma unroll
  for (int p = 0; p < P; ++p) items[tid * P + p] = x[p];
  __syncthreads();
}
__global__ void kern(BatchItem* g, long long* cyc, int Tn) {
  extern __shared__ BatchItem sh[];
  for (int i = threadIdx.x; i < Tn; i += blockDim.x) sh[i] = g[i];
  __syncthreads();
  long long t0 = clock64();
  sortr<8>(sh, Tn);
  long long t1 = clock64();
  for (int i = threadIdx.x; i < Tn; i += blockDim.x) g[i] = sh[i];
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  const int Tn = 2048;
  BatchItem h[Tn];
  uint64_t s = 88172645463325252ull;
  for (int i = 0; i < Tn; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = {s, s * 3, (uint32_t)i, (uint32_t)i}; }
  BatchItem* d; long long* c; cudaMalloc(&d, sizeof(h)); cudaMallocManaged(&c, 8);
  for (int r = 0; r < 3; ++r) {
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    kern<<<1, 256, sizeof(h)>>>(d, c, Tn); cudaDeviceSynchronize();
    printf("sort 2048: %lld cycles (%s)\n", *c, cudaGetErrorString(cudaGetLastError()));
  }
  BatchItem o[Tn]; cudaMemcpy(o, d, sizeof(o), cudaMemcpyDeviceToHost);
  int ok = 1; for (int i = 1; i < Tn; ++i) if (o[i].k < o[i - 1].k) ok = 0;
  printf("sorted: %d\n", ok);
}
