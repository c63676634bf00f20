// eqx_kernels.cu -- sm_100a kernels of the Equinox per-step scheduling path.
//
//   drain_arrivals (engine.cpp:171-197), two launches:
//     drain_hist_kernel  per-(tile, warp, client) counts and each client's first row
//     drain_rank_kernel  every CTA derives its segment offsets from the histogram, ranks its rows
//                        per client (stable), stages the tile client-sorted in shared memory and
//                        writes contiguous per-client runs -> perm (rows grouped by client, FIFO)
//   the counter lift (on_activated, scheduler.cpp:235-253): lift_core, in an extra CTA of the
//     window kernel (fused step) or lift_kernel (standalone drain)
//   admit_requests (engine.cpp:207-271):
//     window_kernel      the first W queued requests of every client scored into [C][W] heads
//     select_topk_kernel one CTA: rounds of block-radix top-K over per-client key streams
//                        (eqx_topk.cuh); writes every event with its payload and request id
//     score_kernel       whole-queue MoPE predict -> map_metrics -> ufc/rfc increments on a side
//                        stream (16-byte streaming loads / stores: the HBM-bound stream)
//   client-sharded step: shard_export / shard_ingest / shard_unpack kernels
//   live queues: live_offsets / gather_live / predict_rows kernels
//   feedback: feedback_kernel
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>
#include <cstdio>

#include "eqx_device.cuh"
#include "eqx_kernels.h"

namespace eqx {

namespace {

__device__ __forceinline__ int4 ldg_stream(const int4* p) {
  int4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ double2 ldg_stream(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t ldg_stream(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void stg_stream(int4* p, int4 v) {
  asm volatile("st.global.cs.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void stg_stream(double2* p, double2 v) {
  asm volatile("st.global.cs.v2.f64 [%0], {%1,%2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ void stg_stream(uint32_t* p, uint32_t v) {
  asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ufc/rfc increments of a queued request from its frozen prediction record (live queues).
__device__ __forceinline__ Scored score_frozen(const Frozen& F, int64_t row, const Policy& P, double now, int32_t in,
                                              double arrival, double w) {
  Scored s;
  s.fallback = 0;
  s.near_tie = 0;
  s.pred = F.pred[row];
  s.bucket = F.bucket[row];
  const double tokens = __dadd_rn(static_cast<double>(in), __dmul_rn(P.ow, static_cast<double>(s.pred)));
  const double denom = __dadd_rn(1.0, __dmul_rn(P.delta, __dadd_rn(__dsub_rn(now, arrival), F.pred_s[row])));
  s.ufc_inc = __ddiv_rn(__dmul_rn(w, tokens), denom);  // scheduler.cpp:21-26
  s.rfc_inc = F.rfc[row];
  return s;
}

// Programmatic dependent launch (sm_90+): wait for the predecessor grid's results / let the
// successor grid get scheduled early.  No-ops for kernels launched without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Copy the compiled model (header + the LUT words in use) into shared memory.
__device__ __forceinline__ void stage_model(const ModelTables* g, int words, unsigned char* smem) {
  const uint32_t* src = reinterpret_cast<const uint32_t*>(g);
  uint32_t* dst = reinterpret_cast<uint32_t*>(smem);
  for (int i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
}

// "Last CTA done" election: every CTA fences its global writes and bumps a counter; the CTA
// that brings it to gridDim.x runs the epilogue (and resets the counter for the next launch).
__device__ __forceinline__ bool last_cta(unsigned int* done) {
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(done, 1u) == gridDim.x - 1) ? 1 : 0;
  __syncthreads();
  if (s_last) __threadfence();
  return s_last != 0;
}

// Lanes holding the same key (the __match_any_sync result) from nbits ballots: MATCH.ANY
// serialises on sm_100, a ballot per key bit does not.  Keys must be < 2^nbits.
__device__ __forceinline__ unsigned peer_mask(uint32_t key, int nbits) {
  unsigned m = 0xffffffffu;
#pragma unroll 4
  for (int b = 0; b < nbits; ++b) {
    const bool bit = (key >> b) & 1u;
    const unsigned bb = __ballot_sync(0xffffffffu, bit);
    m &= bit ? bb : ~bb;
  }
  return m;
}

// peer_mask with the key width fixed at compile time (NB > 0): fully unrolled ballots; NB = 0
// keeps the runtime loop.
template <int NB>
__device__ __forceinline__ unsigned peer_mask_nb(uint32_t key, int nbits) {
  if constexpr (NB == 0) {
    return peer_mask(key, nbits);
  } else {
    unsigned m = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const unsigned bit = (key >> b) & 1u;
      const unsigned bb = __ballot_sync(0xffffffffu, bit);
      m &= bb ^ (bit - 1u);  // bit ? bb : ~bb
    }
    return m;
  }
}

// Block-wide exclusive scan of one uint32 per thread (blockDim.x <= 1024); returns the total.
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* out, uint32_t* warp_buf) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  uint32_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) warp_buf[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < nw ? warp_buf[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += t;
    }
    warp_buf[lane] = w;  // inclusive over warps
  }
  __syncthreads();
  *out = (warp ? warp_buf[warp - 1] : 0u) + incl - v;
  const uint32_t total = warp_buf[nw - 1];
  __syncthreads();
  return total;
}

}  // namespace

// ===================================== drain =============================================

// on_activated in arrival order for every client that goes idle -> backlogged in this drain.
// The lift target is the componentwise min over *other* backlogged clients at that moment.
// Lifted values are >= that min, so the running min only moves when a client that is NOT
// lifted joins the backlog: pre-backlogged clients (qlen_before > 0), the very first arrival
// when nobody was backlogged, and clients with running requests (engine.cpp:182).  Hence
// m(c) = min(base, {vals(r) : r non-lifted arrival, first_row[r] < first_row[c]}).
// Arrival keys are drain rows (one queue) or global trace positions (client-sharded step,
// where the clients' first arrivals live on different ranks).
struct LiftIn {
  int32_t C;
  int32_t counter_lift;
  const int32_t* count;
  const int32_t* qlen_before;
  const int32_t* running;
  double* ufc;
  double* rfc;
  double* counter;
  int32_t* backlogged;
};

template <class Key>
__device__ void lift_core(const LiftIn& a, const Key* first_row) {
  __shared__ double s_min[3][32];
  __shared__ Key s_first[32];
  __shared__ int s_firstc[32], s_flags[32];
  const int32_t C = a.C;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const Key kNone = sizeof(Key) == 8 ? static_cast<Key>(0x7fffffffffffffffLL) : static_cast<Key>(0x7fffffff);
  if (a.counter_lift) {
    double mu = INFINITY, mr = INFINITY, mc = INFINITY;
    int any0 = 0, anyR = 0;
    Key fr = kNone;
    int fc = -1;
    const int NT = blockDim.x;
    for (int c0 = tid; c0 < C; c0 += 4 * NT) {  // 4 clients' loads in flight
      int32_t cnt[4], qb[4], run[4];
      double u[4], r[4], k[4];
      Key f[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = c0 + j * NT;
        const bool in = c < C;
        cnt[j] = in ? a.count[c] : 0;
        qb[j] = in ? a.qlen_before[c] : 0;
        run[j] = in ? a.running[c] : 0;
        u[j] = in ? a.ufc[c] : 0.0;
        r[j] = in ? a.rfc[c] : 0.0;
        k[j] = in ? a.counter[c] : 0.0;
        f[j] = in ? first_row[c] : kNone;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (qb[j] > 0) {
          any0 = 1;
          mu = fmin(mu, u[j]);
          mr = fmin(mr, r[j]);
          mc = fmin(mc, k[j]);
        } else if (cnt[j] > 0 && run[j] != 0) {
          anyR = 1;
        }
        if (cnt[j] > 0 && f[j] < fr) {
          fr = f[j];
          fc = c0 + j * NT;
        }
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      mu = fmin(mu, __shfl_xor_sync(0xffffffffu, mu, o));
      mr = fmin(mr, __shfl_xor_sync(0xffffffffu, mr, o));
      mc = fmin(mc, __shfl_xor_sync(0xffffffffu, mc, o));
      any0 |= __shfl_xor_sync(0xffffffffu, any0, o);
      anyR |= __shfl_xor_sync(0xffffffffu, anyR, o);
      const Key ofr = __shfl_xor_sync(0xffffffffu, fr, o);
      const int ofc = __shfl_xor_sync(0xffffffffu, fc, o);
      if (ofr < fr) {
        fr = ofr;
        fc = ofc;
      }
    }
    if (lane == 0) {
      s_min[0][warp] = mu;
      s_min[1][warp] = mr;
      s_min[2][warp] = mc;
      s_first[warp] = fr;
      s_firstc[warp] = fc;
      s_flags[warp] = any0 | (anyR << 1);
    }
    __syncthreads();
    double bu = INFINITY, br = INFINITY, bc = INFINITY;
    Key f0 = kNone;
    int fc0 = -1, flags = 0;
    for (int w = 0; w < nw; ++w) {
      bu = fmin(bu, s_min[0][w]);
      br = fmin(br, s_min[1][w]);
      bc = fmin(bc, s_min[2][w]);
      flags |= s_flags[w];
      if (s_first[w] < f0) {
        f0 = s_first[w];
        fc0 = s_firstc[w];
      }
    }
    const bool any_s0 = flags & 1, any_r = flags & 2;
    if (!any_s0 && fc0 >= 0) {
      bu = a.ufc[fc0];
      br = a.rfc[fc0];
      bc = a.counter[fc0];
    }
    __syncthreads();  // everyone has read the base before any lift is written
    if ((any_s0 || fc0 >= 0) && !any_r) {  // the common case: one base for every lifted client
      const int NT = blockDim.x;
      for (int c0 = tid; c0 < C; c0 += 4 * NT) {  // 4 clients' loads in flight
        int32_t cnt[4], qb[4], run[4];
        double u[4], r[4], k[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int c = c0 + j * NT;
          const bool in = c < C;
          cnt[j] = in ? a.count[c] : 0;
          qb[j] = in ? a.qlen_before[c] : 0;
          run[j] = in ? a.running[c] : 0;
          u[j] = in ? a.ufc[c] : 0.0;
          r[j] = in ? a.rfc[c] : 0.0;
          k[j] = in ? a.counter[c] : 0.0;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int c = c0 + j * NT;
          if (cnt[j] == 0 || qb[j] > 0 || run[j] != 0) continue;
          if (!any_s0 && c == fc0) continue;
          // std::max(own, min): own unless own < min
          if (u[j] < bu) a.ufc[c] = bu;
          if (r[j] < br) a.rfc[c] = br;
          if (k[j] < bc) a.counter[c] = bc;
        }
      }
    } else if (any_s0 || fc0 >= 0) {
      for (int c = tid; c < C; c += blockDim.x) {
        if (a.count[c] == 0 || a.qlen_before[c] > 0 || a.running[c] != 0) continue;
        if (!any_s0 && c == fc0) continue;
        double u = bu, r = br, k = bc;
        if (any_r) {
          const Key fcr = first_row[c];
          for (int x = 0; x < C; ++x) {  // non-lifted arrivals before c
            if (a.count[x] == 0 || a.qlen_before[x] > 0 || a.running[x] == 0) continue;
            if (first_row[x] < fcr) {
              u = fmin(u, a.ufc[x]);
              r = fmin(r, a.rfc[x]);
              k = fmin(k, a.counter[x]);
            }
          }
        }
        // std::max(own, min): own unless own < min
        if (a.ufc[c] < u) a.ufc[c] = u;
        if (a.rfc[c] < r) a.rfc[c] = r;
        if (a.counter[c] < k) a.counter[c] = k;
      }
    }
  }
  {
    const int NT = blockDim.x;
    for (int c0 = tid; c0 < C; c0 += 4 * NT) {
      int32_t v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = c0 + j * NT;
        v[j] = c < C ? a.qlen_before[c] + a.count[c] : 0;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (c0 + j * NT < C) a.backlogged[c0 + j * NT] = v[j] > 0 ? 1 : 0;
    }
  }
}

// on_activated / set_backlogged for a drained queue (counts from drain_rank_kernel, first
// rows from drain_hist_kernel): a standalone eqx_drain, or the selection kernel's prologue.
__global__ void __launch_bounds__(1024) lift_kernel(const DrainArgs a) {
  const LiftIn l{a.C, a.counter_lift, a.count, a.qlen_before, a.running, a.ufc, a.rfc, a.counter, a.backlogged};
  lift_core<int32_t>(l, a.first_row);
}

#ifdef EQX_PROF
#define EQX_DT_MIN(i) do { if (threadIdx.x == 0) atomicMin(&a.st->dt[i], global_ns()); } while (0)
#define EQX_DT_MAX(i) do { if (threadIdx.x == 0) atomicMax(&a.st->dt[i], global_ns()); } while (0)
#else
#define EQX_DT_MIN(i) do {} while (0)
#define EQX_DT_MAX(i) do {} while (0)
#endif

template <int NB>
__device__ __forceinline__ void drain_hist_body(const DrainArgs& a) {
  extern __shared__ __align__(16) uint32_t sh[];
  EQX_DT_MIN(0);
  pdl_trigger();
  const int32_t C = a.C;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint16_t* wc = reinterpret_cast<uint16_t*>(sh);  // [kDrainWarps][C]
  uint32_t* fr = sh + (kDrainWarps * C + 1) / 2;    // [C] first row of each client in the tile
  for (int i = tid; i < kDrainWarps * C; i += blockDim.x) wc[i] = 0;
  for (int c = tid; c < C; c += blockDim.x) fr[c] = 0xffffffffu;
  __syncthreads();
  const int32_t tile = blockIdx.x;
  const int32_t sub = a.tile_rows / kDrainWarps;
  const int32_t r0 = tile * a.tile_rows + warp * sub;
  const int32_t r1 = min(a.n, r0 + sub);
  uint16_t* my = wc + warp * C;
  bool bad = false;
  for (int32_t rb = r0; rb < r1; rb += 32 * 8) {  // 8 loads in flight per lane, then walk
    int32_t cv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int32_t row = rb + 32 * u + lane;
      cv[u] = row < r1 ? a.client[row] : -1;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {  // per-warp counts: one writer per (warp, client)
      const int32_t row = rb + 32 * u + lane;
      const int32_t c = cv[u];
      const bool ok = static_cast<uint32_t>(c) < static_cast<uint32_t>(C);
      bad |= row < r1 && !ok;
      const unsigned peers = peer_mask_nb<NB>(ok ? static_cast<uint32_t>(c) : static_cast<uint32_t>(C), a.cbits);
      if (ok && lane == __ffs(peers) - 1) {  // the earliest row of the client in these 32
        if (my[c] == 0) atomicMin(&fr[c], static_cast<uint32_t>(row));
        my[c] = static_cast<uint16_t>(my[c] + __popc(peers));
      }
      __syncwarp();
    }
  }
  if (bad) a.st->bad_client = 1;
  __syncthreads();
  for (int c = tid; c < C; c += blockDim.x) a.tfirst[static_cast<int64_t>(tile) * C + c] = fr[c];
  uint16_t* g = a.wcnt + static_cast<int64_t>(tile) * kDrainWarps * C;
  for (int i = tid; i < kDrainWarps * C; i += blockDim.x) g[i] = wc[i];
  for (int c = tid; c < C; c += blockDim.x) {
    uint32_t t = 0;
#pragma unroll 8
    for (int w = 0; w < kDrainWarps; ++w) t += wc[w * C + c];
    a.hist[static_cast<int64_t>(tile) * C + c] = t;  // [tile][client]: drain_scan_kernel's lanes read adjacent clients
  }
  EQX_DT_MAX(1);
}

// The client-key width selects an unrolled peer-mask instantiation (rosters up to 255 clients),
// else the runtime loop.
#define EQX_NB_DISPATCH(BODY)                     \
  switch (a.cbits) {                              \
    case 1: BODY<1>(a); break;                    \
    case 2: BODY<2>(a); break;                    \
    case 3: BODY<3>(a); break;                    \
    case 4: BODY<4>(a); break;                    \
    case 5: BODY<5>(a); break;                    \
    case 6: BODY<6>(a); break;                    \
    case 7: BODY<7>(a); break;                    \
    case 8: BODY<8>(a); break;                    \
    default: BODY<0>(a); break;                   \
  }

__global__ void __launch_bounds__(kDrainThreads) drain_hist_kernel(const DrainArgs a) { EQX_NB_DISPATCH(drain_hist_body) }

// ---- small rosters (C <= kSortMaxClients): per-tile stable counting sort ----------------------
// Thread t owns rows t*8 .. t*8+7 of the tile (in registers).  Counters cnt[c][t] (u16, one
// word of padding per 64 so the raking scan below is conflict-free) count its rows per client;
// the exclusive scan of the counters in (client, thread) order gives every row its slot in the
// client-sorted tile, stable because threads own ascending row ranges.  The tile leaves as
// (client << 16 | tile row) words plus the per-client tile counts; drain_scan_kernel and
// drain_scatter_kernel turn them into perm.  One read of the client column per row.
__global__ void __launch_bounds__(kSortThreads) drain_sort_kernel(const DrainArgs a) {
  extern __shared__ __align__(16) uint32_t sh[];
  EQX_DT_MIN(0);
  pdl_trigger();
  const int32_t C = a.C, Cp = C + (C & 1);  // counter rows padded to even: raking reads word pairs
  const int tid = threadIdx.x;
  const int32_t t0 = blockIdx.x * kSortTile;
  const int32_t rows = min(kSortTile, a.n - t0);
  const int L = Cp * kSortThreads;
  uint16_t* cnt = reinterpret_cast<uint16_t*>(sh);
  const int cwords = (sort_pad(L) + 1) / 2;
  uint32_t* srow = sh + ((cwords + 3) & ~3);
  __shared__ uint32_t warp_buf[32];
  __shared__ uint32_t cstart[kSortMaxClients + 1];
  for (int i = tid; i < cwords; i += kSortThreads) sh[i] = 0u;
  int32_t cv[kSortRows];
  const int32_t r0 = tid * kSortRows;
  if (r0 + kSortRows <= rows) {  // 4 x 16-byte loads
#pragma unroll
    for (int q = 0; q < kSortRows / 4; ++q) {
      const int4 v = ldg_stream(reinterpret_cast<const int4*>(a.client + t0 + r0) + q);
      cv[4 * q] = v.x;
      cv[4 * q + 1] = v.y;
      cv[4 * q + 2] = v.z;
      cv[4 * q + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < kSortRows; ++j) cv[j] = r0 + j < rows ? a.client[t0 + r0 + j] : -1;
  }
  __syncthreads();
  bool bad = false;
#pragma unroll
  for (int j = 0; j < kSortRows; ++j) {
    const int32_t c = cv[j];
    if (static_cast<uint32_t>(c) < static_cast<uint32_t>(C)) {
      cnt[sort_pad(c * kSortThreads + tid)] += 1;
    } else {
      bad |= r0 + j < rows;
      cv[j] = -1;
    }
  }
  if (bad) a.st->bad_client = 1;
  __syncthreads();
  {  // exclusive scan of the counters in (client, thread) order: thread t rakes entries
     // [t Cp, t Cp + Cp) as Cp / 2 words (an even entry and its successor share a word),
     // 8 independent loads at a time
    const int w0 = tid * (Cp / 2), nw = Cp / 2;
    auto waddr = [&](int w) { return (w + ((2 * w) >> 6)); };  // word index of entries 2w, 2w + 1
    uint32_t s = 0;
    for (int k = 0; k < nw; k += 8) {
      uint32_t v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = k + u < nw ? sh[waddr(w0 + k + u)] : 0u;
#pragma unroll
      for (int u = 0; u < 8; ++u) s += (v[u] & 0xffffu) + (v[u] >> 16);
    }
    uint32_t run;
    block_exclusive_scan(s, &run, warp_buf);
    for (int k = 0; k < nw; k += 8) {
      uint32_t v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = k + u < nw ? sh[waddr(w0 + k + u)] : 0u;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t lo = run;
        run += v[u] & 0xffffu;
        const uint32_t hi = run;
        run += v[u] >> 16;
        if (k + u < nw) sh[waddr(w0 + k + u)] = lo | (hi << 16);
      }
    }
  }
  __syncthreads();
  if (tid <= C) cstart[tid] = tid < C ? cnt[sort_pad(tid * kSortThreads)] : 0xffffffffu;
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kSortRows; ++j) {  // walk 2: rows into their slots
    const int32_t c = cv[j];
    if (c >= 0) {
      const int p = sort_pad(c * kSortThreads + tid);
      const uint32_t slot = cnt[p];
      cnt[p] = static_cast<uint16_t>(slot + 1);
      srow[slot] = (static_cast<uint32_t>(c) << 16) | static_cast<uint32_t>(r0 + j);
    }
  }
  __syncthreads();
  // per-client tile counts (the start of the next client, or the number of valid rows) and first rows
  const uint32_t nvalid = cnt[sort_pad((Cp - 1) * kSortThreads + kSortThreads - 1)];
  if (tid < C) {
    const uint32_t st = cstart[tid];
    const uint32_t en = tid + 1 < C ? cstart[tid + 1] : nvalid;
    a.hist[static_cast<int64_t>(blockIdx.x) * C + tid] = en - st;
    a.tfirst[static_cast<int64_t>(blockIdx.x) * C + tid] =
        en > st ? static_cast<uint32_t>(t0) + (srow[st] & 0xffffu) : 0xffffffffu;
  }
  for (int i = tid; i < static_cast<int>(nvalid); i += kSortThreads) a.tsorted[t0 + i] = srow[i];
  EQX_DT_MAX(1);
}

// Sorted tiles -> perm: each tile's client runs go to segment start + rows of the client in
// earlier tiles (drain_scan_kernel) + offset in the run.  Tile 0 writes seg_off / count.
__global__ void __launch_bounds__(kSortThreads) drain_scatter_kernel(const DrainArgs a) {
  __shared__ uint32_t base[kSortMaxClients], toff[kSortMaxClients];
  __shared__ uint32_t warp_buf[32];
  EQX_DT_MIN(3);
  pdl_wait();     // drain_scan_kernel (and through it drain_sort_kernel) is complete
  pdl_trigger();  // the window kernel may get scheduled
  const int32_t C = a.C, tile = blockIdx.x;
  const int tid = threadIdx.x;
  const int32_t t0 = tile * kSortTile;
  uint32_t tot = 0, h = 0, tb = 0;
  if (tid < C) {
    tot = __ldcg(a.ctot + tid);
    h = __ldcg(a.hist + static_cast<int64_t>(tile) * C + tid);
    tb = __ldcg(a.tbase + static_cast<int64_t>(tile) * C + tid);
  }
  uint32_t seg, loc;
  const uint32_t total = block_exclusive_scan(tot, &seg, warp_buf);
  const uint32_t nvalid = block_exclusive_scan(h, &loc, warp_buf);
  if (tid < C) {
    base[tid] = seg + tb;
    toff[tid] = loc;
    if (tile == 0) {
      a.seg_off[tid] = static_cast<int32_t>(seg);
      a.count[tid] = static_cast<int32_t>(tot);
    }
  }
  if (tile == 0 && tid == 0) a.seg_off[C] = static_cast<int32_t>(total);
  __syncthreads();
  uint32_t v[kSortRows];  // every load in flight before the stores
#pragma unroll
  for (int j = 0; j < kSortRows; ++j) {
    const int i = tid + j * kSortThreads;
    v[j] = i < static_cast<int>(nvalid) ? __ldcg(a.tsorted + t0 + i) : 0u;
  }
#pragma unroll
  for (int j = 0; j < kSortRows; ++j) {
    const int i = tid + j * kSortThreads;
    if (i < static_cast<int>(nvalid)) {
      const uint32_t c = v[j] >> 16;
      a.perm[base[c] + (static_cast<uint32_t>(i) - toff[c])] = static_cast<uint32_t>(t0) + (v[j] & 0xffffu);
    }
  }
  EQX_DT_MAX(4);
}

// Per-client prefix over tiles of the drain histogram, once for the whole batch: CTA b owns
// clients 32b..32b+31 (one per lane); its 32 warps split the tiles into contiguous chunks,
// sum them, exchange the chunk sums through shared memory and write every tile's exclusive
// prefix.  tbase[t][c] = rows of client c in tiles < t, ctot[c] = rows of client c; also the
// client's first row (min over the tiles' first rows) and the reset queue heads, so the drain
// needs no memset in front of it.
__global__ void __launch_bounds__(1024) drain_scan_kernel(const DrainArgs a) {
  __shared__ uint32_t part[32][33], pfirst[32][33];
  pdl_wait();     // drain_hist_kernel's histogram is complete
  pdl_trigger();  // drain_rank_kernel may get scheduled
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int32_t C = a.C, nt = a.n_tiles;
  const int32_t c = blockIdx.x * 32 + lane;
  const int32_t per = (nt + 31) / 32;
  const int32_t t0 = min(nt, warp * per), t1 = min(nt, t0 + per);
  uint32_t h[8];  // up to 8 tiles per warp in registers (per <= 8 for <= 256 tiles), else re-read
  uint32_t sum = 0, fmin = 0xffffffffu;
  if (c < C) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      h[u] = t0 + u < t1 ? __ldcg(a.hist + static_cast<int64_t>(t0 + u) * C + c) : 0u;
      const uint32_t f = t0 + u < t1 ? __ldcg(a.tfirst + static_cast<int64_t>(t0 + u) * C + c) : 0xffffffffu;
      sum += h[u];
      fmin = min(fmin, f);
    }
    for (int32_t t = t0 + 8; t < t1; ++t) {
      sum += __ldcg(a.hist + static_cast<int64_t>(t) * C + c);
      fmin = min(fmin, __ldcg(a.tfirst + static_cast<int64_t>(t) * C + c));
    }
  }
  part[warp][lane] = sum;
  pfirst[warp][lane] = fmin;
  __syncthreads();
  uint32_t run = 0, tot = 0, first = 0xffffffffu;
  for (int w = 0; w < 32; ++w) {
    const uint32_t v = part[w][lane];
    run += w < warp ? v : 0u;
    tot += v;
    first = min(first, pfirst[w][lane]);
  }
  if (c < C) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (t0 + u < t1) {
        a.tbase[static_cast<int64_t>(t0 + u) * C + c] = run;
        run += h[u];
      }
    }
    for (int32_t t = t0 + 8; t < t1; ++t) {
      a.tbase[static_cast<int64_t>(t) * C + c] = run;
      run += __ldcg(a.hist + static_cast<int64_t>(t) * C + c);
    }
    if (warp == 0) {
      a.ctot[c] = tot;
      a.first_row[c] = static_cast<int32_t>(first);
      a.head[c] = 0;
      if (a.zero_qlen) a.qlen_before[c] = 0;
    }
  }
}



// Stable scatter of row indices into per-client FIFO segments.  Each CTA owns one tile; each
// of its 8 warps walks a contiguous sub-tile 32 rows at a time in row order, ranking rows of
// the same client (ballot peer masks).  Walk 1 counts per (warp, client); scans over warps
// and clients give every row its slot in a client-sorted copy of the tile in shared memory
// (walk 2), which is then written to perm as contiguous per-client runs (coalesced).
template <int NB>
__device__ __forceinline__ void drain_rank_body(const DrainArgs& a) {
  extern __shared__ __align__(16) uint32_t sh[];
  EQX_DT_MIN(3);
  const int32_t C = a.C;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int32_t tile = blockIdx.x;
  const int32_t sub = a.tile_rows / kDrainWarps;
  const int32_t t0 = tile * a.tile_rows;
  const int32_t t1 = min(a.n, t0 + a.tile_rows);
  const int32_t r0 = t0 + warp * sub;
  const int32_t r1 = min(a.n, r0 + sub);
  const unsigned lt = (1u << lane) - 1u;
  uint32_t* base = sh;                                     // [C] global start of this tile's run
  uint32_t* toff = sh + C;                                 // [C] tile-local start / totals
  uint16_t* wc = reinterpret_cast<uint16_t*>(sh + 2 * C);  // [kDrainWarps][C]
  pdl_wait();     // drain_scan_kernel (and through it drain_hist_kernel) is complete
  pdl_trigger();  // the window kernel may get scheduled
  {  // per-warp client counts from drain_hist_kernel's walk (4 independent L2 loads in flight)
    const uint16_t* g = a.wcnt + static_cast<int64_t>(tile) * kDrainWarps * C;
    const int nwc = kDrainWarps * C, NT = blockDim.x;
    for (int i0 = tid; i0 < nwc; i0 += 4 * NT) {
      uint16_t v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = i0 + u * NT < nwc ? __ldcg(g + i0 + u * NT) : uint16_t(0);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (i0 + u * NT < nwc) wc[i0 + u * NT] = v[u];
    }
  }
  // global offsets: segment start of the client (exclusive scan of the per-client totals) +
  // its rows in earlier tiles (drain_scan_kernel)
  {
    __shared__ uint32_t warp_buf[32];
    const int per = (C + blockDim.x - 1) / blockDim.x;
    const int c0 = min(C, per * tid), c1 = min(C, c0 + per);
    uint32_t s = 0;
    for (int c = c0; c < c1; ++c) {
      const uint32_t t = __ldcg(a.ctot + c);
      toff[c] = t;
      s += t;
    }
    uint32_t run;
    const uint32_t total = block_exclusive_scan(s, &run, warp_buf);
    const uint32_t* tb = a.tbase + static_cast<int64_t>(tile) * C;
    for (int c = c0; c < c1; ++c) {
      const uint32_t t = toff[c];
      if (tile == 0) {
        a.seg_off[c] = static_cast<int32_t>(run);
        a.count[c] = static_cast<int32_t>(t);
      }
      base[c] = run + __ldcg(tb + c);
      run += t;
    }
    if (tile == 0 && tid == 0) a.seg_off[C] = static_cast<int32_t>(total);
  }
  __syncthreads();
  uint16_t* my = wc + warp * C;
  for (int c = tid; c < C; c += blockDim.x) {  // exclusive over warps; total per client
    uint32_t run = 0;
#pragma unroll 8
    for (int w = 0; w < kDrainWarps; ++w) {
      const uint32_t t = wc[w * C + c];
      wc[w * C + c] = static_cast<uint16_t>(run);
      run += t;
    }
    toff[c] = run;
  }
  __syncthreads();
  if (a.staged) {
    // tile-local client offsets: exclusive scan of per-client totals
    __shared__ uint32_t warp_buf[32];
    const int per = (C + blockDim.x - 1) / blockDim.x;
    const int c0 = min(C, per * tid), c1 = min(C, c0 + per);
    uint32_t s = 0;
    for (int c = c0; c < c1; ++c) s += toff[c];
    uint32_t run;
    block_exclusive_scan(s, &run, warp_buf);
    for (int c = c0; c < c1; ++c) {
      const uint32_t t = toff[c];
      toff[c] = run;
      run += t;
    }
    __syncthreads();
    uint32_t* srow = sh + 2 * C + (kDrainWarps / 2) * C;             // [tile_rows]
    uint16_t* scl = reinterpret_cast<uint16_t*>(srow + a.tile_rows);  // [tile_rows]
    for (int32_t rb = r0; rb < r1; rb += 32 * 8) {  // walk 2: slot in the client-sorted tile
      int32_t cv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int32_t row = rb + 32 * u + lane;
        cv[u] = row < r1 ? a.client[row] : -1;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int32_t row = rb + 32 * u + lane;
        const int32_t c = cv[u];
        const bool ok = static_cast<uint32_t>(c) < static_cast<uint32_t>(C);
        const unsigned peers = peer_mask_nb<NB>(ok ? static_cast<uint32_t>(c) : static_cast<uint32_t>(C), a.cbits);
        const int leader = __ffs(peers) - 1;
        uint32_t start = 0;
        if (ok && lane == leader) {
          start = my[c];
          my[c] = static_cast<uint16_t>(start + __popc(peers));
        }
        start = __shfl_sync(0xffffffffu, start, leader);
        if (ok) {
          const uint32_t slot = toff[c] + start + __popc(peers & lt);
          srow[slot] = static_cast<uint32_t>(row);
          scl[slot] = static_cast<uint16_t>(c);
        }
        __syncwarp();
      }
    }
    __syncthreads();
    const int32_t rows = t1 - t0;
    for (int32_t i = tid; i < rows; i += blockDim.x) {  // contiguous per-client runs
      const int32_t c = scl[i];
      a.perm[base[c] + (i - toff[c])] = srow[i];
    }
  } else {
    for (int32_t r = r0; r < r1; r += 32) {  // walk 2: direct scatter (large rosters)
      const int32_t row = r + lane;
      const int32_t c = row < r1 ? a.client[row] : -1;
      const bool ok = static_cast<uint32_t>(c) < static_cast<uint32_t>(C);
      const unsigned peers = peer_mask_nb<NB>(ok ? static_cast<uint32_t>(c) : static_cast<uint32_t>(C), a.cbits);
      const int leader = __ffs(peers) - 1;
      uint32_t start = 0;
      if (ok && lane == leader) {
        start = my[c];
        my[c] = static_cast<uint16_t>(start + __popc(peers));
      }
      start = __shfl_sync(0xffffffffu, start, leader);
      if (ok) a.perm[base[c] + start + __popc(peers & lt)] = static_cast<uint32_t>(row);
      __syncwarp();
    }
  }
  EQX_DT_MAX(4);
}

__global__ void __launch_bounds__(kDrainThreads) drain_rank_kernel(const DrainArgs a) { EQX_NB_DISPATCH(drain_rank_body) }

// ===================================== scoring ===========================================

// A scoring CTA's length-fallback and near-tie counts (fb, nt: warp totals in lane 0; every
// thread of the CTA calls this).  Without a publication target they are added to DevState.
// With one (a.done: the step's selection CTA publishes DevState, see SelectArgs::h_st), thread 0
// adds the CTA's totals to two 64-bit words that also count the CTAs above bit 40: one relaxed
// atomic carries the data and the completion count together, so the selection knows the totals
// are final once both counts reach the grid size -- no fence behind the CTA's output stores.
__device__ __forceinline__ void score_counts(const ScoreArgs& a, uint32_t fb, uint32_t nt) {
  if (!a.done) {
    if ((threadIdx.x & 31) == 0) {
      if (fb) atomicAdd(&a.st->fallbacks, static_cast<unsigned long long>(fb));
      if (nt) atomicAdd(&a.st->near_ties, static_cast<unsigned long long>(nt));
    }
    return;
  }
  __shared__ uint32_t s_fb[32], s_nt[32];
  if ((threadIdx.x & 31) == 0) {
    s_fb[threadIdx.x >> 5] = fb;
    s_nt[threadIdx.x >> 5] = nt;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long f = 0, t = 0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
      f += s_fb[w];
      t += s_nt[w];
    }
#ifdef EQX_PROF
    atomicMax(&a.st->t[5], global_ns());
    __threadfence();  // the timeline stamps before the count
#endif
    atomicAdd(a.done, f + kScoreCtaOne);
    atomicAdd(a.done + 1, t + kScoreCtaOne);
  }
}

// Whole-queue scoring: 4 requests per thread per iteration through 16-byte loads of every
// column, predict + map_metrics through the direct table (read-only cache), FP64 increments,
// streaming stores of pred/bucket/ufc_inc/rfc_inc.
template <int KIND>
__device__ __forceinline__ void score_body(const ScoreArgs& a, const ModelTables& M) {
  const int64_t n = a.n;
  uint32_t fb = 0, nt = 0;
  constexpr bool oracle_like = KIND == kPredOracle || KIND == kPredNoisy;
  const int64_t nvec = a.vec_ok ? n / 4 : 0;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  // software-pipelined: the next vector's loads are in flight while this one is scored
  struct Vec {
    int4 cl, in4, to;
    double2 a01, a23;
    uint32_t tg;
  };
  auto load = [&](int64_t v) {
    Vec x;
    x.cl = ldg_stream(reinterpret_cast<const int4*>(a.client) + v);
    x.in4 = ldg_stream(reinterpret_cast<const int4*>(a.in_tok) + v);
    x.a01 = ldg_stream(reinterpret_cast<const double2*>(a.arrival) + 2 * v);
    x.a23 = ldg_stream(reinterpret_cast<const double2*>(a.arrival) + 2 * v + 1);
    x.tg = ldg_stream(reinterpret_cast<const uint32_t*>(a.tag) + v);
    x.to = oracle_like ? ldg_stream(reinterpret_cast<const int4*>(a.true_out) + v) : make_int4(1, 1, 1, 1);
    return x;
  };
  int64_t v = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  Vec nx{};
  if (v < nvec) nx = load(v);
  for (; v < nvec; v += stride) {
    const Vec x = nx;
    if (v + stride < nvec) nx = load(v + stride);
    const int4 cl = x.cl, in4 = x.in4, to = x.to;
    const double2 a01 = x.a01, a23 = x.a23;
    const uint32_t tg = x.tg;
    const int64_t r0 = 4 * v;
    const int cs[4] = {cl.x, cl.y, cl.z, cl.w};
    const int ins[4] = {in4.x, in4.y, in4.z, in4.w};
    const int tos[4] = {to.x, to.y, to.z, to.w};
    const double arr[4] = {a01.x, a01.y, a23.x, a23.y};
    Scored s[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t id = (KIND == kPredNoisy && a.id) ? a.id[r0 + k] : a.id_base + r0 + k;
      const double w = __ldg(a.weight + cs[k]);
      s[k] = score_request_direct<KIND>(M, a.pol, a.direct, a.direct_n, a.now, ins[k], (tg >> (8 * k)) & 0xffu, tos[k],
                                        id, arr[k], w);
      fb += s[k].fallback;
      nt += s[k].near_tie;
    }
    stg_stream(reinterpret_cast<int4*>(a.pred_out) + v, make_int4(s[0].pred, s[1].pred, s[2].pred, s[3].pred));
    stg_stream(reinterpret_cast<uint32_t*>(a.bucket_out) + v,
               static_cast<uint32_t>(s[0].bucket) | (static_cast<uint32_t>(s[1].bucket) << 8) |
                   (static_cast<uint32_t>(s[2].bucket) << 16) | (static_cast<uint32_t>(s[3].bucket) << 24));
    stg_stream(reinterpret_cast<double2*>(a.ufc_out) + 2 * v, make_double2(s[0].ufc_inc, s[1].ufc_inc));
    stg_stream(reinterpret_cast<double2*>(a.ufc_out) + 2 * v + 1, make_double2(s[2].ufc_inc, s[3].ufc_inc));
    stg_stream(reinterpret_cast<double2*>(a.rfc_out) + 2 * v, make_double2(s[0].rfc_inc, s[1].rfc_inc));
    stg_stream(reinterpret_cast<double2*>(a.rfc_out) + 2 * v + 1, make_double2(s[2].rfc_inc, s[3].rfc_inc));
  }
  for (int64_t r = 4 * nvec + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < n; r += stride) {
    const int32_t c = a.client[r];
    const int64_t id = a.id ? a.id[r] : a.id_base + r;
    const Scored s = score_request_direct<KIND>(M, a.pol, a.direct, a.direct_n, a.now, a.in_tok[r], a.tag[r],
                                                oracle_like ? a.true_out[r] : 1, id, a.arrival[r], a.weight[c]);
    a.pred_out[r] = s.pred;
    a.bucket_out[r] = static_cast<uint8_t>(s.bucket);
    a.ufc_out[r] = s.ufc_inc;
    a.rfc_out[r] = s.rfc_inc;
    fb += s.fallback;
    nt += s.near_tie;
  }
  fb = __reduce_add_sync(0xffffffffu, fb);
  nt = __reduce_add_sync(0xffffffffu, nt);
  score_counts(a, fb, nt);
}

// Live queue: increments at `now` from the frozen prediction records.
__device__ __forceinline__ void score_frozen_body(const ScoreArgs& a) {
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < a.n;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const Scored s = score_frozen(a.frozen, r, a.pol, a.now, a.in_tok[r], a.arrival[r], __ldg(a.weight + a.client[r]));
    a.pred_out[r] = s.pred;
    a.bucket_out[r] = static_cast<uint8_t>(s.bucket);
    a.ufc_out[r] = s.ufc_inc;
    a.rfc_out[r] = s.rfc_inc;
  }
}

__global__ void __launch_bounds__(kScoreThreads, 4) score_kernel(const ScoreArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  if (a.frozen.pred) {
    score_frozen_body(a);
    score_counts(a, 0u, 0u);
    return;
  }
  stage_model(a.model, a.model_words, smem);
  __syncthreads();
  const ModelTables& M = *reinterpret_cast<const ModelTables*>(smem);
  if (threadIdx.x == 0) atomicMin(&a.st->t[4], global_ns());
  if (M.pred_kind == kPredOracle) score_body<kPredOracle>(a, M);
  else if (M.pred_kind == kPredNoisy) score_body<kPredNoisy>(a, M);
  else score_body<kPredMope>(a, M);
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&a.st->t[5], global_ns());
}

// ---- TMA-pipelined whole-queue scoring ---------------------------------------------------
// Persistent CTAs (2 per SM) stream tiles of kScoreTile requests: one elected thread arms an
// mbarrier and issues 1-D bulk copies (cp.async.bulk, the TMA engine) of the tile's columns
// into a kScoreStages-deep shared-memory ring, so several tiles per SM are in flight without
// any thread holding registers for them; all threads score the landed tile from shared memory
// and write the outputs with coalesced 16-byte streaming stores.  Rows past the last full tile
// take the register path (score_body).
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n EQX_WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra EQX_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// PHASE 0: issue the first kScoreStages tiles (thread 0); PHASE 1: consume all tiles.
template <int KIND, int PHASE>
__device__ __forceinline__ void score_tma_body(const ScoreArgs& a, const ModelTables& M, unsigned char* ring,
                                               uint64_t* bars) {
  constexpr bool oracle_like = KIND == kPredOracle || KIND == kPredNoisy;
  constexpr int R = kScoreTile;
  constexpr uint32_t kBytes = R * (4 + 8 + 4 + 1) + (oracle_like ? 4 * R : 0);
  const int tid = threadIdx.x;
  const int64_t n_full = a.n / R;
  auto stage_ptr = [&](int st) { return ring + static_cast<size_t>(st) * kScoreStageBytes; };
  auto issue = [&](int64_t tile, int st) {  // one thread: arm the stage barrier, copy the columns
    unsigned char* b = stage_ptr(st);
    const int64_t r0 = tile * R;
    mbar_expect_tx(&bars[st], kBytes);
    bulk_g2s(b, a.client + r0, 4 * R, &bars[st]);
    bulk_g2s(b + 4 * R, a.arrival + r0, 8 * R, &bars[st]);
    bulk_g2s(b + 12 * R, a.in_tok + r0, 4 * R, &bars[st]);
    bulk_g2s(b + 16 * R, a.tag + r0, R, &bars[st]);
    if constexpr (oracle_like) bulk_g2s(b + 17 * R, a.true_out + r0, 4 * R, &bars[st]);
  };
  if constexpr (PHASE == 0) {
    if (tid == 0) {
      int64_t t = blockIdx.x;
      for (int st = 0; st < kScoreStages && t < n_full; ++st, t += gridDim.x) issue(t, st);
    }
    return;
  }
  uint32_t fb = 0, nt = 0;
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < n_full; tile += gridDim.x, ++it) {
    const int st = it % kScoreStages;
    mbar_wait(&bars[st], static_cast<uint32_t>((it / kScoreStages) & 1));
    const unsigned char* b = stage_ptr(st);
    const int64_t r0 = tile * R;
#pragma unroll
    for (int q = 0; q < R / (4 * kScoreTmaThreads); ++q) {
      const int j = 4 * (tid + q * kScoreTmaThreads);  // tile-local row of this thread's 4 requests
      const int4 cl = *reinterpret_cast<const int4*>(b + 4 * j);
      const double2 a01 = *reinterpret_cast<const double2*>(b + 4 * R + 8 * j);
      const double2 a23 = *reinterpret_cast<const double2*>(b + 4 * R + 8 * j + 16);
      const int4 in4 = *reinterpret_cast<const int4*>(b + 12 * R + 4 * j);
      const uint32_t tg = *reinterpret_cast<const uint32_t*>(b + 16 * R + j);
      int4 to = make_int4(1, 1, 1, 1);
      if constexpr (oracle_like) to = *reinterpret_cast<const int4*>(b + 17 * R + 4 * j);
      const int cs[4] = {cl.x, cl.y, cl.z, cl.w};
      const int ins[4] = {in4.x, in4.y, in4.z, in4.w};
      const int tos[4] = {to.x, to.y, to.z, to.w};
      const double arr[4] = {a01.x, a01.y, a23.x, a23.y};
      const int64_t r = r0 + j;
      Scored sc[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int64_t id = (KIND == kPredNoisy && a.id) ? a.id[r + k] : a.id_base + r + k;
        const double w = __ldg(a.weight + cs[k]);
        sc[k] = score_request_direct<KIND>(M, a.pol, a.direct, a.direct_n, a.now, ins[k], (tg >> (8 * k)) & 0xffu,
                                           tos[k], id, arr[k], w);
        fb += sc[k].fallback;
        nt += sc[k].near_tie;
      }
      const int64_t v = r / 4;
      stg_stream(reinterpret_cast<int4*>(a.pred_out) + v, make_int4(sc[0].pred, sc[1].pred, sc[2].pred, sc[3].pred));
      stg_stream(reinterpret_cast<uint32_t*>(a.bucket_out) + v,
                 static_cast<uint32_t>(sc[0].bucket) | (static_cast<uint32_t>(sc[1].bucket) << 8) |
                     (static_cast<uint32_t>(sc[2].bucket) << 16) | (static_cast<uint32_t>(sc[3].bucket) << 24));
      stg_stream(reinterpret_cast<double2*>(a.ufc_out) + 2 * v, make_double2(sc[0].ufc_inc, sc[1].ufc_inc));
      stg_stream(reinterpret_cast<double2*>(a.ufc_out) + 2 * v + 1, make_double2(sc[2].ufc_inc, sc[3].ufc_inc));
      stg_stream(reinterpret_cast<double2*>(a.rfc_out) + 2 * v, make_double2(sc[0].rfc_inc, sc[1].rfc_inc));
      stg_stream(reinterpret_cast<double2*>(a.rfc_out) + 2 * v + 1, make_double2(sc[2].rfc_inc, sc[3].rfc_inc));
    }
    __syncthreads();  // every thread is done with this stage
    const int64_t next = tile + static_cast<int64_t>(kScoreStages) * gridDim.x;
    if (tid == 0 && next < n_full) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads before async writes
      issue(next, st);
    }
  }
  // rows after the last full tile
  for (int64_t r = n_full * R + static_cast<int64_t>(blockIdx.x) * blockDim.x + tid; r < a.n;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t c = a.client[r];
    const int64_t id = a.id ? a.id[r] : a.id_base + r;
    const Scored sc = score_request_direct<KIND>(M, a.pol, a.direct, a.direct_n, a.now, a.in_tok[r], a.tag[r],
                                                 oracle_like ? a.true_out[r] : 1, id, a.arrival[r], a.weight[c]);
    a.pred_out[r] = sc.pred;
    a.bucket_out[r] = static_cast<uint8_t>(sc.bucket);
    a.ufc_out[r] = sc.ufc_inc;
    a.rfc_out[r] = sc.rfc_inc;
    fb += sc.fallback;
    nt += sc.near_tie;
  }
  fb = __reduce_add_sync(0xffffffffu, fb);
  nt = __reduce_add_sync(0xffffffffu, nt);
  score_counts(a, fb, nt);
}

__global__ void __launch_bounds__(kScoreTmaThreads, 2) score_tma_kernel(const ScoreArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bars[kScoreStages];
  // layout: tile ring | compiled model | direct predict/map table
  unsigned char* ring = smem;
  unsigned char* msm = smem + static_cast<size_t>(kScoreStages) * kScoreStageBytes;
  uint32_t* dsm = reinterpret_cast<uint32_t*>(msm + ((a.model_words * 4 + 127) & ~127));
  if (threadIdx.x == 0) {
    for (int st = 0; st < kScoreStages; ++st) mbar_init(&bars[st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  ScoreArgs b = a;
  b.direct = a.direct_words > 0 ? dsm : a.direct;
  const int kind = __ldg(&a.model->pred_kind);
  // the first tiles' bulk copies start before the tables are staged
  if (kind == kPredOracle) score_tma_body<kPredOracle, 0>(b, *a.model, ring, bars);
  else if (kind == kPredNoisy) score_tma_body<kPredNoisy, 0>(b, *a.model, ring, bars);
  else score_tma_body<kPredMope, 0>(b, *a.model, ring, bars);
  stage_model(a.model, a.model_words, msm);
  for (int i = threadIdx.x; i < a.direct_words; i += blockDim.x) dsm[i] = __ldg(a.direct + i);
  __syncthreads();
  const ModelTables& M = *reinterpret_cast<const ModelTables*>(msm);
  if (threadIdx.x == 0) atomicMin(&a.st->t[4], global_ns());
  if (kind == kPredOracle) score_tma_body<kPredOracle, 1>(b, M, ring, bars);
  else if (kind == kPredNoisy) score_tma_body<kPredNoisy, 1>(b, M, ring, bars);
  else score_tma_body<kPredMope, 1>(b, M, ring, bars);
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&a.st->t[5], global_ns());
}

// ===================================== selection =========================================

// Per-client working state of the loop (shared memory, or global scratch for huge rosters).
struct ClientWork {
  double* ufc;
  double* rfc;
  double* cnt;
  double* w;
  int32_t* pos;     // absolute FIFO position of the current head
  int32_t* end;     // queue length (absolute)
  int32_t* pos0;    // head at step start (window base)
  uint32_t* order;
  int32_t* flags;   // bit0 backlogged, bit1 skipped (backfill)
  int32_t* adm;     // admitted this step
  int32_t* by_order;  // client of each order rank
};

enum : int32_t { kBacklogged = 1, kSkipped = 2 };
enum : int32_t { kDone = 1 };

struct SelShared {
  double red_u[32], red_r[32];
  double max_u, max_r;
  int32_t flags;
  int64_t n_ev, n_adm, n_rej, prefill;
  int32_t members;
  int64_t reserved;
};

__device__ __forceinline__ double hf_key(const Policy& P, double u, double r, double mu, double mr, double cnt) {
  if (P.kind == kFcfs) return 0.0;  // scheduler.cpp:122
  if (P.kind == kVtc) return cnt;   // scheduler.cpp:124
  if (P.norm_mode == 1) return __dadd_rn(__dmul_rn(P.alpha, u), __dmul_rn(P.beta, r));  // :51
  const double uu = mu > 0.0 ? __ddiv_rn(u, mu) : 0.0;  // scheduler.cpp:53-57
  const double rr = mr > 0.0 ? __ddiv_rn(r, mr) : 0.0;
  return __dadd_rn(__dmul_rn(P.alpha, uu), __dmul_rn(P.beta, rr));
}

// Score one queued row into a head-window entry (shared by window_kernel and deep heads).
template <class A>
__device__ __forceinline__ WinEntry make_entry(const A& a, const ModelTables& M, int32_t row, double w) {
  const int64_t id = a.id ? a.id[row] : a.id_base + row;
  const double arr = a.arrival[row];
  const int32_t in = a.in_tok[row];
  const Scored s = a.frozen.pred ? score_frozen(a.frozen, row, a.pol, a.now, in, arr, w)
                                 : score_request(M, a.pol, a.now, in, a.tag[row], a.true_out ? a.true_out[row] : 1,
                                                 id, arr, w);
  WinEntry e;
  e.ufc_inc = s.ufc_inc;
  e.rfc_inc = s.rfc_inc;
  e.abits = ordered_bits(arr);
  e.in = in;
  e.pred = s.pred;
  e.row = row;
  // fits_alone == can_fit on an empty batch: 0 + 1 <= max_batch and in + pred <= tmax
  e.alone = (1 <= a.pol.max_batch) && (static_cast<int64_t>(in) + s.pred <= a.tmax);
  return e;
}

// Head at FIFO position j (window index k) beyond the shared-memory window: scored from HBM
// (rejection streams), or, in a client-sharded step, read from the gathered windows.  A head
// beyond the gathered depth flags DevState::underflow: the host re-runs the step from its
// checkpoint with deeper windows, so a flagged step's picks are never used.  The sentinel
// always fits alone, so the loop still terminates (admissions are bounded by max_batch).
__device__ __noinline__ WinEntry deep_entry(const SelectArgs& a, const ModelTables& M, int32_t c, int32_t j,
                                            int32_t k, double w) {
  if (a.gW > 0) {
    if (k < a.gW) return a.win_g[static_cast<int64_t>(c) * a.gW + k];
    a.st->underflow = 1;
    WinEntry e;
    e.ufc_inc = e.rfc_inc = 0.0;
    e.abits = ~0ull;
    e.in = e.pred = 0;
    e.row = -1;
    e.alone = 1;
    return e;
  }
  return make_entry(a, M, static_cast<int32_t>(a.perm[a.seg_off[c] + j]), w);
}

// First W queued entries of every client (C*W items, one per thread across many CTAs).
__global__ void __launch_bounds__(256) window_kernel(const WindowArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  stage_model(a.model, a.model_words, smem);  // overlaps the drain's tail (programmatic launch)
  pdl_wait();
  pdl_trigger();  // the drain is complete: the selection CTA may start its prologue
  // this step's scoring counts start from zero: the scoring grid waits for this kernel (event)
  // and the selection reads them after its programmatic wait on it
  if (a.score_sig && blockIdx.x == 0 && threadIdx.x < 2) a.score_sig[threadIdx.x] = 0ull;
#ifdef EQX_PROF
  if (threadIdx.x == 0) atomicMin(&a.st->dt[5], global_ns());
#endif
  __syncthreads();
  const ModelTables& M = *reinterpret_cast<const ModelTables*>(smem);
  const int entry_ctas = gridDim.x - (a.do_lift ? 1 : 0);
  if (static_cast<int>(blockIdx.x) >= entry_ctas) {  // the extra CTA: the drain's counter lift
    const LiftIn l{a.C, a.counter_lift, a.count, a.qlen_before, a.running, a.ufc, a.rfc, a.counter, a.backlogged};
    lift_core<int32_t>(l, a.first_row);
    return;
  }
  const int64_t items = static_cast<int64_t>(a.C) * a.W;
  for (int64_t it = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; it < items;
       it += static_cast<int64_t>(entry_ctas) * blockDim.x) {
    const int32_t c = static_cast<int32_t>(it / a.W);
    const int32_t j = a.head[c] + static_cast<int32_t>(it % a.W);
    if (j < a.count[c]) a.win[it] = make_entry(a, M, static_cast<int32_t>(a.perm[a.seg_off[c] + j]), a.weight[c]);
  }
#ifdef EQX_PROF
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&a.st->dt[6], global_ns());
#endif
}

// Outcome flags of a generated key-stream item (the top-K rounds, eqx_topk.cuh, and the
// register pick loops): fits alone, its admission raises a maximum, a max holder leaves the
// backlog with it, the client's generated stream ends with it.
enum : uint32_t { kFlAlone = 1, kFlMaxChg = 2, kFlHolder = 4, kFlExh = 8 };

__device__ __forceinline__ double vtc_inc(const Policy& P, const WinEntry& e, double w) {
  if (P.kind != kVtc) return 0.0;  // scheduler.cpp:169-181
  return P.vtc_use_prediction
             ? __dmul_rn(w, __dadd_rn(static_cast<double>(e.in), __dmul_rn(P.ow, static_cast<double>(e.pred))))
             : __dmul_rn(w, static_cast<double>(e.in));
}

// Max over backlogged clients (scheduler.cpp:40-48) by the whole CTA.
__device__ void cta_maxima(const ClientWork& cw, int32_t C, SelShared& S) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  double mu = 0.0, mr = 0.0;
  const int NT = blockDim.x;
  for (int32_t c0 = tid; c0 < C; c0 += 4 * NT) {  // 4 clients' loads in flight (huge rosters: L2)
    int32_t fl[4];
    double u[4], r[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int32_t c = c0 + k * NT;
      fl[k] = c < C ? cw.flags[c] : 0;
      u[k] = c < C ? cw.ufc[c] : 0.0;
      r[k] = c < C ? cw.rfc[c] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (!(fl[k] & kBacklogged)) continue;
      if (mu < u[k]) mu = u[k];
      if (mr < r[k]) mr = r[k];
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double ou = __shfl_xor_sync(0xffffffffu, mu, o), orr = __shfl_xor_sync(0xffffffffu, mr, o);
    if (mu < ou) mu = ou;
    if (mr < orr) mr = orr;
  }
  if (lane == 0) {
    S.red_u[warp] = mu;
    S.red_r[warp] = mr;
  }
  __syncthreads();
  if (tid == 0) {
    double u = 0.0, r = 0.0;
    for (int w = 0; w < nw; ++w) {
      if (u < S.red_u[w]) u = S.red_u[w];
      if (r < S.red_r[w]) r = S.red_r[w];
    }
    S.max_u = u;
    S.max_r = r;
  }
  __syncthreads();
}



#include "eqx_topk.cuh"

// The selection kernel: one CTA runs the exact admit_requests loop as rounds of block-radix
// top-K over per-client key streams (eqx_topk.cuh).  The prologue stages the model, carves the
// per-client work arrays (shared memory, or global scratch on huge rosters) and loads the
// ledger -- after the window kernel's programmatic completion when that kernel applied the
// drain's counter lift -- and the epilogue writes back ledger, heads, batch and summary.
template <bool kHugeRoster>
__global__ void __launch_bounds__(kTopkThreads, 1) select_topk_kernel(const SelectArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ SelShared S;
  const int32_t C = a.C;
  const int tid = threadIdx.x, NT = blockDim.x;
  stage_model(a.model, a.model_words, smem);
  if (tid == 0) {
    a.st->t[0] = global_ns();
    for (int i = 8; i < 16; ++i) a.st->t[i] = 0;
  }
  // ---- carve per-client work arrays and the top-K scratch ----
  unsigned char* p = smem + ((a.model_words * 4 + 15) & ~15);
  unsigned char* g = reinterpret_cast<unsigned char*>(a.cw_global);
  auto carve = [&](size_t bytes) {
    unsigned char* r = p;
    p += (bytes + 15) & ~size_t(15);
    return r;
  };
  auto take = [&](size_t bytes) {
    if (a.cw_in_smem) return carve(bytes);
    unsigned char* r = g;
    g += (bytes + 15) & ~size_t(15);
    return r;
  };
  ClientWork cw;
  cw.ufc = reinterpret_cast<double*>(take(8ull * C));
  cw.rfc = reinterpret_cast<double*>(take(8ull * C));
  cw.cnt = reinterpret_cast<double*>(take(8ull * C));
  cw.w = reinterpret_cast<double*>(take(8ull * C));
  cw.pos = reinterpret_cast<int32_t*>(take(4ull * C));
  cw.end = reinterpret_cast<int32_t*>(take(4ull * C));
  cw.pos0 = reinterpret_cast<int32_t*>(take(4ull * C));
  cw.order = reinterpret_cast<uint32_t*>(take(4ull * C));
  cw.flags = reinterpret_cast<int32_t*>(take(4ull * C));
  cw.adm = reinterpret_cast<int32_t*>(take(4ull * C));
  cw.by_order = reinterpret_cast<int32_t*>(take(4ull * C));
  TopkScratch TK;
  {
    const size_t items = static_cast<size_t>(a.tk_cap);
    const size_t kc = static_cast<size_t>(a.tk_kcap);
    TK.dsh_max = a.tk_dsh;
    TK.Kcap = a.tk_kcap;
    TK.cap = a.tk_cap;
    TK.k = reinterpret_cast<uint64_t*>(carve(8 * items));  // stream items: always shared memory
    TK.a = reinterpret_cast<uint64_t*>(carve(8 * items));
    TK.u = reinterpret_cast<double*>(carve(8 * items));
    TK.r = reinterpret_cast<double*>(carve(8 * items));
    TK.cn = reinterpret_cast<double*>(carve(8 * items));
    TK.fl = reinterpret_cast<uint8_t*>(carve(items));
    TK.st = reinterpret_cast<uint8_t*>(carve(items));
    TK.sd = reinterpret_cast<uint32_t*>(carve(4 * items));
    TK.sc = reinterpret_cast<int32_t*>(carve(4 * kc));
    TK.snd = reinterpret_cast<int32_t*>(carve(4 * kc));
    TK.spos = reinterpret_cast<int32_t*>(carve(4 * kc));
    TK.sk0 = reinterpret_cast<int32_t*>(carve(4 * kc));
    TK.off = reinterpret_cast<int32_t*>(carve(4 * kc));
    TK.cut = reinterpret_cast<int32_t*>(carve(4 * kc));
    TK.gk = reinterpret_cast<uint64_t*>(carve(8 * kc));
    TK.ga = reinterpret_cast<uint64_t*>(carve(8 * kc));
    TK.go = reinterpret_cast<uint64_t*>(carve(8 * kc));
    TK.gx = reinterpret_cast<int32_t*>(carve(4 * kc));
    TK.rank = reinterpret_cast<int32_t*>(carve(4 * kc));
    TK.srt = reinterpret_cast<int32_t*>(carve(4 * kc));
    TK.ent = reinterpret_cast<WinEntry*>(carve(sizeof(WinEntry) * kc));
    TK.hist = reinterpret_cast<uint32_t*>(carve(4 * 256));
    TK.stage = reinterpret_cast<uint64_t*>(carve(8 * 160 * (kTopkThreads / 32)));
    // head tuples (rosters beyond tk_kcap): shared memory when they fit, else global scratch
    unsigned char* hp = nullptr;
    const size_t cc = static_cast<size_t>((C + 1) & ~1);
    if (C > a.tk_kcap) hp = a.tk_heads ? reinterpret_cast<unsigned char*>(a.tk_heads) : carve(17 * cc + 16);
    TK.hk = reinterpret_cast<uint64_t*>(hp);
    TK.ha = hp ? reinterpret_cast<uint64_t*>(hp + 8 * cc) : nullptr;
    TK.hst = hp ? hp + 16 * cc : nullptr;
  }
  __syncthreads();
  const ModelTables& M = *reinterpret_cast<const ModelTables*>(smem);

  if (a.do_lift) {  // on_activated / set_backlogged of the drain that preceded this step
    const LiftIn l{C, a.counter_lift, a.count, a.qlen_before, a.running, a.ufc, a.rfc, a.counter, a.backlogged};
    lift_core<int32_t>(l, a.first_row);
    __syncthreads();
  }
  // ---- ledger in ----
  if (a.ledger_after_wait) pdl_wait();  // lifted by the window kernel's extra CTA
  // Loads of 2 clients are issued before any store: the work arrays may alias nothing, but the
  // compiler cannot know it, and a load-store-load chain costs one memory round trip per field.
  for (int32_t c0 = tid; c0 < C; c0 += 2 * NT) {
    double u[2], r[2], k[2], w[2];
    int32_t h[2], n[2], bl[2];
    uint32_t o[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int32_t c = c0 + j * NT;
      if (c < C) {
        u[j] = a.ufc[c];
        r[j] = a.rfc[c];
        k[j] = a.counter[c];
        w[j] = a.weight[c];
        h[j] = a.head[c];
        n[j] = a.count[c];
        o[j] = a.order[c];
        bl[j] = a.backlogged[c];
      }
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int32_t c = c0 + j * NT;
      if (c >= C) continue;
      cw.ufc[c] = u[j];
      cw.rfc[c] = r[j];
      cw.cnt[c] = k[j];
      cw.w[c] = w[j];
      cw.pos[c] = h[j];
      cw.pos0[c] = h[j];
      cw.end[c] = n[j];
      cw.order[c] = o[j];
      cw.by_order[o[j]] = c;
      cw.flags[c] = bl[j] ? kBacklogged : 0;
      cw.adm[c] = 0;
    }
  }
  if (!a.ledger_after_wait) pdl_wait();  // window_kernel's [C][W] head entries (read from L2 by the rounds)
  if (tid == 0) {
    S.n_ev = S.n_adm = S.n_rej = S.prefill = 0;
    S.members = a.st->members;
    S.reserved = a.st->reserved;
    S.flags = 0;
  }
  __syncthreads();
  if (tid == 0) a.st->t[1] = global_ns();
  cta_maxima(cw, C, S);
  if (tid == 0) a.st->t[2] = global_ns();
  topk_select<kHugeRoster>(a, M, cw, S, TK);
  if (tid == 0) a.st->t[3] = global_ns();
  pdl_trigger();  // the event fill may get scheduled while the ledger is written back
  // ---- write back ledger, heads, batch, summary ----
  for (int32_t c0 = tid; c0 < C; c0 += 2 * NT) {  // loads first, as for the ledger in
    double u[2], r[2], k[2];
    int32_t h[2], f[2], ad[2], run[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int32_t c = c0 + j * NT;
      if (c < C) {
        u[j] = cw.ufc[c];
        r[j] = cw.rfc[c];
        k[j] = cw.cnt[c];
        h[j] = cw.pos[c];
        f[j] = cw.flags[c];
        ad[j] = cw.adm[c];
        run[j] = a.running[c];
      }
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int32_t c = c0 + j * NT;
      if (c >= C) continue;
      a.ufc[c] = u[j];
      a.rfc[c] = r[j];
      a.counter[c] = k[j];
      a.head[c] = h[j];
      a.backlogged[c] = (f[j] & kBacklogged) ? 1 : 0;
      a.running[c] = run[j] + ad[j];
      if (a.h_ledger) {  // [ufc C][rfc C][counter C] f64, [backlogged C][running C] i32
        double* hd = reinterpret_cast<double*>(a.h_ledger);
        int32_t* hi = reinterpret_cast<int32_t*>(hd + 3 * static_cast<int64_t>(C));
        hd[c] = u[j];
        hd[C + c] = r[j];
        hd[2 * C + c] = k[j];
        hi[c] = (f[j] & kBacklogged) ? 1 : 0;
        hi[C + c] = run[j] + ad[j];
      }
    }
  }
  if (tid == 0) {
    a.st->members = S.members;
    a.st->reserved = S.reserved;
    a.st->n_events = S.n_ev;
    a.st->n_admitted = S.n_adm;
    a.st->n_rejected = S.n_rej;
    a.st->new_prefill = S.prefill;
  }
  if (a.h_st) {  // the step's summary straight to the mapped host copy (no copy kernel)
    __syncthreads();
    if (tid >= 32) return;
    if (tid == 0 && a.score_done) {  // the scoring runs beside the selection on a side stream and is
                                     // normally long done: its counts are final once every CTA has
                                     // added (score_counts); without score_done it finished earlier
      volatile unsigned long long* sig = a.score_done;  // zeroed by this step's window kernel
      unsigned long long f, t;
      const unsigned long long t0 = global_ns();
      while (true) {
        f = sig[0];
        t = sig[1];
        if (static_cast<int64_t>(f / kScoreCtaOne) >= a.score_ctas &&
            static_cast<int64_t>(t / kScoreCtaOne) >= a.score_ctas)
          break;
        if (global_ns() - t0 > 10000000000ull) __trap();  // never silently hang: fail the launch
        __nanosleep(128);
      }
      a.st->fallbacks += f % kScoreCtaOne;
      a.st->near_ties += t % kScoreCtaOne;
    }
    __syncwarp();
    constexpr int kWords = static_cast<int>(sizeof(DevState) / 8), kPer = (kWords + 31) / 32;
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(a.st);
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(a.h_st);
    unsigned long long v[kPer];
#pragma unroll
    for (int k = 0; k < kPer; ++k)  // every load in flight before the PCIe stores
      if (tid + 32 * k < kWords) v[k] = __ldcg(src + tid + 32 * k);
#pragma unroll
    for (int k = 0; k < kPer; ++k)
      if (tid + 32 * k < kWords) dst[tid + 32 * k] = v[k];
  }
}
template __global__ void select_topk_kernel<false>(SelectArgs);
template __global__ void select_topk_kernel<true>(SelectArgs);

// Staged narrow host columns widened in place of the H2D's second half: 8 rows per thread,
// 16-byte loads of each u16 column, 2 x 16-byte stores per i32 column.
__global__ void widen_cols_kernel(const uint16_t* c16, const uint16_t* i16, int64_t n, int32_t* c32, int32_t* i32) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t groups = n / 8;
  for (int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < groups; g += stride) {
    const uint4 a = reinterpret_cast<const uint4*>(c16)[g];
    const uint4 b = reinterpret_cast<const uint4*>(i16)[g];
    const uint32_t aw[4] = {a.x, a.y, a.z, a.w}, bw[4] = {b.x, b.y, b.z, b.w};
    int4 o[4];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      o[k] = make_int4(aw[2 * k] & 0xffff, aw[2 * k] >> 16, aw[2 * k + 1] & 0xffff, aw[2 * k + 1] >> 16);
      o[2 + k] = make_int4(bw[2 * k] & 0xffff, bw[2 * k] >> 16, bw[2 * k + 1] & 0xffff, bw[2 * k + 1] >> 16);
    }
    reinterpret_cast<int4*>(c32)[2 * g] = o[0];
    reinterpret_cast<int4*>(c32)[2 * g + 1] = o[1];
    reinterpret_cast<int4*>(i32)[2 * g] = o[2];
    reinterpret_cast<int4*>(i32)[2 * g + 1] = o[3];
  }
  for (int64_t r = 8 * groups + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < n; r += stride) {
    c32[r] = c16[r];
    i32[r] = i16[r];
  }
}

// Packed arrivals (eqx_pack_arrivals) -> doubles.  Per 256-row block: a base bit pattern and
// the byte offset of the block's data, either 6-byte offsets from the base (packed) or the raw
// doubles (base == ~0: blocks spanning more than 48 bits of the bit pattern, e.g. near zero).
// 8 rows per thread (48 or 64 bytes, 16-byte loads).
__device__ __forceinline__ double unpack_row(const unsigned char* pk, unsigned long long base, int64_t off, int i) {
  if (base == ~0ull) return reinterpret_cast<const double*>(pk + off)[i];
  unsigned long long d = 0;
  for (int j = 5; j >= 0; --j) d = (d << 8) | pk[off + 6 * i + j];
  return __longlong_as_double(static_cast<long long>(base + d));
}
__global__ void unpack_arrivals_kernel(const unsigned char* pk, int64_t n, double* out) {
  const int64_t nb = (n + 255) / 256;
  const unsigned long long* base = reinterpret_cast<const unsigned long long*>(pk + 8);
  const long long* off = reinterpret_cast<const long long*>(pk + 8 + 8 * nb);
  constexpr unsigned long long kM48 = (1ull << 48) - 1;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t groups = n / 8;
  for (int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < groups; g += stride) {
    const int64_t blk = (8 * g) >> 8, i0 = (8 * g) & 255;  // 8 rows never straddle a block
    const unsigned long long b = base[blk];
    const long long o0 = off[blk];
    double2* o = reinterpret_cast<double2*>(out + 8 * g);
    if (b == ~0ull) {
      const double2* p = reinterpret_cast<const double2*>(pk + o0 + 8 * i0);
#pragma unroll
      for (int k = 0; k < 4; ++k) o[k] = p[k];
      continue;
    }
    const ulonglong2* p = reinterpret_cast<const ulonglong2*>(pk + o0 + 6 * i0);
    const ulonglong2 x0 = p[0], x1 = p[1], x2 = p[2];
    const unsigned long long w[6] = {x0.x, x0.y, x1.x, x1.y, x2.x, x2.y};
    const unsigned long long d[8] = {w[0] & kM48,
                                     ((w[0] >> 48) | (w[1] << 16)) & kM48,
                                     ((w[1] >> 32) | (w[2] << 32)) & kM48,
                                     w[2] >> 16,
                                     w[3] & kM48,
                                     ((w[3] >> 48) | (w[4] << 16)) & kM48,
                                     ((w[4] >> 32) | (w[5] << 32)) & kM48,
                                     w[5] >> 16};
#pragma unroll
    for (int k = 0; k < 4; ++k)
      o[k] = make_double2(__longlong_as_double(static_cast<long long>(b + d[2 * k])),
                          __longlong_as_double(static_cast<long long>(b + d[2 * k + 1])));
  }
  for (int64_t r = 8 * groups + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < n; r += stride)
    out[r] = unpack_row(pk, base[r >> 8], off[r >> 8], static_cast<int>(r & 255));
}

// Columns -> mapped host memory by SM stores over PCIe (16-byte words when aligned).
__global__ void pack_cols_kernel(const PackCols p) {
  pdl_wait();  // no-op unless launched programmatically after the kernel producing the columns
  pdl_trigger();
  for (int c = blockIdx.y; c < p.n; c += gridDim.y) {
    const int64_t b = p.bytes[c];
    const unsigned char* src = static_cast<const unsigned char*>(p.src[c]);
    unsigned char* dst = static_cast<unsigned char*>(p.dst[c]);
    const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t nt = static_cast<int64_t>(gridDim.x) * blockDim.x;
    if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
      const int64_t w = b / 16;
      for (int64_t i = tid; i < w; i += nt)
        reinterpret_cast<int4*>(dst)[i] = __ldcg(reinterpret_cast<const int4*>(src) + i);
      for (int64_t i = 16 * w + tid; i < b; i += nt) dst[i] = src[i];
    } else {
      for (int64_t i = tid; i < b; i += nt) dst[i] = src[i];
    }
  }
}

// =================================== live queues ==========================================
// arrivals are appended to the requests still queued.  The new column
// store holds the remaining rows client-grouped in FIFO order (straight from perm/head) followed
// by the arrivals in arrival order, so a drain over it rebuilds every client's FIFO (old rows
// first) and the counter lift sees the remaining counts as drain_arrivals' non-empty queues.
__global__ void __launch_bounds__(1024) live_offsets_kernel(const LiveArgs a) {
  __shared__ uint32_t warp_buf[32];
  const int per = (a.C + blockDim.x - 1) / blockDim.x;
  const int c0 = min(a.C, per * static_cast<int>(threadIdx.x)), c1 = min(a.C, c0 + per);
  uint32_t s = 0;
  for (int c = c0; c < c1; ++c) s += static_cast<uint32_t>(a.count[c] - a.head[c]);
  uint32_t run;
  const uint32_t total = block_exclusive_scan(s, &run, warp_buf);
  for (int c = c0; c < c1; ++c) {
    const int32_t rem = a.count[c] - a.head[c];
    a.live_off[c] = static_cast<int32_t>(run);
    a.qlen_before[c] = rem;
    run += static_cast<uint32_t>(rem);
  }
  if (threadIdx.x == 0) {
    a.live_off[a.C] = static_cast<int32_t>(total);
    *a.n_live = total;
  }
}

__global__ void __launch_bounds__(256) gather_live_kernel(const LiveArgs a) {
  const int64_t n = a.live_off[a.C];
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int32_t lo = 0, hi = a.C;  // client: last c with live_off[c] <= i
    while (hi - lo > 1) {
      const int32_t mid = (lo + hi) >> 1;
      if (a.live_off[mid] <= i) lo = mid;
      else hi = mid;
    }
    const int32_t c = lo;
    const int64_t row = a.perm[a.seg_off[c] + a.head[c] + (i - a.live_off[c])];
    a.n_client[i] = a.o_client[row];
    a.n_arrival[i] = a.o_arrival[row];
    a.n_in[i] = a.o_in[row];
    a.n_tag[i] = a.o_tag[row];
    if (a.n_true) a.n_true[i] = a.o_true ? a.o_true[row] : 1;
    a.n_id[i] = a.o_id[row];
    a.n_pred[i] = a.o_pred[row];
    a.n_bucket[i] = a.o_bucket[row];
    a.n_preds[i] = a.o_preds[row];
    a.n_rfc[i] = a.o_rfc[row];
  }
}

__global__ void __launch_bounds__(256) predict_rows_kernel(const ScoreArgs a, int64_t r0, int64_t r1,
                                                           const LiveArgs L, int32_t fill_id) {
  extern __shared__ __align__(16) unsigned char smem[];
  stage_model(a.model, a.model_words, smem);
  __syncthreads();
  const ModelTables& M = *reinterpret_cast<const ModelTables*>(smem);
  uint32_t fb = 0, nt = 0;
  for (int64_t r = r0 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < r1;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (fill_id) L.n_id[r] = a.id_base + (r - r0);
    const int32_t c = L.n_client[r];
    if (static_cast<uint32_t>(c) >= static_cast<uint32_t>(L.C)) continue;  // the drain flags it
    const double w = a.weight[c];
    // the prediction record of map_metrics at arrival (now / arrival do not enter it)
    const Scored s = score_request(M, a.pol, 0.0, L.n_in[r], L.n_tag[r], L.n_true ? L.n_true[r] : 1, L.n_id[r], 0.0, w);
    L.n_pred[r] = s.pred;
    L.n_bucket[r] = static_cast<uint8_t>(s.bucket);
    L.n_preds[r] = M.prof_pred_s[s.bucket];
    L.n_rfc[r] = s.rfc_inc;
    fb += s.fallback;
    nt += s.near_tie;
  }
  fb = __reduce_add_sync(0xffffffffu, fb);
  nt = __reduce_add_sync(0xffffffffu, nt);
  if ((threadIdx.x & 31) == 0) {
    if (fb) atomicAdd(&a.st->fallbacks, static_cast<unsigned long long>(fb));
    if (nt) atomicAdd(&a.st->near_ties, static_cast<unsigned long long>(nt));
  }
}

// ============================== completion / feedback =====================================
// One engine iteration's feedback (engine.cpp:273-375) in the reference's order: on_tokens for
// every client with decode tokens (scheduler.cpp:185-190), then each completion in order:
// on_complete (scheduler.cpp:192-233: actual minus pending increments, clamped at 0), the
// running-count decrement (engine.cpp:368) and update_map's EMA of the profile entry of the
// observed output length (predictor.cpp:372-383).  Per-client and per-entry chains are
// sequential in completion order (the FP64 rounding and clamps depend on it); different
// clients / entries are independent, so one thread owns each.
__global__ void __launch_bounds__(1024) feedback_kernel(const FeedbackArgs a) {
  const Policy& P = a.pol;
  const int tid = threadIdx.x;
  __shared__ unsigned long long s_clamps;
  if (tid == 0) s_clamps = 0;
  __syncthreads();
  unsigned long long clamps = 0;
  for (int32_t c = tid; c < a.C; c += blockDim.x) {
    const double w = a.weight[c];
    double k = a.counter[c];
    if (a.tokens && P.kind == kVtc && !P.vtc_use_prediction && a.tokens[c] > 0)  // on_tokens
      k = __dadd_rn(k, __dmul_rn(__dmul_rn(w, P.ow), static_cast<double>(a.tokens[c])));
    double u = a.ufc[c], r = a.rfc[c], sv = a.service[c];
    int32_t run = a.running[c];
    for (int64_t i = 0; i < a.n; ++i) {
      if (a.client[i] != c) continue;
      const double wt = __dadd_rn(static_cast<double>(a.in_tok[i]), __dmul_rn(P.ow, static_cast<double>(a.out_tok[i])));
      const double wwt = __dmul_rn(w, wt);
      const double au = __ddiv_rn(wwt, __dadd_rn(1.0, __dmul_rn(P.delta, a.latency_s[i])));
      const double ar = __dmul_rn(__dmul_rn(w, a.tps[i]), a.util[i]);
      u = __dadd_rn(u, __dsub_rn(au, a.pend_ufc[i]));
      if (u < 0.0) {
        u = 0.0;
        ++clamps;
      }
      r = __dadd_rn(r, __dsub_rn(ar, a.pend_rfc[i]));
      if (r < 0.0) {
        r = 0.0;
        ++clamps;
      }
      if (P.kind == kVtc && P.vtc_use_prediction) {
        k = __dadd_rn(k, __dsub_rn(wwt, a.pend_vtc[i]));
        if (k < 0.0) {
          k = 0.0;
          ++clamps;
        }
      }
      sv = __dadd_rn(sv, wwt);
      --run;
    }
    a.ufc[c] = u;
    a.rfc[c] = r;
    a.counter[c] = k;
    a.service[c] = sv;
    a.running[c] = run;
  }
  if (clamps) atomicAdd(&s_clamps, clamps);
  // update_map: lane e of warp 1 owns profile entry e
  if (a.ema_alpha > 0.0 && (tid >> 5) == (blockDim.x > 32 ? 1 : 0)) {
    const int e = tid & 31;
    ModelTables* M = a.model;
    const int np = M->n_prof;
    if (e < np) {
      double lat = M->prof_lat[e], ut = M->prof_util[e], tp = M->prof_tps[e];
      const double al = a.ema_alpha, bl = __dsub_rn(1.0, a.ema_alpha);
      bool hit = false;
      for (int64_t i = 0; i < a.n; ++i) {
        const int32_t out = a.out_tok[i];
        int b = np - 1;  // entry_for (gpu_model.cpp:74-80): first entry with out <= upper
        for (int x = np - 1; x >= 0; --x)
          if (out <= M->prof_upper[x]) b = x;
        if (b != e) continue;
        hit = true;
        lat = __dadd_rn(__dmul_rn(bl, lat), __dmul_rn(al, __dmul_rn(a.latency_s[i], 1000.0)));
        ut = __dadd_rn(__dmul_rn(bl, ut), __dmul_rn(al, a.util[i]));
        tp = __dadd_rn(__dmul_rn(bl, tp), __dmul_rn(al, a.tps[i]));
      }
      if (hit) {
        M->prof_lat[e] = lat;
        M->prof_util[e] = ut;
        M->prof_tps[e] = tp;
        M->prof_pred_s[e] = __ddiv_rn(lat, 1000.0);  // scheduler.cpp:23 reads latency_ms / 1000
      }
    }
  }
  __syncthreads();
  if (tid == 0 && s_clamps) a.st->clamps += static_cast<int64_t>(s_clamps);
}

// ================================ client-sharded step =====================================
// the queue shards by client over ranks; every rank scores its own queue and
// exports its clients' head windows (shard_export_kernel), the records are all-gathered
// (NCCL), and every rank runs the identical exact selection over the gathered windows with a
// replicated ledger (shard_ingest_kernel applies the drain's backlog flags and counter lift
// with global arrival order, shard_unpack_kernel lays the windows out as [C][W]).

__device__ __forceinline__ int32_t rank_of(const ShardMap& m, int32_t c) {
  int32_t r = 0;
  while (r + 1 < m.world && m.off[r + 1] <= c) ++r;
  return r;
}

__global__ void __launch_bounds__(256) shard_export_kernel(const WindowArgs a, int32_t cmax, unsigned char* rec) {
  extern __shared__ __align__(16) unsigned char smem[];
  stage_model(a.model, a.model_words, smem);
  __syncthreads();
  const ModelTables& M = *reinterpret_cast<const ModelTables*>(smem);
  const RecLayout L = rec_layout(cmax, a.W);
  int32_t* r_count = reinterpret_cast<int32_t*>(rec + L.count);
  int64_t* r_first = reinterpret_cast<int64_t*>(rec + L.first);
  WinEntry* r_win = reinterpret_cast<WinEntry*>(rec + L.win);
  int64_t* r_id = reinterpret_cast<int64_t*>(rec + L.id);
  const int64_t items = static_cast<int64_t>(cmax) * a.W;
  for (int64_t it = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; it < items;
       it += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t c = static_cast<int32_t>(it / a.W);
    const int32_t k = static_cast<int32_t>(it % a.W);
    const bool mine = c < a.C;
    const int32_t h = mine ? a.head[c] : 0, cnt = mine ? a.count[c] : 0;
    if (k == 0) {
      r_count[c] = cnt - h;
      int64_t f = 0x7fffffffffffffffLL;
      if (cnt > 0) {
        const int32_t row0 = static_cast<int32_t>(a.perm[a.seg_off[c]]);
        f = a.id ? a.id[row0] : a.id_base + row0;
      }
      r_first[c] = f;
    }
    if (h + k < cnt) {
      const int32_t row = static_cast<int32_t>(a.perm[a.seg_off[c] + h + k]);
      WinEntry e = make_entry(a, M, row, a.weight[c]);
      e.row = -1;
      r_win[it] = e;
      r_id[it] = a.id ? a.id[row] : a.id_base + row;
    }
  }
}

__global__ void __launch_bounds__(1024) shard_ingest_kernel(const ShardMap m, const ShardSelectBufs b) {
  const RecLayout L = rec_layout(m.cmax, m.W);
  const int NT = blockDim.x;
  unsigned long long mine = 0;
  for (int32_t c0 = threadIdx.x; c0 < m.C; c0 += 4 * NT) {  // 4 clients' record loads in flight
    int32_t cnt[4];
    int64_t f[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int32_t c = c0 + j * NT;
      cnt[j] = 0;
      f[j] = 0;
      if (c < m.C) {
        const int32_t r = rank_of(m, c), l = c - m.off[r];
        const unsigned char* base = m.recs + static_cast<int64_t>(r) * m.stride;
        cnt[j] = reinterpret_cast<const int32_t*>(base + L.count)[l];
        f[j] = reinterpret_cast<const int64_t*>(base + L.first)[l];
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int32_t c = c0 + j * NT;
      if (c >= m.C) continue;
      b.count[c] = cnt[j];
      b.first[c] = f[j];
      b.head[c] = 0;
      b.qlen_before[c] = 0;
      mine += static_cast<unsigned long long>(cnt[j]);
    }
  }
  __shared__ unsigned long long total;
  if (threadIdx.x == 0) {
    b.st->underflow = 0;
    total = 0;
  }
  __syncthreads();
#pragma unroll
  for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(&total, mine);  // one shared atomic per warp
  __syncthreads();
  if (threadIdx.x == 0) b.st->n_queued = static_cast<int64_t>(total);
  const LiftIn li{m.C, b.counter_lift, b.count, b.qlen_before, b.running, b.ufc, b.rfc, b.counter, b.backlogged};
  lift_core<int64_t>(li, b.first);
}

__global__ void __launch_bounds__(256) shard_unpack_kernel(const ShardMap m, const ShardSelectBufs b) {
  const RecLayout L = rec_layout(m.cmax, m.W);
  const int64_t items = static_cast<int64_t>(m.C) * m.W;
  for (int64_t it = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; it < items;
       it += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t c = static_cast<int32_t>(it / m.W);
    const int32_t k = static_cast<int32_t>(it % m.W);
    const int32_t r = rank_of(m, c), l = c - m.off[r];
    const unsigned char* base = m.recs + static_cast<int64_t>(r) * m.stride;
    const int64_t src = static_cast<int64_t>(l) * m.W + k;
    WinEntry e = reinterpret_cast<const WinEntry*>(base + L.win)[src];
    e.row = static_cast<int32_t>(it);
    b.win[it] = e;
    b.gid[it] = reinterpret_cast<const int64_t*>(base + L.id)[src];
  }
}

}  // namespace eqx
