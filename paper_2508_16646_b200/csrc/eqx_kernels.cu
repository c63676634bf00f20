// eqx_kernels.cu -- sm_100a kernels of the Equinox per-step scheduling path.
//
//   drain_arrivals (engine.cpp:171-197), two launches:
//     drain_hist_kernel  per-tile client histogram; the last CTA to finish scans the
//                        [client][tile] table into FIFO segment offsets
//     drain_rank_kernel  stable per-client rank inside each tile (warp __match_any_sync walk),
//                        staged in shared memory and written out as contiguous per-client runs
//                        -> perm (row indices grouped by client, arrival order kept); the last
//                        CTA applies the on_activated counter lift (scheduler.cpp:235-253)
//   admit_requests (engine.cpp:207-271), two concurrent launches:
//     select_kernel      one CTA: the exact sequential admission loop over client heads
//                        (select_next / holistic_score / fits_alone / can_fit / on_admit)
//     score_kernel       whole-queue MoPE predict -> map_metrics -> ufc/rfc increments,
//                        16-byte coalesced loads, streaming stores (HBM-bound stream)
//   gather_ids_kernel    event rows -> request ids for the caller.
#include <cstdint>
#include <cuda_runtime.h>

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

__global__ void __launch_bounds__(kDrainThreads) drain_hist_kernel(const DrainArgs a) {
  extern __shared__ __align__(16) uint32_t sh[];
  const int32_t C = a.C;
  for (int c = threadIdx.x; c < C; c += blockDim.x) sh[c] = 0;
  __syncthreads();
  const int32_t tile = blockIdx.x;
  const int32_t r0 = tile * a.tile_rows;
  const int32_t r1 = min(a.n, r0 + a.tile_rows);
  for (int32_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
    const int32_t c = a.client[r];
    if (static_cast<uint32_t>(c) >= static_cast<uint32_t>(C)) {
      a.st->bad_client = 1;
      continue;
    }
    atomicAdd(&sh[c], 1u);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += blockDim.x) a.hist[static_cast<int64_t>(c) * a.n_tiles + tile] = sh[c];
  if (!last_cta(&a.done[0])) return;
  // ---- epilogue (one CTA): exclusive scan of hist in [client][tile] order ----
  __shared__ uint32_t warp_buf[32];
  const int64_t L = a.hist_L;
  const int64_t per = (L + blockDim.x - 1) / blockDim.x;
  const int64_t b0 = ::min(L, per * static_cast<int64_t>(threadIdx.x)), b1 = ::min(L, b0 + per);
  uint32_t sum = 0;
  for (int64_t i = b0; i < b1; ++i) sum += __ldcg(a.hist + i);
  uint32_t run;
  const uint32_t total = block_exclusive_scan(sum, &run, warp_buf);
  for (int64_t i = b0; i < b1; ++i) {
    const uint32_t v = __ldcg(a.hist + i);
    __stcg(a.hist + i, run);
    if (i % a.n_tiles == 0) a.seg_off[i / a.n_tiles] = static_cast<int32_t>(run);
    run += v;
  }
  if (threadIdx.x == 0) {
    a.seg_off[C] = static_cast<int32_t>(total);
    a.done[0] = 0;
  }
}

// on_activated in arrival order for every client that goes idle -> backlogged in this drain.
// The lift target is the componentwise min over *other* backlogged clients at that moment.
// Lifted values are >= that min, so the running min only moves when a client that is NOT
// lifted joins the backlog: pre-backlogged clients (qlen_before > 0), the very first arrival
// when nobody was backlogged, and clients with running requests (engine.cpp:182).  Hence
// m(c) = min(base, {vals(r) : r non-lifted arrival, first_row[r] < first_row[c]}).
__device__ void lift_epilogue(const DrainArgs& a) {
  __shared__ double s_min[3][32];
  __shared__ int s_first[32], s_firstc[32], s_flags[32];
  const int32_t C = a.C;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  // counts and first arrival rows from the segment offsets / perm
  for (int c = tid; c < C; c += blockDim.x) {
    const int32_t s0 = __ldcg(a.seg_off + c), s1 = __ldcg(a.seg_off + c + 1);
    a.count[c] = s1 - s0;
    a.first_row[c] = s1 > s0 ? static_cast<int32_t>(__ldcg(a.perm + s0)) : 0x7fffffff;
  }
  __syncthreads();
  if (a.counter_lift) {
    double mu = INFINITY, mr = INFINITY, mc = INFINITY;
    int any0 = 0, anyR = 0;
    int fr = 0x7fffffff, fc = -1;
    for (int c = tid; c < C; c += blockDim.x) {
      const int32_t cnt = a.count[c];
      if (a.qlen_before[c] > 0) {
        any0 = 1;
        mu = fmin(mu, a.ufc[c]);
        mr = fmin(mr, a.rfc[c]);
        mc = fmin(mc, a.counter[c]);
      } else if (cnt > 0 && a.running[c] != 0) {
        anyR = 1;
      }
      if (cnt > 0 && a.first_row[c] < fr) {
        fr = a.first_row[c];
        fc = c;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      mu = fmin(mu, __shfl_xor_sync(0xffffffffu, mu, o));
      mr = fmin(mr, __shfl_xor_sync(0xffffffffu, mr, o));
      mc = fmin(mc, __shfl_xor_sync(0xffffffffu, mc, o));
      any0 |= __shfl_xor_sync(0xffffffffu, any0, o);
      anyR |= __shfl_xor_sync(0xffffffffu, anyR, o);
      const int ofr = __shfl_xor_sync(0xffffffffu, fr, o);
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
    int f0 = 0x7fffffff, fc0 = -1, flags = 0;
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
    if (any_s0 || fc0 >= 0) {
      for (int c = tid; c < C; c += blockDim.x) {
        if (a.count[c] == 0 || a.qlen_before[c] > 0 || a.running[c] != 0) continue;
        if (!any_s0 && c == fc0) continue;
        double u = bu, r = br, k = bc;
        if (any_r) {
          const int fcr = a.first_row[c];
          for (int x = 0; x < C; ++x) {  // non-lifted arrivals before c
            if (a.count[x] == 0 || a.qlen_before[x] > 0 || a.running[x] == 0) continue;
            if (a.first_row[x] < fcr) {
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
  for (int c = tid; c < C; c += blockDim.x) a.backlogged[c] = (a.qlen_before[c] + a.count[c]) > 0 ? 1 : 0;
}

// Stable scatter of row indices into per-client FIFO segments.  Each CTA owns one tile; each
// of its 8 warps walks a contiguous sub-tile 32 rows at a time in row order, ranking rows of
// the same client with __match_any_sync.  Walk 1 counts per (warp, client); scans over warps
// and clients give every row its slot in a client-sorted copy of the tile in shared memory
// (walk 2), which is then written to perm as contiguous per-client runs (coalesced).
__global__ void __launch_bounds__(kDrainThreads) drain_rank_kernel(const DrainArgs a) {
  extern __shared__ __align__(16) uint32_t sh[];
  const int32_t C = a.C;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int32_t tile = blockIdx.x;
  const int32_t sub = a.tile_rows / 8;
  const int32_t t0 = tile * a.tile_rows;
  const int32_t t1 = min(a.n, t0 + a.tile_rows);
  const int32_t r0 = t0 + warp * sub;
  const int32_t r1 = min(a.n, r0 + sub);
  const unsigned lt = (1u << lane) - 1u;
  uint32_t* base = sh;                                     // [C] global start of this tile's run
  uint32_t* toff = sh + C;                                 // [C] tile-local start / totals
  uint16_t* wc = reinterpret_cast<uint16_t*>(sh + 2 * C);  // [8][C]
  for (int c = tid; c < C; c += blockDim.x) base[c] = a.hist[static_cast<int64_t>(c) * a.n_tiles + tile];
  for (int i = tid; i < 8 * C; i += blockDim.x) wc[i] = 0;
  __syncthreads();
  uint16_t* my = wc + warp * C;
  for (int32_t r = r0; r < r1; r += 32) {  // walk 1: counts per (warp, client)
    const int32_t row = r + lane;
    const int32_t c = row < r1 ? a.client[row] : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, c);
    const int leader = __ffs(peers) - 1;
    if (static_cast<uint32_t>(c) < static_cast<uint32_t>(C) && lane == leader)
      my[c] = static_cast<uint16_t>(my[c] + __popc(peers));
    __syncwarp();
  }
  __syncthreads();
  for (int c = tid; c < C; c += blockDim.x) {  // exclusive over warps; total per client
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
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
    uint32_t* srow = sh + 6 * C;                                      // [tile_rows]
    uint16_t* scl = reinterpret_cast<uint16_t*>(srow + a.tile_rows);  // [tile_rows]
    for (int32_t r = r0; r < r1; r += 32) {  // walk 2: slot in the client-sorted tile
      const int32_t row = r + lane;
      const int32_t c = row < r1 ? a.client[row] : -1;
      const unsigned peers = __match_any_sync(0xffffffffu, c);
      const int leader = __ffs(peers) - 1;
      uint32_t start = 0;
      const bool ok = static_cast<uint32_t>(c) < static_cast<uint32_t>(C);
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
      const unsigned peers = __match_any_sync(0xffffffffu, c);
      const int leader = __ffs(peers) - 1;
      uint32_t start = 0;
      const bool ok = static_cast<uint32_t>(c) < static_cast<uint32_t>(C);
      if (ok && lane == leader) {
        start = my[c];
        my[c] = static_cast<uint16_t>(start + __popc(peers));
      }
      start = __shfl_sync(0xffffffffu, start, leader);
      if (ok) a.perm[base[c] + start + __popc(peers & lt)] = static_cast<uint32_t>(row);
      __syncwarp();
    }
  }
  if (!last_cta(&a.done[1])) return;
  lift_epilogue(a);
  if (threadIdx.x == 0) a.done[1] = 0;
}

// ===================================== scoring ===========================================

// Whole-queue scoring: 8 requests per thread per iteration (two 16-byte vectors of every
// column issued before any compute), streaming stores of pred/bucket/ufc_inc/rfc_inc.
__global__ void __launch_bounds__(kScoreThreads) score_kernel(const ScoreArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  stage_model(a.model, a.model_words, smem);
  __syncthreads();
  const ModelTables& M = *reinterpret_cast<const ModelTables*>(smem);
  if (threadIdx.x == 0) atomicMin(&a.st->t[4], global_ns());
  const int64_t n = a.n;
  uint32_t fb = 0, nt = 0;
  const bool oracle_like = M.pred_kind == kPredOracle || M.pred_kind == kPredNoisy;
  const int64_t nvec = a.vec_ok ? n / 8 : 0;  // groups of 8 rows
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t v = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; v < nvec; v += stride) {
    int4 cl[2], in4[2], to[2];
    double2 ar[4];
    uint32_t tg[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      cl[h] = ldg_stream(reinterpret_cast<const int4*>(a.client) + 2 * v + h);
      in4[h] = ldg_stream(reinterpret_cast<const int4*>(a.in_tok) + 2 * v + h);
      tg[h] = ldg_stream(reinterpret_cast<const uint32_t*>(a.tag) + 2 * v + h);
      to[h] = oracle_like ? ldg_stream(reinterpret_cast<const int4*>(a.true_out) + 2 * v + h)
                          : make_int4(1, 1, 1, 1);
    }
#pragma unroll
    for (int h = 0; h < 4; ++h) ar[h] = ldg_stream(reinterpret_cast<const double2*>(a.arrival) + 4 * v + h);
    const int64_t r0 = 8 * v;
    const int cs[8] = {cl[0].x, cl[0].y, cl[0].z, cl[0].w, cl[1].x, cl[1].y, cl[1].z, cl[1].w};
    const int ins[8] = {in4[0].x, in4[0].y, in4[0].z, in4[0].w, in4[1].x, in4[1].y, in4[1].z, in4[1].w};
    const int tos[8] = {to[0].x, to[0].y, to[0].z, to[0].w, to[1].x, to[1].y, to[1].z, to[1].w};
    const double arr[8] = {ar[0].x, ar[0].y, ar[1].x, ar[1].y, ar[2].x, ar[2].y, ar[3].x, ar[3].y};
    Scored s[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int64_t id = (M.pred_kind == kPredNoisy && a.id) ? a.id[r0 + k] : a.id_base + r0 + k;
      const double w = __ldg(a.weight + cs[k]);
      s[k] = score_request(M, a.pol, a.now, ins[k], (tg[k >> 2] >> (8 * (k & 3))) & 0xffu, tos[k], id, arr[k], w);
      fb += s[k].fallback;
      nt += s[k].near_tie;
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      stg_stream(reinterpret_cast<int4*>(a.pred_out) + 2 * v + h,
                 make_int4(s[4 * h].pred, s[4 * h + 1].pred, s[4 * h + 2].pred, s[4 * h + 3].pred));
      stg_stream(reinterpret_cast<uint32_t*>(a.bucket_out) + 2 * v + h,
                 static_cast<uint32_t>(s[4 * h].bucket) | (static_cast<uint32_t>(s[4 * h + 1].bucket) << 8) |
                     (static_cast<uint32_t>(s[4 * h + 2].bucket) << 16) |
                     (static_cast<uint32_t>(s[4 * h + 3].bucket) << 24));
    }
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      stg_stream(reinterpret_cast<double2*>(a.ufc_out) + 4 * v + h, make_double2(s[2 * h].ufc_inc, s[2 * h + 1].ufc_inc));
      stg_stream(reinterpret_cast<double2*>(a.rfc_out) + 4 * v + h, make_double2(s[2 * h].rfc_inc, s[2 * h + 1].rfc_inc));
    }
  }
  for (int64_t r = 8 * nvec + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < n; r += stride) {
    const int32_t c = a.client[r];
    const int64_t id = a.id ? a.id[r] : a.id_base + r;
    const Scored s = score_request(M, a.pol, a.now, a.in_tok[r], a.tag[r], oracle_like ? a.true_out[r] : 1, id,
                                   a.arrival[r], a.weight[c]);
    a.pred_out[r] = s.pred;
    a.bucket_out[r] = static_cast<uint8_t>(s.bucket);
    a.ufc_out[r] = s.ufc_inc;
    a.rfc_out[r] = s.rfc_inc;
    fb += s.fallback;
    nt += s.near_tie;
  }
  fb = __reduce_add_sync(0xffffffffu, fb);
  nt = __reduce_add_sync(0xffffffffu, nt);
  if ((threadIdx.x & 31) == 0) {
    if (fb) atomicAdd(&a.st->fallbacks, static_cast<unsigned long long>(fb));
    if (nt) atomicAdd(&a.st->near_ties, static_cast<unsigned long long>(nt));
  }
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&a.st->t[5], global_ns());
}

// ===================================== selection =========================================

// Candidate tuple of select_next (scheduler.cpp:139-153): (key, head arrival, client_id rank),
// all as integers.  o = 0xffffffff marks "no candidate".
struct Cand {
  uint64_t k;
  uint64_t a;
  uint32_t o;
};

__device__ __forceinline__ bool better(const Cand& x, const Cand& y) {
  const bool lt = (x.k < y.k) | ((x.k == y.k) & ((x.a < y.a) | ((x.a == y.a) & (x.o < y.o))));
  return (x.o != 0xffffffffu) & ((y.o == 0xffffffffu) | lt);
}

__device__ __forceinline__ Cand no_cand() { return Cand{0ull, 0ull, 0xffffffffu}; }

__device__ __forceinline__ Cand warp_argmin(Cand v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    Cand w;
    w.k = __shfl_xor_sync(0xffffffffu, v.k, o);
    w.a = __shfl_xor_sync(0xffffffffu, v.a, o);
    w.o = __shfl_xor_sync(0xffffffffu, v.o, o);
    if (better(w, v)) v = w;
  }
  return v;
}

// Per-client working state of the loop (shared memory, or global scratch for huge rosters).
struct ClientWork {
  uint64_t* kb;     // ordered bits of the selection key of the current head
  uint64_t* ab;     // ordered bits of the head arrival
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
enum : int32_t { kDone = 1, kDirty = 2, kNeedMax = 4 };

struct SelShared {
  Cand wbest[32];
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

__device__ __forceinline__ WinEntry entry_of_row(const SelectArgs& a, const ModelTables& M, int32_t c,
                                                 int32_t row, double w) {
  const int64_t id = a.id ? a.id[row] : a.id_base + row;
  const double arr = a.arrival[row];
  const int32_t in = a.in_tok[row];
  const Scored s = score_request(M, a.pol, a.now, in, a.tag[row], a.true_out ? a.true_out[row] : 1, id, arr, w);
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

__device__ __forceinline__ WinEntry get_entry(const SelectArgs& a, const ModelTables& M, const WinEntry* win,
                                              const ClientWork& cw, int32_t c, int32_t j) {
  const int32_t k = j - cw.pos0[c];
  if (k < a.W) return win[static_cast<int64_t>(c) * a.W + k];
  return entry_of_row(a, M, c, static_cast<int32_t>(a.perm[a.seg_off[c] + j]), cw.w[c]);  // deep head
}

__device__ __forceinline__ Cand cand_of(const ClientWork& cw, int32_t c) {
  if (cw.pos[c] < cw.end[c] && !(cw.flags[c] & kSkipped)) return Cand{cw.kb[c], cw.ab[c], cw.order[c]};
  return no_cand();
}

// One iteration of admit_requests' loop body for the chosen client (engine.cpp:216-268),
// run by the thread that owns the client.  Returns kDone / kDirty / kNeedMax.
__device__ __forceinline__ int32_t process_pick(const SelectArgs& a, const ModelTables& M, const WinEntry* win,
                                                const ClientWork& cw, SelShared& S, int32_t c) {
  const Policy& P = a.pol;
  const bool maxmode = P.kind == kEquinox && P.norm_mode == 0;
  const int32_t j = cw.pos[c];
  const WinEntry e = get_entry(a, M, win, cw, c, j);
  if (!e.alone) {  // engine.cpp:223-234: Rejected, pop_head, no counter change
    const int64_t k = S.n_ev++;
    if (k < a.ev_cap) {
      a.ev_row[k] = e.row;
      a.ev_kind[k] = 2;
      a.ev_client[k] = c;
      a.ev_pred[k] = e.pred;
      a.ev_ufc[k] = 0.0;
      a.ev_rfc[k] = 0.0;
      a.ev_vtc[k] = 0.0;
      a.ev_wait[k] = 0.0;
    }
    S.n_rej++;
    cw.pos[c] = j + 1;
    if (j + 1 == cw.end[c]) {
      cw.flags[c] &= ~kBacklogged;
      if (maxmode && (cw.ufc[c] == S.max_u || cw.rfc[c] == S.max_r)) return kDirty | kNeedMax;
    } else {
      cw.ab[c] = get_entry(a, M, win, cw, c, j + 1).abits;
    }
    return 0;
  }
  // can_fit (gpu_model.cpp:58-67) with the KV test as the exact integer threshold
  if (!((S.members + 1 <= P.max_batch) && (S.reserved + e.in + e.pred <= a.tmax))) {
    if (P.backfill) {  // engine.cpp:236-238
      cw.flags[c] |= kSkipped;
      return 0;
    }
    return kDone;  // engine.cpp:239
  }
  // admit (engine.cpp:242-268) + on_admit (scheduler.cpp:158-183)
  S.members += 1;
  S.reserved += static_cast<int64_t>(e.in) + e.pred;  // reserved_output = pred, generated = 0
  S.prefill += e.in;
  const double old_u = cw.ufc[c], old_r = cw.rfc[c];
  const double nu = __dadd_rn(old_u, e.ufc_inc), nr = __dadd_rn(old_r, e.rfc_inc);
  cw.ufc[c] = nu;
  cw.rfc[c] = nr;
  double vtc = 0.0;
  if (P.kind == kVtc) {
    const double w = cw.w[c];
    vtc = P.vtc_use_prediction
              ? __dmul_rn(w, __dadd_rn(static_cast<double>(e.in), __dmul_rn(P.ow, static_cast<double>(e.pred))))
              : __dmul_rn(w, static_cast<double>(e.in));
    cw.cnt[c] = __dadd_rn(cw.cnt[c], vtc);
  }
  cw.adm[c] += 1;
  const int64_t k = S.n_ev++;
  if (k < a.ev_cap) {
    a.ev_row[k] = e.row;
    a.ev_kind[k] = 1;
    a.ev_client[k] = c;
    a.ev_pred[k] = e.pred;
    a.ev_ufc[k] = e.ufc_inc;
    a.ev_rfc[k] = e.rfc_inc;
    a.ev_vtc[k] = vtc;
    a.ev_wait[k] = __dsub_rn(a.now, from_ordered_bits(e.abits));
  }
  S.n_adm++;
  cw.pos[c] = j + 1;
  if (j + 1 == cw.end[c]) {  // pop_head emptied the queue: set_backlogged(false)
    cw.flags[c] &= ~kBacklogged;
    if (maxmode && (old_u == S.max_u || old_r == S.max_r)) return kDirty | kNeedMax;
    return 0;
  }
  cw.ab[c] = get_entry(a, M, win, cw, c, j + 1).abits;
  if (maxmode) {
    bool d = false;
    if (S.max_u < nu) {
      S.max_u = nu;
      d = true;
    }
    if (S.max_r < nr) {
      S.max_r = nr;
      d = true;
    }
    if (d) return kDirty;
  }
  cw.kb[c] = ordered_bits(hf_key(P, nu, nr, S.max_u, S.max_r, cw.cnt[c]));
  return 0;
}

__device__ __forceinline__ Cand rescan_owned(const ClientWork& cw, int32_t C, int tid, int nthr) {
  Cand best = no_cand();
  for (int32_t c = tid; c < C; c += nthr) {
    const Cand v = cand_of(cw, c);
    if (better(v, best)) best = v;
  }
  return best;
}

__device__ __forceinline__ Cand recompute_owned(const Policy& P, const ClientWork& cw, int32_t C, int tid, int nthr,
                                                double mu, double mr) {
  Cand best = no_cand();
  for (int32_t c = tid; c < C; c += nthr) {
    cw.kb[c] = ordered_bits(hf_key(P, cw.ufc[c], cw.rfc[c], mu, mr, cw.cnt[c]));
    const Cand v = cand_of(cw, c);
    if (better(v, best)) best = v;
  }
  return best;
}

// Max over backlogged clients (scheduler.cpp:40-48), starting from 0.0 like the reference.
__device__ __forceinline__ void group_maxima(const ClientWork& cw, int32_t C, int tid, int nthr, SelShared& S) {
  double mu = 0.0, mr = 0.0;
  for (int32_t c = tid; c < C; c += nthr) {
    if (!(cw.flags[c] & kBacklogged)) continue;
    if (mu < cw.ufc[c]) mu = cw.ufc[c];
    if (mr < cw.rfc[c]) mr = cw.rfc[c];
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double ou = __shfl_xor_sync(0xffffffffu, mu, o);
    const double orr = __shfl_xor_sync(0xffffffffu, mr, o);
    if (mu < ou) mu = ou;
    if (mr < orr) mr = orr;
  }
  const int nw = nthr >> 5;
  if (nw == 1) {
    if (tid == 0) {
      S.max_u = mu;
      S.max_r = mr;
    }
    __syncwarp();
    return;
  }
  const int lane = tid & 31, warp = tid >> 5;
  if (lane == 0) {
    S.red_u[warp] = mu;
    S.red_r[warp] = mr;
  }
  named_sync(1, nthr);
  if (tid == 0) {
    double u = 0.0, r = 0.0;
    for (int w = 0; w < nw; ++w) {
      if (u < S.red_u[w]) u = S.red_u[w];
      if (r < S.red_r[w]) r = S.red_r[w];
    }
    S.max_u = u;
    S.max_r = r;
  }
  named_sync(1, nthr);
}

__global__ void __launch_bounds__(kSelectMaxThreads, 1) select_kernel(const SelectArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ SelShared S;
  const int32_t C = a.C;
  const int tid = threadIdx.x, NT = blockDim.x;
  stage_model(a.model, a.model_words, smem);
  if (tid == 0) a.st->t[0] = global_ns();
  // ---- carve per-client work arrays + windows ----
  unsigned char* p = smem + ((a.model_words * 4 + 15) & ~15);
  unsigned char* g = reinterpret_cast<unsigned char*>(a.cw_global);
  auto take = [&](size_t bytes) {
    unsigned char** q = a.cw_in_smem ? &p : &g;
    unsigned char* r = *q;
    *q += (bytes + 15) & ~size_t(15);
    return r;
  };
  ClientWork cw;
  cw.kb = reinterpret_cast<uint64_t*>(take(8ull * C));
  cw.ab = reinterpret_cast<uint64_t*>(take(8ull * C));
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
  WinEntry* win = reinterpret_cast<WinEntry*>(p);
  __syncthreads();
  const ModelTables& M = *reinterpret_cast<const ModelTables*>(smem);
  const Policy& P = a.pol;

  // ---- whole CTA: ledger in, head windows (first W queued entries per client) ----
  for (int32_t c = tid; c < C; c += NT) {
    cw.ufc[c] = a.ufc[c];
    cw.rfc[c] = a.rfc[c];
    cw.cnt[c] = a.counter[c];
    cw.w[c] = a.weight[c];
    cw.pos[c] = a.head[c];
    cw.pos0[c] = a.head[c];
    cw.end[c] = a.count[c];
    const uint32_t o = a.order[c];
    cw.order[c] = o;
    cw.by_order[o] = c;
    cw.flags[c] = a.backlogged[c] ? kBacklogged : 0;
    cw.adm[c] = 0;
  }
  __syncthreads();
  const int64_t items = static_cast<int64_t>(C) * a.W;
  constexpr int kU = 4;  // independent gathers in flight per thread
  for (int64_t b = tid; b < items; b += kU * NT) {
    int32_t rows[kU], cs[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t it = b + static_cast<int64_t>(u) * NT;
      rows[u] = -1;
      cs[u] = 0;
      if (it < items) {
        const int32_t c = static_cast<int32_t>(it / a.W);
        const int32_t j = cw.pos0[c] + static_cast<int32_t>(it % a.W);
        cs[u] = c;
        if (j < cw.end[c]) rows[u] = static_cast<int32_t>(a.perm[a.seg_off[c] + j]);
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (rows[u] >= 0) win[b + static_cast<int64_t>(u) * NT] = entry_of_row(a, M, cs[u], rows[u], cw.w[cs[u]]);
  }
  __syncthreads();
  if (tid == 0) {
    a.st->t[1] = global_ns();
    S.n_ev = S.n_adm = S.n_rej = S.prefill = 0;
    S.members = a.st->members;
    S.reserved = a.st->reserved;
  }
  const int nthr = a.sel_threads;
  if (tid >= nthr) return;  // spare warps leave; the loop's barriers are named with nthr
  for (int32_t c = tid; c < C; c += nthr)
    cw.ab[c] = cw.pos[c] < cw.end[c] ? get_entry(a, M, win, cw, c, cw.pos[c]).abits : 0ull;
  named_sync(1, nthr);
  group_maxima(cw, C, tid, nthr, S);
  Cand local = recompute_owned(P, cw, C, tid, nthr, S.max_u, S.max_r);
  const int lane = tid & 31, warp = tid >> 5, nw = nthr >> 5;
  named_sync(1, nthr);
  if (tid == 0) a.st->t[2] = global_ns();

  for (;;) {
    Cand v = warp_argmin(local);
    if (nw > 1) {  // every warp reduces the warp winners redundantly: one barrier per pick
      if (lane == 0) S.wbest[warp] = v;
      named_sync(1, nthr);
      v = warp_argmin(lane < nw ? S.wbest[lane] : no_cand());
    }
    if (v.o == 0xffffffffu) break;  // no candidates (engine.cpp:217)
    const int32_t c = cw.by_order[v.o];
    const int owner = c % nthr;
    int32_t f = 0;
    if (tid == owner) f = process_pick(a, M, win, cw, S, c);
    if (nw == 1) {
      f = __shfl_sync(0xffffffffu, f, owner);
      __syncwarp();
    } else {
      if (tid == owner) S.flags = f;
      named_sync(1, nthr);
      f = S.flags;
    }
    if (f & kDone) break;
    if (f & kDirty) {
      if (f & kNeedMax) group_maxima(cw, C, tid, nthr, S);
      local = recompute_owned(P, cw, C, tid, nthr, S.max_u, S.max_r);
    } else if (tid == owner) {
      local = rescan_owned(cw, C, tid, nthr);
    }
  }
  named_sync(1, nthr);
  if (tid == 0) a.st->t[3] = global_ns();
  // ---- write back ledger, heads, batch, summary ----
  for (int32_t c = tid; c < C; c += nthr) {
    a.ufc[c] = cw.ufc[c];
    a.rfc[c] = cw.rfc[c];
    a.counter[c] = cw.cnt[c];
    a.head[c] = cw.pos[c];
    a.backlogged[c] = (cw.flags[c] & kBacklogged) ? 1 : 0;
    a.running[c] += cw.adm[c];
  }
  if (tid == 0) {
    a.st->members = S.members;
    a.st->reserved = S.reserved;
    a.st->n_events = S.n_ev;
    a.st->n_admitted = S.n_adm;
    a.st->n_rejected = S.n_rej;
    a.st->new_prefill = S.prefill;
  }
}

__global__ void gather_ids_kernel(const int32_t* __restrict__ rows, int64_t n, const int64_t* __restrict__ id,
                                  int64_t id_base, int64_t* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = id ? id[rows[i]] : id_base + rows[i];
}

}  // namespace eqx
