// eqx_kernels.cu -- sm_100a kernels of the Equinox per-step scheduling path.
//
//   drain (engine.cpp:171-197, done once per arrival batch):
//     drain_hist_kernel   per-tile client histogram + first arrival row per client
//     scan_kernel         exclusive scan of the [client][tile] histogram -> FIFO segment offsets
//     drain_rank_kernel   stable per-client rank inside each tile (warp match_any walk) ->
//                         perm: row indices grouped by client, FIFO (arrival) order kept
//     lift_kernel         on_activated counter lift in arrival order (scheduler.cpp:235-253)
//   step (admit_requests, engine.cpp:207-271, plus whole-queue scoring):
//     step_kernel         CTA 0 runs the exact sequential admission loop over client heads
//                         (select_next/holistic_score/can_fit/on_admit semantics); every other
//                         CTA streams the whole queue through predict -> map -> increments
//                         (coalesced 16-byte loads, streaming stores), overlapping the two.
//     gather_ids_kernel   event rows -> request ids for the caller.
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
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t ldg_stream(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void stg_stream(int4* p, int4 v) {
  asm volatile("st.global.cs.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
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

}  // namespace

// ===================================== drain =============================================

__global__ void drain_hist_kernel(const int32_t* __restrict__ client, int32_t n, int32_t C,
                                  int32_t tile_rows, int32_t n_tiles, uint32_t* __restrict__ hist,
                                  int32_t* __restrict__ first_row, int32_t* __restrict__ count,
                                  DevState* st) {
  extern __shared__ uint32_t sh[];
  uint32_t* cnt = sh;
  uint32_t* mn = sh + C;
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    cnt[c] = 0;
    mn[c] = 0xffffffffu;
  }
  __syncthreads();
  const int32_t tile = blockIdx.x;
  const int32_t r0 = tile * tile_rows;
  const int32_t r1 = min(n, r0 + tile_rows);
  for (int32_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
    const int32_t c = client[r];
    if (c < 0 || c >= C) {
      st->bad_client = 1;
      continue;
    }
    atomicAdd(&cnt[c], 1u);
    atomicMin(&mn[c], static_cast<uint32_t>(r));
  }
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    const uint32_t k = cnt[c];
    hist[static_cast<int64_t>(c) * n_tiles + tile] = k;
    if (k) {
      atomicAdd(&count[c], static_cast<int32_t>(k));
      atomicMin(&first_row[c], static_cast<int32_t>(mn[c]));
    }
  }
}

// Single-CTA exclusive scan (1024 threads, 4 elements per thread per round) of L elements in
// place; seg_off[c] = scanned value of (client c, tile 0); seg_off[C] = total.
__global__ void __launch_bounds__(1024) scan_kernel(uint32_t* __restrict__ data, int64_t L,
                                                    int32_t C, int32_t n_tiles,
                                                    int32_t* __restrict__ seg_off) {
  __shared__ uint32_t warp_sums[32];
  __shared__ uint32_t carry_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) carry_s = 0;
  __syncthreads();
  for (int64_t base = 0; base < L; base += 4096) {
    const int64_t i0 = base + 4 * static_cast<int64_t>(tid);
    uint32_t v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = (i0 + k < L) ? data[i0 + k] : 0u;
    const uint32_t local = v[0] + v[1] + v[2] + v[3];
    uint32_t incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) warp_sums[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      uint32_t w = warp_sums[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += t;
      }
      warp_sums[lane] = w;  // inclusive
    }
    __syncthreads();
    const uint32_t carry = carry_s;
    uint32_t run = carry + (warp ? warp_sums[warp - 1] : 0u) + (incl - local);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (i0 + k < L) {
        const int64_t idx = i0 + k;
        data[idx] = run;
        if (idx % n_tiles == 0) seg_off[idx / n_tiles] = static_cast<int32_t>(run);
      }
      run += v[k];
    }
    __syncthreads();
    if (tid == 0) carry_s = carry + warp_sums[31];
    __syncthreads();
  }
  if (tid == 0) seg_off[C] = static_cast<int32_t>(carry_s);
}

// Stable scatter of row indices into per-client FIFO segments.  Each CTA owns one tile; each
// of its 8 warps walks a contiguous sub-tile 32 rows at a time in row order, ranking rows of
// the same client with __match_any_sync.  Walk 1 counts per (warp, client); an exclusive scan
// over warps gives each warp's start inside the tile's slice of the client segment; walk 2
// writes perm.  Per-(warp,client) counters are u16 (sub-tile <= 65535 rows).
__global__ void __launch_bounds__(256) drain_rank_kernel(const int32_t* __restrict__ client,
                                                         int32_t n, int32_t C, int32_t tile_rows,
                                                         int32_t n_tiles,
                                                         const uint32_t* __restrict__ tile_off,
                                                         uint32_t* __restrict__ perm) {
  extern __shared__ uint32_t sh[];
  uint32_t* base = sh;                                       // [C] tile offset per client
  uint16_t* wc = reinterpret_cast<uint16_t*>(sh + C);        // [8][C]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int32_t tile = blockIdx.x;
  for (int c = tid; c < C; c += blockDim.x) base[c] = tile_off[static_cast<int64_t>(c) * n_tiles + tile];
  for (int i = tid; i < 8 * C; i += blockDim.x) wc[i] = 0;
  __syncthreads();
  const int32_t sub = tile_rows / 8;
  const int32_t r0 = tile * tile_rows + warp * sub;
  const int32_t r1 = min(n, r0 + sub);
  uint16_t* my = wc + warp * C;
  const unsigned lt = (1u << lane) - 1u;
  for (int32_t r = r0; r < r1; r += 32) {
    const int32_t row = r + lane;
    const int32_t c = row < r1 ? client[row] : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, c);
    const int leader = __ffs(peers) - 1;
    if (c >= 0 && c < C && lane == leader) my[c] = static_cast<uint16_t>(my[c] + __popc(peers));
    __syncwarp();
  }
  __syncthreads();
  for (int c = tid; c < C; c += blockDim.x) {
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      const uint32_t t = wc[w * C + c];
      wc[w * C + c] = static_cast<uint16_t>(run);
      run += t;
    }
  }
  __syncthreads();
  for (int32_t r = r0; r < r1; r += 32) {
    const int32_t row = r + lane;
    const int32_t c = row < r1 ? client[row] : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, c);
    const int leader = __ffs(peers) - 1;
    uint32_t start = 0;
    if (c >= 0 && c < C && lane == leader) {
      start = my[c];
      my[c] = static_cast<uint16_t>(start + __popc(peers));
    }
    start = __shfl_sync(0xffffffffu, start, leader);
    if (c >= 0 && c < C) perm[base[c] + start + __popc(peers & lt)] = static_cast<uint32_t>(row);
    __syncwarp();
  }
}

// on_activated for every client that goes idle -> backlogged in this drain, in arrival order.
// The lift target is the componentwise min over *other* backlogged clients at that moment.
// Lifted values are >= that min, so the running min only moves when a client that is NOT
// lifted joins the backlog: pre-backlogged clients (qlen_before > 0), the very first arrival
// when nobody was backlogged, and clients with running requests (engine.cpp:182).  Hence
// m(c) = min(base, {vals(r) : r non-lifted arrival, first_row[r] < first_row[c]}).
__global__ void __launch_bounds__(1024) lift_kernel(int32_t C, const int32_t* __restrict__ count,
                                                    const int32_t* __restrict__ first_row,
                                                    const int32_t* __restrict__ qlen_before,
                                                    const int32_t* __restrict__ running,
                                                    double* __restrict__ ufc, double* __restrict__ rfc,
                                                    double* __restrict__ counter,
                                                    int32_t* __restrict__ backlogged,
                                                    int32_t counter_lift) {
  __shared__ double s_min[3][32];
  __shared__ int s_first[32], s_firstc[32];
  __shared__ int s_any0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  if (counter_lift) {
    // base over S0 = {qlen_before > 0} and the first arriving client (argmin first_row)
    double mu = INFINITY, mr = INFINITY, mc = INFINITY;
    int any0 = 0;
    int fr = 0x7fffffff, fc = -1;
    for (int c = tid; c < C; c += blockDim.x) {
      if (qlen_before[c] > 0) {
        any0 = 1;
        mu = fmin(mu, ufc[c]);
        mr = fmin(mr, rfc[c]);
        mc = fmin(mc, counter[c]);
      }
      if (count[c] > 0 && first_row[c] < fr) {
        fr = first_row[c];
        fc = c;
      }
    }
    for (int o = 16; o; o >>= 1) {
      mu = fmin(mu, __shfl_xor_sync(0xffffffffu, mu, o));
      mr = fmin(mr, __shfl_xor_sync(0xffffffffu, mr, o));
      mc = fmin(mc, __shfl_xor_sync(0xffffffffu, mc, o));
      any0 |= __shfl_xor_sync(0xffffffffu, any0, o);
      const int ofr = __shfl_xor_sync(0xffffffffu, fr, o);
      const int ofc = __shfl_xor_sync(0xffffffffu, fc, o);
      if (ofr < fr) {
        fr = ofr;
        fc = ofc;
      }
    }
    if (tid == 0) s_any0 = 0;
    __syncthreads();
    if (lane == 0) {
      s_min[0][warp] = mu;
      s_min[1][warp] = mr;
      s_min[2][warp] = mc;
      s_first[warp] = fr;
      s_firstc[warp] = fc;
      if (any0) atomicOr(&s_any0, 1);
    }
    __syncthreads();
    double bu = INFINITY, br = INFINITY, bc = INFINITY;
    int f0 = 0x7fffffff, fc0 = -1;
    for (int w = 0; w < nw; ++w) {
      bu = fmin(bu, s_min[0][w]);
      br = fmin(br, s_min[1][w]);
      bc = fmin(bc, s_min[2][w]);
      if (s_first[w] < f0) {
        f0 = s_first[w];
        fc0 = s_firstc[w];
      }
    }
    const bool any_s0 = s_any0 != 0;
    if (!any_s0 && fc0 >= 0) {
      bu = ufc[fc0];
      br = rfc[fc0];
      bc = counter[fc0];
    }
    __syncthreads();
    if (any_s0 || fc0 >= 0) {
      for (int c = tid; c < C; c += blockDim.x) {
        if (count[c] == 0 || qlen_before[c] > 0 || running[c] != 0) continue;
        if (!any_s0 && c == fc0) continue;
        double u = bu, r = br, k = bc;
        const int fcr = first_row[c];
        for (int x = 0; x < C; ++x) {  // non-lifted arrivals before c (usually none)
          if (count[x] == 0 || qlen_before[x] > 0 || running[x] == 0) continue;
          if (first_row[x] < fcr) {
            u = fmin(u, ufc[x]);
            r = fmin(r, rfc[x]);
            k = fmin(k, counter[x]);
          }
        }
        // std::max(own, min): own unless own < min
        if (ufc[c] < u) ufc[c] = u;
        if (rfc[c] < r) rfc[c] = r;
        if (counter[c] < k) counter[c] = k;
      }
    }
  }
  for (int c = tid; c < C; c += blockDim.x) backlogged[c] = (qlen_before[c] + count[c]) > 0 ? 1 : 0;
}

// ===================================== step ==============================================

struct Cand {
  double key;
  double arr;
  uint32_t order;
  int32_t c;
};

__device__ __forceinline__ bool better(const Cand& a, const Cand& b) {
  if (a.c < 0) return false;
  if (b.c < 0) return true;
  if (a.key < b.key) return true;
  if (b.key < a.key) return false;
  if (a.arr < b.arr) return true;
  if (b.arr < a.arr) return false;
  return a.order < b.order;
}

__device__ __forceinline__ Cand warp_argmin(Cand v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    Cand w;
    w.key = __shfl_xor_sync(0xffffffffu, v.key, o);
    w.arr = __shfl_xor_sync(0xffffffffu, v.arr, o);
    w.order = __shfl_xor_sync(0xffffffffu, v.order, o);
    w.c = __shfl_xor_sync(0xffffffffu, v.c, o);
    if (better(w, v)) v = w;
  }
  return v;
}

// Per-client working state of the selection loop (smem when it fits, else global scratch).
struct ClientWork {
  double* key;
  double* arr;
  double* ufc;
  double* rfc;
  double* cnt;
  double* w;
  int32_t* pos;   // absolute FIFO position of the current head
  int32_t* end;   // queue length (absolute)
  int32_t* pos0;  // head at step start (window base)
  uint32_t* order;
  int32_t* flags; // bit0 backlogged, bit1 skipped (backfill)
  int32_t* adm;   // admitted this step (running += adm at the end)
};

enum : int32_t { kBacklogged = 1, kSkipped = 2 };
enum : int32_t { kDone = 1, kDirty = 2, kNeedMax = 4 };

__device__ __forceinline__ double hf_key(const Policy& P, double u, double r, double mu, double mr,
                                         double cnt) {
  if (P.kind == kFcfs) return 0.0;  // scheduler.cpp:122
  if (P.kind == kVtc) return cnt;   // scheduler.cpp:124
  if (P.norm_mode == 1) return __dadd_rn(__dmul_rn(P.alpha, u), __dmul_rn(P.beta, r));  // :51
  const double uu = mu > 0.0 ? __ddiv_rn(u, mu) : 0.0;  // scheduler.cpp:53-57
  const double rr = mr > 0.0 ? __ddiv_rn(r, mr) : 0.0;
  return __dadd_rn(__dmul_rn(P.alpha, uu), __dmul_rn(P.beta, rr));
}

struct SelShared {
  Cand wbest[32];
  double red_u[32];
  double red_r[32];
  double max_u, max_r;
  int32_t flags;
  int32_t changed;
  int64_t n_ev, n_adm, n_rej, prefill;
  int32_t members;
  int64_t reserved;
};

__device__ __forceinline__ WinEntry entry_of_row(const StepArgs& a, const ModelTables& M, int32_t c,
                                                 int32_t row) {
  const int64_t id = a.id ? a.id[row] : a.id_base + row;
  const double arr = a.arrival[row];
  const int32_t in = a.in_tok[row];
  const Scored s = score_request(M, a.pol, a.now, in, a.tag[row], a.true_out ? a.true_out[row] : 1, id, arr,
                                 a.weight[c]);
  WinEntry e;
  e.ufc_inc = s.ufc_inc;
  e.rfc_inc = s.rfc_inc;
  e.arrival = arr;
  e.in = in;
  e.pred = s.pred;
  e.row = row;
  e.pad = 0;
  return e;
}

__device__ WinEntry fetch_entry(const StepArgs& a, const ModelTables& M, int32_t c, int32_t j) {
  return entry_of_row(a, M, c, static_cast<int32_t>(a.perm[a.seg_off[c] + j]));
}

__device__ __forceinline__ WinEntry get_entry(const StepArgs& a, const ModelTables& M,
                                              const WinEntry* win, const ClientWork& cw,
                                              int32_t c, int32_t j) {
  const int32_t k = j - cw.pos0[c];
  if (k < a.W) return win[static_cast<int64_t>(c) * a.W + k];
  return fetch_entry(a, M, c, j);
}

// Thread 0 of the selection group: one iteration of admit_requests' while(true) body for the
// chosen client (engine.cpp:216-268).  Returns kDone / kDirty / kNeedMax flags.
__device__ int32_t process_pick(const StepArgs& a, const ModelTables& M, const WinEntry* win,
                                const ClientWork& cw, SelShared& S, const Cand& x) {
  S.changed = -1;
  if (x.c < 0) return kDone;  // no candidates (engine.cpp:217)
  const Policy& P = a.pol;
  const int32_t c = x.c;
  const int32_t j = cw.pos[c];
  const WinEntry e = get_entry(a, M, win, cw, c, j);
  const bool maxmode = P.kind == kEquinox && P.norm_mode == 0;
  // fits_alone (gpu_model.cpp:69-72): can_fit on an empty batch
  const bool alone = (1 <= P.max_batch) &&
                     __dmul_rn(static_cast<double>(static_cast<int64_t>(e.in) + e.pred), P.m) <= P.M;
  if (!alone) {  // engine.cpp:223-234: log Rejected, pop_head, no counter change
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
      cw.arr[c] = get_entry(a, M, win, cw, c, j + 1).arrival;
    }
    S.changed = c;
    return 0;
  }
  // can_fit (gpu_model.cpp:58-67)
  const bool fits = (S.members + 1 <= P.max_batch) &&
                    __dmul_rn(static_cast<double>(S.reserved + e.in + e.pred), P.m) <= P.M;
  if (!fits) {
    if (P.backfill) {  // engine.cpp:236-238
      cw.flags[c] |= kSkipped;
      S.changed = c;
      return 0;
    }
    return kDone;  // engine.cpp:239
  }
  // admit (engine.cpp:242-268) + on_admit (scheduler.cpp:158-183)
  S.members += 1;
  S.reserved += static_cast<int64_t>(e.in) + e.pred;  // reserved_output = pred, generated = 0
  S.prefill += e.in;
  const double old_u = cw.ufc[c], old_r = cw.rfc[c];
  cw.ufc[c] = __dadd_rn(old_u, e.ufc_inc);
  cw.rfc[c] = __dadd_rn(old_r, e.rfc_inc);
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
    a.ev_wait[k] = __dsub_rn(a.now, e.arrival);
  }
  S.n_adm++;
  cw.pos[c] = j + 1;
  if (j + 1 == cw.end[c]) {  // pop_head emptied the queue: set_backlogged(false)
    cw.flags[c] &= ~kBacklogged;
    if (maxmode && (old_u == S.max_u || old_r == S.max_r)) return kDirty | kNeedMax;
    S.changed = c;
    return 0;
  }
  cw.arr[c] = get_entry(a, M, win, cw, c, j + 1).arrival;
  if (maxmode) {
    bool d = false;
    if (S.max_u < cw.ufc[c]) {
      S.max_u = cw.ufc[c];
      d = true;
    }
    if (S.max_r < cw.rfc[c]) {
      S.max_r = cw.rfc[c];
      d = true;
    }
    if (d) return kDirty;
  }
  cw.key[c] = hf_key(P, cw.ufc[c], cw.rfc[c], S.max_u, S.max_r, cw.cnt[c]);
  S.changed = c;
  return 0;
}

__device__ __forceinline__ Cand cand_of(const ClientWork& cw, int32_t c) {
  Cand v;
  const int32_t f = cw.flags[c];
  if (cw.pos[c] < cw.end[c] && !(f & kSkipped)) {
    v.key = cw.key[c];
    v.arr = cw.arr[c];
    v.order = cw.order[c];
    v.c = c;
  } else {
    v.key = 0.0;
    v.arr = 0.0;
    v.order = 0xffffffffu;
    v.c = -1;
  }
  return v;
}

// Max over backlogged clients (scheduler.cpp:40-48) by the selection group; starts at 0.0.
__device__ void group_maxima(const ClientWork& cw, int32_t C, int tid, int nthr, SelShared& S) {
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
  const int lane = tid & 31, warp = tid >> 5, nw = nthr >> 5;
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

__device__ Cand recompute_all(const Policy& P, const ClientWork& cw, int32_t C, int tid, int nthr,
                              const SelShared& S) {
  Cand best;
  best.c = -1;
  best.key = 0.0;
  best.arr = 0.0;
  best.order = 0xffffffffu;
  for (int32_t c = tid; c < C; c += nthr) {
    cw.key[c] = hf_key(P, cw.ufc[c], cw.rfc[c], S.max_u, S.max_r, cw.cnt[c]);
    const Cand v = cand_of(cw, c);
    if (better(v, best)) best = v;
  }
  return best;
}

__device__ Cand rescan_owned(const ClientWork& cw, int32_t C, int tid, int nthr) {
  Cand best;
  best.c = -1;
  best.key = 0.0;
  best.arr = 0.0;
  best.order = 0xffffffffu;
  for (int32_t c = tid; c < C; c += nthr) {
    const Cand v = cand_of(cw, c);
    if (better(v, best)) best = v;
  }
  return best;
}

__device__ void selection(const StepArgs& a, const ModelTables& M, unsigned char* smem) {
  const int32_t C = a.C;
  const int tid = threadIdx.x;
  const int nthr = a.sel_threads;  // multiple of 32, <= blockDim.x
  const int NT = blockDim.x;
  __shared__ SelShared S;
  // ---- carve per-client work arrays + windows ----
  ClientWork cw;
  unsigned char* p = smem;
  auto carve = [&](size_t bytes) {
    unsigned char* q = p;
    p += (bytes + 15) & ~size_t(15);
    return q;
  };
  unsigned char* g = reinterpret_cast<unsigned char*>(a.cw_global);
  auto take = [&](size_t bytes) {
    if (!a.cw_global) return carve(bytes);
    unsigned char* q = g;
    g += (bytes + 15) & ~size_t(15);
    return q;
  };
  cw.key = reinterpret_cast<double*>(take(8ull * C));
  cw.arr = reinterpret_cast<double*>(take(8ull * C));
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
  WinEntry* win = reinterpret_cast<WinEntry*>(carve(0));
  const Policy& P = a.pol;

  // ---- whole CTA: load the ledger, fill each client's head window (first W entries) ----
  for (int32_t c = tid; c < C; c += NT) {
    cw.ufc[c] = a.ufc[c];
    cw.rfc[c] = a.rfc[c];
    cw.cnt[c] = a.counter[c];
    cw.w[c] = a.weight[c];
    cw.pos[c] = a.head[c];
    cw.pos0[c] = a.head[c];
    cw.end[c] = a.count[c];
    cw.order[c] = a.order[c];
    cw.flags[c] = a.backlogged[c] ? kBacklogged : 0;
    cw.adm[c] = 0;
  }
  __syncthreads();
  const int64_t items = static_cast<int64_t>(C) * a.W;
  constexpr int kU = 4;  // 4 independent gathers in flight per thread
  for (int64_t base = tid; base < items; base += kU * NT) {
    int32_t rows[kU], cs[kU];
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      const int64_t it = base + static_cast<int64_t>(k) * NT;
      rows[k] = -1;
      cs[k] = 0;
      if (it < items) {
        const int32_t c = static_cast<int32_t>(it / a.W);
        const int32_t j = cw.pos0[c] + static_cast<int32_t>(it % a.W);
        cs[k] = c;
        if (j < cw.end[c]) rows[k] = static_cast<int32_t>(a.perm[a.seg_off[c] + j]);
      }
    }
#pragma unroll
    for (int k = 0; k < kU; ++k)
      if (rows[k] >= 0) win[base + static_cast<int64_t>(k) * NT] = entry_of_row(a, M, cs[k], rows[k]);
  }
  __syncthreads();
  if (tid >= nthr) return;  // spare warps leave; the loop's barriers are named with nthr
  for (int32_t c = tid; c < C; c += nthr)
    cw.arr[c] = cw.pos[c] < cw.end[c] ? get_entry(a, M, win, cw, c, cw.pos[c]).arrival : 0.0;
  if (tid == 0) {
    S.n_ev = S.n_adm = S.n_rej = S.prefill = 0;
    S.members = a.st->members;
    S.reserved = a.st->reserved;
    S.max_u = S.max_r = 0.0;
  }
  named_sync(1, nthr);
  group_maxima(cw, C, tid, nthr, S);
  Cand local = recompute_all(P, cw, C, tid, nthr, S);
  named_sync(1, nthr);

  const int lane = tid & 31, warp = tid >> 5, nw = nthr >> 5;
  for (;;) {
    const Cand v = warp_argmin(local);
    if (nw > 1) {
      if (lane == 0) S.wbest[warp] = v;
      named_sync(1, nthr);
    }
    if (warp == 0) {
      Cand x = v;
      if (nw > 1) {
        x = lane < nw ? S.wbest[lane] : Cand{0.0, 0.0, 0xffffffffu, -1};
        x = warp_argmin(x);
      }
      if (lane == 0) S.flags = process_pick(a, M, win, cw, S, x);
    }
    named_sync(1, nthr);
    const int32_t f = S.flags;
    if (f & kDone) break;
    if (f & kDirty) {
      if (f & kNeedMax) group_maxima(cw, C, tid, nthr, S);
      local = recompute_all(P, cw, C, tid, nthr, S);
      named_sync(1, nthr);
    } else {
      const int32_t cc = S.changed;
      if (cc >= 0 && (cc % nthr) == tid) local = rescan_owned(cw, C, tid, nthr);
    }
  }
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

// Whole-queue scoring by worker CTAs: 4 requests per thread per iteration through 16-byte
// loads of the SoA columns, streaming stores of pred/bucket/ufc_inc/rfc_inc.
__device__ void score_stream(const StepArgs& a, const ModelTables& M, int worker, int nworkers) {
  const int tid = threadIdx.x;
  const int64_t n = a.n;
  uint32_t fb = 0, nt = 0;
  const bool oracle_like = M.pred_kind == kPredOracle || M.pred_kind == kPredNoisy;
  const int64_t nvec = a.vec_ok ? n / 4 : 0;
  const int64_t stride = static_cast<int64_t>(nworkers) * blockDim.x;
  for (int64_t v = static_cast<int64_t>(worker) * blockDim.x + tid; v < nvec; v += stride) {
    const int4 cl = ldg_stream(reinterpret_cast<const int4*>(a.client) + v);
    const int4 in4 = ldg_stream(reinterpret_cast<const int4*>(a.in_tok) + v);
    const double2 a01 = ldg_stream(reinterpret_cast<const double2*>(a.arrival) + 2 * v);
    const double2 a23 = ldg_stream(reinterpret_cast<const double2*>(a.arrival) + 2 * v + 1);
    const uint32_t tg = ldg_stream(reinterpret_cast<const uint32_t*>(a.tag) + v);
    int4 to = make_int4(1, 1, 1, 1);
    if (oracle_like) to = ldg_stream(reinterpret_cast<const int4*>(a.true_out) + v);
    const int64_t r0 = 4 * v;
    int64_t ids[4] = {a.id_base + r0, a.id_base + r0 + 1, a.id_base + r0 + 2, a.id_base + r0 + 3};
    if (M.pred_kind == kPredNoisy && a.id) {
#pragma unroll
      for (int k = 0; k < 4; ++k) ids[k] = a.id[r0 + k];
    }
    const int cs[4] = {cl.x, cl.y, cl.z, cl.w};
    const int ins[4] = {in4.x, in4.y, in4.z, in4.w};
    const int tos[4] = {to.x, to.y, to.z, to.w};
    const double arr[4] = {a01.x, a01.y, a23.x, a23.y};
    Scored s[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double w = __ldg(a.weight + cs[k]);
      s[k] = score_request(M, a.pol, a.now, ins[k], (tg >> (8 * k)) & 0xffu, tos[k], ids[k], arr[k], w);
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
  // scalar tail (and unaligned inputs)
  for (int64_t r = 4 * nvec + static_cast<int64_t>(worker) * blockDim.x + tid; r < n; r += stride) {
    const int32_t c = a.client[r];
    const int64_t id = a.id ? a.id[r] : a.id_base + r;
    const Scored s = score_request(M, a.pol, a.now, a.in_tok[r], a.tag[r],
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
  if ((tid & 31) == 0) {
    if (fb) atomicAdd(&a.st->fallbacks, static_cast<unsigned long long>(fb));
    if (nt) atomicAdd(&a.st->near_ties, static_cast<unsigned long long>(nt));
  }
}

__global__ void __launch_bounds__(kStepThreads, 1) step_kernel(const StepArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  // Model tables -> shared memory (only the LUT part in use).
  ModelTables* M = reinterpret_cast<ModelTables*>(smem);
  {
    const int lut_words = (a.model_lut_entries);
    const int head_words = static_cast<int>(offsetof(ModelTables, lut) / 4);
    const uint32_t* src = reinterpret_cast<const uint32_t*>(a.model);
    uint32_t* dst = reinterpret_cast<uint32_t*>(smem);
    for (int i = threadIdx.x; i < head_words + lut_words; i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  unsigned char* rest = smem + a.model_smem_bytes;
  if (blockIdx.x == 0) {
    selection(a, *M, rest);
  } else {
    score_stream(a, *M, blockIdx.x - 1, gridDim.x - 1);
  }
}

__global__ void gather_ids_kernel(const int32_t* __restrict__ rows, int64_t n,
                                  const int64_t* __restrict__ id, int64_t id_base,
                                  int64_t* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = id ? id[rows[i]] : id_base + rows[i];
}

}  // namespace eqx
