// eqx_capi.cu -- the C ABI (include/eqx.h): context, model compiler, drain/step orchestration.
//
// Host code here only validates parameters (with the reference's messages), compiles the
// MoPE model + GPU profile into device tables, owns device buffers and launches kernels on
// the context stream.  There is no CPU execution path for the step: every per-request and
// per-pick decision is made by the kernels in eqx_kernels.cu.
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <utility>
#include <vector>

#include <cuda_runtime.h>
#include <map>
#include <mutex>
#include <sys/mman.h>

#include "../../include/eqx.h"
#include "eqx_device.cuh"
#include "eqx_kernels.h"

using namespace eqx;

namespace {

thread_local std::string g_create_error;

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t need) {
    if (need <= bytes && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    const size_t alloc = std::max<size_t>(need, 256);
    cudaError_t e = cudaMalloc(&p, alloc);
    if (e == cudaSuccess) bytes = alloc;
    return e;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  // every buffer of a context is freed with it (eqx_ctx_destroy deletes the context)
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
};

}  // namespace

struct eqx_ctx {
  int device = 0;
  int sm_count = 148;
  size_t smem_optin = 227 * 1024;
  cudaStream_t stream = nullptr;
  std::string err;

  Policy pol{};
  int32_t counter_lift = 1;
  bool policy_set = false;
  eqx_perf perf{64, 0.5 * 1024.0 * 1024.0, 60.0 * 1024.0 * 1024.0 * 1024.0};
  ModelTables model{};
  bool model_set = false, profile_set = false, model_dirty = true;
  int32_t lut_entries = 0;
  DevBuf d_model;

  int32_t C = 0;
  DevBuf d_ufc, d_rfc, d_counter, d_weight, d_order, d_running, d_backlogged;
  DevBuf d_by_order;               // client of client_id rank k (replay reports)
  DevBuf d_head, d_count, d_first, d_qlen_before, d_seg_off;

  int64_t n = 0;
  const int32_t* q_client = nullptr;
  const double* q_arrival = nullptr;
  const int32_t* q_in = nullptr;
  const int32_t* q_true = nullptr;
  const uint8_t* q_tag = nullptr;
  const int64_t* q_id = nullptr;
  int64_t id_base = 0;
  DevBuf own_tag;  // zero tags for device batches without a tag column
  // Host batches are staged through kStages device buffer sets on a copy stream, so the H2D
  // of the next batches (eqx_stage_async) overlaps the current step: with three sets a caller
  // can keep two batches in flight, so the copy engine never idles while the host collects a
  // step.  `free_` is recorded on the main stream after the last launch that reads a set.
  static constexpr int kStages = 3;
  struct Stage {
    DevBuf client, arrival, in, tru, tag, id, c16, i16, apk;  // apk: packed arrivals
    const void* key[6] = {};
    int32_t narrow = 0;
    int64_t n = -1;
    uint64_t seq = 0;  // staging order: a drain consumes the oldest matching staged batch
    bool valid = false;
    cudaEvent_t ready = nullptr, free_ = nullptr, copied = nullptr;
  } stg[kStages];
  int bound_stage = -1;
  uint64_t stage_seq = 0;
  cudaStream_t copy_stream = nullptr;
  cudaStream_t unpack_stream = nullptr;  // widen / unpack kernels of staged batches (the copy stream moves on)
  DevBuf d_perm, d_hist, d_tbase, d_ctot, d_tsorted, d_tfirst;
  bool sort_drain = false;         // small rosters: drain_sort + drain_scan + drain_scatter
  size_t sort_smem = 0;
  bool queue_ready = false;

  DevBuf d_pred, d_bucket, d_ufc_out, d_rfc_out;
  DevBuf d_ev_row, d_ev_kind, d_ev_client, d_ev_pred, d_ev_ufc, d_ev_rfc, d_ev_vtc, d_ev_wait, d_ev_id;
  int64_t ev_cap = 0;
  DevBuf d_state, d_cw;
  DevBuf snap_ufc, snap_rfc, snap_counter, snap_running, snap_backlogged, snap_state;
  bool snap_valid = false;
  DevState* h_state = nullptr;  // pinned
  unsigned long long last_fallbacks = 0, last_near_ties = 0;
  bool step_pending = false;
  bool stepped = false;
  // drain plan (set by drain_prepare, consumed by drain_enqueue)
  int64_t tile_rows = 2048;
  int32_t n_tiles = 1;
  int64_t hist_L = 0;
  size_t hist_smem = 0, rank_smem = 0;
  bool staged = true;
  cudaStream_t stream2 = nullptr;  // side stream for whole-queue scoring
  cudaStream_t stream3 = nullptr;  // the selection's code warm-up (graph step)
  cudaEvent_t ev_warm = nullptr, ev_warm_done = nullptr;
  DevBuf d_warm;                   // the warm-up selection's own small problem (scratch)
  int32_t warm_C = -1;             // clients of the problem d_warm holds
  SelectArgs warm_se{};            // its launch arguments (prepared before a graph capture)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_k[6] = {};        // timing: score start/end, select start/end, drain start/end
  DevBuf d_done;                   // last-CTA counters [0..1] of the drain kernels; bytes 32..47: score_counts
  DevBuf d_win;                    // [C][W] head windows
  DevBuf d_wcnt;                   // per-(tile, warp, client) counts of the drain walk
  DevBuf d_direct;                 // direct predict/map table (see ScoreArgs::direct)
  int32_t direct_n = 0;
  // cached CUDA graphs of drain + step, least recently used evicted (a resident queue, or
  // one per staging buffer set)
  static constexpr int kGraphs = kStages + 1;
  cudaGraphExec_t graphs[kGraphs] = {};
  std::vector<unsigned char> graph_keys[kGraphs];
  uint64_t graph_used[kGraphs] = {};
  uint64_t graph_clock = 0;
  bool owns_stream = true;         // false after eqx_ctx_set_stream (caller's stream)
  // pinned bounce buffer for result reads: async D2H of every column, one sync, host memcpy
  void* h_scratch = nullptr;       // mapped pinned memory
  void* h_scratch_dev = nullptr;   // its device alias
  size_t h_scratch_bytes = 0;
  DevState* h_state_dev = nullptr; // device alias of the mapped h_state
  unsigned char* h_ledger = nullptr;      // mapped host copy of a step's ledger (eqx_step_ledger)
  unsigned char* h_ledger_dev = nullptr;  // its device alias
  size_t h_ledger_cap = 0;
  uint64_t ledger_epoch = 0;              // bumped by every call that changes the device ledger
  uint64_t ledger_pub_epoch = ~0ull;      // the epoch whose ledger h_ledger holds
  // launch-attribute caches (cudaFuncSetAttribute / occupancy queries cost host time per step)
  int smem_attr[13] = {-1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1};  // drain_hist, drain_rank, select kernels (select_fn)
  size_t occ_smem = SIZE_MAX;
  int occ_per_sm = 1;
  // client-sharded step (selection context): gathered windows and their ids
  DevBuf d_first64, d_gid;
  DevBuf d_service;                // ClientState::accumulated_service
  DevBuf d_tk, d_tkh;              // top-K selection: items beyond shared memory, head tuples
  // engine timing (PerfParams, gpu_model.hpp:14-28) for replays
  double prefill_linear_ms = 0.05, prefill_quad_ms = 1e-6, decode_base_ms = 5.0, decode_per_ctx_ms = 0.002,
         refresh_ms = 15.0;
  // live queue (eqx_append): two column stores with frozen prediction records, swapped per append
  struct Live {
    DevBuf client, arrival, in, tag, tru, id, pred, bucket, preds, rfc;
  } live[2];
  int live_cur = -1;
  bool live_mode = false;
  int64_t popped = 0;  // requests popped (admitted / rejected) since the queue was (re)built
  Frozen frozen{};
  DevBuf d_live_off, d_nlive;
  DevBuf d_fb;                     // staged completion batch / token counts
  int32_t shard_W = 0;             // > 0: the last step was a sharded selection
};

namespace {

eqx_status fail(eqx_ctx* ctx, eqx_status st, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return st;
}

cudaError_t ensure_scratch(eqx_ctx* ctx, size_t bytes) {
  if (bytes <= ctx->h_scratch_bytes) return cudaSuccess;
  if (ctx->h_scratch) cudaFreeHost(ctx->h_scratch);
  ctx->h_scratch = nullptr;
  ctx->h_scratch_bytes = 0;
  const size_t want = std::max<size_t>(bytes, 1 << 16);
  cudaError_t e = cudaHostAlloc(&ctx->h_scratch, want, cudaHostAllocMapped);
  if (e == cudaSuccess) e = cudaHostGetDevicePointer(&ctx->h_scratch_dev, ctx->h_scratch, 0);
  if (e == cudaSuccess) ctx->h_scratch_bytes = want;
  return e;
}

// Device columns -> caller arrays through the pinned scratch: the copies are queued back to
// back on the stream, the host waits once, then copies out (pageable D2H copies would each
// stage and synchronise on their own).
struct Col {
  void* dst;
  const void* src;
  size_t bytes;
};

// The selection kernel (one variant: rounds of block-radix top-K, eqx_topk.cuh).
// the selection kernel of a plan: the huge-roster instantiation when the head tuples live in
// global scratch
const void* select_fn(bool huge) {
  return huge ? reinterpret_cast<const void*>(select_topk_kernel<true>)
              : reinterpret_cast<const void*>(select_topk_kernel<false>);
}

// Programmatic dependent launch: the kernel may be scheduled while its predecessor on the
// stream is still finishing; it executes griddepcontrol.wait before touching the predecessor's
// results (pdl_wait in eqx_kernels.cu), so only launch latency and the prologue overlap.
template <class... KArgs, class... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// DevState -> the mapped host copy by a kernel (no copy-engine dependency; capturable).
// pdl: launched programmatically after the kernel that last wrote the state (it waits).
cudaError_t state_to_host(eqx_ctx* ctx, cudaStream_t s, bool pdl = false) {
  PackCols pc;
  std::memset(&pc, 0, sizeof(pc));
  pc.src[0] = ctx->d_state.p;
  pc.dst[0] = ctx->h_state_dev;
  pc.bytes[0] = sizeof(DevState);
  pc.n = 1;
  if (pdl) return launch_pdl(pack_cols_kernel, dim3(1), dim3(64), 0, s, pc);
  pack_cols_kernel<<<1, 64, 0, s>>>(pc);
  return cudaGetLastError();
}

cudaError_t set_smem_attr(eqx_ctx* ctx, int which, const void* fn, size_t bytes) {
  if (ctx->smem_attr[which] == static_cast<int>(bytes)) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
  if (e == cudaSuccess) ctx->smem_attr[which] = static_cast<int>(bytes);
  return e;
}

#define CUDA_TRY(ctx, expr)                                                            \
  do {                                                                                 \
    cudaError_t _e = (expr);                                                           \
    if (_e != cudaSuccess)                                                             \
      return fail((ctx), EQX_ERR_CUDA, std::string("CUDA error: ") + cudaGetErrorString(_e) + \
                                           " at " #expr);                              \
  } while (0)

namespace {
eqx_status read_cols(eqx_ctx* ctx, const Col* cols, int n) {
  size_t total = 0;
  for (int i = 0; i < n; ++i)
    if (cols[i].dst) total += (cols[i].bytes + 15) & ~size_t(15);
  CUDA_TRY(ctx, ensure_scratch(ctx, total));
  cudaStream_t s = ctx->stream;
  size_t off = 0;
  PackCols pc;
  std::memset(&pc, 0, sizeof(pc));
  for (int i = 0; i < n; ++i) {
    if (!cols[i].dst || !cols[i].bytes) continue;
    pc.src[pc.n] = cols[i].src;
    pc.dst[pc.n] = static_cast<char*>(ctx->h_scratch_dev) + off;
    pc.bytes[pc.n] = static_cast<int64_t>(cols[i].bytes);
    ++pc.n;
    off += (cols[i].bytes + 15) & ~size_t(15);
  }
  if (pc.n > 0) {
    pack_cols_kernel<<<dim3(std::max<unsigned>(1, std::min<unsigned>(64, static_cast<unsigned>(total / 4096 + 1))),
                            static_cast<unsigned>(pc.n)),
                       256, 0, s>>>(pc);
    CUDA_TRY(ctx, cudaGetLastError());
  }
  CUDA_TRY(ctx, cudaStreamSynchronize(s));
  off = 0;
  for (int i = 0; i < n; ++i) {
    if (!cols[i].dst || !cols[i].bytes) continue;
    std::memcpy(cols[i].dst, static_cast<char*>(ctx->h_scratch) + off, cols[i].bytes);
    off += (cols[i].bytes + 15) & ~size_t(15);
  }
  return EQX_OK;
}
}  // namespace

// ---- reference predictor semantics, evaluated once per LUT cell (host "model compiler") ----
// RouterModel::length_bucket (predictor.cpp:29-34)
int length_bucket(const eqx_mope& m, int in) {
  for (int i = 0; i < m.n_thresholds; ++i)
    if (in <= m.thresholds[i]) return i;
  return m.num_buckets - 1;
}
// route (predictor.cpp:36-60); row < 0 => tag empty/unseen => length fallback
int route(const eqx_mope& m, int in, int row, bool* fallback) {
  const int len_bucket = length_bucket(m, in);
  if (row < 0) {
    *fallback = true;
    return len_bucket;
  }
  *fallback = false;
  const double* aff = m.rows + static_cast<size_t>(row) * m.num_buckets;
  int bucket = 0;
  double best = -1.0;
  for (int b = 0; b < m.num_buckets; ++b) {
    const double length_score = b == len_bucket ? 1.0 : 0.0;
    const double score = m.mix_weight * length_score + (1.0 - m.mix_weight) * aff[b];
    if (score > best) {
      best = score;
      bucket = b;
    }
  }
  return bucket;
}
// ExpertModel::predict (predictor.cpp:62-71)
int expert_predict(const eqx_mope& m, int e, int in) {
  const int32_t* up = m.bin_upper + static_cast<size_t>(e) * m.n_bins;
  const int32_t* val = m.bin_value + static_cast<size_t>(e) * m.n_bins;
  int idx = m.n_bins - 1;
  for (int i = 0; i < m.n_bins; ++i) {
    if (in <= up[i]) {
      idx = i;
      break;
    }
  }
  return std::clamp(val[idx], m.out_min[e], m.out_max[e]);
}

uint64_t fnv1a(const char* s) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (; *s; ++s) {
    h ^= static_cast<unsigned char>(*s);
    h *= 0x100000001b3ULL;
  }
  return h;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace

extern "C" {

int32_t eqx_abi_version(void) { return EQX_ABI_VERSION; }

namespace {
std::mutex g_host_mu;
std::map<void*, std::pair<void*, size_t>> g_host_maps;  // aligned pointer -> (mapping, length)
constexpr size_t kHuge = size_t(2) << 20;
}  // namespace

void* eqx_host_alloc(int64_t bytes) {
  if (bytes <= 0) return nullptr;
  const size_t size = (size_t(bytes) + kHuge - 1) / kHuge * kHuge;
  const size_t len = size + kHuge;
  void* m = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (m == MAP_FAILED) return nullptr;
  char* al = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(m) + kHuge - 1) & ~(uintptr_t(kHuge) - 1));
  madvise(al, size, MADV_HUGEPAGE);  // advisory: a kernel without THP still gets a working arena
  memset(al, 0, size);               // fault the pages in (huge where THP allows) before pinning
  if (cudaHostRegister(al, size, cudaHostRegisterDefault) != cudaSuccess) {
    cudaGetLastError();
    munmap(m, len);
    return nullptr;
  }
  std::lock_guard<std::mutex> g(g_host_mu);
  g_host_maps[al] = {m, len};
  return al;
}

eqx_status eqx_host_free(void* p) {
  if (!p) return EQX_OK;
  std::pair<void*, size_t> mp;
  {
    std::lock_guard<std::mutex> g(g_host_mu);
    auto it = g_host_maps.find(p);
    if (it == g_host_maps.end()) return EQX_ERR_CONFIG;
    mp = it->second;
    g_host_maps.erase(it);
  }
  cudaHostUnregister(p);
  munmap(mp.first, mp.second);
  return EQX_OK;
}

const char* eqx_last_error(const eqx_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_create_error.c_str();
}

eqx_status eqx_ctx_create(int32_t device, eqx_ctx** out) {
  if (!out) {
    g_create_error = "eqx_ctx_create: out is NULL";
    return EQX_ERR_ARG;
  }
  *out = nullptr;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    g_create_error = std::string("no CUDA device available: ") + cudaGetErrorString(e);
    return EQX_ERR_CUDA;
  }
  if (device < 0 || device >= ndev) {
    g_create_error = "device index out of range";
    return EQX_ERR_ARG;
  }
  cudaDeviceProp prop{};
  cudaSetDevice(device);
  e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) {
    g_create_error = cudaGetErrorString(e);
    return EQX_ERR_CUDA;
  }
  if (prop.major != 10) {
    g_create_error = "libeqx_b200 is built for sm_100a (B200); device " + std::string(prop.name) +
                     " is sm_" + std::to_string(prop.major) + std::to_string(prop.minor);
    return EQX_ERR_CUDA;
  }
  eqx_ctx* ctx = new eqx_ctx();
  ctx->device = device;
  ctx->sm_count = prop.multiProcessorCount;
  ctx->smem_optin = prop.sharedMemPerBlockOptin;
  e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->stream2, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->unpack_stream, cudaStreamNonBlocking);
  for (int b = 0; b < eqx_ctx::kStages && e == cudaSuccess; ++b) {
    e = cudaEventCreateWithFlags(&ctx->stg[b].ready, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->stg[b].free_, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->stg[b].copied, cudaEventDisableTiming);
  }
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming);
  for (int i = 0; i < 6 && e == cudaSuccess; ++i) e = cudaEventCreate(&ctx->ev_k[i]);
  if (e == cudaSuccess) e = ctx->d_done.ensure(64);
  if (e == cudaSuccess) e = cudaMemset(ctx->d_done.p, 0, 64);
  if (e == cudaSuccess) e = ctx->d_state.ensure(sizeof(DevState));
  if (e == cudaSuccess) e = cudaMemset(ctx->d_state.p, 0, sizeof(DevState));
  if (e == cudaSuccess) e = cudaHostAlloc(&ctx->h_state, sizeof(DevState), cudaHostAllocMapped);
  if (e == cudaSuccess) e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->h_state_dev), ctx->h_state, 0);
  if (e == cudaSuccess) e = ctx->d_model.ensure(sizeof(ModelTables));
  if (e != cudaSuccess) {
    g_create_error = cudaGetErrorString(e);
    eqx_ctx_destroy(ctx);
    return EQX_ERR_CUDA;
  }
  ctx->pol.kind = kEquinox;
  ctx->pol.alpha = 0.7;
  ctx->pol.beta = 1.0 - 0.7;
  ctx->pol.delta = 0.1;
  ctx->pol.ow = 4.0;
  ctx->pol.max_batch = ctx->perf.max_batch;
  ctx->pol.m = ctx->perf.mem_per_token_bytes;
  ctx->pol.M = ctx->perf.mem_capacity_bytes;
  *out = ctx;
  return EQX_OK;
}

void eqx_ctx_destroy(eqx_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  DevBuf* bufs[] = {&ctx->d_model, &ctx->d_ufc, &ctx->d_rfc, &ctx->d_counter, &ctx->d_weight,
                    &ctx->d_order, &ctx->d_running, &ctx->d_backlogged, &ctx->d_head,
                    &ctx->d_count, &ctx->d_first, &ctx->d_qlen_before, &ctx->d_seg_off,
                    &ctx->own_tag, &ctx->d_perm, &ctx->d_hist, &ctx->d_tbase, &ctx->d_ctot, &ctx->d_tsorted, &ctx->d_pred,
                    &ctx->d_bucket, &ctx->d_ufc_out, &ctx->d_rfc_out, &ctx->d_ev_row,
                    &ctx->d_ev_kind, &ctx->d_ev_client, &ctx->d_ev_pred, &ctx->d_ev_ufc,
                    &ctx->d_ev_rfc, &ctx->d_ev_vtc, &ctx->d_ev_wait, &ctx->d_ev_id,
                    &ctx->d_state, &ctx->d_cw, &ctx->snap_ufc, &ctx->snap_rfc,
                    &ctx->snap_counter, &ctx->snap_running, &ctx->snap_backlogged, &ctx->snap_state};
  for (DevBuf* b : bufs) b->release();
  if (ctx->h_state) cudaFreeHost(ctx->h_state);
  if (ctx->h_ledger) cudaFreeHost(ctx->h_ledger);
  if (ctx->h_scratch) cudaFreeHost(ctx->h_scratch);
  if (ctx->stream2) cudaStreamSynchronize(ctx->stream2);
  ctx->d_done.release();
  ctx->d_win.release();
  ctx->d_wcnt.release();
  ctx->d_direct.release();
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  for (auto& ev : ctx->ev_k)
    if (ev) cudaEventDestroy(ev);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  if (ctx->stream2) cudaStreamDestroy(ctx->stream2);
  if (ctx->stream3) {
    cudaStreamSynchronize(ctx->stream3);
    cudaStreamDestroy(ctx->stream3);
  }
  if (ctx->ev_warm) cudaEventDestroy(ctx->ev_warm);
  if (ctx->ev_warm_done) cudaEventDestroy(ctx->ev_warm_done);
  if (ctx->copy_stream) {
    cudaStreamSynchronize(ctx->copy_stream);
    cudaStreamDestroy(ctx->copy_stream);
  }
  if (ctx->unpack_stream) {
    cudaStreamSynchronize(ctx->unpack_stream);
    cudaStreamDestroy(ctx->unpack_stream);
  }
  for (auto& st : ctx->stg) {
    DevBuf* sb[] = {&st.client, &st.arrival, &st.in, &st.tru, &st.tag, &st.id};
    for (DevBuf* b : sb) b->release();
    if (st.ready) cudaEventDestroy(st.ready);
    if (st.free_) cudaEventDestroy(st.free_);
    if (st.copied) cudaEventDestroy(st.copied);
  }
  for (auto& g : ctx->graphs)
    if (g) cudaGraphExecDestroy(g);
  ctx->d_first64.release();
  ctx->d_gid.release();
  ctx->d_service.release();
  for (auto& L : ctx->live) {
    DevBuf* lb[] = {&L.client, &L.arrival, &L.in, &L.tag, &L.tru, &L.id, &L.pred, &L.bucket, &L.preds, &L.rfc};
    for (DevBuf* b : lb) b->release();
  }
  ctx->d_live_off.release();
  ctx->d_nlive.release();
  ctx->d_fb.release();
  if (ctx->stream && ctx->owns_stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

void* eqx_ctx_stream(eqx_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }
void* eqx_ctx_copy_stream(eqx_ctx* ctx) { return ctx ? static_cast<void*>(ctx->copy_stream) : nullptr; }

eqx_status eqx_ctx_set_stream(eqx_ctx* ctx, void* stream) {
  if (!ctx) return fail(ctx, EQX_ERR_ARG, "eqx_ctx_set_stream: NULL context");  // stream 0 = legacy default
  cudaSetDevice(ctx->device);
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  if (ctx->owns_stream) CUDA_TRY(ctx, cudaStreamDestroy(ctx->stream));
  ctx->stream = static_cast<cudaStream_t>(stream);
  ctx->owns_stream = false;
  for (int i = 0; i < eqx_ctx::kGraphs; ++i) {  // captured on the old stream's plan
    if (ctx->graphs[i]) cudaGraphExecDestroy(ctx->graphs[i]);
    ctx->graphs[i] = nullptr;
    ctx->graph_keys[i].clear();
  }
  return EQX_OK;
}

// EquinoxParams::validate (scheduler.cpp:11-17)
eqx_status eqx_set_policy(eqx_ctx* ctx, const eqx_policy* p) {
  if (!ctx || !p) return fail(ctx, EQX_ERR_ARG, "eqx_set_policy: NULL argument");
  if (p->kind < EQX_FCFS || p->kind > EQX_EQUINOX) return fail(ctx, EQX_ERR_CONFIG, "unknown policy kind");
  if (p->alpha < 0.0 || p->alpha > 1.0) return fail(ctx, EQX_ERR_CONFIG, "alpha must lie in [0, 1]");
  if (p->delta < 0.0) return fail(ctx, EQX_ERR_CONFIG, "delta must be >= 0");
  if (p->output_weight <= 0.0) return fail(ctx, EQX_ERR_CONFIG, "output_weight must be > 0");
  if (p->norm_mode != EQX_NORM_MAX_OVER_CLIENTS && p->norm_mode != EQX_NORM_NONE)
    return fail(ctx, EQX_ERR_CONFIG, "unknown norm_mode");
  ctx->pol.kind = p->kind;
  ctx->pol.alpha = p->alpha;
  ctx->pol.beta = 1.0 - p->alpha;  // EquinoxParams::beta() (scheduler.hpp:24)
  ctx->pol.delta = p->delta;
  ctx->pol.ow = p->output_weight;
  ctx->pol.norm_mode = p->norm_mode;
  ctx->pol.vtc_use_prediction = p->vtc_use_prediction ? 1 : 0;
  ctx->pol.backfill = p->backfill ? 1 : 0;
  ctx->counter_lift = p->counter_lift ? 1 : 0;
  ctx->policy_set = true;
  return EQX_OK;
}

// PerfParams::validate (gpu_model.cpp:9-24) for the admission fields
eqx_status eqx_set_perf(eqx_ctx* ctx, const eqx_perf* p) {
  if (!ctx || !p) return fail(ctx, EQX_ERR_ARG, "eqx_set_perf: NULL argument");
  if (p->mem_per_token_bytes <= 0.0)
    return fail(ctx, EQX_ERR_CONFIG, "perf parameter 'mem_per_token_bytes' must be > 0");
  if (p->mem_capacity_bytes <= 0.0)
    return fail(ctx, EQX_ERR_CONFIG, "perf parameter 'mem_capacity_bytes' must be > 0");
  if (p->max_batch <= 0) return fail(ctx, EQX_ERR_CONFIG, "perf parameter 'max_batch' must be > 0");
  ctx->perf = *p;
  ctx->pol.max_batch = p->max_batch;
  ctx->pol.m = p->mem_per_token_bytes;
  ctx->pol.M = p->mem_capacity_bytes;
  return EQX_OK;
}

eqx_status eqx_set_profile(eqx_ctx* ctx, const eqx_profile* p) {
  if (!ctx || !p) return fail(ctx, EQX_ERR_ARG, "eqx_set_profile: NULL argument");
  if (p->n <= 0) return fail(ctx, EQX_ERR_CONFIG, "engine needs a non-empty GPU profile");
  if (p->n > kMaxProfile)
    return fail(ctx, EQX_ERR_CONFIG, "GPU profile has more than " + std::to_string(kMaxProfile) + " buckets");
  ModelTables& M = ctx->model;
  M.n_prof = p->n;
  for (int i = 0; i < p->n; ++i) {
    M.prof_upper[i] = p->bucket_upper[i];
    M.prof_lat[i] = p->latency_ms[i];
    M.prof_util[i] = p->gpu_util[i];
    M.prof_tps[i] = p->tps[i];
    M.prof_pred_s[i] = p->latency_ms[i] / 1000.0;  // scheduler.cpp:23
  }
  ctx->profile_set = true;
  ctx->model_dirty = true;
  return EQX_OK;
}

eqx_status eqx_set_predictor(eqx_ctx* ctx, const eqx_predictor* p) {
  if (!ctx || !p) return fail(ctx, EQX_ERR_ARG, "eqx_set_predictor: NULL argument");
  ModelTables& M = ctx->model;
  M.pred_kind = p->kind;
  if (p->kind == EQX_PRED_ORACLE) {
    M.n_cuts = 0;
    M.n_tag_states = 1;
    ctx->lut_entries = 1;
    M.lut[0] = 1;
  } else if (p->kind == EQX_PRED_NOISY_ORACLE) {
    if (p->noisy_l1 < 0.0) return fail(ctx, EQX_ERR_CONFIG, "noisy oracle target_l1 must be >= 0");
    M.noisy_l1 = p->noisy_l1;
    M.noisy_key = mix_keys(p->noisy_seed, fnv1a("noisy_oracle"));
    M.n_cuts = 0;
    M.n_tag_states = 1;
    ctx->lut_entries = 1;
    M.lut[0] = 1;
  } else if (p->kind == EQX_PRED_MOPE || p->kind == EQX_PRED_SINGLE_PROXY) {
    const eqx_mope& m = p->mope;
    if (m.n_experts <= 0) return fail(ctx, EQX_ERR_CONFIG, "MoPE predictor constructed without trained experts");
    if (m.n_bins <= 0) return fail(ctx, EQX_ERR_PARSE, "malformed MoPE model: expert without bins");
    if (p->kind == EQX_PRED_MOPE) {
      if (m.num_buckets <= 0 || m.num_buckets > m.n_experts)
        return fail(ctx, EQX_ERR_PARSE, "malformed MoPE model: num_buckets does not match the experts");
      if (m.n_thresholds < 0 || m.n_thresholds > 64) return fail(ctx, EQX_ERR_PARSE, "malformed MoPE model: thresholds");
      for (int t = 0; t < m.n_tags; ++t)
        if (m.tag_row[t] >= m.n_rows) return fail(ctx, EQX_ERR_PARSE, "malformed MoPE model: tag row out of range");
      if (m.n_tags + 1 > kMaxTagStates) return fail(ctx, EQX_ERR_CONFIG, "more than 255 distinct category tags");
    }
    // Merged cut points: every threshold / bin bound any comparison `in <= x` can test.
    std::vector<int> cuts;
    if (p->kind == EQX_PRED_MOPE) cuts.assign(m.thresholds, m.thresholds + m.n_thresholds);
    const int ne = p->kind == EQX_PRED_MOPE ? m.n_experts : 1;
    for (int e = 0; e < ne; ++e)
      for (int i = 0; i < m.n_bins; ++i) cuts.push_back(m.bin_upper[e * m.n_bins + i]);
    std::sort(cuts.begin(), cuts.end());
    cuts.erase(std::unique(cuts.begin(), cuts.end()), cuts.end());
    if (static_cast<int>(cuts.size()) > kMaxCuts) return fail(ctx, EQX_ERR_CONFIG, "MoPE model has too many distinct cut points");
    const int nt = p->kind == EQX_PRED_MOPE ? m.n_tags + 1 : 1;
    const int ni = static_cast<int>(cuts.size()) + 1;
    if (ni * nt > kMaxLut) return fail(ctx, EQX_ERR_CONFIG, "MoPE lookup table too large");
    M.n_cuts = static_cast<int>(cuts.size());
    M.n_tag_states = nt;
    for (int i = 0; i < M.n_cuts; ++i) M.cuts[i] = cuts[i];
    // Interval k = {in : cuts[k-1] < in <= cuts[k]}: every `in <= x` test is constant on it,
    // so evaluating the reference functions at one representative is exact for all members.
    for (int k = 0; k < ni; ++k) {
      int rep;
      if (k < M.n_cuts) rep = cuts[k];
      else rep = (M.n_cuts == 0) ? 1 : (cuts.back() == INT_MAX ? INT_MAX : cuts.back() + 1);
      for (int t = 0; t < nt; ++t) {
        int pred;
        bool fb = false;
        if (p->kind == EQX_PRED_MOPE) {
          const int row = t == 0 ? -1 : m.tag_row[t - 1];
          const int b = route(m, rep, row, &fb);
          pred = expert_predict(m, b, rep);
        } else {
          pred = expert_predict(m, 0, rep);
        }
        pred = std::max(1, pred);  // engine.cpp:179
        M.lut[k * nt + t] = fb ? -pred : pred;
      }
    }
    ctx->lut_entries = ni * nt;
  } else {
    return fail(ctx, EQX_ERR_CONFIG, "unknown predictor kind");
  }
  ctx->model_set = true;
  ctx->model_dirty = true;
  return EQX_OK;
}

eqx_status eqx_set_clients(eqx_ctx* ctx, int32_t n, const char* names, const double* weight,
                           const double* ufc, const double* rfc, const double* counter,
                           const int32_t* running) {
  if (ctx) ++ctx->ledger_epoch;  // the published step ledger (eqx_step_ledger) is stale
  if (!ctx || n < 0 || (n > 0 && (!names || !weight))) return fail(ctx, EQX_ERR_ARG, "eqx_set_clients: bad arguments");
  cudaSetDevice(ctx->device);
  std::vector<std::string> ids;
  const char* q = names;
  for (int i = 0; i < n; ++i) {
    ids.emplace_back(q);
    q += ids.back().size() + 1;
    if (!(weight[i] > 0.0)) return fail(ctx, EQX_ERR_CONFIG, "client '" + ids.back() + "' has non-positive weight");
  }
  // lexicographic rank by std::string operator< (bytewise), index breaks exact duplicates the
  // way select_next keeps the earlier candidate (scheduler.cpp:139-153)
  std::vector<int> idx(n);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return ids[a] < ids[b]; });
  std::vector<uint32_t> order(n);
  for (int r = 0; r < n; ++r) order[idx[r]] = static_cast<uint32_t>(r);
  std::vector<double> zeros(n, 0.0);
  std::vector<int32_t> izeros(n, 0);
  const size_t d8 = 8ull * std::max(n, 1), d4 = 4ull * std::max(n, 1);
  CUDA_TRY(ctx, ctx->d_ufc.ensure(d8));
  CUDA_TRY(ctx, ctx->d_rfc.ensure(d8));
  CUDA_TRY(ctx, ctx->d_counter.ensure(d8));
  CUDA_TRY(ctx, ctx->d_weight.ensure(d8));
  CUDA_TRY(ctx, ctx->d_order.ensure(d4));
  CUDA_TRY(ctx, ctx->d_by_order.ensure(d4));
  CUDA_TRY(ctx, ctx->d_running.ensure(d4));
  CUDA_TRY(ctx, ctx->d_backlogged.ensure(d4));
  CUDA_TRY(ctx, ctx->d_head.ensure(d4));
  CUDA_TRY(ctx, ctx->d_count.ensure(d4));
  CUDA_TRY(ctx, ctx->d_first.ensure(d4));
  CUDA_TRY(ctx, ctx->d_qlen_before.ensure(d4));
  CUDA_TRY(ctx, ctx->d_seg_off.ensure(4ull * (n + 1)));
  CUDA_TRY(ctx, ctx->d_service.ensure(d8));
  cudaStream_t s = ctx->stream;
  CUDA_TRY(ctx, cudaMemsetAsync(ctx->d_service.p, 0, d8, s));
  if (n > 0) {
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->d_ufc.p, ufc ? ufc : zeros.data(), 8ull * n, cudaMemcpyHostToDevice, s));
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->d_rfc.p, rfc ? rfc : zeros.data(), 8ull * n, cudaMemcpyHostToDevice, s));
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->d_counter.p, counter ? counter : zeros.data(), 8ull * n, cudaMemcpyHostToDevice, s));
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->d_weight.p, weight, 8ull * n, cudaMemcpyHostToDevice, s));
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->d_order.p, order.data(), 4ull * n, cudaMemcpyHostToDevice, s));
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->d_by_order.p, idx.data(), 4ull * n, cudaMemcpyHostToDevice, s));
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->d_running.p, running ? running : izeros.data(), 4ull * n, cudaMemcpyHostToDevice, s));
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->d_backlogged.p, 0, d4, s));
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->d_head.p, 0, d4, s));
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->d_count.p, 0, d4, s));
  }
  CUDA_TRY(ctx, cudaStreamSynchronize(s));  // host vectors above are about to go away
  ctx->C = n;
  ctx->queue_ready = false;
  ctx->stepped = false;
  return EQX_OK;
}

eqx_status eqx_get_clients(eqx_ctx* ctx, int32_t n, double* ufc, double* rfc, double* counter,
                           int32_t* backlogged, int32_t* running) {
  if (!ctx || n != ctx->C) return fail(ctx, EQX_ERR_ARG, "eqx_get_clients: roster size mismatch");
  cudaSetDevice(ctx->device);
  const size_t d8 = 8ull * n, d4 = 4ull * n;
  const Col cols[] = {{ufc, ctx->d_ufc.p, d8}, {rfc, ctx->d_rfc.p, d8}, {counter, ctx->d_counter.p, d8},
                      {backlogged, ctx->d_backlogged.p, d4}, {running, ctx->d_running.p, d4}};
  return read_cols(ctx, cols, n > 0 ? 5 : 0);
}

eqx_status eqx_step_ledger(eqx_ctx* ctx, int32_t n, double* ufc, double* rfc, double* counter,
                           int32_t* backlogged, int32_t* running) {
  if (!ctx || n != ctx->C) return fail(ctx, EQX_ERR_ARG, "eqx_step_ledger: roster size mismatch");
  if (ctx->step_pending || !ctx->h_ledger || ctx->ledger_pub_epoch != ctx->ledger_epoch)
    return fail(ctx, EQX_ERR_CONFIG, "eqx_step_ledger: no collected step ledger (use eqx_get_clients)");
  const double* hd = reinterpret_cast<const double*>(ctx->h_ledger);
  const int32_t* hi = reinterpret_cast<const int32_t*>(hd + 3 * static_cast<int64_t>(n));
  if (ufc) std::memcpy(ufc, hd, 8ull * n);
  if (rfc) std::memcpy(rfc, hd + n, 8ull * n);
  if (counter) std::memcpy(counter, hd + 2 * static_cast<int64_t>(n), 8ull * n);
  if (backlogged) std::memcpy(backlogged, hi, 4ull * n);
  if (running) std::memcpy(running, hi + n, 4ull * n);
  return EQX_OK;
}

eqx_status eqx_ledger_checkpoint(eqx_ctx* ctx) {
  if (!ctx) return fail(ctx, EQX_ERR_ARG, "eqx_ledger_checkpoint: NULL context");
  cudaSetDevice(ctx->device);
  cudaStream_t s = ctx->stream;
  const size_t d8 = 8ull * std::max(ctx->C, 1), d4 = 4ull * std::max(ctx->C, 1);
  CUDA_TRY(ctx, ctx->snap_ufc.ensure(d8));
  CUDA_TRY(ctx, ctx->snap_rfc.ensure(d8));
  CUDA_TRY(ctx, ctx->snap_counter.ensure(d8));
  CUDA_TRY(ctx, ctx->snap_running.ensure(d4));
  CUDA_TRY(ctx, ctx->snap_backlogged.ensure(d4));
  CUDA_TRY(ctx, ctx->snap_state.ensure(sizeof(DevState)));
  if (ctx->C > 0) {
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->snap_ufc.p, ctx->d_ufc.p, 8ull * ctx->C, cudaMemcpyDeviceToDevice, s));
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->snap_rfc.p, ctx->d_rfc.p, 8ull * ctx->C, cudaMemcpyDeviceToDevice, s));
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->snap_counter.p, ctx->d_counter.p, 8ull * ctx->C, cudaMemcpyDeviceToDevice, s));
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->snap_running.p, ctx->d_running.p, 4ull * ctx->C, cudaMemcpyDeviceToDevice, s));
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->snap_backlogged.p, ctx->d_backlogged.p, 4ull * ctx->C, cudaMemcpyDeviceToDevice, s));
  }
  CUDA_TRY(ctx, cudaMemcpyAsync(ctx->snap_state.p, ctx->d_state.p, offsetof(DevState, n_events), cudaMemcpyDeviceToDevice, s));
  CUDA_TRY(ctx, cudaStreamSynchronize(s));
  ctx->snap_valid = true;
  return EQX_OK;
}

eqx_status eqx_ledger_restore_async(eqx_ctx* ctx) {
  if (ctx) ++ctx->ledger_epoch;  // the published step ledger (eqx_step_ledger) is stale
  if (!ctx || !ctx->snap_valid) return fail(ctx, EQX_ERR_CONFIG, "eqx_ledger_restore_async: no checkpoint");
  cudaSetDevice(ctx->device);
  cudaStream_t s = ctx->stream;
  // one copy kernel for the six arrays (six memcpy nodes cost ~2 us of device time each)
  PackCols pc;
  std::memset(&pc, 0, sizeof(pc));
  auto add = [&](void* dst, const void* src, size_t bytes) {
    pc.src[pc.n] = src;
    pc.dst[pc.n] = dst;
    pc.bytes[pc.n] = static_cast<int64_t>(bytes);
    ++pc.n;
  };
  if (ctx->C > 0) {
    add(ctx->d_ufc.p, ctx->snap_ufc.p, 8ull * ctx->C);
    add(ctx->d_rfc.p, ctx->snap_rfc.p, 8ull * ctx->C);
    add(ctx->d_counter.p, ctx->snap_counter.p, 8ull * ctx->C);
    add(ctx->d_running.p, ctx->snap_running.p, 4ull * ctx->C);
    add(ctx->d_backlogged.p, ctx->snap_backlogged.p, 4ull * ctx->C);
  }
  add(ctx->d_state.p, ctx->snap_state.p, offsetof(DevState, n_events));
  static_assert(kMaxPackCols >= 6, "restore copies six arrays");
  const unsigned gx = std::max<unsigned>(1, std::min<unsigned>(32, static_cast<unsigned>(8ull * ctx->C / 4096 + 1)));
  pack_cols_kernel<<<dim3(gx, pc.n), 256, 0, s>>>(pc);
  CUDA_TRY(ctx, cudaGetLastError());
  return EQX_OK;
}

eqx_status eqx_set_batch(eqx_ctx* ctx, int32_t members, int64_t reserved) {
  if (!ctx || members < 0 || reserved < 0) return fail(ctx, EQX_ERR_ARG, "eqx_set_batch: bad arguments");
  cudaSetDevice(ctx->device);
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  ctx->h_state->members = members;
  ctx->h_state->reserved = reserved;
  CUDA_TRY(ctx, cudaMemcpyAsync(ctx->d_state.p, ctx->h_state, offsetof(DevState, n_events),
                                cudaMemcpyHostToDevice, ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return EQX_OK;
}

// H2D of a host batch into staging set b on the copy stream (after the set's last reader).
static eqx_status stage_fill(eqx_ctx* ctx, const eqx_requests* r, int b) {
  eqx_ctx::Stage& st = ctx->stg[b];
  cudaStream_t cs = ctx->copy_stream;
  const int64_t n = r->n;
  const size_t nn = static_cast<size_t>(std::max<int64_t>(n, 1));
  st.valid = false;
  CUDA_TRY(ctx, st.client.ensure(4 * nn));
  CUDA_TRY(ctx, st.arrival.ensure(8 * nn));
  CUDA_TRY(ctx, st.in.ensure(4 * nn));
  CUDA_TRY(ctx, st.tag.ensure(nn + 16));
  if (r->true_output_tokens) CUDA_TRY(ctx, st.tru.ensure(4 * nn));
  if (r->id) CUDA_TRY(ctx, st.id.ensure(8 * nn));
  const bool n16 = (r->narrow & EQX_NARROW_U16) != 0, packed = (r->narrow & EQX_PACKED_ARRIVALS) != 0;
  if (n16) {
    CUDA_TRY(ctx, st.c16.ensure(2 * nn + 16));
    CUDA_TRY(ctx, st.i16.ensure(2 * nn + 16));
  }
  int64_t pk_bytes = 0;  // the packed column's size is its first word
  if (packed && n > 0) std::memcpy(&pk_bytes, r->arrival_s, 8);
  if (packed && n > 0) {  // the header's block offsets must stay inside the column (device reads)
    const int64_t nb = (n + 255) / 256, hdr = (8 + 16 * nb + 15) & ~int64_t(15);
    bool ok = pk_bytes >= hdr + 6 * n && pk_bytes <= hdr + 16 * nb + 8 * n;
    const unsigned char* hp = static_cast<const unsigned char*>(static_cast<const void*>(r->arrival_s));
    for (int64_t b = 0; b < nb && ok; ++b) {
      uint64_t base;
      int64_t off;
      std::memcpy(&base, hp + 8 + 8 * b, 8);
      std::memcpy(&off, hp + 8 + 8 * nb + 8 * b, 8);
      const int64_t rows = std::min<int64_t>(256, n - 256 * b);
      ok = off >= hdr && (off & 15) == 0 && off + (base == ~0ull ? 8 : 6) * rows <= pk_bytes;
    }
    if (!ok) return fail(ctx, EQX_ERR_ARG, "packed arrivals: not an eqx_pack_arrivals column of n rows");
  }
  if (packed) CUDA_TRY(ctx, st.apk.ensure(static_cast<size_t>(pk_bytes) + 16));
  CUDA_TRY(ctx, cudaStreamWaitEvent(cs, st.free_, 0));
  auto h2d = [&](void* dst, const void* src, size_t bytes) {
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, cs);
  };
  // every H2D first on the copy stream; the widen / unpack kernels run on their own stream behind
  // an event, so the copy engine moves straight on to the next batch
  if (n > 0) {
    CUDA_TRY(ctx, n16 ? h2d(st.c16.p, r->client, 2 * n) : h2d(st.client.p, r->client, 4 * n));
    CUDA_TRY(ctx, packed ? h2d(st.apk.p, r->arrival_s, static_cast<size_t>(pk_bytes))
                         : h2d(st.arrival.p, r->arrival_s, 8 * n));
    CUDA_TRY(ctx, n16 ? h2d(st.i16.p, r->input_tokens, 2 * n) : h2d(st.in.p, r->input_tokens, 4 * n));
    if (r->tag) CUDA_TRY(ctx, h2d(st.tag.p, r->tag, n));
    else CUDA_TRY(ctx, cudaMemsetAsync(st.tag.p, 0, n, cs));
    if (r->true_output_tokens) CUDA_TRY(ctx, h2d(st.tru.p, r->true_output_tokens, 4 * n));
    if (r->id) CUDA_TRY(ctx, h2d(st.id.p, r->id, 8 * n));
  }
  if (n > 0 && (n16 || packed)) {
    cudaStream_t us = ctx->unpack_stream;
    CUDA_TRY(ctx, cudaEventRecord(st.copied, cs));
    CUDA_TRY(ctx, cudaStreamWaitEvent(us, st.copied, 0));
    const int blocks = static_cast<int>(std::min<int64_t>((n / 8 + 255) / 256 + 1, 4ll * ctx->sm_count));
    if (packed) unpack_arrivals_kernel<<<blocks, 256, 0, us>>>(st.apk.as<unsigned char>(), n, st.arrival.as<double>());
    if (n16)
      widen_cols_kernel<<<blocks, 256, 0, us>>>(st.c16.as<uint16_t>(), st.i16.as<uint16_t>(), n,
                                                st.client.as<int32_t>(), st.in.as<int32_t>());
    CUDA_TRY(ctx, cudaGetLastError());
    CUDA_TRY(ctx, cudaEventRecord(st.ready, us));
  } else {
    CUDA_TRY(ctx, cudaEventRecord(st.ready, cs));
  }
  const void* key[6] = {r->client, r->arrival_s, r->input_tokens, r->tag, r->true_output_tokens, r->id};
  std::memcpy(st.key, key, sizeof(key));
  st.narrow = r->narrow;
  st.n = n;
  st.seq = ++ctx->stage_seq;
  st.valid = true;
  return EQX_OK;
}

// Staging target: the least recently filled set holding no unconsumed batch, preferring one
// the live queue is not bound to (its copy then need not wait for the step in flight); with
// every set unconsumed, the oldest.
static int stage_target(const eqx_ctx* ctx) {
  int best = -1, rank_best = 0;
  for (int k = 0; k < eqx_ctx::kStages; ++k) {
    const eqx_ctx::Stage& st = ctx->stg[k];
    const int rank = st.valid ? 2 : (k == ctx->bound_stage ? 1 : 0);
    if (best < 0 || rank < rank_best || (rank == rank_best && st.seq < ctx->stg[best].seq)) {
      best = k;
      rank_best = rank;
    }
  }
  return best;
}

static bool stage_matches(const eqx_ctx::Stage& st, const eqx_requests* r) {
  const void* key[6] = {r->client, r->arrival_s, r->input_tokens, r->tag, r->true_output_tokens, r->id};
  return st.valid && st.n == r->n && st.narrow == r->narrow && std::memcmp(st.key, key, sizeof(key)) == 0;
}

// Layout (see include/eqx.h): [u64 total bytes][u64 base[nb]][u64 off[nb]] then per block,
// 16-byte aligned at off[b]: 6-byte offsets (packed) or the raw doubles (base[b] == ~0).
int64_t eqx_pack_arrivals(const double* a, int64_t n, void* out, int64_t cap) {
  if (n < 0 || (n > 0 && !a)) return -1;
  const int64_t nb = (n + 255) / 256;
  auto packable = [&](int64_t r0, int64_t r1, uint64_t* base) {
    uint64_t b0, prev;
    std::memcpy(&b0, a + r0, 8);
    prev = b0;
    for (int64_t r = r0; r < r1; ++r) {
      uint64_t v;
      std::memcpy(&v, a + r, 8);
      // non-negative (sign clear), not NaN, non-decreasing bit patterns, 48-bit span
      if ((v >> 63) || v > 0x7ff0000000000000ull || v < prev || v - b0 >= (uint64_t(1) << 48)) return false;
      prev = v;
    }
    *base = b0;
    return true;
  };
  int64_t cur = (8 + 16 * nb + 15) & ~int64_t(15), total = cur;
  for (int64_t b = 0; b < nb; ++b) {  // size pass
    const int64_t r0 = 256 * b, r1 = std::min<int64_t>(n, r0 + 256);
    uint64_t base;
    total += ((packable(r0, r1, &base) ? 6 : 8) * (r1 - r0) + 15) & ~int64_t(15);
  }
  if (!out) return total;
  if (cap < total) return -2;
  unsigned char* o = static_cast<unsigned char*>(out);
  std::memset(o, 0, static_cast<size_t>(total));
  std::memcpy(o, &total, 8);
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t r0 = 256 * b, r1 = std::min<int64_t>(n, r0 + 256);
    uint64_t base = ~0ull;
    const bool pk = packable(r0, r1, &base);
    if (!pk) base = ~0ull;
    std::memcpy(o + 8 + 8 * b, &base, 8);
    std::memcpy(o + 8 + 8 * nb + 8 * b, &cur, 8);
    for (int64_t r = r0; r < r1; ++r) {
      uint64_t v;
      std::memcpy(&v, a + r, 8);
      if (pk) {
        const uint64_t d = v - base;
        std::memcpy(o + cur + 6 * (r - r0), &d, 6);  // little endian: the low 6 bytes
      } else {
        std::memcpy(o + cur + 8 * (r - r0), &v, 8);
      }
    }
    cur += ((pk ? 6 : 8) * (r1 - r0) + 15) & ~int64_t(15);
  }
  return total;
}

// The main stream is done with the bound staging set once everything enqueued so far ran.
static eqx_status release_stage(eqx_ctx* ctx) {
  if (ctx->bound_stage >= 0) CUDA_TRY(ctx, cudaEventRecord(ctx->stg[ctx->bound_stage].free_, ctx->stream));
  return EQX_OK;
}

eqx_status eqx_stage_async(eqx_ctx* ctx, const eqx_requests* r) {
  if (!ctx || !r) return fail(ctx, EQX_ERR_ARG, "eqx_stage_async: NULL argument");
  if (r->location != EQX_HOST) return fail(ctx, EQX_ERR_ARG, "eqx_stage_async: only host batches are staged");
  if (r->narrow & ~(EQX_NARROW_U16 | EQX_PACKED_ARRIVALS))
    return fail(ctx, EQX_ERR_ARG, "eqx_stage_async: unknown narrow flags");
  if ((r->narrow & EQX_NARROW_U16) &&
      (reinterpret_cast<uintptr_t>(r->client) & 1 || reinterpret_cast<uintptr_t>(r->input_tokens) & 1))
    return fail(ctx, EQX_ERR_ARG, "eqx_stage_async: narrow columns must be 2-byte aligned");
  if (r->n < 0 || r->n >= (int64_t(1) << 31) - 1) return fail(ctx, EQX_ERR_ARG, "eqx_stage_async: n out of range");
  if (r->n > 0 && (!r->client || !r->arrival_s || !r->input_tokens))
    return fail(ctx, EQX_ERR_ARG, "eqx_stage_async: missing request column");
  cudaSetDevice(ctx->device);
  return stage_fill(ctx, r, stage_target(ctx));
}

static eqx_status drain_prepare(eqx_ctx* ctx, const eqx_requests* r) {
  if (!ctx || !r) return fail(ctx, EQX_ERR_ARG, "eqx_drain: NULL argument");
  if (!ctx->model_set || !ctx->profile_set)
    return fail(ctx, EQX_ERR_CONFIG, "eqx_drain: predictor and GPU profile must be set first");
  if (r->n < 0 || r->n >= (int64_t(1) << 31) - 1) return fail(ctx, EQX_ERR_ARG, "eqx_drain: n out of range");
  const int64_t n = r->n;
  const int32_t C = ctx->C;
  if (n > 0 && C == 0) return fail(ctx, EQX_ERR_CONFIG, "eqx_drain: requests but no clients");
  const bool needs_true = ctx->model.pred_kind == kPredOracle || ctx->model.pred_kind == kPredNoisy;
  if (n > 0 && (!r->client || !r->arrival_s || !r->input_tokens || (needs_true && !r->true_output_tokens)))
    return fail(ctx, EQX_ERR_ARG, "eqx_drain: missing request column");
  if (r->narrow && r->location == EQX_DEVICE)
    return fail(ctx, EQX_ERR_ARG, "eqx_drain: narrow (uint16 / packed) columns are for host batches only");
  if (r->narrow & ~(EQX_NARROW_U16 | EQX_PACKED_ARRIVALS)) return fail(ctx, EQX_ERR_ARG, "eqx_drain: unknown narrow flags");
  if ((r->narrow & EQX_NARROW_U16) &&
      (reinterpret_cast<uintptr_t>(r->client) & 1 || reinterpret_cast<uintptr_t>(r->input_tokens) & 1))
    return fail(ctx, EQX_ERR_ARG, "eqx_drain: narrow columns must be 2-byte aligned");
  cudaSetDevice(ctx->device);
  cudaStream_t s = ctx->stream;
  const size_t nn = static_cast<size_t>(std::max<int64_t>(n, 1));
  // bind (device) or copy (host) the columns
  if (r->location == EQX_DEVICE) {
    ctx->bound_stage = -1;
    ctx->q_client = r->client;
    ctx->q_arrival = r->arrival_s;
    ctx->q_in = r->input_tokens;
    ctx->q_true = r->true_output_tokens;
    ctx->q_id = r->id;
    if (r->tag) {
      ctx->q_tag = r->tag;
    } else {
      CUDA_TRY(ctx, ctx->own_tag.ensure(nn + 16));
      CUDA_TRY(ctx, cudaMemsetAsync(ctx->own_tag.p, 0, nn, s));
      ctx->q_tag = ctx->own_tag.as<uint8_t>();
    }
  } else {
    // host batch: a matching staged copy (eqx_stage_async), else stage it now
    int b = -1;
    for (int k = 0; k < eqx_ctx::kStages; ++k)
      if (stage_matches(ctx->stg[k], r) && (b < 0 || ctx->stg[k].seq < ctx->stg[b].seq)) b = k;
    if (b < 0) {
      if (std::getenv("EQX_DEBUG_STAGE")) std::fprintf(stderr, "eqx: drain of an unstaged host batch\n");
      b = stage_target(ctx);
      eqx_status e = stage_fill(ctx, r, b);
      if (e != EQX_OK) return e;
    }
    eqx_ctx::Stage& st = ctx->stg[b];
    st.valid = false;  // consumed
    CUDA_TRY(ctx, cudaStreamWaitEvent(s, st.ready, 0));
    ctx->bound_stage = b;
    ctx->q_client = st.client.as<int32_t>();
    ctx->q_arrival = st.arrival.as<double>();
    ctx->q_in = st.in.as<int32_t>();
    ctx->q_tag = st.tag.as<uint8_t>();
    ctx->q_true = r->true_output_tokens ? st.tru.as<int32_t>() : nullptr;
    ctx->q_id = r->id ? st.id.as<int64_t>() : nullptr;
  }
  ctx->id_base = r->id_base;
  ctx->n = n;
  ctx->popped = 0;
  // scores + events sized to the queue
  CUDA_TRY(ctx, ctx->d_pred.ensure(4 * nn + 16));
  CUDA_TRY(ctx, ctx->d_bucket.ensure(nn + 16));
  CUDA_TRY(ctx, ctx->d_ufc_out.ensure(8 * nn + 16));
  CUDA_TRY(ctx, ctx->d_rfc_out.ensure(8 * nn + 16));
  ctx->ev_cap = static_cast<int64_t>(nn);
  CUDA_TRY(ctx, ctx->d_ev_row.ensure(4 * nn));
  CUDA_TRY(ctx, ctx->d_ev_kind.ensure(4 * nn));
  CUDA_TRY(ctx, ctx->d_ev_client.ensure(4 * nn));
  CUDA_TRY(ctx, ctx->d_ev_pred.ensure(4 * nn));
  CUDA_TRY(ctx, ctx->d_ev_ufc.ensure(8 * nn));
  CUDA_TRY(ctx, ctx->d_ev_rfc.ensure(8 * nn));
  CUDA_TRY(ctx, ctx->d_ev_vtc.ensure(8 * nn));
  CUDA_TRY(ctx, ctx->d_ev_wait.ensure(8 * nn));
  CUDA_TRY(ctx, ctx->d_ev_id.ensure(8 * nn));
  CUDA_TRY(ctx, ctx->d_perm.ensure(4 * nn));
  // tiling: one wave of tiles (~n / #SMs rows each, a multiple of 32 warps x 32 rows), so the
  // [client][tile] histogram stays ~C x #SMs entries and its scan is short.  Each tile is
  // staged in shared memory (coalesced per-client runs) when it fits.
  int64_t tile_rows = (n + ctx->sm_count - 1) / std::max(ctx->sm_count, 1);
  tile_rows = std::max<int64_t>(1024, (tile_rows + 1023) / 1024 * 1024);
  // small rosters: per-tile counting sort (one read of the client column, no peer masks)
  ctx->sort_drain = C <= kSortMaxClients;
  if (ctx->sort_drain) {
    tile_rows = kSortTile;
    CUDA_TRY(ctx, ctx->d_tsorted.ensure(4 * nn));
    const size_t cbytes = (2ull * sort_pad((C + (C & 1)) * kSortThreads) + 2 + 15) & ~size_t(15);
    ctx->sort_smem = cbytes + 4ull * kSortTile;
    CUDA_TRY(ctx, set_smem_attr(ctx, 11, reinterpret_cast<const void*>(drain_sort_kernel), ctx->sort_smem));
  }
  if (tile_rows / kDrainWarps > 65535) return fail(ctx, EQX_ERR_CONFIG, "queue too long for the drain tiling");
  const int32_t n_tiles = static_cast<int32_t>(std::max<int64_t>(1, (n + tile_rows - 1) / tile_rows));
  const int64_t L = static_cast<int64_t>(C) * n_tiles;
  CUDA_TRY(ctx, ctx->d_hist.ensure(4 * std::max<int64_t>(L, 1)));
  CUDA_TRY(ctx, ctx->d_tbase.ensure(4 * std::max<int64_t>(L, 1)));
  CUDA_TRY(ctx, ctx->d_tfirst.ensure(4 * std::max<int64_t>(L, 1)));
  CUDA_TRY(ctx, ctx->d_ctot.ensure(4 * std::max<int64_t>(C, 1)));
  ctx->tile_rows = tile_rows;
  ctx->n_tiles = n_tiles;
  ctx->hist_L = L;
  const size_t rank_base = (8ull + 2ull * kDrainWarps) * C + 64;
  ctx->staged = rank_base + 6ull * tile_rows <= ctx->smem_optin;
  ctx->hist_smem = 2ull * kDrainWarps * C + 4ull * C + 16;  // per-warp counts + per-client first rows
  CUDA_TRY(ctx, ctx->d_wcnt.ensure(std::max<size_t>(2ull * kDrainWarps * C * n_tiles, 64)));
  ctx->rank_smem = rank_base + (ctx->staged ? 6ull * tile_rows : 0);
  if (ctx->rank_smem > ctx->smem_optin || ctx->hist_smem > ctx->smem_optin)
    return fail(ctx, EQX_ERR_CONFIG, "too many clients per device (" + std::to_string(C) + ")");
  CUDA_TRY(ctx, set_smem_attr(ctx, 0, reinterpret_cast<const void*>(drain_hist_kernel), ctx->hist_smem));
  CUDA_TRY(ctx, set_smem_attr(ctx, 1, reinterpret_cast<const void*>(drain_rank_kernel), ctx->rank_smem));
  ctx->queue_ready = true;
  return EQX_OK;
}

static DrainArgs drain_args(eqx_ctx* ctx) {
  DrainArgs d;
  std::memset(&d, 0, sizeof(d));
  d.client = ctx->q_client;
  d.n = static_cast<int32_t>(ctx->n);
  d.C = ctx->C;
  d.cbits = 1;
  while ((1 << d.cbits) <= d.C) ++d.cbits;
  d.tile_rows = static_cast<int32_t>(ctx->tile_rows);
  d.n_tiles = ctx->n_tiles;
  d.staged = ctx->staged ? 1 : 0;
  d.hist = ctx->d_hist.as<uint32_t>();
  d.tbase = ctx->d_tbase.as<uint32_t>();
  d.ctot = ctx->d_ctot.as<uint32_t>();
  d.tsorted = ctx->d_tsorted.as<uint32_t>();
  d.tfirst = ctx->d_tfirst.as<uint32_t>();
  d.head = ctx->d_head.as<int32_t>();
  d.zero_qlen = 1;
  d.hist_L = ctx->hist_L;
  d.seg_off = ctx->d_seg_off.as<int32_t>();
  d.perm = ctx->d_perm.as<uint32_t>();
  d.count = ctx->d_count.as<int32_t>();
  d.first_row = ctx->d_first.as<int32_t>();
  d.qlen_before = ctx->d_qlen_before.as<int32_t>();
  d.running = ctx->d_running.as<int32_t>();
  d.ufc = ctx->d_ufc.as<double>();
  d.rfc = ctx->d_rfc.as<double>();
  d.counter = ctx->d_counter.as<double>();
  d.backlogged = ctx->d_backlogged.as<int32_t>();
  d.counter_lift = ctx->counter_lift;
  d.done = ctx->d_done.as<unsigned int>();
  d.wcnt = ctx->d_wcnt.as<uint16_t>();
  d.st = ctx->d_state.as<DevState>();
  return d;
}

// Pure stream work of a drain (3 kernels, no memsets); capturable into a CUDA graph.
// lift: also apply on_activated / set_backlogged now (a standalone drain); a drain fused into a
// step leaves that to the selection kernel's prologue (SelectArgs::do_lift).
static eqx_status drain_enqueue(eqx_ctx* ctx, bool lift, bool keep_qlen = false) {
  if (ctx) ++ctx->ledger_epoch;  // the published step ledger (eqx_step_ledger) is stale
  cudaStream_t s = ctx->stream;
  const int32_t C = ctx->C;
  if (C == 0) return EQX_OK;
  // heads, qlen_before (unless the queue is kept) and first rows are written by
  // drain_scan_kernel: no memset nodes in front of the drain
#ifdef EQX_PROF
  {
    char* dt = reinterpret_cast<char*>(ctx->d_state.p) + offsetof(DevState, dt);
    CUDA_TRY(ctx, cudaMemsetAsync(dt, 0, 8 * 8, s));
    CUDA_TRY(ctx, cudaMemsetAsync(dt, 0xff, 8, s));
    CUDA_TRY(ctx, cudaMemsetAsync(dt + 24, 0xff, 8, s));
    CUDA_TRY(ctx, cudaMemsetAsync(dt + 40, 0xff, 8, s));
  }
#endif
  DrainArgs d = drain_args(ctx);
  d.zero_qlen = keep_qlen ? 0 : 1;
  if (ctx->sort_drain) {
    drain_sort_kernel<<<ctx->n_tiles, kSortThreads, ctx->sort_smem, s>>>(d);
    CUDA_TRY(ctx, launch_pdl(drain_scan_kernel, dim3((C + 31) / 32), dim3(1024), 0, s, d));
    CUDA_TRY(ctx, launch_pdl(drain_scatter_kernel, dim3(ctx->n_tiles), dim3(kSortThreads), 0, s, d));
  } else {
    drain_hist_kernel<<<ctx->n_tiles, kDrainThreads, ctx->hist_smem, s>>>(d);
    CUDA_TRY(ctx, launch_pdl(drain_scan_kernel, dim3((C + 31) / 32), dim3(1024), 0, s, d));
    CUDA_TRY(ctx, launch_pdl(drain_rank_kernel, dim3(ctx->n_tiles), dim3(kDrainThreads), ctx->rank_smem, s, d));
  }
  if (lift) lift_kernel<<<1, 1024, 0, s>>>(d);
  CUDA_TRY(ctx, cudaGetLastError());
  return EQX_OK;
}

// Largest T with double(T) * m <= M (the can_fit KV test, gpu_model.cpp:64-66).  double(T)
// and the IEEE product are monotone in T, so the test is exactly T <= tmax for integer T.
static int64_t kv_threshold(double m, double M) {
  auto ok = [&](int64_t t) { return static_cast<double>(t) * m <= M; };
  const int64_t cap = int64_t(1) << 61;
  if (ok(cap)) return cap;
  int64_t lo = 0, hi = 1;  // ok(lo) holds (0 * m = 0 <= M for M > 0)
  while (ok(hi)) {
    lo = hi;
    hi *= 2;
  }
  while (hi - lo > 1) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (ok(mid)) lo = mid;
    else hi = mid;
  }
  return lo;
}

struct StepPlan {
  ScoreArgs sc;
  WindowArgs wi;
  SelectArgs se;
  size_t score_smem, select_smem, window_smem;
  int score_grid, select_threads, window_grid;
  int score_tma;  // 1: score_tma_kernel (bulk-copy tiles), 0: score_kernel
};

// gW > 0 plans the selection of a client-sharded step over gathered [C][gW] head windows
// (no local queue; see eqx_shard_select_async).
static eqx_status step_prepare(eqx_ctx* ctx, double now, StepPlan& pl, int32_t gW = 0) {
  if (!ctx) return fail(ctx, EQX_ERR_ARG, "eqx_step_async: NULL context");
  if (!ctx->model_set || !ctx->profile_set)
    return fail(ctx, EQX_ERR_CONFIG, "eqx_step: predictor and GPU profile must be set first");
  if (!gW && !ctx->queue_ready) return fail(ctx, EQX_ERR_CONFIG, "eqx_step: no drained queue (call eqx_drain first)");
  cudaSetDevice(ctx->device);
  cudaStream_t s = ctx->stream;
  const int32_t C = ctx->C;
  const size_t model_bytes = offsetof(ModelTables, lut) + 4ull * ctx->lut_entries;
  if (ctx->model_dirty) {  // compiled model tables -> device, only after they changed
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->d_model.p, &ctx->model, model_bytes, cudaMemcpyHostToDevice, s));
    // direct table: the LUT + entry_for evaluated for every small input (MoPE / single proxy)
    // or every small prediction (oracle); same functions, so the same results.
    const ModelTables& M = ctx->model;
    auto entry_for = [&](int pred) {
      int b = M.n_prof - 1;
      for (int e = M.n_prof - 1; e >= 0; --e)
        if (pred <= M.prof_upper[e]) b = e;
      return b;
    };
    std::vector<uint32_t> tab;
    ctx->direct_n = 0;
    if (M.pred_kind == kPredMope || M.pred_kind == kPredSingle) {
      const int dn = 2048;
      bool ok = true;
      tab.resize(static_cast<size_t>(M.n_tag_states) * dn);
      for (int t = 0; t < M.n_tag_states && ok; ++t) {
        for (int in = 0; in < dn; ++in) {
          int iv = 0;
          for (int i = 0; i < M.n_cuts; ++i) iv += M.cuts[i] < in ? 1 : 0;
          const int e = M.lut[iv * M.n_tag_states + t];
          const int pred = e < 0 ? -e : e;
          if (pred >= 65536) {
            ok = false;
            break;
          }
          tab[static_cast<size_t>(t) * dn + in] = static_cast<uint32_t>(pred) |
                                                  (static_cast<uint32_t>(entry_for(pred)) << 16) |
                                                  (static_cast<uint32_t>(e < 0 ? 1 : 0) << 24);
        }
      }
      if (ok && !std::getenv("EQX_NO_DIRECT")) ctx->direct_n = dn;  // EQX_NO_DIRECT: experiments
    } else if (M.pred_kind == kPredOracle) {
      const int dn = 8192;
      tab.resize(dn);
      for (int p = 0; p < dn; ++p) tab[p] = static_cast<uint32_t>(entry_for(p));
      ctx->direct_n = dn;
    }
    if (ctx->direct_n) {
      CUDA_TRY(ctx, ctx->d_direct.ensure(tab.size() * 4));
      CUDA_TRY(ctx, cudaMemcpyAsync(ctx->d_direct.p, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice, s));
    }
    CUDA_TRY(ctx, cudaStreamSynchronize(s));
    ctx->model_dirty = false;
  }
  const int32_t model_words = static_cast<int32_t>((model_bytes + 3) / 4);
  const size_t model_smem = (static_cast<size_t>(model_words) * 4 + 15) & ~size_t(15);
  std::memset(&pl, 0, sizeof(pl));
  // ---- whole-queue scoring ----
  ScoreArgs& sc = pl.sc;
  sc.n = ctx->n;
  sc.client = ctx->q_client;
  sc.arrival = ctx->q_arrival;
  sc.in_tok = ctx->q_in;
  sc.true_out = ctx->q_true;
  sc.tag = ctx->q_tag;
  sc.id = ctx->q_id;
  sc.id_base = ctx->id_base;
  sc.weight = ctx->d_weight.as<double>();
  sc.pred_out = ctx->d_pred.as<int32_t>();
  sc.bucket_out = ctx->d_bucket.as<uint8_t>();
  sc.ufc_out = ctx->d_ufc_out.as<double>();
  sc.rfc_out = ctx->d_rfc_out.as<double>();
  sc.st = ctx->d_state.as<DevState>();
  sc.model = ctx->d_model.as<ModelTables>();
  sc.model_words = model_words;
  sc.direct = ctx->d_direct.as<uint32_t>();
  sc.direct_n = ctx->direct_n;
  sc.vec_ok = aligned16(sc.client) && aligned16(sc.arrival) && aligned16(sc.in_tok) &&
              (reinterpret_cast<uintptr_t>(sc.tag) % 8 == 0) && (!sc.true_out || aligned16(sc.true_out));
  sc.pol = ctx->pol;
  sc.frozen = ctx->live_mode ? ctx->frozen : Frozen{};
  sc.now = now;
  pl.score_smem = model_smem;
  int per_sm = 1;
  if (ctx->occ_smem != pl.score_smem) {
    CUDA_TRY(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctx->occ_per_sm, score_kernel, kScoreThreads,
                                                                pl.score_smem));
    ctx->occ_smem = pl.score_smem;
  }
  per_sm = ctx->occ_per_sm;
  const int64_t want = (ctx->n / 8 + kScoreThreads - 1) / kScoreThreads;  // two 4-request vectors per thread
  pl.score_grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, static_cast<int64_t>(ctx->sm_count) * std::max(per_sm, 1))));
  {  // TMA-pipelined variant: 16-byte aligned columns (bulk copies) and at least one full tile
    const char* m = std::getenv("EQX_SCORE");
    // opt-in (EQX_SCORE=tma): measured slower than the register-streaming kernel (profiles/)
    const bool tma_ok = sc.vec_ok && (reinterpret_cast<uintptr_t>(sc.tag) % 16 == 0) && ctx->n >= kScoreTile &&
                        (m && std::string(m) == "tma");
    pl.score_tma = tma_ok ? 1 : 0;
    if (tma_ok) {
      // ring | model | direct table (staged in shared memory when it fits two CTAs per SM)
      const int32_t dwords = ctx->direct_n ? (ctx->model.pred_kind == kPredOracle ? ctx->direct_n
                                                                                  : ctx->direct_n * ctx->model.n_tag_states)
                                           : 0;
      size_t tsmem = static_cast<size_t>(kScoreStages) * kScoreStageBytes +
                     ((static_cast<size_t>(model_words) * 4 + 127) & ~size_t(127));
      sc.direct_words = (tsmem + 4ull * dwords) * 2 <= ctx->smem_optin ? dwords : 0;
      tsmem += 4ull * sc.direct_words;
      pl.score_smem = tsmem;
      CUDA_TRY(ctx, set_smem_attr(ctx, 7, reinterpret_cast<const void*>(score_tma_kernel), tsmem));
      const int64_t tiles = ctx->n / kScoreTile;
      pl.score_grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(tiles, 2ll * ctx->sm_count)));
    }
  }
  // ---- selection ----
  SelectArgs& a = pl.se;
  a.client = ctx->q_client;
  a.arrival = ctx->q_arrival;
  a.in_tok = ctx->q_in;
  a.true_out = ctx->q_true;
  a.tag = ctx->q_tag;
  a.id = ctx->q_id;
  a.id_base = ctx->id_base;
  a.perm = ctx->d_perm.as<uint32_t>();
  a.seg_off = ctx->d_seg_off.as<int32_t>();
  a.count = ctx->d_count.as<int32_t>();
  a.head = ctx->d_head.as<int32_t>();
  a.C = C;
  a.ufc = ctx->d_ufc.as<double>();
  a.rfc = ctx->d_rfc.as<double>();
  a.counter = ctx->d_counter.as<double>();
  a.weight = ctx->d_weight.as<double>();
  a.order = ctx->d_order.as<uint32_t>();
  a.running = ctx->d_running.as<int32_t>();
  a.backlogged = ctx->d_backlogged.as<int32_t>();
  a.ev_row = ctx->d_ev_row.as<int32_t>();
  a.ev_kind = ctx->d_ev_kind.as<int32_t>();
  a.ev_client = ctx->d_ev_client.as<int32_t>();
  a.ev_pred = ctx->d_ev_pred.as<int32_t>();
  a.ev_ufc = ctx->d_ev_ufc.as<double>();
  a.ev_rfc = ctx->d_ev_rfc.as<double>();
  a.ev_vtc = ctx->d_ev_vtc.as<double>();
  a.ev_wait = ctx->d_ev_wait.as<double>();
  a.ev_id = ctx->d_ev_id.as<int64_t>();
  a.ev_cap = ctx->ev_cap;
  a.st = ctx->d_state.as<DevState>();
  a.model = ctx->d_model.as<ModelTables>();
  a.model_words = model_words;
  a.tmax = kv_threshold(ctx->perf.mem_per_token_bytes, ctx->perf.mem_capacity_bytes);
  a.do_lift = 0;
  a.first_row = ctx->d_first.as<int32_t>();
  a.qlen_before = ctx->d_qlen_before.as<int32_t>();
  a.counter_lift = ctx->counter_lift;
  a.pol = ctx->pol;
  a.frozen = ctx->live_mode ? ctx->frozen : Frozen{};
  a.now = now;
  // Rounds of block-radix top-K over per-client key streams (select_topk_kernel, eqx_topk.cuh)
  {
    const size_t static_smem = 12288;
    const int32_t kcap = kTopkThreads;
    const size_t cw_bytes = 11ull * 16 + static_cast<size_t>(C) * (4 * 8 + 7 * 4);
    const size_t k_bytes = static_cast<size_t>(kcap) * (6 * 4 + 3 * 8 + 3 * 4 + sizeof(WinEntry)) + 15 * 16 + 4 * 256 +
                           8 * 160 * (kTopkThreads / 32);
    const size_t heads_bytes = C > kcap ? 17 * static_cast<size_t>((C + 1) & ~1) + 16 : 0;
    const size_t per_item = 5 * 8 + 2 + 4;  // k, a, u, r, cn, fl, st, sd
    const size_t min_items = 1024;
    // shared memory: model | per-client work | ranked list | head tuples | stream items (the
    // rest); per-client work and head tuples fall back to global scratch on huge rosters
    const size_t fixed = static_smem + model_smem + k_bytes + min_items * per_item + 8 * 16;
    size_t smem = model_smem + k_bytes;
    a.cw_in_smem = fixed + cw_bytes + heads_bytes <= ctx->smem_optin ||
                   (heads_bytes > 0 && fixed + cw_bytes <= ctx->smem_optin && cw_bytes >= heads_bytes);
    if (a.cw_in_smem) {
      a.cw_global = nullptr;
      smem += cw_bytes;
    } else {
      CUDA_TRY(ctx, ctx->d_cw.ensure(cw_bytes));
      a.cw_global = ctx->d_cw.p;
    }
    a.tk_heads = nullptr;
    if (heads_bytes > 0) {
      if (static_smem + smem + heads_bytes + min_items * per_item + 8 * 16 <= ctx->smem_optin) {
        smem += heads_bytes;
      } else {
        CUDA_TRY(ctx, ctx->d_tkh.ensure(heads_bytes));
        a.tk_heads = ctx->d_tkh.p;
      }
    }
    // head windows stay in HBM/L2 (window_kernel output): deep enough for a client taking every
    // free slot on small rosters, a few entries per client on huge ones
    int64_t W = std::min<int64_t>(static_cast<int64_t>(ctx->perf.max_batch) + 2,
                                  std::max<int64_t>(4, (1 << 16) / std::max(C, 1)));
    if (gW > 0) W = std::min<int64_t>(W, gW);
    a.W = static_cast<int32_t>(W);
    a.gW = gW;
    // stream items per round: the rest of shared memory, at most 4096; the depth per client (a
    // power of two <= 64) is fitted per round on the device
    const int64_t cap = std::min<int64_t>(4096, static_cast<int64_t>((ctx->smem_optin - static_smem - smem - 8 * 16) / per_item));
    smem += static_cast<size_t>(cap) * per_item + 8 * 16;
    a.tk_cap = static_cast<int32_t>(cap);
    a.tk_dsh = 6;
    a.tk_kcap = kcap;
    // K of the first round (then doubled while lists run out, else about twice what a round
    // consumed): 256 measured best across cfg2 / cfg3 / cfg4's 10k roster (64: cfg3 -15%, cfg2
    // and the 10k roster +12% / +30%; 128 / 512: cfg3 +9% / +26%)
    a.tk_k0 = 256;
    pl.select_threads = kTopkThreads;
    pl.select_smem = smem;
    CUDA_TRY(ctx, ctx->d_win.ensure(std::max<size_t>(static_cast<size_t>(gW > 0 ? gW : a.W) * C * sizeof(WinEntry), 64)));
    a.win_g = ctx->d_win.as<WinEntry>();
  }
  WindowArgs& wi = pl.wi;
  wi.arrival = ctx->q_arrival;
  wi.in_tok = ctx->q_in;
  wi.true_out = ctx->q_true;
  wi.tag = ctx->q_tag;
  wi.id = ctx->q_id;
  wi.id_base = ctx->id_base;
  wi.perm = ctx->d_perm.as<uint32_t>();
  wi.seg_off = ctx->d_seg_off.as<int32_t>();
  wi.count = ctx->d_count.as<int32_t>();
  wi.head = ctx->d_head.as<int32_t>();
  wi.weight = ctx->d_weight.as<double>();
  wi.C = C;
  wi.W = a.W;
  wi.win = ctx->d_win.as<WinEntry>();
  wi.model = ctx->d_model.as<ModelTables>();
  wi.st = ctx->d_state.as<DevState>();
  wi.model_words = model_words;
  wi.tmax = a.tmax;
  wi.pol = ctx->pol;
  wi.frozen = ctx->live_mode ? ctx->frozen : Frozen{};
  wi.now = now;
  wi.do_lift = 0;  // eqx_drain_step_async moves the lift here
  wi.counter_lift = ctx->counter_lift;
  wi.qlen_before = ctx->d_qlen_before.as<int32_t>();
  wi.running = ctx->d_running.as<int32_t>();
  wi.first_row = ctx->d_first.as<int32_t>();
  wi.ufc = ctx->d_ufc.as<double>();
  wi.rfc = ctx->d_rfc.as<double>();
  wi.counter = ctx->d_counter.as<double>();
  wi.backlogged = ctx->d_backlogged.as<int32_t>();
  pl.window_smem = model_smem;
  const int64_t witems = static_cast<int64_t>(C) * a.W;
  pl.window_grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((witems + 255) / 256, 8ll * ctx->sm_count)));
  CUDA_TRY(ctx, set_smem_attr(ctx, a.tk_heads ? 12 : 10, select_fn(a.tk_heads != nullptr), pl.select_smem));
  return EQX_OK;
}

// The selection kernel's instructions are fetched cold once per step when the L2 was flushed
// (bench.py's timed steps; ~12 us of cfg2's selection loop).  The graph step therefore starts
// with a warm-up launch of the same kernel on a small problem of its own (up to 64 clients x 8
// queued heads in scratch memory: every phase of a regenerating round runs once) on a third
// stream, concurrently with the drain; the real selection then fetches its code from L2.  The
// warm-up reads and writes only its scratch.
static eqx_status warm_args(eqx_ctx* ctx, const StepPlan& pl, SelectArgs& w) {
  const int32_t C = std::max(1, std::min<int32_t>(64, ctx->C));
  constexpr int32_t W = 8;
  // layout: windows | ufc rfc counter weight (f64) | order count head running backlogged (i32)
  //         | 128 events x 8 columns | DevState | per-client work (cw_global plans)
  const size_t wb = sizeof(WinEntry) * C * W, ld = 8ull * C, li = 4ull * C, ev = 128;
  const size_t o_win = 0, o_u = o_win + ((wb + 15) & ~15), o_r = o_u + ld, o_k = o_r + ld, o_w = o_k + ld,
               o_ord = o_w + ld, o_cnt = o_ord + li, o_head = o_cnt + li, o_run = o_head + li, o_bl = o_run + li,
               o_ev = (o_bl + li + 15) & ~size_t(15), o_st = o_ev + 8 * 8 * ev,
               o_cw = (o_st + sizeof(DevState) + 255) & ~size_t(255);
  const size_t total = o_cw + 64 * 1024;
  if (ctx->warm_C != C) {
    CUDA_TRY(ctx, ctx->d_warm.ensure(total));
    std::vector<unsigned char> h(o_cw, 0);
    WinEntry* win = reinterpret_cast<WinEntry*>(h.data() + o_win);
    for (int32_t c = 0; c < C; ++c)
      for (int32_t k = 0; k < W; ++k) {
        WinEntry& e = win[c * W + k];
        e.ufc_inc = 100.0 + 7.0 * ((c * 13 + k * 5) % 17);
        e.rfc_inc = 50.0 + 3.0 * ((c * 7 + k * 11) % 13);
        const double arr = 1e-3 * (k * C + c);
        uint64_t b;
        std::memcpy(&b, &arr, 8);
        e.abits = b | 0x8000000000000000ull;  // ordered bits of a non-negative double
        e.in = 16 + (c + k) % 32;
        e.pred = 8 + (c * 3 + k) % 24;
        e.row = c * W + k;
        e.alone = 1;
      }
    for (int32_t c = 0; c < C; ++c) {
      reinterpret_cast<double*>(h.data() + o_u)[c] = 1000.0 * ((c * 37) % C);
      reinterpret_cast<double*>(h.data() + o_r)[c] = 100.0 * ((c * 11) % C);
      reinterpret_cast<double*>(h.data() + o_w)[c] = 1.0;
      reinterpret_cast<uint32_t*>(h.data() + o_ord)[c] = static_cast<uint32_t>(c);
      reinterpret_cast<int32_t*>(h.data() + o_cnt)[c] = W;
      reinterpret_cast<int32_t*>(h.data() + o_bl)[c] = 1;
    }
    CUDA_TRY(ctx, cudaMemcpy(ctx->d_warm.p, h.data(), o_cw, cudaMemcpyHostToDevice));
    ctx->warm_C = C;
  }
  char* b = static_cast<char*>(ctx->d_warm.p);
  w = pl.se;
  w.C = C;
  w.W = W;
  w.gW = 0;
  w.win_g = reinterpret_cast<const WinEntry*>(b + o_win);
  w.do_lift = 0;
  w.ledger_after_wait = 0;
  w.frozen = Frozen{};
  w.count = reinterpret_cast<const int32_t*>(b + o_cnt);
  w.head = reinterpret_cast<int32_t*>(b + o_head);
  w.ufc = reinterpret_cast<double*>(b + o_u);
  w.rfc = reinterpret_cast<double*>(b + o_r);
  w.counter = reinterpret_cast<double*>(b + o_k);
  w.weight = reinterpret_cast<const double*>(b + o_w);
  w.order = reinterpret_cast<const uint32_t*>(b + o_ord);
  w.running = reinterpret_cast<int32_t*>(b + o_run);
  w.backlogged = reinterpret_cast<int32_t*>(b + o_bl);
  int32_t* evi = reinterpret_cast<int32_t*>(b + o_ev);
  w.ev_row = evi;
  w.ev_kind = evi + ev;
  w.ev_client = evi + 2 * ev;
  w.ev_pred = evi + 3 * ev;
  double* evd = reinterpret_cast<double*>(b + o_ev + 4 * 4 * ev);
  w.ev_ufc = evd;
  w.ev_rfc = evd + ev;
  w.ev_vtc = evd + 2 * ev;
  w.ev_wait = evd + 3 * ev;
  w.ev_cap = ev;
  w.st = reinterpret_cast<DevState*>(b + o_st);
  w.tk_heads = nullptr;
  w.cw_global = w.cw_in_smem ? nullptr : static_cast<void*>(b + o_cw);
  return EQX_OK;
}

// The mapped host buffer a step's selection writes the ledger to (eqx_step_ledger); allocated
// outside any graph capture.
static eqx_status ensure_step_ledger(eqx_ctx* ctx) {
  const size_t lb = 32ull * std::max(ctx->C, 1);
  if (ctx->h_ledger_cap >= lb) return EQX_OK;
  if (ctx->h_ledger) cudaFreeHost(ctx->h_ledger);
  ctx->h_ledger = nullptr;
  ctx->h_ledger_dev = nullptr;
  ctx->h_ledger_cap = 0;
  void* p = nullptr;
  CUDA_TRY(ctx, cudaHostAlloc(&p, lb, cudaHostAllocMapped));
  ctx->h_ledger = static_cast<unsigned char*>(p);
  ctx->h_ledger_cap = lb;
  void* d = nullptr;
  CUDA_TRY(ctx, cudaHostGetDevicePointer(&d, p, 0));
  ctx->h_ledger_dev = static_cast<unsigned char*>(d);
  return EQX_OK;
}

// Stream work of a step.  Scoring (HBM-bound, whole queue) runs on the side stream
// concurrently with [optional drain ->] selection on the main stream; both join before the
// summary D2H.  Capturable into a CUDA graph (fork/join through events).
static eqx_status step_enqueue(eqx_ctx* ctx, const StepPlan& pl, bool with_drain) {
  cudaStream_t s = ctx->stream, s2 = ctx->stream2;
  char* st = reinterpret_cast<char*>(ctx->d_state.p);
  // Timing (events, the scoring-CTA stamps of eqx_phase_times) belongs to split launches and the
  // instrumented build; a captured graph carries only the work.
  const bool timing = !with_drain;
#ifndef EQX_PROF
  const bool stamps = timing;
#else
  const bool stamps = true;
#endif
  if (stamps) {
    CUDA_TRY(ctx, cudaMemsetAsync(st + offsetof(DevState, t) + 4 * 8, 0xff, 8, s));
    CUDA_TRY(ctx, cudaMemsetAsync(st + offsetof(DevState, t) + 5 * 8, 0, 8, s));
  }
  if (timing) CUDA_TRY(ctx, cudaEventRecord(ctx->ev_k[4], s));
  const bool warm = with_drain && ctx->C > 0 && ctx->stream3;
  if (warm) {  // the selection's code warm-up, concurrent with the drain (see warm_args)
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev_warm, s));
    CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->stream3, ctx->ev_warm, 0));
    SelectArgs w = ctx->warm_se;
    void* args[] = {&w};
    CUDA_TRY(ctx, cudaLaunchKernel(select_fn(pl.se.tk_heads != nullptr), dim3(1), dim3(pl.select_threads), args, pl.select_smem, ctx->stream3));
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev_warm_done, ctx->stream3));
  }
  if (with_drain) {
    eqx_status e = drain_enqueue(ctx, false);
    if (e != EQX_OK) return e;
  }
  // Split launches record the per-kernel timing events; the graph path (with_drain) leaves the
  // drain -> window -> selection chain bare so its programmatic (PDL) edges survive capture.
  // The selection CTA writes the host-visible DevState itself, with the scoring's counts once
  // every scoring CTA has added them (score_counts): no copy kernel after the join.  An empty
  // queue launches no scoring: the copy kernel remains.
  const bool publish = ctx->n > 0;
  ScoreArgs sc = pl.sc;
  SelectArgs se = pl.se;
  WindowArgs wi = pl.wi;
  if (publish) {
    sc.done = reinterpret_cast<unsigned long long*>(ctx->d_done.as<unsigned char>() + 32);
    se.h_st = ctx->h_state_dev;
    se.score_done = sc.done;
    se.score_ctas = pl.score_grid;
    wi.score_sig = sc.done;
    if (ctx->h_ledger_dev && ctx->h_ledger_cap >= 32ull * ctx->C) {
      se.h_ledger = ctx->h_ledger_dev;
      ctx->ledger_pub_epoch = ++ctx->ledger_epoch;
    }
  }
  if (timing) CUDA_TRY(ctx, cudaEventRecord(ctx->ev_k[5], s));
  CUDA_TRY(ctx, launch_pdl(window_kernel, dim3(pl.window_grid), dim3(256), pl.window_smem, s, wi));
  // Whole-queue scoring forks off after the windows: the selection CTA (PDL) is resident by
  // then, so the scoring grid fills the other SMs while the one-warp selection loop runs
  // (nothing in the selection reads the per-request scores; the state copy joins them).
  CUDA_TRY(ctx, cudaEventRecord(ctx->ev_fork, s));
  CUDA_TRY(ctx, cudaStreamWaitEvent(s2, ctx->ev_fork, 0));
  if (timing) CUDA_TRY(ctx, cudaEventRecord(ctx->ev_k[0], s2));
  if (ctx->n > 0) {
    if (pl.score_tma) score_tma_kernel<<<pl.score_grid, kScoreTmaThreads, pl.score_smem, s2>>>(sc);
    else score_kernel<<<pl.score_grid, kScoreThreads, pl.score_smem, s2>>>(sc);
  }
  CUDA_TRY(ctx, cudaGetLastError());
  if (timing) CUDA_TRY(ctx, cudaEventRecord(ctx->ev_k[1], s2));
  CUDA_TRY(ctx, cudaEventRecord(ctx->ev_join, s2));
  if (timing) CUDA_TRY(ctx, cudaEventRecord(ctx->ev_k[2], s));
  {  // PDL: the selection CTA stages its model, lifts and loads the ledger while the windows fill
    void* args[] = {&se};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(pl.select_threads);
    cfg.dynamicSmemBytes = pl.select_smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CUDA_TRY(ctx, cudaLaunchKernelExC(&cfg, select_fn(pl.se.tk_heads != nullptr), args));
  }
  if (timing) CUDA_TRY(ctx, cudaEventRecord(ctx->ev_k[3], s));
  CUDA_TRY(ctx, cudaGetLastError());
  // the selection wrote every event with its payload and request id (topk_event); the state
  // copy follows the scoring (DevState::fallbacks / near_ties) and the warm-up
  CUDA_TRY(ctx, cudaStreamWaitEvent(s, ctx->ev_join, 0));
  if (warm) CUDA_TRY(ctx, cudaStreamWaitEvent(s, ctx->ev_warm_done, 0));
  if (!publish) CUDA_TRY(ctx, state_to_host(ctx, s, true));
  return EQX_OK;
}

eqx_status eqx_drain(eqx_ctx* ctx, const eqx_requests* r) {
  eqx_status st = drain_prepare(ctx, r);
  if (st != EQX_OK) return st;
  ctx->live_mode = false;  // replaces the queue
  ctx->shard_W = 0;
  st = drain_enqueue(ctx, true);
  if (st != EQX_OK) return st;
  return release_stage(ctx);
}

eqx_status eqx_step_async(eqx_ctx* ctx, double now) {
  StepPlan pl;
  eqx_status st = step_prepare(ctx, now, pl);
  if (st == EQX_OK) st = ensure_step_ledger(ctx);
  if (st != EQX_OK) return st;
  ctx->shard_W = 0;
  st = step_enqueue(ctx, pl, false);
  if (st != EQX_OK) return st;
  ctx->step_pending = true;
  ctx->stepped = true;
  return release_stage(ctx);
}

eqx_status eqx_drain_step_async(eqx_ctx* ctx, const eqx_requests* r, double now) {
  eqx_status st = drain_prepare(ctx, r);
  if (st != EQX_OK) return st;
  ctx->live_mode = false;  // replaces the queue
  ctx->shard_W = 0;
  StepPlan pl;
  st = step_prepare(ctx, now, pl);
  if (st != EQX_OK) return st;
  // the fused drain leaves on_activated / set_backlogged to an extra CTA of the window kernel
  // (the selection CTA, launched programmatically behind it, reads the ledger after its wait)
  pl.wi.do_lift = 1;
  pl.window_grid += 1;
  pl.se.do_lift = 0;
  pl.se.ledger_after_wait = 1;
  cudaStream_t s = ctx->stream;
  // One CUDA-graph launch replays drain + scoring + selection.  The key covers every launch
  // parameter (pointers, sizes, policy, `now`, smem/tiling plan); two graphs are cached, for a
  // resident queue or the staging buffer sets of host batches (whose H2D and release events
  // stay outside the graph).
  {
    eqx_status le = ensure_step_ledger(ctx);
    if (le != EQX_OK) return le;
  }
  if (ctx->C > 0) {  // the selection code warm-up's problem and stream (outside any capture)
    eqx_status we = warm_args(ctx, pl, ctx->warm_se);
    if (we != EQX_OK) return we;
    if (!ctx->stream3) {
      CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->stream3, cudaStreamNonBlocking));
      CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->ev_warm, cudaEventDisableTiming));
      CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->ev_warm_done, cudaEventDisableTiming));
    }
  }
  std::vector<unsigned char> key(sizeof(StepPlan) + 9 * sizeof(int64_t));
  std::memcpy(key.data(), &pl, sizeof(StepPlan));
  const int64_t extra[9] = {ctx->tile_rows, ctx->n_tiles, ctx->counter_lift, static_cast<int64_t>(ctx->hist_smem),
                            static_cast<int64_t>(ctx->rank_smem), ctx->staged,
                            static_cast<int64_t>(reinterpret_cast<uintptr_t>(ctx->q_id)), ctx->id_base,
                            static_cast<int64_t>(reinterpret_cast<uintptr_t>(ctx->h_ledger_dev))};
  std::memcpy(key.data() + sizeof(StepPlan), extra, sizeof(extra));
  int slot = -1;
  for (int i = 0; i < eqx_ctx::kGraphs; ++i)
    if (ctx->graphs[i] && ctx->graph_keys[i] == key) slot = i;
  if (slot < 0) {
    slot = 0;
    for (int i = 1; i < eqx_ctx::kGraphs; ++i)
      if (ctx->graph_used[i] < ctx->graph_used[slot]) slot = i;
    if (ctx->graphs[slot]) cudaGraphExecDestroy(ctx->graphs[slot]);
    ctx->graphs[slot] = nullptr;
    cudaGraph_t g = nullptr;
    CUDA_TRY(ctx, cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    st = step_enqueue(ctx, pl, true);
    cudaError_t ce = cudaStreamEndCapture(s, &g);
    if (st != EQX_OK) {
      if (g) cudaGraphDestroy(g);
      return st;
    }
    CUDA_TRY(ctx, ce);
    cudaError_t ie = cudaGraphInstantiate(&ctx->graphs[slot], g, 0);
    cudaGraphDestroy(g);
    CUDA_TRY(ctx, ie);
    ctx->graph_keys[slot] = key;
  }
  ctx->graph_used[slot] = ++ctx->graph_clock;
  CUDA_TRY(ctx, cudaGraphLaunch(ctx->graphs[slot], s));
  // a replay drains (the ledger changes) and, on a non-empty queue, publishes the step ledger
  // exactly as the captured step_enqueue did (the graph key holds h_ledger_dev)
  ++ctx->ledger_epoch;
  if (ctx->n > 0 && ctx->h_ledger_dev && ctx->h_ledger_cap >= 32ull * ctx->C) ctx->ledger_pub_epoch = ++ctx->ledger_epoch;
  if (r->location != EQX_DEVICE) st = release_stage(ctx);
  if (st != EQX_OK) return st;
  ctx->step_pending = true;
  ctx->stepped = true;
  return EQX_OK;
}

// ---- batched engine replays -------------------------------------------
eqx_status eqx_set_timing(eqx_ctx* ctx, double prefill_linear_ms, double prefill_quad_ms, double decode_base_ms,
                          double decode_per_ctx_ms, double refresh_ms) {
  if (!ctx) return fail(ctx, EQX_ERR_ARG, "eqx_set_timing: NULL context");
  // PerfParams::validate (gpu_model.cpp:9-24)
  if (prefill_linear_ms < 0.0 || prefill_quad_ms < 0.0 || decode_base_ms < 0.0 || decode_per_ctx_ms < 0.0 ||
      refresh_ms < 0.0)
    return fail(ctx, EQX_ERR_CONFIG, "perf timing parameters must be >= 0");
  ctx->prefill_linear_ms = prefill_linear_ms;
  ctx->prefill_quad_ms = prefill_quad_ms;
  ctx->decode_base_ms = decode_base_ms;
  ctx->decode_per_ctx_ms = decode_per_ctx_ms;
  ctx->refresh_ms = refresh_ms;
  return EQX_OK;
}

eqx_status eqx_replay(eqx_ctx* ctx, const eqx_replays* R, eqx_replay_out* O) {
  if (ctx) ++ctx->ledger_epoch;  // the published step ledger (eqx_step_ledger) is stale
  if (!ctx || !R || !O) return fail(ctx, EQX_ERR_ARG, "eqx_replay: NULL argument");
  if (!ctx->policy_set || !ctx->model_set || !ctx->profile_set)
    return fail(ctx, EQX_ERR_CONFIG, "eqx_replay: policy, predictor and GPU profile must be set first");
  const int32_t nr = R->n_replays, C = ctx->C;
  if (nr < 0 || !R->row_off || (nr > 0 && (!R->alpha || !R->client || !R->arrival_s || !R->input_tokens ||
                                           !R->true_output_tokens)))
    return fail(ctx, EQX_ERR_ARG, "eqx_replay: missing replay columns");
  if (C < 1) return fail(ctx, EQX_ERR_CONFIG, "eqx_replay: empty roster");
  if (R->ema_alpha <= 0.0 || R->ema_alpha > 1.0) return fail(ctx, EQX_ERR_CONFIG, "ema_alpha must lie in (0, 1]");
  if (R->prediction_overhead_ms < 0.0) return fail(ctx, EQX_ERR_CONFIG, "prediction_overhead_ms must be >= 0");
  if (R->max_sim_time_s < 0.0) return fail(ctx, EQX_ERR_CONFIG, "max_sim_time_s must be >= 0");
  for (int32_t i = 0; i < nr; ++i) {
    if (R->alpha[i] < 0.0 || R->alpha[i] > 1.0) return fail(ctx, EQX_ERR_CONFIG, "alpha must lie in [0, 1]");
    if (R->row_off[i + 1] < R->row_off[i]) return fail(ctx, EQX_ERR_ARG, "eqx_replay: row offsets must be ordered");
  }
  if (nr == 0) return EQX_OK;
  const int64_t rows = R->row_off[nr] - R->row_off[0];
  if (R->row_off[0] != 0) return fail(ctx, EQX_ERR_ARG, "eqx_replay: row_off[0] must be 0");
  for (int64_t i = 0; i < rows; ++i)
    if (R->client[i] < 0 || R->client[i] >= C) return fail(ctx, EQX_ERR_CONFIG, "request references unknown client");
  cudaSetDevice(ctx->device);
  cudaStream_t s = ctx->stream;
  if (ctx->model_dirty) {  // upload the compiled model tables
    StepPlan pl;
    const bool qr = ctx->queue_ready;
    const int64_t n0 = ctx->n;
    ctx->queue_ready = true;
    eqx_status st = step_prepare(ctx, 0.0, pl);
    ctx->queue_ready = qr;
    ctx->n = n0;
    if (st != EQX_OK) return st;
  }
  const int64_t cap = std::max<int64_t>(R->ev_cap, 1);
  const size_t rr = static_cast<size_t>(std::max<int64_t>(rows, 1)), n8 = static_cast<size_t>(nr);
  // one device block: inputs | scratch | outputs
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += (bytes + 15) & ~size_t(15);
    return o;
  };
  const size_t o_off = take(8 * (n8 + 1)), o_client = take(4 * rr), o_arr = take(8 * rr), o_in = take(4 * rr),
               o_true = take(4 * rr), o_tag = take(rr), o_id = take(8 * rr), o_alpha = take(8 * n8),
               o_crow = take(4 * rr), o_fpred = take(4 * rr), o_fpreds = take(8 * rr), o_frfc = take(8 * rr),
               o_cl = take(sizeof(ReplayClient) * n8 * C), o_mb = take(sizeof(ReplayMember) * n8 * ctx->perf.max_batch),
               o_prof = take(8 * n8 * 4 * kMaxProfile), o_evid = take(8 * n8 * cap), o_evk = take(4 * n8 * cap),
               o_evt = take(8 * n8 * cap), o_nev = take(8 * n8), o_comp = take(8 * n8), o_end = take(8 * n8),
               o_clamp = take(8 * n8), o_stat = take(4 * n8), o_u = take(8 * n8 * C), o_r = take(8 * n8 * C),
               o_k = take(8 * n8 * C), o_ttft = take(8 * rr), o_jain = take(8 * n8), o_tput = take(8 * n8);
  const int64_t wcap = std::max<int64_t>(R->win_cap, 0);
  const size_t w8 = static_cast<size_t>(wcap), c8 = static_cast<size_t>(C);
  const bool full = R->log_all != 0;
  const size_t o_dur = take(8 * n8), o_given = take(R->predicted ? 4 * rr : 0), o_plat = take(full ? 8 * rr : 0),
               o_i0 = take(full ? 4 * n8 * cap : 0), o_d0 = take(full ? 8 * n8 * cap : 0),
               o_d1 = take(full ? 8 * n8 * cap : 0), o_d2 = take(full ? 8 * n8 * cap : 0);
  const size_t o_lat = take(8 * rr), o_rep = take(sizeof(eqx_replay_report) * n8),
               o_rcl = take(sizeof(eqx_replay_client) * n8 * c8), o_win = take(8 * 4 * n8 * w8),
               o_winc = take(8 * 4 * n8 * w8 * c8), o_diff = take(8 * 2 * n8 * w8), o_rate = take(8 * n8 * c8 * w8);
  CUDA_TRY(ctx, ctx->d_fb.ensure(off));
  char* b = static_cast<char*>(ctx->d_fb.p);
  auto up = [&](size_t o, const void* src, size_t bytes) {
    return src ? cudaMemcpyAsync(b + o, src, bytes, cudaMemcpyHostToDevice, s) : cudaMemsetAsync(b + o, 0, bytes, s);
  };
  CUDA_TRY(ctx, up(o_off, R->row_off, 8 * (n8 + 1)));
  CUDA_TRY(ctx, up(o_client, R->client, 4 * rows));
  CUDA_TRY(ctx, up(o_arr, R->arrival_s, 8 * rows));
  CUDA_TRY(ctx, up(o_in, R->input_tokens, 4 * rows));
  CUDA_TRY(ctx, up(o_true, R->true_output_tokens, 4 * rows));
  CUDA_TRY(ctx, up(o_tag, R->tag, rows));
  CUDA_TRY(ctx, up(o_alpha, R->alpha, 8 * n8));
  if (R->duration_s) CUDA_TRY(ctx, up(o_dur, R->duration_s, 8 * n8));
  if (R->predicted) CUDA_TRY(ctx, up(o_given, R->predicted, 4 * rows));
  std::vector<int64_t> ids;
  if (!R->id) {  // trace positions within each replay
    ids.resize(rr);
    for (int32_t i = 0; i < nr; ++i)
      for (int64_t k = R->row_off[i]; k < R->row_off[i + 1]; ++k) ids[k] = k - R->row_off[i];
  }
  CUDA_TRY(ctx, up(o_id, R->id ? static_cast<const void*>(R->id) : ids.data(), 8 * rows));
  if (O->rate && wcap > 0) CUDA_TRY(ctx, cudaMemsetAsync(b + o_rate, 0, 8 * n8 * c8 * w8, s));
  // slots past a replay's own count (events, window samples) read back as zeros, not as stale
  // scratch: the outputs a caller asked for start cleared
  auto clear = [&](const void* want, size_t o, size_t bytes) {
    return want && bytes ? cudaMemsetAsync(b + o, 0, bytes, s) : cudaSuccess;
  };
  CUDA_TRY(ctx, clear(O->ev_id, o_evid, 8 * n8 * cap));
  CUDA_TRY(ctx, clear(O->ev_kind, o_evk, 4 * n8 * cap));
  CUDA_TRY(ctx, clear(O->ev_time, o_evt, 8 * n8 * cap));
  if (full) {
    CUDA_TRY(ctx, clear(O->ev_i0, o_i0, 4 * n8 * cap));
    CUDA_TRY(ctx, clear(O->ev_d0, o_d0, 8 * n8 * cap));
    CUDA_TRY(ctx, clear(O->ev_d1, o_d1, 8 * n8 * cap));
    CUDA_TRY(ctx, clear(O->ev_d2, o_d2, 8 * n8 * cap));
  }
  if (wcap > 0) {
    CUDA_TRY(ctx, clear(O->win, o_win, 8 * 4 * n8 * w8));
    CUDA_TRY(ctx, clear(O->win_clients, o_winc, 8 * 4 * n8 * w8 * c8));
    CUDA_TRY(ctx, clear(O->diff, o_diff, 8 * 2 * n8 * w8));
  }
  ReplayArgs A;
  std::memset(&A, 0, sizeof(A));
  A.n_replays = nr;
  A.C = C;
  A.row_off = reinterpret_cast<const int64_t*>(b + o_off);
  A.client = reinterpret_cast<const int32_t*>(b + o_client);
  A.arrival = reinterpret_cast<const double*>(b + o_arr);
  A.in_tok = reinterpret_cast<const int32_t*>(b + o_in);
  A.true_out = reinterpret_cast<const int32_t*>(b + o_true);
  A.tag = reinterpret_cast<const uint8_t*>(b + o_tag);
  A.id = reinterpret_cast<const int64_t*>(b + o_id);
  A.alpha = reinterpret_cast<const double*>(b + o_alpha);
  A.weight = ctx->d_weight.as<double>();
  A.order = ctx->d_order.as<uint32_t>();
  A.model = ctx->d_model.as<ModelTables>();
  A.pol = ctx->pol;
  A.counter_lift = ctx->counter_lift;
  A.max_sim_time_s = R->max_sim_time_s;
  A.ema_alpha = R->ema_alpha;
  A.prefill_linear_ms = ctx->prefill_linear_ms;
  A.prefill_quad_ms = ctx->prefill_quad_ms;
  A.decode_base_ms = ctx->decode_base_ms;
  A.decode_per_ctx_ms = ctx->decode_per_ctx_ms;
  A.refresh_ms = ctx->refresh_ms;
  A.crow = reinterpret_cast<int32_t*>(b + o_crow);
  A.f_pred = reinterpret_cast<int32_t*>(b + o_fpred);
  A.f_preds = reinterpret_cast<double*>(b + o_fpreds);
  A.f_rfc = reinterpret_cast<double*>(b + o_frfc);
  A.cl = reinterpret_cast<ReplayClient*>(b + o_cl);
  A.mb = reinterpret_cast<ReplayMember*>(b + o_mb);
  A.prof = reinterpret_cast<double*>(b + o_prof);
  A.ev_cap = cap;
  A.ev_id = reinterpret_cast<int64_t*>(b + o_evid);
  A.ev_kind = reinterpret_cast<int32_t*>(b + o_evk);
  A.ev_time = reinterpret_cast<double*>(b + o_evt);
  A.n_events = reinterpret_cast<int64_t*>(b + o_nev);
  A.completed = reinterpret_cast<int64_t*>(b + o_comp);
  A.sim_end = reinterpret_cast<double*>(b + o_end);
  A.clamps = reinterpret_cast<int64_t*>(b + o_clamp);
  A.status = reinterpret_cast<int32_t*>(b + o_stat);
  A.out_ufc = reinterpret_cast<double*>(b + o_u);
  A.out_rfc = reinterpret_cast<double*>(b + o_r);
  A.out_counter = reinterpret_cast<double*>(b + o_k);
  A.f_ttft = reinterpret_cast<double*>(b + o_ttft);
  A.jain_ttft_p90 = reinterpret_cast<double*>(b + o_jain);
  A.throughput_tps = reinterpret_cast<double*>(b + o_tput);
  A.window_s = R->report_window_s > 0.0 ? R->report_window_s : 1.0;  // EngineConfig default
  A.win_cap = wcap;
  A.f_lat = reinterpret_cast<double*>(b + o_lat);
  A.report = reinterpret_cast<eqx_replay_report*>(b + o_rep);
  A.rclients = reinterpret_cast<eqx_replay_client*>(b + o_rcl);
  A.win = O->win && wcap > 0 ? reinterpret_cast<double*>(b + o_win) : nullptr;
  A.win_clients = O->win_clients && wcap > 0 ? reinterpret_cast<double*>(b + o_winc) : nullptr;
  A.diff = O->diff && wcap > 0 ? reinterpret_cast<double*>(b + o_diff) : nullptr;
  A.rate = O->rate && wcap > 0 ? reinterpret_cast<double*>(b + o_rate) : nullptr;
  A.duration = R->duration_s ? reinterpret_cast<const double*>(b + o_dur) : nullptr;
  A.overhead_s = R->prediction_overhead_ms / 1000.0;  // eligible_at's operand (engine.cpp:167)
  A.given_pred = R->predicted ? reinterpret_cast<const int32_t*>(b + o_given) : nullptr;
  A.by_order = ctx->d_by_order.as<uint32_t>();
  A.log_all = full ? 1 : 0;
  A.f_plat = full ? reinterpret_cast<double*>(b + o_plat) : nullptr;
  A.ev_i0 = full ? reinterpret_cast<int32_t*>(b + o_i0) : nullptr;
  A.ev_d0 = full ? reinterpret_cast<double*>(b + o_d0) : nullptr;
  A.ev_d1 = full ? reinterpret_cast<double*>(b + o_d1) : nullptr;
  A.ev_d2 = full ? reinterpret_cast<double*>(b + o_d2) : nullptr;
  CUDA_TRY(ctx, cudaEventRecord(ctx->ev_k[2], s));
  {  // one warp per replay; the instantiation of the context's policy (explicit in eqx_replay.cu)
    const bool big = C > kMaxReplayClients;
    const void* rk = ctx->pol.kind == kFcfs
                         ? (big ? reinterpret_cast<const void*>(replay_kernel<kFcfs, true>)
                                : reinterpret_cast<const void*>(replay_kernel<kFcfs, false>))
                     : ctx->pol.kind == kVtc ? (big ? reinterpret_cast<const void*>(replay_kernel<kVtc, true>)
                                                    : reinterpret_cast<const void*>(replay_kernel<kVtc, false>))
                     : (big ? reinterpret_cast<const void*>(replay_kernel<kEquinox, true>)
                            : reinterpret_cast<const void*>(replay_kernel<kEquinox, false>));
    void* args[] = {&A};
    CUDA_TRY(ctx, cudaLaunchKernel(rk, dim3((nr + 3) / 4), dim3(128), args, 0, s));
  }
  CUDA_TRY(ctx, cudaGetLastError());
  CUDA_TRY(ctx, cudaEventRecord(ctx->ev_k[3], s));
  const Col cols[] = {{O->n_events, b + o_nev, 8 * n8},       {O->ev_id, b + o_evid, 8 * n8 * cap},
                      {O->ev_kind, b + o_evk, 4 * n8 * cap},    {O->ev_time, b + o_evt, 8 * n8 * cap},
                      {O->ufc, b + o_u, 8 * n8 * C},           {O->rfc, b + o_r, 8 * n8 * C},
                      {O->counter, b + o_k, 8 * n8 * C},       {O->completed, b + o_comp, 8 * n8}};
  eqx_status st = read_cols(ctx, cols, 8);
  if (st != EQX_OK) return st;
  const Col cols2[] = {{O->sim_end, b + o_end, 8 * n8},
                       {O->counter_clamps, b + o_clamp, 8 * n8},
                       {O->status, b + o_stat, 4 * n8},
                       {O->jain_ttft_p90, b + o_jain, 8 * n8},
                       {O->throughput_tps, b + o_tput, 8 * n8},
                       {O->report, b + o_rep, sizeof(eqx_replay_report) * n8},
                       {O->clients, b + o_rcl, sizeof(eqx_replay_client) * n8 * c8},
                       {wcap > 0 ? O->win : nullptr, b + o_win, 8 * 4 * n8 * w8}};
  st = read_cols(ctx, cols2, 8);
  if (st != EQX_OK) return st;
  const Col cols3[] = {{wcap > 0 ? O->win_clients : nullptr, b + o_winc, 8 * 4 * n8 * w8 * c8},
                       {wcap > 0 ? O->diff : nullptr, b + o_diff, 8 * 2 * n8 * w8},
                       {wcap > 0 ? O->rate : nullptr, b + o_rate, 8 * n8 * c8 * w8}};
  st = read_cols(ctx, cols3, 3);
  if (st != EQX_OK) return st;
  const size_t np = static_cast<size_t>(ctx->model.n_prof);
  const Col cols4[] = {{full ? O->ev_i0 : nullptr, b + o_i0, 4 * n8 * cap},
                       {full ? O->ev_d0 : nullptr, b + o_d0, 8 * n8 * cap},
                       {full ? O->ev_d1 : nullptr, b + o_d1, 8 * n8 * cap},
                       {full ? O->ev_d2 : nullptr, b + o_d2, 8 * n8 * cap},
                       {O->profile, b + o_prof, 8 * 3 * np * n8}};
  return read_cols(ctx, cols4, 5);
}

// ---- live queues -----------------------------------------------------
eqx_status eqx_append(eqx_ctx* ctx, const eqx_requests* r) {
  if (ctx) ++ctx->ledger_epoch;  // the published step ledger (eqx_step_ledger) is stale
  if (!ctx || !r) return fail(ctx, EQX_ERR_ARG, "eqx_append: NULL argument");
  if (!ctx->model_set || !ctx->profile_set)
    return fail(ctx, EQX_ERR_CONFIG, "eqx_append: predictor and GPU profile must be set first");
  if (ctx->queue_ready && !ctx->live_mode)
    return fail(ctx, EQX_ERR_CONFIG, "eqx_append: the context holds a queue from eqx_drain (which replaces queues)");
  const int64_t m = r->n;
  if (m < 0) return fail(ctx, EQX_ERR_ARG, "eqx_append: negative batch size");
  if (r->narrow) return fail(ctx, EQX_ERR_ARG, "eqx_append: narrow (uint16) columns are for eqx_stage_async / eqx_drain");
  const int32_t C = ctx->C;
  if (m > 0 && C == 0) return fail(ctx, EQX_ERR_CONFIG, "eqx_append: requests but no clients");
  const bool needs_true = ctx->model.pred_kind == kPredOracle || ctx->model.pred_kind == kPredNoisy;
  if (m > 0 && (!r->client || !r->arrival_s || !r->input_tokens || (needs_true && !r->true_output_tokens)))
    return fail(ctx, EQX_ERR_ARG, "eqx_append: missing request column");
  cudaSetDevice(ctx->device);
  cudaStream_t s = ctx->stream;
  // 1. remaining rows of the live queue (client-grouped FIFO order)
  const int old = ctx->live_cur;
  const bool have_old = ctx->live_mode && old >= 0;
  LiveArgs L;
  std::memset(&L, 0, sizeof(L));
  L.C = C;
  int64_t n_live = 0;
  CUDA_TRY(ctx, ctx->d_live_off.ensure(4ull * (C + 1)));
  CUDA_TRY(ctx, ctx->d_nlive.ensure(64));
  L.live_off = ctx->d_live_off.as<int32_t>();
  L.qlen_before = ctx->d_qlen_before.as<int32_t>();
  L.n_live = ctx->d_nlive.as<int64_t>();
  if (have_old && C > 0) {
    L.perm = ctx->d_perm.as<uint32_t>();
    L.seg_off = ctx->d_seg_off.as<int32_t>();
    L.count = ctx->d_count.as<int32_t>();
    L.head = ctx->d_head.as<int32_t>();
    live_offsets_kernel<<<1, 1024, 0, s>>>(L);
    CUDA_TRY(ctx, cudaGetLastError());
    CUDA_TRY(ctx, cudaMemcpyAsync(&n_live, L.n_live, 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(ctx, cudaStreamSynchronize(s));
  } else if (C > 0) {
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->d_qlen_before.p, 0, 4ull * C, s));
  }
  // 2. the new column store: remaining rows, then the arrivals
  const int nb = have_old ? (old ^ 1) : 0;
  eqx_ctx::Live& N = ctx->live[nb];
  const int64_t total = n_live + m;
  if (total >= (int64_t(1) << 31) - 1) return fail(ctx, EQX_ERR_ARG, "eqx_append: live queue too long");
  const size_t tt = static_cast<size_t>(std::max<int64_t>(total, 1));
  CUDA_TRY(ctx, N.client.ensure(4 * tt + 16));
  CUDA_TRY(ctx, N.arrival.ensure(8 * tt + 16));
  CUDA_TRY(ctx, N.in.ensure(4 * tt + 16));
  CUDA_TRY(ctx, N.tag.ensure(tt + 16));
  CUDA_TRY(ctx, N.id.ensure(8 * tt + 16));
  CUDA_TRY(ctx, N.pred.ensure(4 * tt + 16));
  CUDA_TRY(ctx, N.bucket.ensure(tt + 16));
  CUDA_TRY(ctx, N.preds.ensure(8 * tt + 16));
  CUDA_TRY(ctx, N.rfc.ensure(8 * tt + 16));
  if (needs_true) CUDA_TRY(ctx, N.tru.ensure(4 * tt + 16));
  L.n_client = N.client.as<int32_t>();
  L.n_arrival = N.arrival.as<double>();
  L.n_in = N.in.as<int32_t>();
  L.n_tag = N.tag.as<uint8_t>();
  L.n_true = needs_true ? N.tru.as<int32_t>() : nullptr;
  L.n_id = N.id.as<int64_t>();
  L.n_pred = N.pred.as<int32_t>();
  L.n_bucket = N.bucket.as<uint8_t>();
  L.n_preds = N.preds.as<double>();
  L.n_rfc = N.rfc.as<double>();
  if (n_live > 0) {
    eqx_ctx::Live& O = ctx->live[old];
    L.o_client = O.client.as<int32_t>();
    L.o_arrival = O.arrival.as<double>();
    L.o_in = O.in.as<int32_t>();
    L.o_tag = O.tag.as<uint8_t>();
    L.o_true = needs_true ? O.tru.as<int32_t>() : nullptr;
    L.o_id = O.id.as<int64_t>();
    L.o_pred = O.pred.as<int32_t>();
    L.o_bucket = O.bucket.as<uint8_t>();
    L.o_preds = O.preds.as<double>();
    L.o_rfc = O.rfc.as<double>();
    const int grid = static_cast<int>(std::min<int64_t>((n_live + 255) / 256, 8ll * ctx->sm_count));
    gather_live_kernel<<<grid, 256, 0, s>>>(L);
    CUDA_TRY(ctx, cudaGetLastError());
  }
  if (m > 0) {
    const cudaMemcpyKind k = r->location == EQX_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    CUDA_TRY(ctx, cudaMemcpyAsync(L.n_client + n_live, r->client, 4 * m, k, s));
    CUDA_TRY(ctx, cudaMemcpyAsync(L.n_arrival + n_live, r->arrival_s, 8 * m, k, s));
    CUDA_TRY(ctx, cudaMemcpyAsync(L.n_in + n_live, r->input_tokens, 4 * m, k, s));
    if (r->tag) CUDA_TRY(ctx, cudaMemcpyAsync(L.n_tag + n_live, r->tag, m, k, s));
    else CUDA_TRY(ctx, cudaMemsetAsync(L.n_tag + n_live, 0, m, s));
    if (needs_true) CUDA_TRY(ctx, cudaMemcpyAsync(L.n_true + n_live, r->true_output_tokens, 4 * m, k, s));
    if (r->id) CUDA_TRY(ctx, cudaMemcpyAsync(L.n_id + n_live, r->id, 8 * m, k, s));
    // 3. prediction records against the current profile (drain_arrivals: predict + map_metrics)
    StepPlan pl;
    const bool qr = ctx->queue_ready;
    const int64_t n0 = ctx->n;
    ctx->queue_ready = true;  // plan only: uploads the model tables if they changed
    eqx_status st = step_prepare(ctx, 0.0, pl);
    ctx->queue_ready = qr;
    ctx->n = n0;
    if (st != EQX_OK) return st;
    ScoreArgs sc = pl.sc;
    sc.frozen = Frozen{};
    sc.id_base = r->id_base;
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((m + 255) / 256, 8ll * ctx->sm_count)));
    predict_rows_kernel<<<grid, 256, pl.window_smem, s>>>(sc, n_live, total, L, r->id ? 0 : 1);
    CUDA_TRY(ctx, cudaGetLastError());
  }
  ctx->live_cur = nb;
  ctx->live_mode = true;
  ctx->frozen = Frozen{L.n_pred, L.n_bucket, L.n_preds, L.n_rfc};
  // 4. per-client FIFOs over the new store; the lift treats the remaining counts as non-empty
  //    queues (on_activated only for clients idle before the batch, engine.cpp:182)
  eqx_requests q{};
  q.n = total;
  q.id = L.n_id;
  q.client = L.n_client;
  q.arrival_s = L.n_arrival;
  q.input_tokens = L.n_in;
  q.true_output_tokens = L.n_true;
  q.tag = L.n_tag;
  q.location = EQX_DEVICE;
  eqx_status st = drain_prepare(ctx, &q);
  if (st != EQX_OK) return st;
  ctx->shard_W = 0;
  return drain_enqueue(ctx, true, true);
}

// ---- completion / feedback ------------------------------------------
eqx_status eqx_feedback(eqx_ctx* ctx, const int64_t* tokens, const eqx_completions* done, double ema_alpha) {
  if (ctx) ++ctx->ledger_epoch;  // the published step ledger (eqx_step_ledger) is stale
  if (!ctx) return fail(ctx, EQX_ERR_ARG, "eqx_feedback: NULL context");
  if (!ctx->policy_set || !ctx->profile_set) return fail(ctx, EQX_ERR_CONFIG, "eqx_feedback: policy and profile must be set first");
  const int64_t n = done ? done->n : 0;
  if (n < 0) return fail(ctx, EQX_ERR_ARG, "eqx_feedback: negative completion count");
  if (n > 0 && (ema_alpha <= 0.0 || ema_alpha > 1.0))
    return fail(ctx, EQX_ERR_CONFIG, "ema_alpha must lie in (0, 1]");  // predictor.cpp:374-376
  if (n > 0 && (!done->client || !done->input_tokens || !done->output_tokens || !done->latency_s || !done->tps ||
                !done->gpu_util || !done->pending_ufc || !done->pending_rfc))
    return fail(ctx, EQX_ERR_ARG, "eqx_feedback: missing completion column");
  const int32_t C = ctx->C;
  if (n > 0 && done->location == EQX_HOST)
    for (int64_t i = 0; i < n; ++i)
      if (done->client[i] < 0 || done->client[i] >= C)
        return fail(ctx, EQX_ERR_ENGINE, "completion for unknown client index " + std::to_string(done->client[i]));
  cudaSetDevice(ctx->device);
  cudaStream_t s = ctx->stream;
  FeedbackArgs f;
  std::memset(&f, 0, sizeof(f));
  f.n = n;
  // host columns: one staging block [tokens C][client, in, out n][latency, tps, util, pending x3 n]
  const size_t nn = static_cast<size_t>(n);
  const size_t need = 8ull * C + 12 * nn + 48 * nn + 16 * 12;  // + 16-byte alignment of 10 sections
  CUDA_TRY(ctx, ctx->d_fb.ensure(need));
  char* base = static_cast<char*>(ctx->d_fb.p);
  if (tokens) {
    CUDA_TRY(ctx, cudaMemcpyAsync(base, tokens, 8ull * C, cudaMemcpyHostToDevice, s));
    f.tokens = reinterpret_cast<const int64_t*>(base);
  }
  if (n > 0) {
    if (done->location == EQX_DEVICE) {
      f.client = done->client;
      f.in_tok = done->input_tokens;
      f.out_tok = done->output_tokens;
      f.latency_s = done->latency_s;
      f.tps = done->tps;
      f.util = done->gpu_util;
      f.pend_ufc = done->pending_ufc;
      f.pend_rfc = done->pending_rfc;
      f.pend_vtc = done->pending_vtc;
    } else {
      char* p = base + ((8ull * C + 15) & ~size_t(15));
      auto put = [&](const void* src, size_t bytes) -> const void* {
        if (!src) return nullptr;
        char* d = p;
        p += (bytes + 15) & ~size_t(15);
        return cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, s) == cudaSuccess ? d : nullptr;
      };
      f.client = static_cast<const int32_t*>(put(done->client, 4 * nn));
      f.in_tok = static_cast<const int32_t*>(put(done->input_tokens, 4 * nn));
      f.out_tok = static_cast<const int32_t*>(put(done->output_tokens, 4 * nn));
      f.latency_s = static_cast<const double*>(put(done->latency_s, 8 * nn));
      f.tps = static_cast<const double*>(put(done->tps, 8 * nn));
      f.util = static_cast<const double*>(put(done->gpu_util, 8 * nn));
      f.pend_ufc = static_cast<const double*>(put(done->pending_ufc, 8 * nn));
      f.pend_rfc = static_cast<const double*>(put(done->pending_rfc, 8 * nn));
      f.pend_vtc = static_cast<const double*>(put(done->pending_vtc, 8 * nn));
      if (!f.client || !f.in_tok || !f.out_tok || !f.latency_s || !f.tps || !f.util || !f.pend_ufc || !f.pend_rfc ||
          (done->pending_vtc && !f.pend_vtc))
        return fail(ctx, EQX_ERR_CUDA, "eqx_feedback: completion upload failed");
    }
    if (!f.pend_vtc) {  // only VTC with predictions reads it
      if (ctx->pol.kind == kVtc && ctx->pol.vtc_use_prediction)
        return fail(ctx, EQX_ERR_ARG, "eqx_feedback: pending_vtc is required for vtc+pred");
      f.pend_vtc = f.pend_ufc;
    }
  }
  f.C = C;
  f.ema_alpha = n > 0 ? ema_alpha : 0.0;
  f.weight = ctx->d_weight.as<double>();
  f.ufc = ctx->d_ufc.as<double>();
  f.rfc = ctx->d_rfc.as<double>();
  f.counter = ctx->d_counter.as<double>();
  f.service = ctx->d_service.as<double>();
  f.running = ctx->d_running.as<int32_t>();
  f.model = ctx->d_model.as<ModelTables>();
  f.st = ctx->d_state.as<DevState>();
  f.pol = ctx->pol;
  if (ctx->model_dirty) {  // the device profile must exist before update_map edits it
    StepPlan pl;
    const bool qr = ctx->queue_ready;
    ctx->queue_ready = true;  // step_prepare only uploads the tables here
    const int64_t n0 = ctx->n;
    eqx_status st = step_prepare(ctx, 0.0, pl);
    ctx->queue_ready = qr;
    ctx->n = n0;
    if (st != EQX_OK) return st;
  }
  if (C > 0 || n > 0) feedback_kernel<<<1, 1024, 0, s>>>(f);
  CUDA_TRY(ctx, cudaGetLastError());
  CUDA_TRY(ctx, cudaStreamSynchronize(s));  // host columns may go away
  return EQX_OK;
}

eqx_status eqx_get_service(eqx_ctx* ctx, int32_t n, double* service, int64_t* counter_clamps) {
  if (!ctx || n != ctx->C) return fail(ctx, EQX_ERR_ARG, "eqx_get_service: roster size mismatch");
  cudaSetDevice(ctx->device);
  const Col cols[] = {{service, ctx->d_service.p, 8ull * n},
                      {counter_clamps, reinterpret_cast<char*>(ctx->d_state.p) + offsetof(DevState, clamps), 8}};
  return read_cols(ctx, cols, 2);
}

eqx_status eqx_set_service(eqx_ctx* ctx, int32_t n, const double* service) {
  if (!ctx || n != ctx->C || (n > 0 && !service)) return fail(ctx, EQX_ERR_ARG, "eqx_set_service: roster size mismatch");
  cudaSetDevice(ctx->device);
  if (n > 0) CUDA_TRY(ctx, cudaMemcpyAsync(ctx->d_service.p, service, 8ull * n, cudaMemcpyHostToDevice, ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return EQX_OK;
}

eqx_status eqx_get_profile(eqx_ctx* ctx, int32_t n, double* latency_ms, double* gpu_util, double* tps) {
  if (!ctx || !ctx->profile_set || n != ctx->model.n_prof)
    return fail(ctx, EQX_ERR_ARG, "eqx_get_profile: profile size mismatch");
  cudaSetDevice(ctx->device);
  if (ctx->model_dirty) {  // not uploaded yet: the host copy is current
    for (int e = 0; e < n; ++e) {
      if (latency_ms) latency_ms[e] = ctx->model.prof_lat[e];
      if (gpu_util) gpu_util[e] = ctx->model.prof_util[e];
      if (tps) tps[e] = ctx->model.prof_tps[e];
    }
    return EQX_OK;
  }
  char* m = static_cast<char*>(ctx->d_model.p);
  const size_t b = 8ull * n;
  const Col cols[] = {{latency_ms, m + offsetof(ModelTables, prof_lat), b},
                      {gpu_util, m + offsetof(ModelTables, prof_util), b},
                      {tps, m + offsetof(ModelTables, prof_tps), b}};
  return read_cols(ctx, cols, 3);
}

// ---- client-sharded step ---------------------------------------------------
int64_t eqx_shard_record_bytes(int32_t cmax, int32_t W) {
  if (cmax < 0 || W < 1) return -1;
  return rec_layout(cmax, W).bytes;
}

eqx_status eqx_shard_export_async(eqx_ctx* ctx, double now, int32_t cmax, int32_t W, void* rec) {
  if (ctx) ++ctx->ledger_epoch;  // the published step ledger (eqx_step_ledger) is stale
  if (!ctx || !rec) return fail(ctx, EQX_ERR_ARG, "eqx_shard_export_async: NULL argument");
  if (W < 1) return fail(ctx, EQX_ERR_ARG, "eqx_shard_export_async: window depth must be >= 1");
  if (cmax < ctx->C) return fail(ctx, EQX_ERR_ARG, "eqx_shard_export_async: cmax is smaller than the shard's client count");
  if (reinterpret_cast<uintptr_t>(rec) & 15u) return fail(ctx, EQX_ERR_ARG, "eqx_shard_export_async: record must be 16-byte aligned");
  StepPlan pl;
  eqx_status st = step_prepare(ctx, now, pl);
  if (st != EQX_OK) return st;
  cudaStream_t s = ctx->stream, s2 = ctx->stream2;
  CUDA_TRY(ctx, cudaEventRecord(ctx->ev_fork, s));
  CUDA_TRY(ctx, cudaStreamWaitEvent(s2, ctx->ev_fork, 0));
  CUDA_TRY(ctx, cudaEventRecord(ctx->ev_k[0], s2));
  if (ctx->n > 0) {
    if (pl.score_tma) score_tma_kernel<<<pl.score_grid, kScoreTmaThreads, pl.score_smem, s2>>>(pl.sc);
    else score_kernel<<<pl.score_grid, kScoreThreads, pl.score_smem, s2>>>(pl.sc);
  }
  CUDA_TRY(ctx, cudaGetLastError());
  CUDA_TRY(ctx, cudaEventRecord(ctx->ev_k[1], s2));
  CUDA_TRY(ctx, cudaEventRecord(ctx->ev_join, s2));
  WindowArgs wi = pl.wi;
  wi.W = W;
  const int64_t items = static_cast<int64_t>(cmax) * W;
  if (items > 0) {
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((items + 255) / 256, 8ll * ctx->sm_count)));
    shard_export_kernel<<<grid, 256, pl.window_smem, s>>>(wi, cmax, static_cast<unsigned char*>(rec));
    CUDA_TRY(ctx, cudaGetLastError());
  }
  CUDA_TRY(ctx, cudaStreamWaitEvent(s, ctx->ev_join, 0));
  ctx->stepped = true;
  ctx->shard_W = 0;
  return release_stage(ctx);
}

eqx_status eqx_shard_select_async(eqx_ctx* ctx, const void* recs, int32_t world, int64_t stride,
                                  const int32_t* client_off, int32_t cmax, int32_t W, double now) {
  if (ctx) ++ctx->ledger_epoch;  // the published step ledger (eqx_step_ledger) is stale
  if (!ctx || !recs || !client_off) return fail(ctx, EQX_ERR_ARG, "eqx_shard_select_async: NULL argument");
  if (world < 1 || world > kMaxWorld) return fail(ctx, EQX_ERR_ARG, "eqx_shard_select_async: world size out of range (1..64)");
  if (W < 1 || cmax < 0) return fail(ctx, EQX_ERR_ARG, "eqx_shard_select_async: bad window depth / cmax");
  if (stride < rec_layout(cmax, W).bytes || (stride & 15))
    return fail(ctx, EQX_ERR_ARG, "eqx_shard_select_async: record stride too small or not 16-byte aligned");
  const int32_t C = ctx->C;
  if (client_off[0] != 0 || client_off[world] != C)
    return fail(ctx, EQX_ERR_ARG, "eqx_shard_select_async: client offsets must span [0, C]");
  ShardMap m;
  std::memset(&m, 0, sizeof(m));
  for (int r = 0; r <= world; ++r) {
    if (r > 0 && (client_off[r] < client_off[r - 1] || client_off[r] - client_off[r - 1] > cmax))
      return fail(ctx, EQX_ERR_ARG, "eqx_shard_select_async: client blocks must be ordered and <= cmax");
    m.off[r] = client_off[r];
  }
  m.recs = static_cast<const unsigned char*>(recs);
  m.stride = stride;
  m.world = world;
  m.cmax = cmax;
  m.W = W;
  m.C = C;
  cudaSetDevice(ctx->device);
  const size_t items = static_cast<size_t>(std::max<int64_t>(static_cast<int64_t>(C) * W, 1));
  CUDA_TRY(ctx, ctx->d_first64.ensure(8ull * std::max(C, 1)));
  CUDA_TRY(ctx, ctx->d_gid.ensure(8 * items));
  CUDA_TRY(ctx, ctx->d_ev_row.ensure(4 * items));
  CUDA_TRY(ctx, ctx->d_ev_kind.ensure(4 * items));
  CUDA_TRY(ctx, ctx->d_ev_client.ensure(4 * items));
  CUDA_TRY(ctx, ctx->d_ev_pred.ensure(4 * items));
  CUDA_TRY(ctx, ctx->d_ev_ufc.ensure(8 * items));
  CUDA_TRY(ctx, ctx->d_ev_rfc.ensure(8 * items));
  CUDA_TRY(ctx, ctx->d_ev_vtc.ensure(8 * items));
  CUDA_TRY(ctx, ctx->d_ev_wait.ensure(8 * items));
  CUDA_TRY(ctx, ctx->d_ev_id.ensure(8 * items));
  ctx->ev_cap = static_cast<int64_t>(items);
  ctx->queue_ready = false;  // the selection context holds no local queue
  ctx->n = 0;
  StepPlan pl;
  eqx_status st = step_prepare(ctx, now, pl, W);
  if (st != EQX_OK) return st;
  pl.se.id = ctx->d_gid.as<int64_t>();  // event ids: the gathered heads' global trace positions
  pl.se.id_base = 0;
  cudaStream_t s = ctx->stream;
  ShardSelectBufs b;
  b.count = ctx->d_count.as<int32_t>();
  b.first = ctx->d_first64.as<int64_t>();
  b.head = ctx->d_head.as<int32_t>();
  b.qlen_before = ctx->d_qlen_before.as<int32_t>();
  b.running = ctx->d_running.as<int32_t>();
  b.ufc = ctx->d_ufc.as<double>();
  b.rfc = ctx->d_rfc.as<double>();
  b.counter = ctx->d_counter.as<double>();
  b.backlogged = ctx->d_backlogged.as<int32_t>();
  b.counter_lift = ctx->counter_lift;
  b.win = ctx->d_win.as<WinEntry>();
  b.gid = ctx->d_gid.as<int64_t>();
  b.st = ctx->d_state.as<DevState>();
  if (C > 0) {
    shard_ingest_kernel<<<1, 1024, 0, s>>>(m, b);
    const int grid = static_cast<int>(std::min<int64_t>((static_cast<int64_t>(C) * W + 255) / 256, 8ll * ctx->sm_count));
    shard_unpack_kernel<<<grid, 256, 0, s>>>(m, b);
    CUDA_TRY(ctx, cudaGetLastError());
  }
  CUDA_TRY(ctx, cudaEventRecord(ctx->ev_k[2], s));
  {  // the local scoring joined the stream in eqx_shard_export_async: the selection publishes the
     // summary to the mapped host copy with no wait and no copy kernel behind it
    SelectArgs se = pl.se;
    se.h_st = ctx->h_state_dev;
    void* args[] = {&se};
    CUDA_TRY(ctx, cudaLaunchKernel(select_fn(pl.se.tk_heads != nullptr), dim3(1), dim3(pl.select_threads), args, pl.select_smem, s));
  }
  CUDA_TRY(ctx, cudaEventRecord(ctx->ev_k[3], s));
  CUDA_TRY(ctx, cudaGetLastError());
  ctx->q_id = ctx->d_gid.as<int64_t>();
  ctx->id_base = 0;
  ctx->shard_W = W;
  ctx->step_pending = true;
  ctx->stepped = true;
  return EQX_OK;
}

eqx_status eqx_step_collect(eqx_ctx* ctx, eqx_step_summary* out) {
  if (!ctx) return fail(ctx, EQX_ERR_ARG, "eqx_step_collect: NULL context");
  cudaSetDevice(ctx->device);
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  const DevState& h = *ctx->h_state;
  if (h.bad_client) {
    // the flag is sticky on the device: clear it so the next drain of valid queues succeeds, and
    // end this step (its schedule is void)
    ctx->step_pending = false;
    ctx->h_state->bad_client = 0;
    CUDA_TRY(ctx, cudaMemset(reinterpret_cast<char*>(ctx->d_state.p) + offsetof(DevState, bad_client), 0,
                             sizeof(int32_t)));
    return fail(ctx, EQX_ERR_CONFIG, "request references unknown client index");
  }
  if (out) {
    out->n_events = h.n_events;
    out->n_admitted = h.n_admitted;
    out->n_rejected = h.n_rejected;
    out->new_prefill_tokens = h.new_prefill;
    out->length_fallbacks = static_cast<int64_t>(h.fallbacks - ctx->last_fallbacks);
    out->noisy_near_ties = static_cast<int64_t>(h.near_ties - ctx->last_near_ties);
    out->batch_members = h.members;
    out->batch_reserved_kv_tokens = h.reserved;
    if (ctx->shard_W > 0) {
      out->queued = h.n_queued - h.n_events;
    } else {
      ctx->popped += h.n_events;
      out->queued = ctx->n - ctx->popped;
    }
    out->window_underflow = ctx->shard_W > 0 ? h.underflow : 0;
  }
  ctx->last_fallbacks = h.fallbacks;
  ctx->last_near_ties = h.near_ties;
  ctx->step_pending = false;
  return EQX_OK;
}

eqx_status eqx_phase_times(eqx_ctx* ctx, double* out_us, int32_t n) {
  if (!ctx || !out_us) return fail(ctx, EQX_ERR_ARG, "eqx_phase_times: NULL argument");
  cudaSetDevice(ctx->device);
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  const unsigned long long* t = ctx->h_state->t;
  const double base = static_cast<double>(t[0]);
  for (int i = 0; i < n && i < 6; ++i) out_us[i] = (static_cast<double>(t[i]) - base) * 1e-3;
  for (int i = 6; i < n && i < 16; ++i) out_us[i] = static_cast<double>(t[i]);  // counts / cycles
  const unsigned long long* dt = ctx->h_state->dt;  // EQX_PROF drain timeline (us from hist start)
  for (int i = 16; i < n && i < 22; ++i) out_us[i] = (static_cast<double>(dt[i - 16]) - static_cast<double>(dt[0])) * 1e-3;
  if (n > 22) out_us[22] = (base - static_cast<double>(dt[0])) * 1e-3;  // selection start after drain start
  if (n > 24) {  // window kernel first CTA past its wait / last CTA done, after drain start
    out_us[23] = (static_cast<double>(dt[5]) - static_cast<double>(dt[0])) * 1e-3;
    out_us[24] = (static_cast<double>(dt[6]) - static_cast<double>(dt[0])) * 1e-3;
  }
  if (n > 26) {  // selection epilogue done / last event-fill CTA done, after drain start
    out_us[25] = (static_cast<double>(t[12]) - static_cast<double>(dt[0])) * 1e-3;
    out_us[26] = (static_cast<double>(dt[7]) - static_cast<double>(dt[0])) * 1e-3;
  }
  for (int i = 27; i < n && i < 35; ++i) out_us[i] = static_cast<double>(ctx->h_state->tk[i - 27]);  // raw counters
  return EQX_OK;
}

eqx_status eqx_kernel_times(eqx_ctx* ctx, float* out_ms) {
  if (!ctx || !out_ms) return fail(ctx, EQX_ERR_ARG, "eqx_kernel_times: NULL argument");
  cudaSetDevice(ctx->device);
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  // pairs never recorded (e.g. a replay-only context) read as -1
  for (int i = 0; i < 3; ++i)
    if (cudaEventElapsedTime(&out_ms[i], ctx->ev_k[2 * i], ctx->ev_k[2 * i + 1]) != cudaSuccess) out_ms[i] = -1.0f;
  cudaGetLastError();
  return EQX_OK;
}

eqx_status eqx_step(eqx_ctx* ctx, double now, eqx_step_summary* out) {
  eqx_status st = eqx_step_async(ctx, now);
  if (st != EQX_OK) return st;
  return eqx_step_collect(ctx, out);
}

eqx_status eqx_copy_events(eqx_ctx* ctx, int64_t cap, int64_t* id, int32_t* kind, int32_t* client,
                           int32_t* pred, double* ufc_inc, double* rfc_inc, double* vtc_inc,
                           double* wait_s) {
  if (!ctx || !ctx->stepped) return fail(ctx, EQX_ERR_CONFIG, "eqx_copy_events: no step has run");
  cudaSetDevice(ctx->device);
  cudaStream_t s = ctx->stream;
  CUDA_TRY(ctx, cudaStreamSynchronize(s));
  const int64_t n = std::min<int64_t>(std::min<int64_t>(cap, ctx->h_state->n_events), ctx->ev_cap);
  if (n <= 0) return EQX_OK;
  // request ids were gathered inside the step (the selection): the id column may live in a
  // staging set the copy stream refills once the step released it
  const size_t n8 = 8ull * n, n4 = 4ull * n;
  const Col cols[] = {{id, ctx->d_ev_id.p, n8},        {kind, ctx->d_ev_kind.p, n4},
                      {client, ctx->d_ev_client.p, n4}, {pred, ctx->d_ev_pred.p, n4},
                      {ufc_inc, ctx->d_ev_ufc.p, n8},   {rfc_inc, ctx->d_ev_rfc.p, n8},
                      {vtc_inc, ctx->d_ev_vtc.p, n8},   {wait_s, ctx->d_ev_wait.p, n8}};
  return read_cols(ctx, cols, 8);
}

eqx_status eqx_copy_scores(eqx_ctx* ctx, int64_t cap, int32_t* pred, uint8_t* bucket,
                           double* ufc_inc, double* rfc_inc) {
  if (!ctx || !ctx->stepped) return fail(ctx, EQX_ERR_CONFIG, "eqx_copy_scores: no step has run");
  if (ctx->shard_W > 0)
    return fail(ctx, EQX_ERR_CONFIG, "eqx_copy_scores: a sharded selection context holds no queue (scores live on the ranks' contexts)");
  cudaSetDevice(ctx->device);
  cudaStream_t s = ctx->stream;
  const int64_t n = std::min<int64_t>(cap, ctx->n);
  const size_t nn = n > 0 ? static_cast<size_t>(n) : 0;
  const Col cols[] = {{pred, ctx->d_pred.p, 4 * nn}, {bucket, ctx->d_bucket.p, nn},
                      {ufc_inc, ctx->d_ufc_out.p, 8 * nn}, {rfc_inc, ctx->d_rfc_out.p, 8 * nn}};
  (void)s;
  return read_cols(ctx, cols, 4);
}

// bindings/module.cpp:144-172 scalar helpers (host utilities; not part of the step)
double eqx_ufc_increment(double weight, int32_t in, int32_t pred, double wait_s, double lat_ms,
                         double delta, double ow) {
  const double tokens = static_cast<double>(in) + ow * static_cast<double>(pred);
  const double predict_s = lat_ms / 1000.0;
  return weight * tokens / (1.0 + delta * (wait_s + predict_s));
}

double eqx_rfc_increment(double weight, double tps, double util) { return weight * tps * util; }

}  // extern "C"
