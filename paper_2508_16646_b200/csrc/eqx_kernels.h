// eqx_kernels.h -- kernel entry points and argument blocks (device-side view).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "eqx_device.cuh"
#include "../../include/eqx.h"

namespace eqx {

constexpr int kDrainThreads = 1024;  // 32 warps per tile
// small rosters: tile-local counting sort, one thread per 16 consecutive rows
constexpr int kSortThreads = 512;
constexpr int kSortRows = 16;
constexpr int kSortTile = kSortThreads * kSortRows;  // 8192 rows
constexpr int kSortMaxClients = 128;
__host__ __device__ constexpr int sort_pad(int L) { return L + 2 * (L >> 6); }  // one word per 64 counters
constexpr int kDrainWarps = kDrainThreads / 32;
constexpr int kScoreThreads = 256;
constexpr unsigned long long kScoreCtaOne = 1ull << 40;  // one CTA in score_counts' packed words
constexpr int kScoreTmaThreads = 256;                        // score_tma_kernel block
constexpr int kScoreTile = 1024;                             // requests per bulk-copied tile
constexpr int kScoreStages = 3;                              // tiles in flight per CTA
constexpr int kScoreStageBytes = kScoreTile * (4 + 8 + 4 + 1 + 4);  // columns (+ true_out)
constexpr int kTopkThreads = 512;                           // select_topk_kernel block

// Prediction records frozen when a request joined a live queue (drain_arrivals stores
// map_metrics' PredictionRecord with the request, engine.cpp:178-180): later update_map EMA
// steps do not change them.  pred == nullptr: no live queue (predict at step time).
struct Frozen {
  const int32_t* pred;    // predicted output tokens (after the engine's max(1, .))
  const uint8_t* bucket;  // profile entry
  const double* pred_s;   // predicted_latency_ms / 1000.0 (scheduler.cpp:23)
  const double* rfc;      // rfc_increment(prediction, weight) = (w * tps) * util
};

// One head-of-queue entry as the selection loop consumes it (40 B, shared memory).
struct WinEntry {
  double ufc_inc;
  double rfc_inc;
  uint64_t abits;   // order-preserving bits of arrival_time_s (-0.0 canonicalised to +0.0)
  int32_t in;
  int32_t pred;
  int32_t row;
  int32_t alone;    // fits_alone(in, pred) (gpu_model.cpp:69-72)
};


struct DrainArgs {
  const int32_t* client;
  int32_t n;
  int32_t C;
  int32_t cbits;        // bits of a client key (keys 0..C; C marks rows outside the roster)
  int32_t tile_rows;
  int32_t n_tiles;
  int32_t staged;       // 1: smem-staged coalesced scatter (when the tile fits in smem)
  uint32_t* hist;       // per-tile client counts [n_tiles][C]
  uint32_t* tbase;      // [n_tiles][C] rows of the client in earlier tiles (drain_scan_kernel)
  uint32_t* ctot;       // [C] rows of the client in the batch (drain_scan_kernel)
  uint32_t* tsorted;    // [n] small rosters: each tile's rows sorted by client, (client << 16) | row - t0
  uint32_t* tfirst;     // [n_tiles][C] first row of the client in the tile (0xffffffff: none)
  int32_t* head;        // [C] queue heads, reset by drain_scan_kernel
  int32_t zero_qlen;    // drain_scan_kernel also resets qlen_before (a drain that replaces the queue)
  int64_t hist_L;
  int32_t* seg_off;     // [C+1]
  uint32_t* perm;       // [n] row indices grouped by client, FIFO order
  int32_t* count;       // [C] queued requests per client
  int32_t* first_row;   // [C] first arrival row of the client in this drain
  int32_t* qlen_before;
  const int32_t* running;
  double* ufc;
  double* rfc;
  double* counter;
  int32_t* backlogged;
  int32_t counter_lift;
  unsigned int* done;   // [2] last-CTA counters (hist, rank), reset by their last CTA
  uint16_t* wcnt;       // [n_tiles][kDrainWarps][C] per-warp client counts (hist -> rank)
  DevState* st;
};

struct ScoreArgs {
  Frozen frozen;         // live queue: frozen prediction records (see Frozen)
  int64_t n;
  const int32_t* client;
  const double* arrival;
  const int32_t* in_tok;
  const int32_t* true_out;
  const uint8_t* tag;
  const int64_t* id;
  int64_t id_base;
  const double* weight;
  int32_t* pred_out;
  uint8_t* bucket_out;
  double* ufc_out;
  double* rfc_out;
  DevState* st;
  unsigned long long* done;  // [2] fallback / near-tie totals + CTA counts for the selection's
                             // DevState publication (score_counts), or nullptr
  const ModelTables* model;
  int32_t model_words;  // uint32 words of ModelTables to stage in smem (header + used LUT)
  // Direct tables compiled on the host from the same LUT/profile (bit-identical results):
  //   direct[tag * direct_n + in] = pred | bucket << 16 | fallback << 24  (MoPE/single proxy)
  //   direct[pred]                = bucket                              (oracle / noisy)
  // Inputs outside [0, direct_n) take the interval/profile search.
  const uint32_t* direct;
  int32_t direct_n;
  int32_t direct_words;  // uint32 words of `direct` (staged in shared memory by score_tma_kernel)
  int32_t vec_ok;
  Policy pol;
  double now;
};

// Head windows: the first W queued entries of every client, scored once per step by many
// CTAs (window_kernel) and bulk-loaded into the selection CTA's shared memory.
struct WindowArgs {
  Frozen frozen;         // live queue: frozen prediction records (see Frozen)
  unsigned long long* score_sig;  // [2] the step's score_counts words, zeroed by CTA 0 (or nullptr)
  const double* arrival;
  const int32_t* in_tok;
  const int32_t* true_out;
  const uint8_t* tag;
  const int64_t* id;
  int64_t id_base;
  const uint32_t* perm;
  const int32_t* seg_off;
  const int32_t* count;
  const int32_t* head;
  const double* weight;
  int32_t C;
  int32_t W;
  WinEntry* win;         // [C][W]
  const ModelTables* model;
  int32_t model_words;
  int64_t tmax;
  Policy pol;
  double now;
  DevState* st;          // EQX_PROF timeline stamps (dt[5] window start, dt[6] window end)
  // drain + step: the last CTA runs the drain's counter lift (on_activated / set_backlogged)
  // beside the window entries, off the selection CTA's critical path
  int32_t do_lift, counter_lift;
  const int32_t* qlen_before;
  const int32_t* running;
  const int32_t* first_row;
  double* ufc;
  double* rfc;
  double* counter;
  int32_t* backlogged;
};

struct SelectArgs {
  Frozen frozen;         // live queue: frozen prediction records (see Frozen)
  // queue columns (head entries are scored in-kernel with the same device function)
  const int32_t* client;
  const double* arrival;
  const int32_t* in_tok;
  const int32_t* true_out;
  const uint8_t* tag;
  const int64_t* id;
  int64_t id_base;
  const uint32_t* perm;
  const int32_t* seg_off;
  const int32_t* count;
  int32_t* head;
  int32_t C;
  int32_t W;             // head-window depth per client (window_kernel's [C][W] entries)
  const WinEntry* win_g; // [C][W] windows produced by window_kernel ([C][gW] when gathered)
  int32_t gW;            // > 0: client-sharded step; win_g holds the gathered [C][gW] windows and
                         // a head beyond them raises DevState::underflow instead of reading HBM
  int32_t do_lift;       // run the drain's counter lift / backlog flags first (drain + step)
  int32_t ledger_after_wait;  // the preceding window kernel lifted the ledger: load it after the
                              // programmatic wait
  const int32_t* first_row;
  const int32_t* qlen_before;
  int32_t counter_lift;
  int32_t cw_in_smem;
  void* cw_global;       // per-client work arrays when they do not fit in smem
  // top-K rounds (select_topk_kernel, eqx_topk.cuh)
  int32_t tk_dsh;        // log2 of the largest key-stream depth per client
  int32_t tk_kcap;       // largest K of one round (<= threads)
  int32_t tk_k0;         // K of the first round
  int32_t tk_cap;        // stream items per round
  void* tk_heads;        // [C] head tuples in global scratch (rosters beyond tk_kcap clients whose
                         // tuples do not fit in shared memory; nullptr: shared memory)
  // ledger
  double* ufc;
  double* rfc;
  double* counter;
  const double* weight;
  const uint32_t* order;  // rank of client_id (bytewise), ties by index
  int32_t* running;
  int32_t* backlogged;
  // events
  int32_t* ev_row;
  int32_t* ev_kind;
  int32_t* ev_client;
  int32_t* ev_pred;
  double* ev_ufc;
  double* ev_rfc;
  double* ev_vtc;
  double* ev_wait;
  int64_t* ev_id;
  int64_t ev_cap;
  DevState* st;
  DevState* h_st;        // mapped host copy the epilogue writes the step's DevState to (or nullptr)
  unsigned char* h_ledger;  // mapped host copy of the written-back ledger (eqx_step_ledger layout), or nullptr
  unsigned long long* score_done;  // ... with the scoring's counts from here (ScoreArgs::done)
  int32_t score_ctas;
  const ModelTables* model;
  int32_t model_words;
  int64_t tmax;          // largest T with double(T) * m <= M (exact, host binary search)
  Policy pol;
  double now;
};

// ---- client-sharded step ------------------------------------------------
// One rank's exchange record: for cmax client slots (the rank's clients, padded to the largest
// shard so every rank contributes the same byte count to the all-gather) the drained queue
// length, the trace position (id) of the client's first arrival in the drain, and the first W
// queued requests scored at the step's `now`, with their ids.  16-byte aligned sections.
struct RecLayout {
  int64_t count, first, win, id, bytes;
};
__host__ __device__ inline RecLayout rec_layout(int64_t cmax, int64_t W) {
  auto a16 = [](int64_t x) { return (x + 15) & ~int64_t(15); };
  RecLayout L;
  L.count = 0;
  L.first = a16(4 * cmax);
  L.win = L.first + a16(8 * cmax);
  L.id = L.win + a16(static_cast<int64_t>(sizeof(WinEntry)) * cmax * W);
  L.bytes = L.id + a16(8 * cmax * W);
  return L;
}

constexpr int kMaxWorld = 64;

// The gathered records of `world` ranks: rank r's record at recs + r * stride covers global
// clients [off[r], off[r+1]) (contiguous client_id-rank blocks).
struct ShardMap {
  const unsigned char* recs;
  int64_t stride;
  int32_t world;
  int32_t cmax;
  int32_t W;
  int32_t C;
  int32_t off[kMaxWorld + 1];
};

struct ShardSelectBufs {
  int32_t* count;        // [C]
  int64_t* first;        // [C] trace position of the first arrival
  int32_t* head;         // [C] reset to 0 (cold step)
  int32_t* qlen_before;  // [C] reset to 0 (the drain replaces the queue)
  const int32_t* running;
  double* ufc;
  double* rfc;
  double* counter;
  int32_t* backlogged;
  int32_t counter_lift;
  WinEntry* win;         // [C][W] gathered windows, row = c * W + k
  int64_t* gid;          // [C][W] request ids
  DevState* st;
};

__global__ void shard_export_kernel(WindowArgs a, int32_t cmax, unsigned char* rec);
__global__ void shard_ingest_kernel(ShardMap m, ShardSelectBufs b);
__global__ void shard_unpack_kernel(ShardMap m, ShardSelectBufs b);

// ---- completion / feedback ------------------------------------------
struct FeedbackArgs {
  int64_t n;               // completions, in engine order (complete_finished)
  const int32_t* client;
  const int32_t* in_tok;
  const int32_t* out_tok;
  const double* latency_s;
  const double* tps;
  const double* util;
  const double* pend_ufc;
  const double* pend_rfc;
  const double* pend_vtc;
  const int64_t* tokens;   // [C] on_tokens of one iteration (nullptr: none)
  int32_t C;
  double ema_alpha;        // update_map; <= 0: skip
  const double* weight;
  double* ufc;
  double* rfc;
  double* counter;
  double* service;         // ClientState::accumulated_service
  int32_t* running;
  ModelTables* model;      // the device copy: update_map edits its profile metrics
  DevState* st;
  Policy pol;
};
__global__ void feedback_kernel(FeedbackArgs a);

// Device -> mapped pinned host memory without the DMA engines (a step's results must not
// queue behind the next batch's H2D prefetch on the copy engines).
constexpr int kMaxPackCols = 8;
struct PackCols {
  const void* src[kMaxPackCols];
  void* dst[kMaxPackCols];  // device-side aliases of mapped host memory
  int64_t bytes[kMaxPackCols];
  int32_t n;
};
__global__ void pack_cols_kernel(PackCols p);
// packed arrivals (eqx_pack_arrivals) -> the f64 arrival column, on the copy stream
__global__ void unpack_arrivals_kernel(const unsigned char* pk, int64_t n, double* out);
// u16 host columns (eqx_requests::narrow) -> the i32 client / input_tokens columns, on the copy stream
__global__ void widen_cols_kernel(const uint16_t* c16, const uint16_t* i16, int64_t n, int32_t* c32, int32_t* i32);

// ---- live queues: append arrivals to the remaining queue ------------
struct LiveArgs {
  // remaining rows of the current queue, per client FIFO through perm/seg_off/head/count
  const uint32_t* perm;
  const int32_t* seg_off;
  const int32_t* count;
  const int32_t* head;
  int32_t C;
  int32_t* live_off;      // [C+1] exclusive scan of the remaining counts
  int32_t* qlen_before;   // [C] remaining count (drain_arrivals' "queue non-empty")
  int64_t* n_live;        // total remaining
  // old columns -> new columns (client-grouped remaining rows first)
  const int32_t* o_client; const double* o_arrival; const int32_t* o_in; const uint8_t* o_tag;
  const int32_t* o_true; const int64_t* o_id;
  const int32_t* o_pred; const uint8_t* o_bucket; const double* o_preds; const double* o_rfc;
  int32_t* n_client; double* n_arrival; int32_t* n_in; uint8_t* n_tag; int32_t* n_true; int64_t* n_id;
  int32_t* n_pred; uint8_t* n_bucket; double* n_preds; double* n_rfc;
};
__global__ void live_offsets_kernel(LiveArgs a);
__global__ void gather_live_kernel(LiveArgs a);
// Prediction records of rows [r0, r1) of the new columns (drain_arrivals' predict + map_metrics
// against the current profile); ids default to id_base + (row - r0) when `fill_id`.
__global__ void predict_rows_kernel(ScoreArgs a, int64_t r0, int64_t r1, LiveArgs L, int32_t fill_id);

// ---- batched engine replays (eqx_replay.cu) ---------------------------
constexpr int kMaxReplayClients = 16;  // rosters up to this size keep the ledger in registers /
                                       // local memory; larger ones in global scratch (kBig)
struct ReplayClient {
  double ufc, rfc, counter, weight;
  double service;            // ClientState::accumulated_service
  double bucket, merged;     // service of the current rate window; previous + current window
  int32_t running, backlogged;
  uint32_t order;            // rank of client_id (select_next tie-break)
  int32_t qbase, qhead, qend;  // FIFO over the client's rows: [qhead, qend) of crow
  int32_t skip;              // admit_requests' skipped set (large rosters): stamp of the call
};
struct ReplayMember {
  int32_t row, client, in, generated, reserved_out, pad;
  double admit_s, busy_at, ovh_at;
  double p_ufc, p_rfc, p_vtc;  // PendingContribution
};
struct ReplayArgs {
  int32_t n_replays;
  int32_t C;
  const int64_t* row_off;     // [n_replays + 1] into the concatenated traces
  const int32_t* client;
  const double* arrival;
  const int32_t* in_tok;
  const int32_t* true_out;
  const uint8_t* tag;
  const int64_t* id;
  const double* alpha;        // [n_replays]
  const double* weight;       // [C]
  const uint32_t* order;      // [C]
  const ModelTables* model;
  Policy pol;
  int32_t counter_lift;
  double max_sim_time_s, ema_alpha;
  double prefill_linear_ms, prefill_quad_ms, decode_base_ms, decode_per_ctx_ms, refresh_ms;
  // scratch
  int32_t* crow;
  int32_t* f_pred;
  double* f_preds;
  double* f_rfc;
  ReplayClient* cl;           // [n_replays][C]
  ReplayMember* mb;           // [n_replays][max_batch]
  double* prof;               // [n_replays][4][kMaxProfile]
  // outputs
  int64_t ev_cap;             // per replay
  int64_t* ev_id;
  int32_t* ev_kind;
  double* ev_time;
  int64_t* n_events;
  int64_t* completed;
  double* sim_end;
  int64_t* clamps;
  int32_t* status;            // 0 ok, 2 KV memory bound violated (EngineError)
  double* out_ufc;            // [n_replays][C]
  double* out_rfc;
  double* out_counter;
  // build_report's sweep metrics (metrics.cpp:155-229; experiments.cpp:354-360)
  double* f_ttft;             // [rows] first-token latency per request (-1: none)
  double* jain_ttft_p90;      // [n_replays]
  double* throughput_tps;     // [n_replays]
  // reporting (engine.cpp:379-430, metrics.cpp:151-229)
  double window_s;
  int64_t win_cap;
  double* f_lat;              // [rows] end-to-end latency of completed requests (-1: none)
  eqx_replay_report* report;  // [n_replays]
  eqx_replay_client* rclients;  // [n_replays][C]
  double* win;                // [n_replays][win_cap][4]
  double* win_clients;        // [n_replays][win_cap][C][4]
  double* diff;               // [n_replays][win_cap][2]
  double* rate;               // [n_replays][C][win_cap] (zeroed by the host)
  // ABI 3: horizons, eligibility, caller predictions, the whole event log
  const double* duration;     // [n_replays] Trace::duration_s (nullptr: last arrival)
  double overhead_s;          // prediction_overhead_ms / 1000.0 (engine.cpp:165-168)
  const int32_t* given_pred;  // [rows] Predictor::predict per row (nullptr: the device predictor)
  const uint32_t* by_order;   // [C] client of client_id rank k
  int32_t log_all;
  int32_t* ev_i0;             // [n_replays][ev_cap] payloads (nullptr: not kept)
  double* ev_d0;
  double* ev_d1;
  double* ev_d2;
  double* f_plat;             // [rows] frozen predicted_latency_ms (log_all)
};
template <int KIND, bool kBig>
__global__ void replay_kernel(ReplayArgs a);  // KIND: kFcfs / kVtc / kEquinox; kBig: C > 16

__global__ void drain_hist_kernel(DrainArgs a);
__global__ void lift_kernel(DrainArgs a);
__global__ void drain_scan_kernel(DrainArgs a);
__global__ void drain_sort_kernel(DrainArgs a);     // small rosters: per-tile stable counting sort
__global__ void drain_scatter_kernel(DrainArgs a);  // small rosters: sorted tiles -> perm
__global__ void drain_rank_kernel(DrainArgs a);
__global__ void score_kernel(ScoreArgs a);
__global__ void score_tma_kernel(ScoreArgs a);
__global__ void window_kernel(WindowArgs a);
template <bool kHugeRoster>  // true: head tuples in global scratch (tk_heads != nullptr)
__global__ void select_topk_kernel(SelectArgs a);  // the admission loop as rounds of block-radix top-K (eqx_topk.cuh)

}  // namespace eqx
