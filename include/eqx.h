/*
 * eqx.h -- C ABI of the B200-native Equinox per-step scheduling path (libeqx_b200.so).
 *
 * The reference (arXiv 2508.16646, /root/reference/proj) exposes this path only through C++
 * (`equinox::SchedulerPolicy`, `run_simulation`) and a pybind11 module; it has no C ABI or
 * plugin registry.  These entry points sit *beneath* that API: a host mirror
 * (C++ or Python) drives them exactly where the reference engine runs
 * `SimulationRun::drain_arrivals` (engine.cpp:171-197) and `SimulationRun::admit_requests`
 * (engine.cpp:207-271).  Plain pointers and sizes only; no exceptions cross the ABI; every
 * call returns an eqx_status and leaves a message retrievable with eqx_last_error().
 *
 * Status -> reference exception mapping (errors.hpp:10-31, module.cpp:53-56):
 *   EQX_ERR_CONFIG -> ConfigError (ValueError in Python)     EQX_ERR_PARSE -> ParseError
 *   EQX_ERR_ENGINE -> EngineError (RuntimeError)             EQX_ERR_CUDA  -> EngineError
 *
 * Threading: one context per engine instance, owning one CUDA stream; not thread-safe
 * (scheduler.hpp:97-100).  Several contexts may share a device (replicas).
 */
#ifndef EQX_H
#define EQX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EQX_ABI_VERSION 3

typedef enum {
  EQX_OK = 0,
  EQX_ERR_CONFIG = 1, /* invalid parameter: ConfigError */
  EQX_ERR_PARSE = 2,  /* malformed model/profile tables: ParseError */
  EQX_ERR_ENGINE = 3, /* consistency violation: EngineError */
  EQX_ERR_CUDA = 4,   /* CUDA runtime/driver failure (reported as EngineError) */
  EQX_ERR_ARG = 5     /* NULL/out-of-range argument to this ABI */
} eqx_status;

/* PolicyKind (scheduler.hpp:66), NormMode (scheduler.hpp:14) */
enum { EQX_FCFS = 0, EQX_VTC = 1, EQX_EQUINOX = 2 };
enum { EQX_NORM_MAX_OVER_CLIENTS = 0, EQX_NORM_NONE = 1 };
/* Predictor implementations (predictor.hpp:34-129) */
enum { EQX_PRED_ORACLE = 0, EQX_PRED_MOPE = 1, EQX_PRED_NOISY_ORACLE = 2, EQX_PRED_SINGLE_PROXY = 3 };
/* LogEvent (engine.hpp:33): a step logs admissions and rejections; a replay with log_all set
 * logs the engine's whole event log */
enum { EQX_EV_ADMITTED = 1, EQX_EV_REJECTED = 2, EQX_EV_ARRIVED = 3, EQX_EV_FIRST_TOKEN = 4, EQX_EV_COMPLETED = 5 };
/* where the pointers of an eqx_requests batch live */
enum { EQX_HOST = 0, EQX_DEVICE = 1 };

typedef struct eqx_ctx eqx_ctx;

/* PolicySpec (scheduler.hpp:71-81) + EquinoxParams (scheduler.hpp:18-26)
 * + EngineConfig::backfill (engine.hpp:25). */
typedef struct {
  int32_t kind;
  double alpha, delta, output_weight;
  int32_t norm_mode;
  int32_t vtc_use_prediction;
  int32_t counter_lift;
  int32_t backfill;
} eqx_policy;

/* The admission-control fields of PerfParams (gpu_model.hpp:14-28). */
typedef struct {
  int32_t max_batch;
  double mem_per_token_bytes;
  double mem_capacity_bytes;
} eqx_perf;

/* GpuProfile (gpu_model.hpp:61-77): entries in roster order, bucket_upper per entry. */
typedef struct {
  int32_t n;
  const int32_t* bucket_upper;
  const double* latency_ms;
  const double* gpu_util;
  const double* tps;
} eqx_profile;

/* MopeModel (predictor.hpp:56-92) as flat tables.  keyword_scores rows are addressed through
 * tag_row: request tag id t in [1, n_tags] uses row tag_row[t-1] (-1 = tag unseen by the
 * router -> length fallback, predictor.cpp:43-47); tag id 0 = untagged.  All experts share
 * n_bins (train_mope fits them over shared bins, predictor.cpp:313).  SINGLE_PROXY uses
 * expert 0 (ExpertModel, predictor.hpp:118-129). */
typedef struct {
  int32_t n_thresholds;
  const int32_t* thresholds;
  double mix_weight;
  int32_t num_buckets;
  int32_t n_rows;
  const double* rows; /* [n_rows][num_buckets] */
  int32_t n_experts;
  int32_t n_bins;
  const int32_t* bin_upper; /* [n_experts][n_bins] */
  const int32_t* bin_value; /* [n_experts][n_bins] */
  const int32_t* out_min;   /* [n_experts] */
  const int32_t* out_max;   /* [n_experts] */
  int32_t n_tags;
  const int32_t* tag_row;   /* [n_tags] */
} eqx_mope;

typedef struct {
  int32_t kind;        /* EQX_PRED_* */
  eqx_mope mope;       /* MOPE, SINGLE_PROXY */
  double noisy_l1;     /* NOISY_ORACLE: NoisyOraclePredictor(target_l1, seed) */
  uint64_t noisy_seed;
} eqx_predictor;

/* A batch of queued requests in arrival order (Request, workload.hpp:16-23), struct of arrays.
 * location EQX_DEVICE means every pointer is device memory on the context's device; those
 * arrays are used in place (no copy) and must outlive the queue.  EQX_HOST arrays are copied. */
typedef struct {
  int64_t n;
  const int64_t* id;              /* NULL: id = id_base + row */
  int64_t id_base;
  const int32_t* client;          /* roster index of client_id */
  const double* arrival_s;        /* arrival_time_s, non-decreasing */
  const int32_t* input_tokens;
  const int32_t* true_output_tokens; /* ORACLE / NOISY_ORACLE only; may be NULL otherwise */
  const uint8_t* tag;             /* category_tag as a tag id (see eqx_mope.tag_row) */
  int32_t location;               /* EQX_HOST / EQX_DEVICE */
  int32_t narrow;                 /* ABI 3, EQX_HOST batches of eqx_stage_async / eqx_drain only, bit
                                     flags (0 = every column as typed above):
                                     EQX_NARROW_U16: client and input_tokens point to uint16_t
                                     arrays (rosters up to 65536 clients, inputs below 65536
                                     tokens -- the caller's lossless choice);
                                     EQX_PACKED_ARRIVALS: arrival_s points to the output of
                                     eqx_pack_arrivals for these n rows (about 6 instead of 8
                                     bytes per request, lossless).
                                     Both: 11 instead of 17 bytes per request cross PCIe; the
                                     copy stream widens / unpacks them on the device */
} eqx_requests;

#define EQX_NARROW_U16 1
#define EQX_PACKED_ARRIVALS 2

/* Lossless packing of an arrival_s column for eqx_requests::narrow & EQX_PACKED_ARRIVALS.
 * Layout: the packed size in bytes (u64), then per block of 256 rows a base (u64) and the byte
 * offset of the block's data (u64), then the blocks' data, 16-byte aligned.  A block whose rows
 * are non-negative and non-decreasing with bit patterns within 2^48 of its first row's (about 2 s
 * of arrivals at 40 s: non-negative doubles order like their bit patterns) stores that pattern
 * as the base and each row's offset from it in 6 bytes (little endian).  Any other block (near
 * zero, or a wide span) stores its doubles (base = all ones).
 * out == NULL: returns the packed size of this column.  Otherwise writes it and returns the
 * size, -1 for bad arguments, -2 when cap is smaller than the packed size.  Host-only; no
 * context needed. */
int64_t eqx_pack_arrivals(const double* arrival_s, int64_t n, void* out, int64_t cap);

typedef struct {
  int64_t n_events;          /* admitted + rejected, in log order */
  int64_t n_admitted;
  int64_t n_rejected;
  int64_t new_prefill_tokens; /* admit_requests() return value (engine.cpp:270) */
  int64_t length_fallbacks;   /* MopePredictor::length_fallbacks() over scored requests */
  int64_t noisy_near_ties;    /* NOISY_ORACLE: predictions within 1e-9 of a .5 boundary */
  int32_t batch_members;      /* BatchState::members.size() after the step */
  int64_t batch_reserved_kv_tokens; /* BatchState::reserved_kv_tokens() after the step */
  int64_t queued;             /* requests still queued after the step */
  int32_t window_underflow;   /* sharded step only: a gathered head window ran out -- the
                                 events are not valid; restore the ledger, re-export deeper */
} eqx_step_summary;

/* ---- context ---------------------------------------------------------------------------- */
int32_t eqx_abi_version(void);
eqx_status eqx_ctx_create(int32_t device, eqx_ctx** out);
void eqx_ctx_destroy(eqx_ctx* ctx);
/* Message for the last failing call on ctx (ctx may be NULL for eqx_ctx_create failures). */
const char* eqx_last_error(const eqx_ctx* ctx);
/* The cudaStream_t the context launches on (as void*), for event timing by the caller. */
void* eqx_ctx_stream(eqx_ctx* ctx);
/* The stream host batches are staged on (eqx_stage_async), for timing by the caller. */
void* eqx_ctx_copy_stream(eqx_ctx* ctx);
/* Launch on the caller's cudaStream_t from now on (e.g. the stream a torch.distributed / NCCL
 * collective runs on), so contexts and collectives order without host synchronisation.  The
 * context no longer owns (or destroys) a stream. */
eqx_status eqx_ctx_set_stream(eqx_ctx* ctx, void* stream);

/* ---- configuration (SchedulerPolicy ctor, scheduler.cpp:92-100; validate() :11-17) ------ */
eqx_status eqx_set_policy(eqx_ctx* ctx, const eqx_policy* policy);
eqx_status eqx_set_perf(eqx_ctx* ctx, const eqx_perf* perf);
eqx_status eqx_set_profile(eqx_ctx* ctx, const eqx_profile* profile);
eqx_status eqx_set_predictor(eqx_ctx* ctx, const eqx_predictor* predictor);
/* Client roster + ledger (ClientState, scheduler.hpp:35-43).  names: n NUL-terminated
 * client_id strings concatenated (ties in selection break on their bytes, scheduler.cpp:144).
 * running[c] = requests of client c currently in the batch (engine.cpp:182 running_count_). */
eqx_status eqx_set_clients(eqx_ctx* ctx, int32_t n, const char* names, const double* weight,
                           const double* ufc, const double* rfc, const double* counter,
                           const int32_t* running);
eqx_status eqx_get_clients(eqx_ctx* ctx, int32_t n, double* ufc, double* rfc, double* counter,
                           int32_t* backlogged, int32_t* running);
/* The ledger as the last collected step left it, read from mapped host memory the step's
 * selection CTA wrote it to (no device copy, no synchronisation): same arrays as
 * eqx_get_clients.  Valid after eqx_step_collect of a step on a non-empty queue until the next
 * call that changes the ledger on the device (drain, restore, set_clients, append, feedback,
 * sharded steps, replays); EQX_ERR_CONFIG otherwise. */
eqx_status eqx_step_ledger(eqx_ctx* ctx, int32_t n, double* ufc, double* rfc, double* counter,
                           int32_t* backlogged, int32_t* running);
/* Existing batch: BatchState::members.size() and reserved_kv_tokens() (gpu_model.cpp:40-46). */
eqx_status eqx_set_batch(eqx_ctx* ctx, int32_t members, int64_t reserved_kv_tokens);

/* Device-side snapshot of the ledger (ufc, rfc, counter, running, backlogged) and the batch
 * state, and its asynchronous restore on the context stream (what-if / replica replays). */
eqx_status eqx_ledger_checkpoint(eqx_ctx* ctx);
eqx_status eqx_ledger_restore_async(eqx_ctx* ctx);

/* Pinned host arena for request columns: 2 MiB-aligned, MADV_HUGEPAGE-backed and registered
 * with the driver, so the staging DMA walks huge pages (a steady ~54 GB/s H2D on a B200 box,
 * where cudaHostAlloc'd buffers measured 18-49 GB/s depending on the allocation).  Returns NULL
 * on failure.  Free with eqx_host_free; no context needed. */
void* eqx_host_alloc(int64_t bytes);
eqx_status eqx_host_free(void* p);

/* ---- the hot path ------------------------------------------------------------------------ */
/* Prefetch a HOST batch: its H2D copy runs on the context's copy stream into the next of three
 * device staging buffers, overlapping whatever the context is computing (a serving loop keeps
 * up to two batches staged ahead of the step it collects).  A later eqx_drain /
 * eqx_drain_step_async of the same batch (same pointers and n) uses the staged copy.  Host
 * buffers should be pinned for the copy to be asynchronous; they must stay unchanged until
 * that drain.  A step's results stay readable until the batch after next is drained. */
eqx_status eqx_stage_async(eqx_ctx* ctx, const eqx_requests* arrivals);
/* drain_arrivals (engine.cpp:171-197) for a whole batch of arrivals: the batch becomes the
 * per-client FIFO queues (client-grouped index in HBM), clients that go idle -> backlogged get
 * the counter lift (on_activated, scheduler.cpp:235-253) in arrival order, and every
 * arriving client is marked backlogged.  Replaces any previously queued requests. */
eqx_status eqx_drain(eqx_ctx* ctx, const eqx_requests* arrivals);
/* admit_requests (engine.cpp:207-271) at simulated time `now`, plus per-request scoring of the
 * whole queue: MoPE gate+experts -> map_metrics -> ufc/rfc increments (the prediction
 * record as of drain).  Enqueued on the context stream; results stay on the device. */
eqx_status eqx_step_async(eqx_ctx* ctx, double now);
/* eqx_drain + eqx_step_async in one call.  For a resident queue (EQX_DEVICE columns) the
 * whole launch sequence is captured once into a CUDA graph and replayed while every launch
 * parameter (pointers, sizes, policy, `now`) is unchanged. */
eqx_status eqx_drain_step_async(eqx_ctx* ctx, const eqx_requests* arrivals, double now);
/* Waits for the last step and returns its summary. */
eqx_status eqx_step_collect(eqx_ctx* ctx, eqx_step_summary* out);
/* Convenience: eqx_step_async + eqx_step_collect. */
eqx_status eqx_step(eqx_ctx* ctx, double now, eqx_step_summary* out);

/* ---- batched engine replays (config 5, the alpha sweep) ---------------
 * run_simulation (engine.cpp:119-146) for many independent traces at once, one replay per
 * GPU warp, with the context's policy / perf / timing / profile / predictor / roster and a
 * per-replay EquinoxParams::alpha.  Each replay starts from zero ledgers (engine.cpp:148-157)
 * and its own copy of the profile.  Rosters of any size (one warp per replay; rosters beyond 16
 * clients keep the ledger in global scratch).  The
 * reporting side runs on the device too: the engine's window samples (advance_clock /
 * emit_window_samples, engine.cpp:379-430) and build_report (metrics.cpp:151-229) with the
 * policy's output_weight and report_window_s as its window. */
typedef struct {
  int32_t n_replays;
  const int64_t* row_off;            /* [n_replays + 1], row_off[0] = 0: rows of replay r */
  const int32_t* client;             /* concatenated traces, each in arrival order */
  const double* arrival_s;
  const int32_t* input_tokens;
  const int32_t* true_output_tokens;
  const uint8_t* tag;                /* may be NULL (untagged) */
  const int64_t* id;                 /* may be NULL: trace positions within each replay */
  const double* alpha;               /* [n_replays] */
  double max_sim_time_s;             /* <= 0: each trace's last arrival */
  double ema_alpha;                  /* EngineConfig::ema_alpha (update_map) */
  int64_t ev_cap;                    /* admitted / rejected events kept per replay */
  double report_window_s;            /* EngineConfig::report_window_s; <= 0: 1.0 (default) */
  int64_t win_cap;                   /* window samples kept per replay in the series outputs */
  /* ABI 3 */
  const double* duration_s;          /* [n_replays] Trace::duration_s, the horizon when
                                        max_sim_time_s <= 0 (engine.cpp:120-121); NULL: each
                                        trace's last arrival */
  double prediction_overhead_ms;     /* EngineConfig::prediction_overhead_ms: a request is
                                        eligible at arrival + overhead / 1000 (engine.cpp:165-168) */
  const int32_t* predicted;          /* optional [rows]: Predictor::predict(req) of every row, made by
                                        the caller's predictor (the engine applies max(1, .)); NULL:
                                        the context's predictor on the device */
  int32_t log_all;                   /* 1: ev_* is the engine's whole log (EventLog, engine.hpp:
                                        36-57) -- arrived / admitted / first_token / completed /
                                        rejected, with payloads in ev_i0 / ev_d0..2 */
} eqx_replays;

/* build_report's SimReport summary (metrics.hpp:63-81) + the SimResult totals of one replay. */
typedef struct {
  double max_diff, avg_diff, var_diff; /* service_difference over report windows (C >= 2) */
  double jain_hf;                      /* Jain index of final_hf (metric_hf over all clients) */
  double jain_ttft_p90;                /* Jain index of the per-client p90 TTFT */
  double throughput_tps;               /* completed (in + out) tokens per second */
  double mean_gpu_util;                /* busy_ms_total / (sim_end_s * 1000) */
  double ttft_p50, ttft_p90;           /* nearest-rank percentiles over all first tokens */
  double latency_p50, latency_p90;     /* ... over completed requests' end-to-end latency */
  int64_t ttft_count, latency_count;
  double sim_end_s, busy_ms_total, overhead_ms_total;
  int64_t completed, rejected, total_completed_tokens;
  int64_t n_windows;                   /* engine window samples (gpu_series / counter_series) */
  int64_t n_diff;                      /* service-difference samples (diff_series) */
  int64_t n_rate;                      /* service-rate windows per client */
  int64_t max_resident_kv_tokens;      /* SimResult::max_resident_kv_tokens (with status 2: the
                                          resident tokens that exceeded the capacity) */
  int64_t drained;                     /* requests that entered the queues (drain_arrivals) */
} eqx_replay_report;

/* ClientReport (metrics.hpp:55-60) + the final reporting HF of one client of one replay. */
typedef struct {
  double final_hf;
  double accumulated_service;
  double mean_service_rate;
  double ttft_p50, ttft_p90;
  int64_t ttft_count;
  int64_t backlogged;                  /* ClientState::backlogged at the end of the run (ABI 3) */
} eqx_replay_client;

typedef struct {                     /* host arrays; any may be NULL */
  int64_t* n_events;                 /* [n_replays] (may exceed ev_cap) */
  int64_t* ev_id;                    /* [n_replays][ev_cap] */
  int32_t* ev_kind;                  /* EQX_EV_* */
  double* ev_time;                   /* LogEntry::time_s */
  double *ufc, *rfc, *counter;       /* [n_replays][C] SimResult::final_clients */
  int64_t* completed;                /* SimResult::completed */
  double* sim_end;                   /* SimResult::sim_end_s */
  int64_t* counter_clamps;
  int32_t* status;                   /* 0 ok; 2: KV memory bound violated (EngineError) */
  double* jain_ttft_p90;             /* build_report: Jain index of per-client p90 TTFT */
  double* throughput_tps;            /* build_report: completed (in + out) tokens per second */
  eqx_replay_report* report;         /* [n_replays] */
  eqx_replay_client* clients;        /* [n_replays][C], roster order */
  double* win;                       /* [n_replays][win_cap][4] time, busy_ms, overhead_ms, gpu_util */
  double* win_clients;               /* [n_replays][win_cap][C][4] ufc, rfc, hf, service_cum */
  double* diff;                      /* [n_replays][win_cap][2] time, max-min service */
  double* rate;                      /* [n_replays][C][win_cap] service rate of window w
                                        (time = window_s * (w + 1)) */
  /* ABI 3: event payloads ([n_replays][ev_cap]; LogEntry fields, engine.hpp:39-51).
   *   arrived / rejected: ev_i0 = input_tokens; ev_time = arrival_time_s for arrivals
   *   admitted:  ev_i0 = predicted_output_tokens, ev_d0 = predicted_latency_ms
   *   completed: ev_i0 = output_tokens, ev_d0 = latency_s, ev_d1 = tps, ev_d2 = gpu_util */
  int32_t* ev_i0;
  double *ev_d0, *ev_d1, *ev_d2;
  double* profile;                   /* [n_replays][3][n_profile]: SimResult::profile after the
                                        update_map feedback -- latency_ms, gpu_util, tps */
} eqx_replay_out;

/* PerfParams timing fields (gpu_model.hpp:14-28) used by replays. */
eqx_status eqx_set_timing(eqx_ctx* ctx, double prefill_linear_ms, double prefill_quad_ms, double decode_base_ms,
                          double decode_per_ctx_ms, double refresh_ms);
eqx_status eqx_replay(eqx_ctx* ctx, const eqx_replays* replays, eqx_replay_out* out);

/* ---- request traces (the trace formats) --------------------------------
 * load_trace (workload.cpp:312-400) -- the reference's CSV format with its validation and
 * ParseError messages ("trace line N: ..."), stable re-sort of out-of-order rows (one warning),
 * client roster in first-appearance order -- plus write_trace_csv / trace_hash (FNV-1a of the
 * canonical CSV, 16 hex digits; workload.cpp:405-428) and a binary struct-of-arrays format that
 * records the hash and loads straight into the pinned host arena (eqx_host_alloc).  Columns are
 * the eqx_requests layout: pass them to eqx_stage_async / eqx_drain as EQX_HOST columns.
 * Errors: EQX_ERR_PARSE with the reference's message in err (ParseError). */
typedef struct eqx_trace eqx_trace;
typedef struct {
  int64_t n;
  int32_t n_clients, n_tags, n_warnings;
  int32_t pinned;                    /* columns live in the pinned host arena */
  double duration_s;                 /* last arrival (Trace::duration_s) */
  const int32_t* client;             /* roster index, arrival order */
  const double* arrival_s;
  const int32_t* input_tokens;
  const int32_t* output_tokens;      /* true_output_tokens */
  const int32_t* tag;                /* index into tag_names; -1 = untagged */
  const char* client_names;          /* n_clients NUL-terminated client_id strings */
  const char* tag_names;             /* n_tags NUL-terminated category_tag strings */
  const char* warnings;              /* n_warnings NUL-terminated strings */
  char stored_hash[17];              /* hash recorded in a binary trace ("" for CSV) */
} eqx_trace_view;
eqx_status eqx_trace_load_csv(const char* path, eqx_trace** out, char* err, int32_t err_len);
eqx_status eqx_trace_load_bin(const char* path, eqx_trace** out, char* err, int32_t err_len);
eqx_status eqx_trace_create(int64_t n, const int32_t* client, const double* arrival_s, const int32_t* input_tokens,
                            const int32_t* output_tokens, const int32_t* tag, int32_t n_clients,
                            const char* client_names, int32_t n_tags, const char* tag_names, eqx_trace** out);
eqx_status eqx_trace_view_get(eqx_trace* t, eqx_trace_view* v);
eqx_status eqx_trace_hash(eqx_trace* t, char out[17]);
eqx_status eqx_trace_save_csv(eqx_trace* t, const char* path);
eqx_status eqx_trace_save_bin(eqx_trace* t, const char* path);
void eqx_trace_free(eqx_trace* t);

/* ---- live queues ------------------------------------------------------
 * drain_arrivals (engine.cpp:171-197) for a batch of arrivals that joins the requests still
 * queued (unlike eqx_drain, which replaces the queue): each arrival's prediction record is made
 * now against the current profile and frozen with it (update_map later does not change it),
 * clients idle before the batch (empty queue, no running requests) get on_activated in arrival
 * order, every arriving client becomes backlogged.  Then eqx_step_async / eqx_step schedule
 * from the live queue, repeatedly; eqx_feedback between steps.  ids default to id_base + i. */
eqx_status eqx_append(eqx_ctx* ctx, const eqx_requests* arrivals);

/* ---- completion / feedback -------------------------------------------
 * A batch of completed requests, in the engine's completion order (complete_finished,
 * engine.cpp:327-375): RequestActuals (scheduler.hpp:89-95) plus the PendingContribution the
 * admission registered (scheduler.hpp:131-138; the event payloads of eqx_copy_events). */
typedef struct {
  int64_t n;
  const int32_t* client;          /* roster index */
  const int32_t* input_tokens;
  const int32_t* output_tokens;   /* RequestActuals::output_tokens */
  const double* latency_s;
  const double* tps;
  const double* gpu_util;
  const double* pending_ufc;
  const double* pending_rfc;
  const double* pending_vtc;      /* VTC with predictions only; may be NULL otherwise */
  int32_t location;               /* EQX_HOST / EQX_DEVICE */
} eqx_completions;

/* One engine iteration's feedback, in the reference's order: on_tokens for every client with
 * tokens[c] > 0 (scheduler.cpp:185-190; tokens may be NULL), then for each completion
 * on_complete (scheduler.cpp:192-233), the running-count decrement (engine.cpp:368) and
 * update_map with ema_alpha (predictor.cpp:372-383) on the context's profile, which later
 * drains map against.  done may be NULL. */
eqx_status eqx_feedback(eqx_ctx* ctx, const int64_t* tokens, const eqx_completions* done, double ema_alpha);
/* ClientState::accumulated_service per client and SchedulerPolicy::counter_clamps(). */
eqx_status eqx_get_service(eqx_ctx* ctx, int32_t n, double* service, int64_t* counter_clamps);
eqx_status eqx_set_service(eqx_ctx* ctx, int32_t n, const double* service);
/* The profile metrics as update_map left them (GpuProfile entries in roster order). */
eqx_status eqx_get_profile(eqx_ctx* ctx, int32_t n, double* latency_ms, double* gpu_util, double* tps);

/* ---- client-sharded step over several GPUs ------------------------------
 * The queue shards by client: rank r owns the contiguous client_id-rank block
 * [client_off[r], client_off[r+1]) of the global roster and every queued request of those
 * clients (ids must be global trace positions, the reference's arrival order,
 * workload.cpp:235-237).  Per step:
 *   1. each rank: eqx_drain (its requests, local client indices) then eqx_shard_export_async,
 *      which scores the whole local queue and writes the rank's exchange record -- queue
 *      length, first-arrival trace position and the first W queued requests of each of its
 *      clients (scored at `now`, with ids) -- into device memory `rec`;
 *   2. all-gather the records (ncclAllGather / torch.distributed.all_gather_into_tensor);
 *   3. every rank: eqx_shard_select_async on a context holding the *global* roster and a
 *      replicated ledger -- it applies the drain's backlog flags and counter lift in global
 *      arrival order (on_activated, scheduler.cpp:235-253) and runs admit_requests
 *      (engine.cpp:207-271) over the gathered heads.  All ranks compute the same schedule with
 *      no further exchange.  A client that would need a head beyond W sets
 *      eqx_step_summary.window_underflow: restore the ledger (eqx_ledger_restore_async) and
 *      repeat with a larger W.  W = free batch slots + 1 never underflows without rejections.
 * Records are rec_bytes = eqx_shard_record_bytes(cmax, W) bytes, cmax = the largest block. */
int64_t eqx_shard_record_bytes(int32_t cmax, int32_t W);
eqx_status eqx_shard_export_async(eqx_ctx* ctx, double now, int32_t cmax, int32_t W, void* rec);
/* recs: device pointer to `world` records, rank r's at recs + r * stride; client_off: host
 * array of world + 1 offsets.  Events: eqx_copy_events (ids are the global trace ids). */
eqx_status eqx_shard_select_async(eqx_ctx* ctx, const void* recs, int32_t world, int64_t stride,
                                  const int32_t* client_off, int32_t cmax, int32_t W, double now);

/* ---- results (host copies; any pointer may be NULL) ------------------------------------- */
/* Event log of the last step in order: request id, EQX_EV_*, client, predicted output tokens
 * and the PendingContribution of admissions (scheduler.hpp:131-138: ufc/rfc/vtc increment and
 * ScheduleContext::wait_s); rejections carry zeros. */
eqx_status eqx_copy_events(eqx_ctx* ctx, int64_t cap, int64_t* id, int32_t* kind,
                           int32_t* client, int32_t* pred, double* ufc_inc, double* rfc_inc,
                           double* vtc_inc, double* wait_s);
/* Per-request scores of the queue (row order of the drained batch): predicted output tokens,
 * profile bucket, ufc_increment and rfc_increment at the step's `now`. */
eqx_status eqx_copy_scores(eqx_ctx* ctx, int64_t cap, int32_t* pred, uint8_t* bucket,
                           double* ufc_inc, double* rfc_inc);

/* Profiling: phase timestamps of the last step in microseconds relative to the selection
 * CTA's start: [0] 0, [1] head windows filled, [2] selection loop start, [3] loop end,
 * [4] first scoring CTA start, [5] last scoring CTA end. */
eqx_status eqx_phase_times(eqx_ctx* ctx, double* out_us, int32_t n);

/* Profiling: CUDA-event durations (ms) of the last non-graph step: [0] score_kernel (side
 * stream), [1] select_kernel (or the last eqx_replay's replay_kernel), [2] drain launched
 * inside eqx_drain_step_async; -1 for a pair never recorded. */
eqx_status eqx_kernel_times(eqx_ctx* ctx, float* out_ms);

/* ---- host scalar utilities (bindings/module.cpp:144-172 `ufc_increment`/`rfc_increment`) - */
double eqx_ufc_increment(double weight, int32_t input_tokens, int32_t predicted_output_tokens,
                         double wait_s, double predicted_latency_ms, double delta,
                         double output_weight);
double eqx_rfc_increment(double weight, double tps, double gpu_util);

#ifdef __cplusplus
}
#endif
#endif /* EQX_H */
