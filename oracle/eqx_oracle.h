/*
 * eqx_oracle.h -- TEST INFRASTRUCTURE ONLY (never linked into the product).
 *
 * Plain-C description of one Equinox scheduling step, shared by
 *   - oracle/eqx_oracle.c   : the CPU restatement of the reference algorithm, and
 *   - oracle/ref_step.cpp   : a driver that runs the *reference's own* C++ code
 *                             (compiled from /root/reference/proj/src into oracle/_ref/).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load either library.
 *
 * One "step" = SimulationRun::drain_arrivals (engine.cpp:171-197) over every request in
 * `reqs` (all treated as arrivals at or before `now`, drained in array order) followed by
 * SimulationRun::admit_requests (engine.cpp:207-271) against a pre-existing batch, with a
 * pre-seeded per-client ledger.  This is the "step oracle" of SURVEY.md section 8(c).
 */
#ifndef EQX_ORACLE_H
#define EQX_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { EQXO_FCFS = 0, EQXO_VTC = 1, EQXO_EQUINOX = 2 };           /* scheduler.hpp:66 */
enum { EQXO_NORM_MAX = 0, EQXO_NORM_NONE = 1 };                   /* scheduler.hpp:14 */
enum { EQXO_PRED_ORACLE = 0, EQXO_PRED_MOPE = 1, EQXO_PRED_NOISY = 2,
       EQXO_PRED_SINGLE = 3 };                                     /* predictor.hpp:34-129 */
enum { EQXO_EV_ADMIT = 1, EQXO_EV_REJECT = 2 };                   /* engine.hpp LogEvent */

/* MoPE model tables (predictor.hpp:56-92). keyword rows are addressed by tag id. */
typedef struct {
  int32_t n_thresholds;
  const int32_t* thresholds;      /* RouterModel::input_len_thresholds */
  double mix_weight;              /* RouterModel::mix_weight */
  int32_t num_buckets;            /* RouterModel::num_buckets */
  int32_t n_rows;                 /* keyword_scores rows */
  const double* rows;             /* [n_rows][num_buckets] */
  int32_t n_experts;
  int32_t n_bins;                 /* every expert shares the same bin count */
  const int32_t* bin_upper;       /* [n_experts][n_bins] */
  const int32_t* bin_value;       /* [n_experts][n_bins] */
  const int32_t* out_min;         /* [n_experts] */
  const int32_t* out_max;         /* [n_experts] */
} eqxo_mope;

typedef struct {
  /* policy (scheduler.hpp:18-26, 71-81; engine.hpp:25) */
  int32_t kind;
  double alpha, delta, output_weight;
  int32_t norm_mode;
  int32_t vtc_use_prediction, counter_lift, backfill;
  /* perf (gpu_model.hpp:14-28) */
  int32_t max_batch;
  double mem_per_token_bytes, mem_capacity_bytes;
  /* profile (gpu_model.hpp:61-77) */
  int32_t n_profile;
  const int32_t* prof_upper;
  const double *prof_lat, *prof_util, *prof_tps;
  /* predictor */
  int32_t pred_kind;
  eqxo_mope mope;                 /* MOPE; SINGLE uses expert 0 of it */
  double noisy_l1;                /* NOISY */
  uint64_t noisy_seed;
  /* clients: ledger before the step */
  int32_t n_clients;
  const char* client_names;       /* n_clients NUL-terminated strings, concatenated */
  const double *weight, *ufc0, *rfc0, *counter0;
  const int32_t* running;         /* requests of this client already in the batch */
  /* existing batch (gpu_model.hpp:30-46) */
  int32_t n_members;
  const int32_t *mem_in, *mem_generated, *mem_reserved;
  /* requests, in arrival (= drain) order */
  int64_t n_req;
  const int64_t* id;
  const int32_t* client;
  const double* arrival;
  const int32_t* in_tokens;
  const int32_t* true_out;
  const int32_t* tag;             /* -1 = untagged; else index into tag_names */
  int32_t n_tags;
  const char* tag_names;          /* n_tags NUL-terminated strings (ref driver) */
  const int32_t* tag_row;         /* [n_tags] keyword row for that tag, -1 = unseen */
  double now;
  double duration_s;              /* replays: Trace::duration_s (<= 0: the last arrival) */
  double prediction_overhead_ms;  /* replays: EngineConfig::prediction_overhead_ms */
} eqxo_step_in;

typedef struct {
  /* per request (n_req): the prediction record frozen at drain + increments at `now` */
  int32_t* pred;
  int32_t* bucket;                /* profile entry index */
  double *lat, *util, *tps;
  double *ufc_inc, *rfc_inc;
  /* events in log order (capacity n_req) */
  int64_t n_events;
  int64_t* ev_id;
  int32_t* ev_kind;
  int32_t* ev_client;
  double *ev_ufc_inc, *ev_rfc_inc, *ev_vtc_inc, *ev_wait;  /* PendingContribution */
  /* ledger after the step (n_clients) */
  double *ufc, *rfc, *counter;
  int32_t* backlogged;
  int64_t n_admitted, n_rejected, new_prefill, length_fallbacks;
  double ns_drain, ns_admit;      /* wall time of each phase (timing only) */
} eqxo_step_out;

/* 0 on success; nonzero + message in err on invalid configuration. */
int eqxo_step(const eqxo_step_in* in, eqxo_step_out* out, char* err, int err_len);

/* ---- completion / feedback path ------------------------------------
 * One engine iteration's feedback, in engine order (engine.cpp:273-375): on_tokens for every
 * client with generated tokens (scheduler.cpp:185-190), then for each completion in order
 * on_complete (scheduler.cpp:192-233), running_count decrement (engine.cpp:368) and update_map
 * (predictor.cpp:372-383).  Ledger and profile arrays are updated in place. */
typedef struct {
  int32_t kind;
  double alpha, delta, output_weight;
  int32_t vtc_use_prediction;
  int32_t n_clients;
  const double* weight;
  double *ufc, *rfc, *counter, *service;  /* ClientState::accumulated_service */
  int32_t* running;
  int32_t n_profile;
  const int32_t* prof_upper;
  double *prof_lat, *prof_util, *prof_tps;
  double ema_alpha;
  const int64_t* tokens;                  /* [n_clients] decode tokens of the iteration */
  int64_t n_done;
  const int32_t *client, *in_tokens, *out_tokens;
  const double *latency_s, *tps, *util;
  const double *pend_ufc, *pend_rfc, *pend_vtc; /* PendingContribution of each completion */
  int64_t clamps;                         /* out: counter_clamps() increments */
} eqxo_feedback;

int eqxo_feedback_run(eqxo_feedback* f);

#ifdef __cplusplus
}
#endif
#endif
