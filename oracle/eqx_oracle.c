/*
 * eqx_oracle.c -- TEST INFRASTRUCTURE ONLY: CPU restatement of the reference's per-step
 * scheduling path, used by tests/ (as the checker), __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg.  It is never linked into or called by the product.
 *
 * Parity is pinned two ways:
 *   1. tests/test_oracle.py checks this file against the reference's own compiled code
 *      (oracle/_ref/libeqx_ref.so, built from /root/reference/proj/src) on seeded traces, and
 *   2. against the committed golden vectors in tests/golden/ produced by that same library
 *      (oracle/gen_golden.py) plus the reference unit-test known answers.
 *
 * Every function cites the reference lines it restates.  Arithmetic is FP64 in the
 * reference's exact operation order; the Makefile builds with -ffp-contract=off so no FMA is
 * formed (the reference's CMake sets no -march).
 */
#include "eqx_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ---- rng.hpp:13-75 (SplitMix64, FNV-1a, keyed streams) ------------------------------- */
static uint64_t splitmix_next(uint64_t* state) {
  *state += 0x9e3779b97f4a7c15ULL;
  uint64_t z = *state;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

static uint64_t fnv1a(const char* s) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (; *s; ++s) {
    h ^= (unsigned char)*s;
    h *= 0x100000001b3ULL;
  }
  return h;
}

static uint64_t mix_keys(uint64_t a, uint64_t b) {
  uint64_t z = a + 0x9e3779b97f4a7c15ULL * (b + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* ---- predictor.cpp:17-23  NoisyOraclePredictor::predict (+ rng.hpp:44-48 laplace) ---- */
static int noisy_predict(double l1, uint64_t seed, int64_t id, int true_out) {
  uint64_t st = mix_keys(mix_keys(seed, fnv1a("noisy_oracle")), (uint64_t)id);
  const double u = ((double)(splitmix_next(&st) >> 11) + 0.5) * 0x1.0p-53 - 0.5;
  const double mag = -log1p(-2.0 * fabs(u));
  const double noise = u < 0 ? -l1 * mag : l1 * mag;
  const double predicted = round((double)true_out + noise);
  return (int)(predicted > 1.0 ? predicted : 1.0);
}

/* ---- predictor.cpp:29-34  RouterModel::length_bucket --------------------------------- */
static int length_bucket(const eqxo_mope* m, int in) {
  for (int i = 0; i < m->n_thresholds; ++i)
    if (in <= m->thresholds[i]) return i;
  return m->num_buckets - 1;
}

/* ---- predictor.cpp:36-60  route(); returns bucket, sets *fallback -------------------- */
static int route(const eqxo_mope* m, int in, int row, int* fallback) {
  const int len_bucket = length_bucket(m, in);
  if (row < 0) { /* tag empty or not in keyword_scores */
    *fallback = 1;
    return len_bucket;
  }
  *fallback = 0;
  const double* aff = m->rows + (size_t)row * (size_t)m->num_buckets;
  int bucket = 0;
  double best = -1.0;
  for (int b = 0; b < m->num_buckets; ++b) {
    const double length_score = b == len_bucket ? 1.0 : 0.0;
    const double score = m->mix_weight * length_score + (1.0 - m->mix_weight) * aff[b];
    if (score > best) { /* ties keep the shorter bucket */
      best = score;
      bucket = b;
    }
  }
  return bucket;
}

/* ---- predictor.cpp:62-71  ExpertModel::predict --------------------------------------- */
static int expert_predict(const eqxo_mope* m, int e, int in) {
  const int32_t* up = m->bin_upper + (size_t)e * (size_t)m->n_bins;
  const int32_t* val = m->bin_value + (size_t)e * (size_t)m->n_bins;
  int idx = m->n_bins - 1;
  for (int i = 0; i < m->n_bins; ++i) {
    if (in <= up[i]) {
      idx = i;
      break;
    }
  }
  int v = val[idx]; /* std::clamp(v, out_min, out_max) */
  if (v < m->out_min[e]) v = m->out_min[e];
  else if (m->out_max[e] < v) v = m->out_max[e];
  return v;
}

/* ---- gpu_model.cpp:74-80  GpuProfile::entry_for -------------------------------------- */
static int entry_for(const eqxo_step_in* in, int out_tokens) {
  for (int e = 0; e < in->n_profile; ++e)
    if (out_tokens <= in->prof_upper[e]) return e;
  return in->n_profile - 1;
}

/* ---- scheduler.cpp:19-27  ufc_increment ---------------------------------------------- */
static double ufc_increment(int in_tokens, int pred, double wait_s, double lat_ms, double w,
                            double delta, double ow) {
  const double tokens = (double)in_tokens + ow * (double)pred;
  const double predict_s = lat_ms / 1000.0;
  return w * tokens / (1.0 + delta * (wait_s + predict_s));
}

/* ---- scheduler.cpp:29-31  rfc_increment ---------------------------------------------- */
static double rfc_increment(double tps, double util, double w) { return w * tps * util; }

/* ---- gpu_model.cpp:58-72  can_fit / fits_alone (reserved_kv_tokens :40-46 tracked) ---- */
static int can_fit(int64_t members, int64_t reserved, int in_tokens, int pred,
                   const eqxo_step_in* in) {
  if ((int)members + 1 > in->max_batch) return 0;
  const double claimed = (double)(reserved + in_tokens + pred);
  return claimed * in->mem_per_token_bytes <= in->mem_capacity_bytes;
}

typedef struct {
  double ufc, rfc, counter;
  int backlogged;
} ledger_t;

/* ---- scheduler.cpp:235-253  on_activated (counter lift) ----------------------------- */
static void on_activated(ledger_t* L, int n, int client, int counter_lift) {
  if (!counter_lift) return;
  double min_ufc = INFINITY, min_rfc = INFINITY, min_counter = INFINITY;
  int any = 0;
  for (int i = 0; i < n; ++i) {
    if (i == client || !L[i].backlogged) continue;
    any = 1;
    min_ufc = L[i].ufc < min_ufc ? L[i].ufc : min_ufc; /* std::min(a, b): b < a ? b : a */
    min_rfc = L[i].rfc < min_rfc ? L[i].rfc : min_rfc;
    min_counter = L[i].counter < min_counter ? L[i].counter : min_counter;
  }
  if (!any) return;
  /* std::max(a, b) returns a unless a < b */
  if (L[client].ufc < min_ufc) L[client].ufc = min_ufc;
  if (L[client].rfc < min_rfc) L[client].rfc = min_rfc;
  if (L[client].counter < min_counter) L[client].counter = min_counter;
}

/* byte-wise std::string operator< (char_traits<char>::compare == memcmp semantics) */
static int str_less(const char* a, const char* b) {
  const size_t la = strlen(a), lb = strlen(b);
  const int c = memcmp(a, b, la < lb ? la : lb);
  return c < 0 || (c == 0 && la < lb);
}

int eqxo_step(const eqxo_step_in* in, eqxo_step_out* out, char* err, int err_len) {
  const int C = in->n_clients;
  const int64_t N = in->n_req;
#define FAIL(msg)                                   \
  do {                                              \
    if (err && err_len > 0) snprintf(err, (size_t)err_len, "%s", msg); \
    return 1;                                       \
  } while (0)
  /* scheduler.cpp:11-17 EquinoxParams::validate; :92-100 weights; gpu_model.cpp validate */
  if (in->alpha < 0.0 || in->alpha > 1.0) FAIL("alpha must lie in [0, 1]");
  if (in->delta < 0.0) FAIL("delta must be >= 0");
  if (in->output_weight <= 0.0) FAIL("output_weight must be > 0");
  for (int c = 0; c < C; ++c)
    if (in->weight[c] <= 0.0) FAIL("client has non-positive weight");
  if (in->n_profile < 1) FAIL("profile lookup on empty GpuProfile");

  const char** names = (const char**)malloc(sizeof(char*) * (size_t)(C > 0 ? C : 1));
  {
    const char* p = in->client_names;
    for (int c = 0; c < C; ++c) {
      names[c] = p;
      p += strlen(p) + 1;
    }
  }
  ledger_t* L = (ledger_t*)calloc((size_t)(C > 0 ? C : 1), sizeof(ledger_t));
  for (int c = 0; c < C; ++c) {
    L[c].ufc = in->ufc0[c];
    L[c].rfc = in->rfc0[c];
    L[c].counter = in->counter0[c];
  }
  int32_t* running = (int32_t*)malloc(sizeof(int32_t) * (size_t)(C > 0 ? C : 1));
  memcpy(running, in->running, sizeof(int32_t) * (size_t)C);

  /* per-client FIFO queues as index lists in drain order */
  int64_t* qoff = (int64_t*)calloc((size_t)C + 1, sizeof(int64_t));
  for (int64_t r = 0; r < N; ++r) qoff[in->client[r] + 1]++;
  for (int c = 0; c < C; ++c) qoff[c + 1] += qoff[c];
  int64_t* qidx = (int64_t*)malloc(sizeof(int64_t) * (size_t)(N > 0 ? N : 1));
  int64_t* fill = (int64_t*)calloc((size_t)(C > 0 ? C : 1), sizeof(int64_t));
  int64_t* head = (int64_t*)calloc((size_t)(C > 0 ? C : 1), sizeof(int64_t));
  int64_t* tail = (int64_t*)calloc((size_t)(C > 0 ? C : 1), sizeof(int64_t));

  /* ---- engine.cpp:171-197 drain_arrivals ---- */
  int64_t fallbacks = 0;
  for (int64_t r = 0; r < N; ++r) {
    const int c = in->client[r];
    int p;
    switch (in->pred_kind) {
      case EQXO_PRED_ORACLE: p = in->true_out[r]; break; /* predictor.hpp:34-38 */
      case EQXO_PRED_NOISY: p = noisy_predict(in->noisy_l1, in->noisy_seed, in->id[r], in->true_out[r]); break;
      case EQXO_PRED_SINGLE: p = expert_predict(&in->mope, 0, in->in_tokens[r]); break;
      default: { /* predictor.cpp:355-360 MopePredictor::predict */
        int fb = 0;
        const int row = in->tag[r] >= 0 ? in->tag_row[in->tag[r]] : -1;
        const int b = route(&in->mope, in->in_tokens[r], row, &fb);
        fallbacks += fb;
        p = expert_predict(&in->mope, b, in->in_tokens[r]);
      }
    }
    if (p < 1) p = 1; /* engine.cpp:179 std::max(1, predict) */
    const int e = entry_for(in, p); /* predictor.cpp:362-370 map_metrics */
    out->pred[r] = p;
    out->bucket[r] = e;
    out->lat[r] = in->prof_lat[e];
    out->util[r] = in->prof_util[e];
    out->tps[r] = in->prof_tps[e];
    const double w = in->weight[c];
    out->ufc_inc[r] = ufc_increment(in->in_tokens[r], p, in->now - in->arrival[r], out->lat[r], w,
                                    in->delta, in->output_weight);
    out->rfc_inc[r] = rfc_increment(out->tps[r], out->util[r], w);
    if (head[c] == tail[c] && running[c] == 0) on_activated(L, C, c, in->counter_lift);
    qidx[qoff[c] + fill[c]++] = r;
    tail[c]++;
    L[c].backlogged = 1;
  }

  /* ---- engine.cpp:207-271 admit_requests ---- */
  int64_t members = in->n_members, reserved = 0, n_ev = 0, n_adm = 0, n_rej = 0, prefill = 0;
  for (int i = 0; i < in->n_members; ++i) /* gpu_model.cpp:40-46 */
    reserved += in->mem_in[i] + (in->mem_reserved[i] > in->mem_generated[i] ? in->mem_reserved[i]
                                                                             : in->mem_generated[i]);
  unsigned char* skipped = (unsigned char*)calloc((size_t)(C > 0 ? C : 1), 1);
  const double beta = 1.0 - in->alpha; /* scheduler.hpp:24 */
  for (;;) {
    /* scheduler.cpp:40-48 backlogged_maxima (constant during one select_next) */
    double max_ufc = 0.0, max_rfc = 0.0;
    for (int i = 0; i < C; ++i) {
      if (!L[i].backlogged) continue;
      if (max_ufc < L[i].ufc) max_ufc = L[i].ufc;
      if (max_rfc < L[i].rfc) max_rfc = L[i].rfc;
    }
    /* scheduler.cpp:131-156 select_next over candidates in client order */
    int best = -1;
    double best_key = INFINITY, best_arr = 0.0;
    for (int i = 0; i < C; ++i) {
      if (head[i] == tail[i] || skipped[i]) continue;
      const double arr = in->arrival[qidx[qoff[i] + head[i]]];
      double key; /* scheduler.cpp:119-129 selection_key */
      if (in->kind == EQXO_FCFS) key = 0.0;
      else if (in->kind == EQXO_VTC) key = L[i].counter;
      else if (in->norm_mode == EQXO_NORM_NONE) key = in->alpha * L[i].ufc + beta * L[i].rfc;
      else { /* scheduler.cpp:50-57 combine */
        const double u = max_ufc > 0.0 ? L[i].ufc / max_ufc : 0.0;
        const double v = max_rfc > 0.0 ? L[i].rfc / max_rfc : 0.0;
        key = in->alpha * u + beta * v;
      }
      int better = 0;
      if (best < 0 || key < best_key) better = 1;
      else if (key == best_key) {
        if (arr < best_arr) better = 1;
        else if (arr == best_arr && str_less(names[i], names[best])) better = 1;
      }
      if (better) {
        best = i;
        best_key = key;
        best_arr = arr;
      }
    }
    if (best < 0) break;
    const int c = best;
    const int64_t r = qidx[qoff[c] + head[c]];
    const int tin = in->in_tokens[r];
    const int p = out->pred[r];
    if (!can_fit(0, 0, tin, p, in)) { /* fits_alone: reject, pop, no counter change */
      out->ev_id[n_ev] = in->id[r];
      out->ev_kind[n_ev] = EQXO_EV_REJECT;
      out->ev_client[n_ev] = c;
      out->ev_ufc_inc[n_ev] = out->ev_rfc_inc[n_ev] = out->ev_vtc_inc[n_ev] = out->ev_wait[n_ev] = 0.0;
      ++n_ev;
      ++n_rej;
      if (++head[c] == tail[c]) L[c].backlogged = 0; /* engine.cpp:199-203 pop_head */
      continue;
    }
    if (!can_fit(members, reserved, tin, p, in)) {
      if (in->backfill) {
        skipped[c] = 1;
        continue;
      }
      break;
    }
    if (++head[c] == tail[c]) L[c].backlogged = 0;
    ++members;
    reserved += tin + p; /* reserved_output = pred, generated = 0 */
    ++running[c];
    prefill += tin;
    /* scheduler.cpp:158-183 on_admit */
    const double w = in->weight[c];
    const double wait = in->now - in->arrival[r];
    const double ui = ufc_increment(tin, p, wait, out->lat[r], w, in->delta, in->output_weight);
    const double ri = rfc_increment(out->tps[r], out->util[r], w);
    L[c].ufc += ui;
    L[c].rfc += ri;
    double vi = 0.0;
    if (in->kind == EQXO_VTC) {
      vi = in->vtc_use_prediction ? w * ((double)tin + in->output_weight * (double)p) : w * (double)tin;
      L[c].counter += vi;
    }
    out->ev_id[n_ev] = in->id[r];
    out->ev_kind[n_ev] = EQXO_EV_ADMIT;
    out->ev_client[n_ev] = c;
    out->ev_ufc_inc[n_ev] = ui;
    out->ev_rfc_inc[n_ev] = ri;
    out->ev_vtc_inc[n_ev] = vi;
    out->ev_wait[n_ev] = wait;
    ++n_ev;
    ++n_adm;
  }
  for (int c = 0; c < C; ++c) {
    out->ufc[c] = L[c].ufc;
    out->rfc[c] = L[c].rfc;
    out->counter[c] = L[c].counter;
    out->backlogged[c] = L[c].backlogged;
  }
  out->n_events = n_ev;
  out->n_admitted = n_adm;
  out->n_rejected = n_rej;
  out->new_prefill = prefill;
  out->length_fallbacks = in->pred_kind == EQXO_PRED_MOPE ? fallbacks : 0;
  out->ns_drain = out->ns_admit = 0.0;
  free(names); free(L); free(running); free(qoff); free(qidx); free(fill); free(head);
  free(tail); free(skipped);
  return 0;
#undef FAIL
}

/* Stand-alone entry points used by tests for per-function known answers. */
double eqxo_ufc_increment(double w, int in, int pred, double wait_s, double lat_ms, double delta,
                          double ow) {
  return ufc_increment(in, pred, wait_s, lat_ms, w, delta, ow);
}
double eqxo_rfc_increment(double w, double tps, double util) { return rfc_increment(tps, util, w); }
int eqxo_noisy_predict(double l1, uint64_t seed, int64_t id, int true_out) {
  return noisy_predict(l1, seed, id, true_out);
}
int eqxo_route(const eqxo_mope* m, int in, int row, int* fallback) { return route(m, in, row, fallback); }

/* ---- completion / feedback (restatement of scheduler.cpp:185-233, predictor.cpp:372-383,
 *      engine.cpp:287-293 and 327-375) ---- */
static int entry_for_idx(int n, const int32_t* upper, int out) { /* gpu_model.cpp:74-80 */
  for (int e = 0; e < n; ++e)
    if (out <= upper[e]) return e;
  return n - 1;
}

int eqxo_feedback_run(eqxo_feedback* f) {
  if (f->ema_alpha <= 0.0 || f->ema_alpha > 1.0) return 1; /* ConfigError (predictor.cpp:374-376) */
  const double ow = f->output_weight;
  f->clamps = 0;
  /* run_iteration: on_tokens per client in index order (engine.cpp:289-293) */
  if (f->tokens && f->kind == EQXO_VTC && !f->vtc_use_prediction) {
    for (int c = 0; c < f->n_clients; ++c)
      if (f->tokens[c] > 0) f->counter[c] += f->weight[c] * ow * (double)f->tokens[c];
  }
  /* complete_finished: completions in order */
  for (int64_t i = 0; i < f->n_done; ++i) {
    const int c = f->client[i];
    const double w = f->weight[c];
    const double wt = (double)f->in_tokens[i] + ow * (double)f->out_tokens[i];
    const double actual_ufc = w * wt / (1.0 + f->delta * f->latency_s[i]);
    const double actual_rfc = w * f->tps[i] * f->util[i];
    f->ufc[c] += actual_ufc - f->pend_ufc[i];
    if (f->ufc[c] < 0.0) { f->ufc[c] = 0.0; ++f->clamps; }
    f->rfc[c] += actual_rfc - f->pend_rfc[i];
    if (f->rfc[c] < 0.0) { f->rfc[c] = 0.0; ++f->clamps; }
    if (f->kind == EQXO_VTC && f->vtc_use_prediction) {
      f->counter[c] += w * wt - f->pend_vtc[i];
      if (f->counter[c] < 0.0) { f->counter[c] = 0.0; ++f->clamps; }
    }
    f->service[c] += w * wt;
    if (f->running) f->running[c] -= 1;
    /* update_map with ObservedMetrics{out, latency_s * 1000, util, tps} */
    const int e = entry_for_idx(f->n_profile, f->prof_upper, f->out_tokens[i]);
    const double a = f->ema_alpha;
    f->prof_lat[e] = (1.0 - a) * f->prof_lat[e] + a * (f->latency_s[i] * 1000.0);
    f->prof_util[e] = (1.0 - a) * f->prof_util[e] + a * f->util[i];
    f->prof_tps[e] = (1.0 - a) * f->prof_tps[e] + a * f->tps[i];
  }
  return 0;
}
