// ref_step.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin driver over the reference's *public* C++ API (compiled from the unmodified sources
// under /root/reference/proj/src by oracle/Makefile into oracle/_ref/libeqx_ref.so).  It
// exposes plain C entry points so tests/ and bench.py (--impl reference, cpu_baseline) can
// run the reference algorithm on the same arrays the GPU path consumes.  No reference code is
// copied here: every decision is made by a reference function.
//
//   ref_step     -- drain_arrivals + admit_requests (engine.cpp:171-271) re-driven line for
//                   line through SchedulerPolicy / Predictor / map_metrics / can_fit /
//                   fits_alone, with a pre-seeded ledger and batch (SURVEY.md 8(c) mode 1).
//   ref_train_mope_json / ref_build_profile / ref_corpus -- model + profile fixtures.
//   ref_replay   -- run_simulation (engine.cpp:458-463) on an array trace (mode 2).
//   ref_units    -- the reference unit-test formulas (ufc/rfc/holistic/route/can_fit).

#include <chrono>
#include <cstring>
#include <deque>
#include <exception>
#include <fstream>
#include <memory>
#include <set>
#include <string>
#include <vector>

#include "equinox/engine.hpp"
#include "equinox/errors.hpp"
#include "equinox/gpu_model.hpp"
#include "equinox/metrics.hpp"
#include "equinox/predictor.hpp"
#include "equinox/rng.hpp"
#include "equinox/scheduler.hpp"
#include "equinox/workload.hpp"

#include "eqx_oracle.h"

using namespace equinox;

namespace {

std::vector<std::string> split_names(const char* buf, int n) {
  std::vector<std::string> out;
  out.reserve(static_cast<std::size_t>(n));
  const char* p = buf;
  for (int i = 0; i < n; ++i) {
    out.emplace_back(p);
    p += out.back().size() + 1;
  }
  return out;
}

void set_err(char* err, int len, const char* msg) {
  if (err && len > 0) {
    std::strncpy(err, msg, static_cast<std::size_t>(len) - 1);
    err[len - 1] = '\0';
  }
}

MopeModel model_from(const eqxo_mope& m, const std::vector<std::string>& tag_names,
                     const int32_t* tag_row, int n_tags) {
  MopeModel model;
  model.router.input_len_thresholds.assign(m.thresholds, m.thresholds + m.n_thresholds);
  model.router.mix_weight = m.mix_weight;
  model.router.num_buckets = m.num_buckets;
  for (int t = 0; t < n_tags; ++t) {
    if (tag_row[t] < 0) continue;
    const double* row = m.rows + static_cast<std::size_t>(tag_row[t]) * m.num_buckets;
    model.router.keyword_scores[tag_names[static_cast<std::size_t>(t)]] =
        std::vector<double>(row, row + m.num_buckets);
  }
  for (int e = 0; e < m.n_experts; ++e) {
    ExpertModel ex;
    ex.bucket = e;
    ex.bin_upper.assign(m.bin_upper + e * m.n_bins, m.bin_upper + (e + 1) * m.n_bins);
    ex.bin_value.assign(m.bin_value + e * m.n_bins, m.bin_value + (e + 1) * m.n_bins);
    ex.out_min = m.out_min[e];
    ex.out_max = m.out_max[e];
    model.experts.push_back(std::move(ex));
  }
  return model;
}

struct Queued {
  Request req;
  PredictionRecord prediction;
};

}  // namespace

extern "C" {

int ref_step(const eqxo_step_in* in, eqxo_step_out* out, char* err, int err_len) {
  try {
    const auto names = split_names(in->client_names, in->n_clients);
    const auto tags = split_names(in->tag_names, in->n_tags);

    PolicySpec spec;
    spec.kind = static_cast<PolicyKind>(in->kind);
    spec.equinox.alpha = in->alpha;
    spec.equinox.delta = in->delta;
    spec.equinox.output_weight = in->output_weight;
    spec.equinox.norm_mode =
        in->norm_mode == EQXO_NORM_NONE ? NormMode::None : NormMode::MaxOverClients;
    spec.vtc_use_prediction = in->vtc_use_prediction != 0;
    spec.counter_lift = in->counter_lift != 0;

    std::vector<ClientState> roster(static_cast<std::size_t>(in->n_clients));
    for (int c = 0; c < in->n_clients; ++c) {
      roster[c].client_id = names[c];
      roster[c].weight = in->weight[c];
      roster[c].ufc = in->ufc0[c];
      roster[c].rfc = in->rfc0[c];
      roster[c].counter = in->counter0[c];
    }
    SchedulerPolicy policy(spec, roster);

    PerfParams perf;
    perf.max_batch = in->max_batch;
    perf.mem_per_token_bytes = in->mem_per_token_bytes;
    perf.mem_capacity_bytes = in->mem_capacity_bytes;

    GpuProfile profile;
    for (int e = 0; e < in->n_profile; ++e) {
      profile.entries.push_back(
          {in->prof_upper[e], in->prof_lat[e], in->prof_util[e], in->prof_tps[e]});
    }

    std::unique_ptr<Predictor> predictor;
    MopePredictor* mope_ptr = nullptr;
    switch (in->pred_kind) {
      case EQXO_PRED_ORACLE:
        predictor = std::make_unique<OraclePredictor>();
        break;
      case EQXO_PRED_NOISY:
        predictor = std::make_unique<NoisyOraclePredictor>(in->noisy_l1, in->noisy_seed);
        break;
      case EQXO_PRED_MOPE: {
        auto p = std::make_unique<MopePredictor>(
            model_from(in->mope, tags, in->tag_row, in->n_tags));
        mope_ptr = p.get();
        predictor = std::move(p);
        break;
      }
      case EQXO_PRED_SINGLE: {
        MopeModel m = model_from(in->mope, tags, in->tag_row, in->n_tags);
        predictor = std::make_unique<SingleProxyPredictor>(m.experts.at(0));
        break;
      }
      default:
        throw ConfigError("unknown predictor kind");
    }

    BatchState batch;
    for (int i = 0; i < in->n_members; ++i) {
      batch.members.push_back({-1 - i, in->mem_in[i], in->mem_generated[i], in->mem_reserved[i]});
    }

    // Requests are materialised before the timed region (the engine holds them in its Trace).
    std::vector<Request> reqs(static_cast<std::size_t>(in->n_req));
    for (int64_t r = 0; r < in->n_req; ++r) {
      Request& q = reqs[static_cast<std::size_t>(r)];
      q.id = in->id[r];
      q.client_id = names[static_cast<std::size_t>(in->client[r])];
      q.arrival_time_s = in->arrival[r];
      q.input_tokens = in->in_tokens[r];
      q.true_output_tokens = in->true_out[r];
      if (in->tag[r] >= 0) q.category_tag = tags[static_cast<std::size_t>(in->tag[r])];
    }

    std::vector<std::deque<Queued>> queues(static_cast<std::size_t>(in->n_clients));
    std::vector<int> running(in->running, in->running + in->n_clients);
    std::vector<PredictionRecord> frozen(static_cast<std::size_t>(in->n_req));

    // ---- drain_arrivals (engine.cpp:171-197) ----
    const auto t0 = std::chrono::steady_clock::now();
    for (int64_t r = 0; r < in->n_req; ++r) {
      const Request& req = reqs[static_cast<std::size_t>(r)];
      const std::size_t ci = static_cast<std::size_t>(in->client[r]);
      const int predicted = std::max(1, predictor->predict(req));
      Queued queued{req, map_metrics(predicted, profile)};
      frozen[static_cast<std::size_t>(r)] = queued.prediction;
      if (queues[ci].empty() && running[ci] == 0) policy.on_activated(ci);
      queues[ci].push_back(std::move(queued));
      policy.set_backlogged(ci, true);
    }
    const auto t1 = std::chrono::steady_clock::now();

    // ---- admit_requests (engine.cpp:207-271) ----
    int64_t n_ev = 0, n_adm = 0, n_rej = 0, new_prefill = 0;
    auto pop_head = [&](std::size_t ci) {
      queues[ci].pop_front();
      if (queues[ci].empty()) policy.set_backlogged(ci, false);
    };
    std::set<std::size_t> skipped;
    while (true) {
      std::vector<HeadCandidate> candidates;
      for (std::size_t i = 0; i < queues.size(); ++i) {
        if (queues[i].empty() || skipped.count(i) != 0) continue;
        candidates.push_back({i, queues[i].front().req.arrival_time_s});
      }
      const auto choice = policy.select_next(candidates);
      if (!choice) break;
      const std::size_t ci = *choice;
      const Queued head = queues[ci].front();
      const int tin = head.req.input_tokens;
      const int predicted = head.prediction.predicted_output_tokens;
      if (!fits_alone(tin, predicted, perf)) {
        out->ev_id[n_ev] = head.req.id;
        out->ev_kind[n_ev] = EQXO_EV_REJECT;
        out->ev_client[n_ev] = static_cast<int32_t>(ci);
        out->ev_ufc_inc[n_ev] = out->ev_rfc_inc[n_ev] = out->ev_vtc_inc[n_ev] = 0.0;
        out->ev_wait[n_ev] = 0.0;
        ++n_ev;
        ++n_rej;
        pop_head(ci);
        continue;
      }
      if (!can_fit(batch, tin, predicted, perf)) {
        if (in->backfill) {
          skipped.insert(ci);
          continue;
        }
        break;
      }
      pop_head(ci);
      batch.members.push_back({head.req.id, tin, 0, predicted});
      ++running[ci];
      new_prefill += tin;
      ScheduleContext ctx;
      ctx.now_s = in->now;
      ctx.wait_s = in->now - head.req.arrival_time_s;
      ctx.prediction = head.prediction;
      const ClientState before = policy.clients()[ci];
      policy.on_admit(ci, head.req, ctx);
      const ClientState& after = policy.clients()[ci];
      out->ev_id[n_ev] = head.req.id;
      out->ev_kind[n_ev] = EQXO_EV_ADMIT;
      out->ev_client[n_ev] = static_cast<int32_t>(ci);
      // PendingContribution values, recomputed by the same reference functions on_admit uses.
      out->ev_ufc_inc[n_ev] = ufc_increment(head.req, ctx, before.weight, spec.equinox);
      out->ev_rfc_inc[n_ev] = rfc_increment(ctx.prediction, before.weight);
      // vtc_inc as on_admit forms it (scheduler.cpp:169-181); the ledger itself is reported
      // from the reference object below.
      double vtc = 0.0;
      if (spec.kind == PolicyKind::Vtc) {
        vtc = spec.vtc_use_prediction
                  ? before.weight * (static_cast<double>(tin) +
                                     spec.equinox.output_weight * static_cast<double>(predicted))
                  : before.weight * static_cast<double>(tin);
      }
      (void)after;
      out->ev_vtc_inc[n_ev] = vtc;
      out->ev_wait[n_ev] = ctx.wait_s;
      ++n_ev;
      ++n_adm;
    }
    const auto t2 = std::chrono::steady_clock::now();

    // ---- per-request outputs (prediction record + increments at `now`) ----
    for (int64_t r = 0; r < in->n_req; ++r) {
      const PredictionRecord& p = frozen[static_cast<std::size_t>(r)];
      const Request& req = reqs[static_cast<std::size_t>(r)];
      out->pred[r] = p.predicted_output_tokens;
      const ProfileEntry* e = &profile.entry_for(p.predicted_output_tokens);
      out->bucket[r] = static_cast<int32_t>(e - profile.entries.data());
      out->lat[r] = p.predicted_latency_ms;
      out->util[r] = p.predicted_gpu_util;
      out->tps[r] = p.predicted_tps;
      ScheduleContext ctx;
      ctx.now_s = in->now;
      ctx.wait_s = in->now - req.arrival_time_s;
      ctx.prediction = p;
      const double w = in->weight[in->client[r]];
      out->ufc_inc[r] = ufc_increment(req, ctx, w, spec.equinox);
      out->rfc_inc[r] = rfc_increment(p, w);
    }
    for (int c = 0; c < in->n_clients; ++c) {
      const ClientState& s = policy.clients()[static_cast<std::size_t>(c)];
      out->ufc[c] = s.ufc;
      out->rfc[c] = s.rfc;
      out->counter[c] = s.counter;
      out->backlogged[c] = s.backlogged ? 1 : 0;
    }
    out->n_events = n_ev;
    out->n_admitted = n_adm;
    out->n_rejected = n_rej;
    out->new_prefill = new_prefill;
    out->length_fallbacks = mope_ptr ? mope_ptr->length_fallbacks() : 0;
    out->ns_drain = std::chrono::duration<double, std::nano>(t1 - t0).count();
    out->ns_admit = std::chrono::duration<double, std::nano>(t2 - t1).count();
    return 0;
  } catch (const std::exception& e) {
    set_err(err, err_len, e.what());
    return 1;
  }
}

// Trains the reference MoPE on the builtin corpus (experiments.cpp:58-73) and returns its
// JSON (predictor.cpp:408-430).  Returns the needed length; writes when buf is big enough.
int64_t ref_train_mope_json(int corpus_size, uint64_t seed, int experts, char* buf,
                            int64_t buf_len) {
  const Trace corpus = make_prediction_corpus(corpus_size, seed);
  std::vector<double> pct;
  for (int i = 1; i < experts; ++i) pct.push_back(100.0 * i / static_cast<double>(experts));
  const std::string s = train_mope(corpus, pct).to_json().dump();
  if (buf && buf_len > static_cast<int64_t>(s.size())) std::memcpy(buf, s.c_str(), s.size() + 1);
  return static_cast<int64_t>(s.size()) + 1;
}

// build_profile (gpu_model.cpp:87-126) with default PerfParams except the given fields.
int ref_build_profile(const int32_t* bounds, int n, int ref_input, int32_t* upper,
                      double* lat, double* util, double* tps) {
  try {
    const GpuProfile p = build_profile(PerfParams{}, std::vector<int>(bounds, bounds + n), ref_input);
    for (int i = 0; i < n; ++i) {
      upper[i] = p.entries[i].bucket_upper;
      lat[i] = p.entries[i].latency_ms;
      util[i] = p.entries[i].gpu_util;
      tps[i] = p.entries[i].tps;
    }
    return 0;
  } catch (...) {
    return 1;
  }
}

// make_prediction_corpus (workload.cpp:430-476): in/out/tag(0 short,1 medium,2 long).
int ref_corpus(int n, uint64_t seed, int32_t* in_tok, int32_t* out_tok, int32_t* tag) {
  const Trace t = make_prediction_corpus(n, seed);
  for (int i = 0; i < n; ++i) {
    in_tok[i] = t.requests[i].input_tokens;
    out_tok[i] = t.requests[i].true_output_tokens;
    const std::string& g = t.requests[i].category_tag;
    tag[i] = g == "short" ? 0 : g == "medium" ? 1 : 2;
  }
  return 0;
}

// NoisyOraclePredictor::predict (predictor.cpp:17-23) for a vector of (id, true_out).
void ref_noisy_predict(double l1, uint64_t seed, int64_t n, const int64_t* id,
                       const int32_t* true_out, int32_t* pred) {
  NoisyOraclePredictor p(l1, seed);
  Request r;
  for (int64_t i = 0; i < n; ++i) {
    r.id = id[i];
    r.true_output_tokens = true_out[i];
    pred[i] = std::max(1, p.predict(r));
  }
}

// glibc log1p as the reference links it (rng.hpp:46), for device-libm pinning.
void ref_log1p(int64_t n, const double* x, double* y) {
  for (int64_t i = 0; i < n; ++i) y[i] = std::log1p(x[i]);
}

// Reference unit-test formulas (test_scheduler.cpp:50-110; test_gpu_model.cpp:28-44).
double ref_ufc_increment(double w, int in, int pred, double wait_s, double lat_ms,
                         double delta, double ow) {
  Request req;
  req.input_tokens = in;
  ScheduleContext ctx;
  ctx.wait_s = wait_s;
  ctx.prediction.predicted_output_tokens = pred;
  ctx.prediction.predicted_latency_ms = lat_ms;
  EquinoxParams p;
  p.delta = delta;
  p.output_weight = ow;
  return ufc_increment(req, ctx, w, p);
}

double ref_rfc_increment(double w, double tps, double util) {
  PredictionRecord r;
  r.predicted_tps = tps;
  r.predicted_gpu_util = util;
  return rfc_increment(r, w);
}

// Full engine replay (run_simulation) of an array trace with default PerfParams/profile
// overrides; writes the admission/rejection event sequence.  Returns #events or -1.
int64_t ref_replay(const eqxo_step_in* in, double max_sim_time_s, double ema_alpha,
                   int64_t* ev_id, int32_t* ev_kind, double* ev_time, int64_t ev_cap,
                   double* final_ufc, double* final_rfc, double* final_counter, char* err,
                   int err_len) {
  try {
    const auto names = split_names(in->client_names, in->n_clients);
    const auto tags = split_names(in->tag_names, in->n_tags);
    Trace trace;
    for (int c = 0; c < in->n_clients; ++c) {
      ClientSpec s;
      s.client_id = names[c];
      s.weight = in->weight[c];
      s.arrivals.kind = ArrivalKind::Replay;
      trace.clients.push_back(s);
    }
    double last = 0.0;
    for (int64_t r = 0; r < in->n_req; ++r) {
      Request q;
      q.id = in->id[r];
      q.client_id = names[static_cast<std::size_t>(in->client[r])];
      q.arrival_time_s = in->arrival[r];
      q.input_tokens = in->in_tokens[r];
      q.true_output_tokens = in->true_out[r];
      if (in->tag[r] >= 0) q.category_tag = tags[static_cast<std::size_t>(in->tag[r])];
      last = q.arrival_time_s;
      trace.requests.push_back(q);
    }
    trace.duration_s = in->duration_s > 0.0 ? in->duration_s : last;
    EngineConfig cfg;
    cfg.policy.kind = static_cast<PolicyKind>(in->kind);
    cfg.policy.equinox.alpha = in->alpha;
    cfg.policy.equinox.delta = in->delta;
    cfg.policy.equinox.output_weight = in->output_weight;
    cfg.policy.equinox.norm_mode =
        in->norm_mode == EQXO_NORM_NONE ? NormMode::None : NormMode::MaxOverClients;
    cfg.policy.vtc_use_prediction = in->vtc_use_prediction != 0;
    cfg.policy.counter_lift = in->counter_lift != 0;
    cfg.perf.max_batch = in->max_batch;
    cfg.perf.mem_per_token_bytes = in->mem_per_token_bytes;
    cfg.perf.mem_capacity_bytes = in->mem_capacity_bytes;
    cfg.backfill = in->backfill != 0;
    cfg.max_sim_time_s = max_sim_time_s;
    cfg.ema_alpha = ema_alpha;
    GpuProfile profile;
    for (int e = 0; e < in->n_profile; ++e) {
      profile.entries.push_back(
          {in->prof_upper[e], in->prof_lat[e], in->prof_util[e], in->prof_tps[e]});
    }
    std::unique_ptr<Predictor> predictor;
    if (in->pred_kind == EQXO_PRED_MOPE) {
      predictor = std::make_unique<MopePredictor>(model_from(in->mope, tags, in->tag_row, in->n_tags));
    } else if (in->pred_kind == EQXO_PRED_NOISY) {
      predictor = std::make_unique<NoisyOraclePredictor>(in->noisy_l1, in->noisy_seed);
    } else {
      predictor = std::make_unique<OraclePredictor>();
    }
    const SimResult res = run_simulation(trace, cfg, *predictor, profile);
    int64_t n = 0;
    for (const auto& e : res.log.entries) {
      if (e.event != LogEvent::Admitted && e.event != LogEvent::Rejected) continue;
      if (n < ev_cap) {
        ev_id[n] = e.request_id;
        ev_kind[n] = e.event == LogEvent::Admitted ? EQXO_EV_ADMIT : EQXO_EV_REJECT;
        ev_time[n] = e.time_s;
      }
      ++n;
    }
    for (std::size_t c = 0; c < res.final_clients.size(); ++c) {
      final_ufc[c] = res.final_clients[c].ufc;
      final_rfc[c] = res.final_clients[c].rfc;
      final_counter[c] = res.final_clients[c].counter;
    }
    return n;
  } catch (const std::exception& e) {
    set_err(err, err_len, e.what());
    return -1;
  }
}

}  // extern "C"

// ref_feedback -- the completion / feedback path through the reference objects: every
// admission registers its PendingContribution with SchedulerPolicy::on_admit (the prediction
// record from map_metrics against the profile), then one iteration's on_tokens in client order
// (engine.cpp:289-293), then for each completion in order SchedulerPolicy::on_complete and
// update_map (engine.cpp:327-375).  `f` carries the pre-admission ledger and profile in and the
// final state out; pend_out[3][n_adm] = the registered pending (ufc, rfc, vtc) increments and
// mid_out[3][C] = the ledger (ufc, rfc, counter) after the admissions.
extern "C" int ref_feedback(eqxo_feedback* f, const char* client_names, double now, int64_t n_adm,
                            const int64_t* adm_id, const int32_t* adm_client, const int32_t* adm_in,
                            const int32_t* adm_pred, const double* adm_wait, const int32_t* done_adm,
                            double* pend_out, double* mid_out, char* err, int err_len) {
  try {
    const auto names = split_names(client_names, f->n_clients);
    PolicySpec spec;
    spec.kind = static_cast<PolicyKind>(f->kind);
    spec.equinox.alpha = f->alpha;
    spec.equinox.delta = f->delta;
    spec.equinox.output_weight = f->output_weight;
    spec.vtc_use_prediction = f->vtc_use_prediction != 0;
    std::vector<ClientState> roster(static_cast<std::size_t>(f->n_clients));
    for (int c = 0; c < f->n_clients; ++c) {
      roster[c].client_id = names[c];
      roster[c].weight = f->weight[c];
      roster[c].ufc = f->ufc[c];
      roster[c].rfc = f->rfc[c];
      roster[c].counter = f->counter[c];
      roster[c].accumulated_service = f->service[c];
    }
    SchedulerPolicy policy(spec, roster);
    GpuProfile profile;
    for (int e = 0; e < f->n_profile; ++e)
      profile.entries.push_back({f->prof_upper[e], f->prof_lat[e], f->prof_util[e], f->prof_tps[e]});
    std::vector<Request> reqs(static_cast<std::size_t>(n_adm));
    for (int64_t a = 0; a < n_adm; ++a) {
      Request& r = reqs[static_cast<std::size_t>(a)];
      r.id = adm_id[a];
      r.client_id = names[adm_client[a]];
      r.input_tokens = adm_in[a];
      ScheduleContext ctx;
      ctx.now_s = now;
      ctx.wait_s = adm_wait[a];
      ctx.prediction = map_metrics(adm_pred[a], profile);
      const ClientState before = policy.clients()[static_cast<std::size_t>(adm_client[a])];
      policy.on_admit(static_cast<std::size_t>(adm_client[a]), r, ctx);
      const ClientState& after = policy.clients()[static_cast<std::size_t>(adm_client[a])];
      pend_out[a] = ufc_increment(r, ctx, before.weight, spec.equinox);
      pend_out[n_adm + a] = rfc_increment(ctx.prediction, before.weight);
      pend_out[2 * n_adm + a] = after.counter - before.counter;  // vtc_inc (0 unless VTC)
    }
    for (int c = 0; c < f->n_clients; ++c) {
      const ClientState& s = policy.clients()[static_cast<std::size_t>(c)];
      mid_out[c] = s.ufc;
      mid_out[f->n_clients + c] = s.rfc;
      mid_out[2 * f->n_clients + c] = s.counter;
    }
    if (f->tokens)
      for (int c = 0; c < f->n_clients; ++c)
        if (f->tokens[c] > 0) policy.on_tokens(static_cast<std::size_t>(c), f->tokens[c]);
    for (int64_t i = 0; i < f->n_done; ++i) {
      const int64_t a = done_adm[i];
      RequestActuals act;
      act.output_tokens = f->out_tokens[i];
      act.latency_s = f->latency_s[i];
      act.tps = f->tps[i];
      act.gpu_util = f->util[i];
      policy.on_complete(static_cast<std::size_t>(adm_client[a]), reqs[static_cast<std::size_t>(a)], act);
      ObservedMetrics obs;
      obs.output_tokens = act.output_tokens;
      obs.latency_ms = act.latency_s * 1000.0;
      obs.gpu_util = act.gpu_util;
      obs.tps = act.tps;
      update_map(profile, obs, f->ema_alpha);
    }
    for (int c = 0; c < f->n_clients; ++c) {
      const ClientState& s = policy.clients()[static_cast<std::size_t>(c)];
      f->ufc[c] = s.ufc;
      f->rfc[c] = s.rfc;
      f->counter[c] = s.counter;
      f->service[c] = s.accumulated_service;
    }
    for (int e = 0; e < f->n_profile; ++e) {
      f->prof_lat[e] = profile.entries[static_cast<std::size_t>(e)].latency_ms;
      f->prof_util[e] = profile.entries[static_cast<std::size_t>(e)].gpu_util;
      f->prof_tps[e] = profile.entries[static_cast<std::size_t>(e)].tps;
    }
    f->clamps = policy.counter_clamps();
    return 0;
  } catch (const std::exception& e) {
    set_err(err, err_len, e.what());
    return 1;
  }
}

// ref_multi -- several engine steps on live queues through the reference objects: at step k
// the arrivals in rows [step_end[k-1], step_end[k]) are drained (engine.cpp:171-197: predict,
// map_metrics against the *current* profile, on_activated for idle clients, push,
// set_backlogged), admit_requests runs at step_now[k] (engine.cpp:207-271) on the queues left
// by earlier steps plus the new arrivals, and then every batch member whose
// (request_id * 7 + k) % complete_mod == 0 completes in batch order (engine.cpp:327-375:
// on_complete, update_map, running count, member erase) with actuals
// {true_output_tokens, step_now[k] - arrival + act_extra, act_tps, act_util} (row-indexed).
// ids must be the row indices.  Events go to ev_* with their step in ev_step; returns the
// event count, or -1 on error.
extern "C" int64_t ref_multi(const eqxo_step_in* in, int32_t n_steps, const int64_t* step_end,
                             const double* step_now, const double* act_extra, const double* act_tps,
                             const double* act_util, double ema_alpha, int32_t complete_mod, int64_t* ev_id,
                             int32_t* ev_kind, int32_t* ev_step, double* ev_ufc, double* ev_rfc, int64_t cap,
                             double* ufc, double* rfc, double* counter, double* prof_lat, double* prof_util,
                             double* prof_tps, char* err, int err_len) {
  try {
    const auto names = split_names(in->client_names, in->n_clients);
    const auto tags = split_names(in->tag_names, in->n_tags);
    PolicySpec spec;
    spec.kind = static_cast<PolicyKind>(in->kind);
    spec.equinox.alpha = in->alpha;
    spec.equinox.delta = in->delta;
    spec.equinox.output_weight = in->output_weight;
    spec.equinox.norm_mode = in->norm_mode == EQXO_NORM_NONE ? NormMode::None : NormMode::MaxOverClients;
    spec.vtc_use_prediction = in->vtc_use_prediction != 0;
    spec.counter_lift = in->counter_lift != 0;
    std::vector<ClientState> roster(static_cast<std::size_t>(in->n_clients));
    for (int c = 0; c < in->n_clients; ++c) {
      roster[c].client_id = names[c];
      roster[c].weight = in->weight[c];
      roster[c].ufc = in->ufc0[c];
      roster[c].rfc = in->rfc0[c];
      roster[c].counter = in->counter0[c];
    }
    SchedulerPolicy policy(spec, roster);
    PerfParams perf;
    perf.max_batch = in->max_batch;
    perf.mem_per_token_bytes = in->mem_per_token_bytes;
    perf.mem_capacity_bytes = in->mem_capacity_bytes;
    GpuProfile profile;
    for (int e = 0; e < in->n_profile; ++e)
      profile.entries.push_back({in->prof_upper[e], in->prof_lat[e], in->prof_util[e], in->prof_tps[e]});
    std::unique_ptr<Predictor> predictor;
    switch (in->pred_kind) {
      case EQXO_PRED_ORACLE: predictor = std::make_unique<OraclePredictor>(); break;
      case EQXO_PRED_NOISY: predictor = std::make_unique<NoisyOraclePredictor>(in->noisy_l1, in->noisy_seed); break;
      case EQXO_PRED_MOPE:
        predictor = std::make_unique<MopePredictor>(model_from(in->mope, tags, in->tag_row, in->n_tags));
        break;
      case EQXO_PRED_SINGLE: {
        MopeModel m = model_from(in->mope, tags, in->tag_row, in->n_tags);
        predictor = std::make_unique<SingleProxyPredictor>(m.experts.at(0));
        break;
      }
      default: throw ConfigError("unknown predictor kind");
    }
    std::vector<Request> reqs(static_cast<std::size_t>(in->n_req));
    for (int64_t r = 0; r < in->n_req; ++r) {
      Request& q = reqs[static_cast<std::size_t>(r)];
      q.id = in->id[r];
      q.client_id = names[static_cast<std::size_t>(in->client[r])];
      q.arrival_time_s = in->arrival[r];
      q.input_tokens = in->in_tokens[r];
      q.true_output_tokens = in->true_out[r];
      if (in->tag[r] >= 0) q.category_tag = tags[static_cast<std::size_t>(in->tag[r])];
    }
    std::vector<std::deque<Queued>> queues(static_cast<std::size_t>(in->n_clients));
    std::vector<int> running(static_cast<std::size_t>(in->n_clients), 0);
    BatchState batch;
    std::vector<std::size_t> member_client;
    int64_t n_ev = 0, row = 0;
    for (int32_t k = 0; k < n_steps; ++k) {
      const double now = step_now[k];
      for (; row < step_end[k]; ++row) {  // drain_arrivals
        const Request& req = reqs[static_cast<std::size_t>(row)];
        const std::size_t ci = static_cast<std::size_t>(in->client[row]);
        const int predicted = std::max(1, predictor->predict(req));
        Queued queued{req, map_metrics(predicted, profile)};
        if (queues[ci].empty() && running[ci] == 0) policy.on_activated(ci);
        queues[ci].push_back(std::move(queued));
        policy.set_backlogged(ci, true);
      }
      auto pop_head = [&](std::size_t ci) {
        queues[ci].pop_front();
        if (queues[ci].empty()) policy.set_backlogged(ci, false);
      };
      std::set<std::size_t> skipped;
      while (true) {  // admit_requests
        std::vector<HeadCandidate> candidates;
        for (std::size_t i = 0; i < queues.size(); ++i) {
          if (queues[i].empty() || skipped.count(i) != 0) continue;
          candidates.push_back({i, queues[i].front().req.arrival_time_s});
        }
        const auto choice = policy.select_next(candidates);
        if (!choice) break;
        const std::size_t ci = *choice;
        const Queued head = queues[ci].front();
        const int tin = head.req.input_tokens;
        const int predicted = head.prediction.predicted_output_tokens;
        if (!fits_alone(tin, predicted, perf)) {
          if (n_ev < cap) {
            ev_id[n_ev] = head.req.id;
            ev_kind[n_ev] = EQXO_EV_REJECT;
            ev_step[n_ev] = k;
            ev_ufc[n_ev] = ev_rfc[n_ev] = 0.0;
          }
          ++n_ev;
          pop_head(ci);
          continue;
        }
        if (!can_fit(batch, tin, predicted, perf)) {
          if (in->backfill) {
            skipped.insert(ci);
            continue;
          }
          break;
        }
        pop_head(ci);
        batch.members.push_back({head.req.id, tin, 0, predicted});
        member_client.push_back(ci);
        ++running[ci];
        ScheduleContext ctx;
        ctx.now_s = now;
        ctx.wait_s = now - head.req.arrival_time_s;
        ctx.prediction = head.prediction;
        const double w = policy.clients()[ci].weight;
        policy.on_admit(ci, head.req, ctx);
        if (n_ev < cap) {
          ev_id[n_ev] = head.req.id;
          ev_kind[n_ev] = EQXO_EV_ADMIT;
          ev_step[n_ev] = k;
          ev_ufc[n_ev] = ufc_increment(head.req, ctx, w, spec.equinox);
          ev_rfc[n_ev] = rfc_increment(ctx.prediction, w);
        }
        ++n_ev;
      }
      // completions, in batch order
      std::size_t i = 0;
      while (i < batch.members.size()) {
        const int64_t id = batch.members[i].request_id;
        if ((id * 7 + k) % complete_mod != 0) {
          ++i;
          continue;
        }
        const Request& req = reqs[static_cast<std::size_t>(id)];
        const std::size_t ci = member_client[i];
        RequestActuals act;
        act.output_tokens = req.true_output_tokens;
        act.latency_s = now - req.arrival_time_s + act_extra[id];
        act.tps = act_tps[id];
        act.gpu_util = act_util[id];
        policy.on_complete(ci, req, act);
        ObservedMetrics obs;
        obs.output_tokens = act.output_tokens;
        obs.latency_ms = act.latency_s * 1000.0;
        obs.gpu_util = act.gpu_util;
        obs.tps = act.tps;
        update_map(profile, obs, ema_alpha);
        --running[ci];
        batch.members.erase(batch.members.begin() + static_cast<std::ptrdiff_t>(i));
        member_client.erase(member_client.begin() + static_cast<std::ptrdiff_t>(i));
      }
    }
    for (int c = 0; c < in->n_clients; ++c) {
      const ClientState& s = policy.clients()[static_cast<std::size_t>(c)];
      ufc[c] = s.ufc;
      rfc[c] = s.rfc;
      counter[c] = s.counter;
    }
    for (int e = 0; e < in->n_profile; ++e) {
      prof_lat[e] = profile.entries[static_cast<std::size_t>(e)].latency_ms;
      prof_util[e] = profile.entries[static_cast<std::size_t>(e)].gpu_util;
      prof_tps[e] = profile.entries[static_cast<std::size_t>(e)].tps;
    }
    return n_ev;
  } catch (const std::exception& e) {
    set_err(err, err_len, e.what());
    return -1;
  }
}

// ref_replay_report -- run_simulation as ref_replay does, then build_report (metrics.cpp:155-229)
// for the two numbers run_sweep_alpha aggregates (experiments.cpp:354-360): the Jain index of
// the per-client p90 TTFT and the completed-token throughput.
extern "C" int ref_replay_report(const eqxo_step_in* in, double max_sim_time_s, double ema_alpha,
                                 double* jain_ttft_p90, double* throughput_tps, int64_t* completed,
                                 double* sim_end, char* err, int err_len) {
  try {
    const auto names = split_names(in->client_names, in->n_clients);
    const auto tags = split_names(in->tag_names, in->n_tags);
    Trace trace;
    for (int c = 0; c < in->n_clients; ++c) {
      ClientSpec cs;
      cs.client_id = names[c];
      cs.weight = in->weight[c];
      cs.arrivals.kind = ArrivalKind::Replay;
      trace.clients.push_back(cs);
    }
    double last = 0.0;
    for (int64_t r = 0; r < in->n_req; ++r) {
      Request q;
      q.id = in->id[r];
      q.client_id = names[static_cast<std::size_t>(in->client[r])];
      q.arrival_time_s = in->arrival[r];
      q.input_tokens = in->in_tokens[r];
      q.true_output_tokens = in->true_out[r];
      if (in->tag[r] >= 0) q.category_tag = tags[static_cast<std::size_t>(in->tag[r])];
      last = q.arrival_time_s;
      trace.requests.push_back(q);
    }
    trace.duration_s = in->duration_s > 0.0 ? in->duration_s : last;
    EngineConfig cfg;
    cfg.policy.kind = static_cast<PolicyKind>(in->kind);
    cfg.policy.equinox.alpha = in->alpha;
    cfg.policy.equinox.delta = in->delta;
    cfg.policy.equinox.output_weight = in->output_weight;
    cfg.policy.equinox.norm_mode = in->norm_mode == EQXO_NORM_NONE ? NormMode::None : NormMode::MaxOverClients;
    cfg.policy.vtc_use_prediction = in->vtc_use_prediction != 0;
    cfg.policy.counter_lift = in->counter_lift != 0;
    cfg.perf.max_batch = in->max_batch;
    cfg.perf.mem_per_token_bytes = in->mem_per_token_bytes;
    cfg.perf.mem_capacity_bytes = in->mem_capacity_bytes;
    cfg.backfill = in->backfill != 0;
    cfg.max_sim_time_s = max_sim_time_s;
    cfg.ema_alpha = ema_alpha;
    GpuProfile profile;
    for (int e = 0; e < in->n_profile; ++e)
      profile.entries.push_back({in->prof_upper[e], in->prof_lat[e], in->prof_util[e], in->prof_tps[e]});
    std::unique_ptr<Predictor> predictor;
    if (in->pred_kind == EQXO_PRED_MOPE) {
      predictor = std::make_unique<MopePredictor>(model_from(in->mope, tags, in->tag_row, in->n_tags));
    } else if (in->pred_kind == EQXO_PRED_NOISY) {
      predictor = std::make_unique<NoisyOraclePredictor>(in->noisy_l1, in->noisy_seed);
    } else {
      predictor = std::make_unique<OraclePredictor>();
    }
    const SimResult res = run_simulation(trace, cfg, *predictor, profile);
    const SimReport rep = build_report(trace, res, cfg.policy.equinox.output_weight, cfg.report_window_s);
    *jain_ttft_p90 = rep.jain_ttft_p90;
    *throughput_tps = rep.throughput_tps;
    *completed = rep.completed;
    *sim_end = rep.sim_end_s;
    return 0;
  } catch (const std::exception& e) {
    set_err(err, err_len, e.what());
    return 1;
  }
}

// ref_replay_full -- run_simulation + build_report (metrics.cpp:151-229) with every reported
// quantity the device replay produces: the SimReport summary (rep[22], the field order of
// eqx_replay_report, integers as doubles), per-client reports (cli[C][6], roster order:
// final_hf, accumulated_service, mean_service_rate, ttft p50, p90, count), and the series,
// each cut at win_cap windows: gpu_series (win[w][4]), counter_series (winc[w][C][4]),
// diff_series (diff[w][2]) and service_rate_series values (rate[C][win_cap]).
extern "C" int ref_replay_full(const eqxo_step_in* in, double max_sim_time_s, double ema_alpha, double window_s,
                               int64_t win_cap, double* rep, double* cli, double* win, double* winc, double* diff,
                               double* rate, char* err, int err_len) {
  try {
    const auto names = split_names(in->client_names, in->n_clients);
    const auto tags = split_names(in->tag_names, in->n_tags);
    Trace trace;
    for (int c = 0; c < in->n_clients; ++c) {
      ClientSpec cs;
      cs.client_id = names[c];
      cs.weight = in->weight[c];
      cs.arrivals.kind = ArrivalKind::Replay;
      trace.clients.push_back(cs);
    }
    double last = 0.0;
    for (int64_t r = 0; r < in->n_req; ++r) {
      Request q;
      q.id = in->id[r];
      q.client_id = names[static_cast<std::size_t>(in->client[r])];
      q.arrival_time_s = in->arrival[r];
      q.input_tokens = in->in_tokens[r];
      q.true_output_tokens = in->true_out[r];
      if (in->tag[r] >= 0) q.category_tag = tags[static_cast<std::size_t>(in->tag[r])];
      last = q.arrival_time_s;
      trace.requests.push_back(q);
    }
    trace.duration_s = in->duration_s > 0.0 ? in->duration_s : last;
    EngineConfig cfg;
    cfg.policy.kind = static_cast<PolicyKind>(in->kind);
    cfg.policy.equinox.alpha = in->alpha;
    cfg.policy.equinox.delta = in->delta;
    cfg.policy.equinox.output_weight = in->output_weight;
    cfg.policy.equinox.norm_mode = in->norm_mode == EQXO_NORM_NONE ? NormMode::None : NormMode::MaxOverClients;
    cfg.policy.vtc_use_prediction = in->vtc_use_prediction != 0;
    cfg.policy.counter_lift = in->counter_lift != 0;
    cfg.perf.max_batch = in->max_batch;
    cfg.perf.mem_per_token_bytes = in->mem_per_token_bytes;
    cfg.perf.mem_capacity_bytes = in->mem_capacity_bytes;
    cfg.backfill = in->backfill != 0;
    cfg.max_sim_time_s = max_sim_time_s;
    cfg.ema_alpha = ema_alpha;
    cfg.report_window_s = window_s;
    GpuProfile profile;
    for (int e = 0; e < in->n_profile; ++e)
      profile.entries.push_back({in->prof_upper[e], in->prof_lat[e], in->prof_util[e], in->prof_tps[e]});
    std::unique_ptr<Predictor> predictor;
    if (in->pred_kind == EQXO_PRED_MOPE) {
      predictor = std::make_unique<MopePredictor>(model_from(in->mope, tags, in->tag_row, in->n_tags));
    } else if (in->pred_kind == EQXO_PRED_NOISY) {
      predictor = std::make_unique<NoisyOraclePredictor>(in->noisy_l1, in->noisy_seed);
    } else {
      predictor = std::make_unique<OraclePredictor>();
    }
    const SimResult res = run_simulation(trace, cfg, *predictor, profile);
    const SimReport r = build_report(trace, res, cfg.policy.equinox.output_weight, cfg.report_window_s);
    const std::size_t C = trace.clients.size();
    std::size_t n_rate = 0;
    for (const auto& kv : r.per_client) n_rate = std::max(n_rate, kv.second.service_rate_series.size());
    const double v[22] = {r.max_diff,
                          r.avg_diff,
                          r.var_diff,
                          r.jain_hf,
                          r.jain_ttft_p90,
                          r.throughput_tps,
                          r.mean_gpu_util,
                          r.ttft_overall.p50,
                          r.ttft_overall.p90,
                          r.latency_overall.p50,
                          r.latency_overall.p90,
                          static_cast<double>(r.ttft_overall.count),
                          static_cast<double>(r.latency_overall.count),
                          r.sim_end_s,
                          res.busy_ms_total,
                          res.overhead_ms_total,
                          static_cast<double>(r.completed),
                          static_cast<double>(r.rejected),
                          static_cast<double>(r.total_completed_tokens),
                          static_cast<double>(res.gpu_series.size()),
                          static_cast<double>(r.diff_series.size()),
                          static_cast<double>(n_rate)};
    std::memcpy(rep, v, sizeof(v));
    for (std::size_t c = 0; c < C; ++c) {
      const ClientReport& pc = r.per_client.at(names[c]);
      double* o = cli + 6 * c;
      o[0] = res.final_hf[c];
      o[1] = pc.accumulated_service;
      o[2] = pc.mean_service_rate;
      o[3] = pc.ttft.p50;
      o[4] = pc.ttft.p90;
      o[5] = static_cast<double>(pc.ttft.count);
      for (std::size_t w = 0; w < pc.service_rate_series.size() && static_cast<int64_t>(w) < win_cap; ++w)
        rate[c * static_cast<std::size_t>(win_cap) + w] = pc.service_rate_series[w].value;
    }
    for (std::size_t w = 0; w < res.gpu_series.size() && static_cast<int64_t>(w) < win_cap; ++w) {
      const GpuWindowSample& g = res.gpu_series[w];
      win[4 * w + 0] = g.time_s;
      win[4 * w + 1] = g.busy_ms;
      win[4 * w + 2] = g.overhead_ms;
      win[4 * w + 3] = g.gpu_util;
    }
    for (std::size_t k = 0; k < res.counter_series.size(); ++k) {
      const std::size_t w = k / C;
      if (static_cast<int64_t>(w) >= win_cap) break;
      const CounterSample& cs = res.counter_series[k];
      double* o = winc + 4 * (w * C + cs.client_index);
      o[0] = cs.ufc;
      o[1] = cs.rfc;
      o[2] = cs.hf;
      o[3] = cs.service_cum;
    }
    for (std::size_t w = 0; w < r.diff_series.size() && static_cast<int64_t>(w) < win_cap; ++w) {
      diff[2 * w] = r.diff_series[w].time_s;
      diff[2 * w + 1] = r.diff_series[w].value;
    }
    return 0;
  } catch (const std::exception& e) {
    set_err(err, err_len, e.what());
    return 1;
  }
}

// ---- traces ------------------------------------------------------------
// ref_trace_load -- load_trace (workload.cpp:312-400) + trace_hash; columns into caller arrays
// of capacity cap (n returned even when larger), roster / tag strings NUL-packed.  Returns 0, or
// 1 with the ParseError / ConfigError message in err.
extern "C" int ref_trace_load(const char* path, int64_t cap, int64_t* n, int32_t* client, double* arrival,
                              int32_t* in_tokens, int32_t* out_tokens, char* tags, int64_t tags_cap,
                              char* names, int64_t names_cap, int32_t* n_clients, int32_t* n_warnings,
                              double* duration, char* hash, char* err, int err_len) {
  try {
    const Trace t = load_trace(path);
    *n = static_cast<int64_t>(t.requests.size());
    *n_clients = static_cast<int32_t>(t.clients.size());
    *n_warnings = static_cast<int32_t>(t.warnings.size());
    *duration = t.duration_s;
    std::string nb, tb;
    for (const auto& c : t.clients) nb += c.client_id + std::string(1, '\0');
    for (int64_t i = 0; i < *n && i < cap; ++i) {
      const Request& r = t.requests[static_cast<std::size_t>(i)];
      if (r.id != i) throw EngineError("load_trace ids are not positions");
      int32_t ci = -1;
      for (std::size_t c = 0; c < t.clients.size(); ++c)
        if (t.clients[c].client_id == r.client_id) ci = static_cast<int32_t>(c);
      client[i] = ci;
      arrival[i] = r.arrival_time_s;
      in_tokens[i] = r.input_tokens;
      out_tokens[i] = r.true_output_tokens;
      tb += r.category_tag + std::string(1, '\0');
    }
    std::memcpy(names, nb.data(), std::min<std::size_t>(nb.size(), static_cast<std::size_t>(names_cap)));
    std::memcpy(tags, tb.data(), std::min<std::size_t>(tb.size(), static_cast<std::size_t>(tags_cap)));
    const std::string h = trace_hash(t);
    std::memcpy(hash, h.c_str(), 17);
    return 0;
  } catch (const std::exception& e) {
    set_err(err, err_len, e.what());
    return 1;
  }
}

// ref_scenario_csv -- generate_scenario (workload.cpp:254-298) written with write_trace_csv to
// path; hash = trace_hash of the generated trace.
extern "C" int ref_scenario_csv(const char* preset, uint64_t seed, double duration_s, const char* path, char* hash,
                                char* err, int err_len) {
  try {
    const Trace t = generate_scenario(std::string_view(preset), seed, duration_s);
    std::ofstream out(path, std::ios::binary);
    write_trace_csv(t, out);
    out.close();
    const std::string h = trace_hash(t);
    std::memcpy(hash, h.c_str(), 17);
    return 0;
  } catch (const std::exception& e) {
    set_err(err, err_len, e.what());
    return 1;
  }
}

// The whole SimResult of run_simulation (engine.cpp:119-146) with its event log: per entry the
// kind as EQX_EV_* (admitted 1, rejected 2, arrived 3, first_token 4, completed 5), request
// id, time and the payload fields as include/eqx.h lays them out (i0: input / predicted /
// output tokens; d0..d2: predicted_latency_ms, or latency_s / tps / gpu_util), the profile
// after update_map (prof[3][P]: latency_ms, gpu_util, tps), final clients (cl[C][5]: ufc,
// rfc, counter, accumulated_service, backlogged) and totals (sim_end, busy, overhead, max resident KV
// tokens, completed, rejected, clamps).  Returns the number of log entries or -1.
extern "C" int64_t ref_replay_log(const eqxo_step_in* in, double max_sim_time_s, double ema_alpha, double window_s,
                                  int64_t cap, int64_t* id, int32_t* kind, double* t, int32_t* i0, double* d0,
                                  double* d1, double* d2, double* prof, double* cl, double* tot, char* err,
                                  int err_len) {
  try {
    const auto names = split_names(in->client_names, in->n_clients);
    const auto tags = split_names(in->tag_names, in->n_tags);
    Trace trace;
    for (int c = 0; c < in->n_clients; ++c) {
      ClientSpec cs;
      cs.client_id = names[c];
      cs.weight = in->weight[c];
      cs.arrivals.kind = ArrivalKind::Replay;
      trace.clients.push_back(cs);
    }
    double last = 0.0;
    for (int64_t r = 0; r < in->n_req; ++r) {
      Request q;
      q.id = in->id[r];
      q.client_id = names[static_cast<std::size_t>(in->client[r])];
      q.arrival_time_s = in->arrival[r];
      q.input_tokens = in->in_tokens[r];
      q.true_output_tokens = in->true_out[r];
      if (in->tag[r] >= 0) q.category_tag = tags[static_cast<std::size_t>(in->tag[r])];
      last = q.arrival_time_s;
      trace.requests.push_back(q);
    }
    trace.duration_s = in->duration_s > 0.0 ? in->duration_s : last;
    EngineConfig cfg;
    cfg.policy.kind = static_cast<PolicyKind>(in->kind);
    cfg.policy.equinox.alpha = in->alpha;
    cfg.policy.equinox.delta = in->delta;
    cfg.policy.equinox.output_weight = in->output_weight;
    cfg.policy.equinox.norm_mode = in->norm_mode == EQXO_NORM_NONE ? NormMode::None : NormMode::MaxOverClients;
    cfg.policy.vtc_use_prediction = in->vtc_use_prediction != 0;
    cfg.policy.counter_lift = in->counter_lift != 0;
    cfg.perf.max_batch = in->max_batch;
    cfg.perf.mem_per_token_bytes = in->mem_per_token_bytes;
    cfg.perf.mem_capacity_bytes = in->mem_capacity_bytes;
    cfg.backfill = in->backfill != 0;
    cfg.max_sim_time_s = max_sim_time_s;
    cfg.ema_alpha = ema_alpha;
    cfg.report_window_s = window_s;
    cfg.prediction_overhead_ms = in->prediction_overhead_ms;
    GpuProfile profile;
    for (int e = 0; e < in->n_profile; ++e)
      profile.entries.push_back({in->prof_upper[e], in->prof_lat[e], in->prof_util[e], in->prof_tps[e]});
    std::unique_ptr<Predictor> predictor;
    if (in->pred_kind == EQXO_PRED_MOPE) {
      predictor = std::make_unique<MopePredictor>(model_from(in->mope, tags, in->tag_row, in->n_tags));
    } else if (in->pred_kind == EQXO_PRED_NOISY) {
      predictor = std::make_unique<NoisyOraclePredictor>(in->noisy_l1, in->noisy_seed);
    } else {
      predictor = std::make_unique<OraclePredictor>();
    }
    const SimResult res = run_simulation(trace, cfg, *predictor, profile);
    int64_t n = 0;
    for (const auto& e : res.log.entries) {
      if (n < cap) {
        int k = 0, a = 0;
        double x = 0.0, y = 0.0, z = 0.0;
        switch (e.event) {
          case LogEvent::Admitted: k = 1; a = e.predicted_output_tokens; x = e.predicted_latency_ms; break;
          case LogEvent::Rejected: k = 2; a = e.input_tokens; break;
          case LogEvent::Arrived: k = 3; a = e.input_tokens; break;
          case LogEvent::FirstToken: k = 4; break;
          case LogEvent::Completed: k = 5; a = e.output_tokens; x = e.latency_s; y = e.tps; z = e.gpu_util; break;
        }
        id[n] = e.request_id;
        kind[n] = k;
        t[n] = e.time_s;
        i0[n] = a;
        d0[n] = x;
        d1[n] = y;
        d2[n] = z;
      }
      ++n;
    }
    const std::size_t P = res.profile.entries.size();
    for (std::size_t e = 0; e < P; ++e) {
      prof[e] = res.profile.entries[e].latency_ms;
      prof[P + e] = res.profile.entries[e].gpu_util;
      prof[2 * P + e] = res.profile.entries[e].tps;
    }
    for (std::size_t c = 0; c < res.final_clients.size(); ++c) {
      cl[5 * c] = res.final_clients[c].ufc;
      cl[5 * c + 1] = res.final_clients[c].rfc;
      cl[5 * c + 2] = res.final_clients[c].counter;
      cl[5 * c + 3] = res.final_clients[c].accumulated_service;
      cl[5 * c + 4] = res.final_clients[c].backlogged ? 1.0 : 0.0;
    }
    tot[0] = res.sim_end_s;
    tot[1] = res.busy_ms_total;
    tot[2] = res.overhead_ms_total;
    tot[3] = static_cast<double>(res.max_resident_kv_tokens);
    tot[4] = static_cast<double>(res.completed);
    tot[5] = static_cast<double>(res.rejected);
    tot[6] = static_cast<double>(res.counter_clamps);
    return n;
  } catch (const std::exception& e) {
    if (err && err_len > 0) std::snprintf(err, err_len, "%s", e.what());
    return -1;
  }
}
