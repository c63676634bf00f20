// engine_b200.cpp -- the reference engine's translation unit (proj/src/engine.cpp) replaced by
// the B200 path: `equinox::run_simulation` with the reference's signature (engine.hpp:94-95),
// whose discrete-event loop runs on the GPU through the C ABI (include/eqx.h, eqx_replay with
// the whole event log).  Linked in place of engine.cpp, every other reference translation unit
// (workload, predictor, scheduler, metrics, run_config, experiments, the pybind module) calls
// it unchanged -- this is the drop-in INTEGRATION.md section 1 describes.
//
// What stays on the host: parameter validation (the reference's own validate() rules, same
// exception types and messages), the caller's Predictor (a virtual plugin the engine calls once
// per request in arrival order, engine.cpp:177-179 -- its predictions go to the device as a
// column), and the conversion of the device's column outputs into SimResult.  Everything the
// engine computes -- drain_arrivals, admit_requests, run_iteration, complete_finished, the
// counters, update_map, the window samples -- runs in replay_kernel (csrc/eqx_replay.cu).
//
// The remaining engine.cpp entry points (EngineConfig::validate, log_event_name,
// EventLog::to_ndjson, measure_actuals) are defined here as well, with the reference's
// behaviour, so that this file replaces engine.cpp one for one.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "eqx.h"
#include "equinox/engine.hpp"
#include "equinox/errors.hpp"
#include "json.hpp"

namespace equinox {

void EngineConfig::validate() const {
  perf.validate();
  policy.equinox.validate();
  if (report_window_s <= 0.0) throw ConfigError("report_window_s must be > 0");
  if (max_sim_time_s < 0.0) throw ConfigError("max_sim_time_s must be >= 0");
  if (ema_alpha <= 0.0 || ema_alpha > 1.0) throw ConfigError("ema_alpha must lie in (0, 1]");
  if (prediction_overhead_ms < 0.0) throw ConfigError("prediction_overhead_ms must be >= 0");
}

std::string_view log_event_name(LogEvent e) {
  static constexpr std::string_view names[] = {"arrived", "admitted", "first_token", "completed", "rejected"};
  const auto i = static_cast<std::size_t>(e);
  return i < 5 ? names[i] : std::string_view("unknown");
}

// One JSON object per line; nlohmann's object keys are ordered, so the bytes depend only on the
// fields each event kind carries (engine.hpp:39-51).
std::string EventLog::to_ndjson() const {
  std::string out;
  for (const LogEntry& e : entries) {
    nlohmann::json j = {{"time_s", e.time_s},
                        {"request_id", e.request_id},
                        {"client_id", e.client_id},
                        {"event", log_event_name(e.event)}};
    if (e.event == LogEvent::Arrived || e.event == LogEvent::Rejected || e.event == LogEvent::Completed)
      j["input_tokens"] = e.input_tokens;
    if (e.event == LogEvent::Admitted) {
      j["predicted_output_tokens"] = e.predicted_output_tokens;
      j["predicted_latency_ms"] = e.predicted_latency_ms;
    } else if (e.event == LogEvent::Completed) {
      j["output_tokens"] = e.output_tokens;
      j["latency_s"] = e.latency_s;
      j["tps"] = e.tps;
      j["gpu_util"] = e.gpu_util;
    }
    out += j.dump();
    out += '\n';
  }
  return out;
}

RequestActuals measure_actuals(const EventLog& log, std::int64_t request_id) {
  const LogEntry *arrived = nullptr, *admitted = nullptr, *completed = nullptr;
  for (const LogEntry& e : log.entries) {
    if (e.request_id != request_id) continue;
    if (e.event == LogEvent::Arrived) arrived = &e;
    else if (e.event == LogEvent::Admitted) admitted = &e;
    else if (e.event == LogEvent::Completed) completed = &e;
  }
  if (!arrived || !admitted || !completed)
    throw EngineError("request " + std::to_string(request_id) + " has no completed lifecycle in the log");
  RequestActuals a;
  a.output_tokens = completed->output_tokens;
  a.gpu_util = completed->gpu_util;
  a.latency_s = completed->time_s - arrived->time_s;
  a.exec_s = completed->time_s - admitted->time_s;
  a.tps = (static_cast<double>(arrived->input_tokens) + a.output_tokens) / a.exec_s;
  return a;
}

namespace {

// One context per call: runs are independent (the experiment runner calls run_simulation from
// several threads, experiments.cpp:134-162), so nothing is shared between calls.
struct Ctx {
  eqx_ctx* p = nullptr;
  Ctx() {
    int dev = 0;
    if (const char* d = std::getenv("EQX_DEVICE")) dev = std::atoi(d);
    if (eqx_ctx_create(dev, &p) != EQX_OK) {
      const char* m = eqx_last_error(nullptr);
      throw EngineError(std::string("B200 engine: ") + (m ? m : "no CUDA device"));
    }
  }
  ~Ctx() { eqx_ctx_destroy(p); }
  void check(eqx_status st) const {
    if (st == EQX_OK) return;
    const std::string m = eqx_last_error(p) ? eqx_last_error(p) : "";
    if (st == EQX_ERR_CONFIG) throw ConfigError(m);
    if (st == EQX_ERR_PARSE) throw ParseError(m);
    throw EngineError(m);
  }
};

LogEvent event_of(int32_t k) {
  switch (k) {
    case EQX_EV_ADMITTED: return LogEvent::Admitted;
    case EQX_EV_REJECTED: return LogEvent::Rejected;
    case EQX_EV_ARRIVED: return LogEvent::Arrived;
    case EQX_EV_FIRST_TOKEN: return LogEvent::FirstToken;
    default: return LogEvent::Completed;
  }
}

}  // namespace

SimResult run_simulation(const Trace& trace, const EngineConfig& config, Predictor& predictor,
                         const GpuProfile& initial_profile) {
  // ---- the reference's construction-time checks, in its order (engine.cpp:96-118) ----
  std::vector<ClientState> roster;
  roster.reserve(trace.clients.size());
  for (const ClientSpec& spec : trace.clients) {
    ClientState c;
    c.client_id = spec.client_id;
    c.weight = spec.weight;
    roster.push_back(std::move(c));
  }
  { SchedulerPolicy check(config.policy, roster); }  // EquinoxParams + weights (scheduler.cpp:92-100)
  config.validate();
  if (initial_profile.empty()) throw ConfigError("engine needs a non-empty GPU profile");
  std::map<std::string, int32_t> index;
  for (std::size_t i = 0; i < trace.clients.size(); ++i) index[trace.clients[i].client_id] = static_cast<int32_t>(i);
  const int64_t n = static_cast<int64_t>(trace.requests.size());
  std::vector<int32_t> client(n), in_tok(n), true_out(n), predicted(n);
  std::vector<double> arrival(n);
  for (int64_t i = 0; i < n; ++i) {
    const Request& r = trace.requests[i];
    const auto it = index.find(r.client_id);
    if (it == index.end())
      throw ConfigError("request " + std::to_string(r.id) + " references unknown client '" + r.client_id + "'");
    client[i] = it->second;
    arrival[i] = r.arrival_time_s;
    in_tok[i] = r.input_tokens;
    true_out[i] = r.true_output_tokens;
  }
  SimResult result;
  result.profile = initial_profile;
  const int32_t C = static_cast<int32_t>(roster.size());
  if (C == 0) {  // nothing can arrive: the loop never admits (the horizon still advances nothing)
    result.sim_end_s = 0.0;
    return result;
  }
  // the caller's predictor, once per request in arrival order (engine.cpp:177-179)
  for (int64_t i = 0; i < n; ++i) predicted[i] = predictor.predict(trace.requests[i]);

  // ---- the B200 engine ----
  Ctx ctx;
  const PolicySpec& ps = config.policy;
  eqx_policy pol{};
  pol.kind = ps.kind == PolicyKind::Fcfs ? EQX_FCFS : ps.kind == PolicyKind::Vtc ? EQX_VTC : EQX_EQUINOX;
  pol.alpha = ps.equinox.alpha;
  pol.delta = ps.equinox.delta;
  pol.output_weight = ps.equinox.output_weight;
  pol.norm_mode = ps.equinox.norm_mode == NormMode::None ? EQX_NORM_NONE : EQX_NORM_MAX_OVER_CLIENTS;
  pol.vtc_use_prediction = ps.vtc_use_prediction ? 1 : 0;
  pol.counter_lift = ps.counter_lift ? 1 : 0;
  pol.backfill = config.backfill ? 1 : 0;
  ctx.check(eqx_set_policy(ctx.p, &pol));
  const eqx_perf perf{config.perf.max_batch, config.perf.mem_per_token_bytes, config.perf.mem_capacity_bytes};
  ctx.check(eqx_set_perf(ctx.p, &perf));
  ctx.check(eqx_set_timing(ctx.p, config.perf.prefill_linear_ms, config.perf.prefill_quad_ms,
                           config.perf.decode_base_ms, config.perf.decode_per_ctx_ms, config.perf.refresh_ms));
  const std::size_t P = initial_profile.entries.size();
  std::vector<int32_t> up(P);
  std::vector<double> lat(P), util(P), tps(P);
  for (std::size_t e = 0; e < P; ++e) {
    up[e] = initial_profile.entries[e].bucket_upper;
    lat[e] = initial_profile.entries[e].latency_ms;
    util[e] = initial_profile.entries[e].gpu_util;
    tps[e] = initial_profile.entries[e].tps;
  }
  const eqx_profile prof{static_cast<int32_t>(P), up.data(), lat.data(), util.data(), tps.data()};
  ctx.check(eqx_set_profile(ctx.p, &prof));
  eqx_predictor pred{};
  pred.kind = EQX_PRED_ORACLE;  // unused: the caller's predictions come as a column
  ctx.check(eqx_set_predictor(ctx.p, &pred));
  std::string names;
  std::vector<double> weight(C);
  for (int32_t c = 0; c < C; ++c) {
    names += roster[c].client_id;
    names.push_back('\0');
    weight[c] = roster[c].weight;
  }
  ctx.check(eqx_set_clients(ctx.p, C, names.data(), weight.data(), nullptr, nullptr, nullptr, nullptr));

  // window samples: one per report window up to the horizon, plus the flushed partial one and
  // the windows the last iteration crosses; retried with the exact count if that falls short
  const double horizon = config.max_sim_time_s > 0.0 ? config.max_sim_time_s : trace.duration_s;
  int64_t win_cap = static_cast<int64_t>(std::ceil(std::max(horizon, 0.0) / config.report_window_s)) + 8;
  const int64_t ev_cap = 4 * n + 4;  // arrived + admitted + first_token + completed per request
  const int64_t row_off[2] = {0, n};
  const double alpha = ps.equinox.alpha, duration = trace.duration_s;
  std::vector<int64_t> ev_id(ev_cap);
  std::vector<int32_t> ev_kind(ev_cap), ev_i0(ev_cap);
  std::vector<double> ev_time(ev_cap), ev_d0(ev_cap), ev_d1(ev_cap), ev_d2(ev_cap);
  std::vector<double> ufc(C), rfc(C), counter(C), prof_out(3 * P), win, win_clients;
  std::vector<eqx_replay_client> cl(C);
  eqx_replay_report rep{};
  int64_t n_events = 0, clamps = 0, completed = 0;
  int32_t status = 0;
  double sim_end = 0.0;
  for (;;) {
    win.assign(4 * win_cap, 0.0);
    win_clients.assign(4 * win_cap * C, 0.0);
    eqx_replays R{};
    R.n_replays = 1;
    R.row_off = row_off;
    R.client = client.data();
    R.arrival_s = arrival.data();
    R.input_tokens = in_tok.data();
    R.true_output_tokens = true_out.data();
    R.alpha = &alpha;
    R.max_sim_time_s = config.max_sim_time_s;
    R.ema_alpha = config.ema_alpha;
    R.ev_cap = ev_cap;
    R.report_window_s = config.report_window_s;
    R.win_cap = win_cap;
    R.duration_s = &duration;
    R.prediction_overhead_ms = config.prediction_overhead_ms;
    R.predicted = predicted.data();
    R.log_all = 1;
    eqx_replay_out O{};
    O.n_events = &n_events;
    O.ev_id = ev_id.data();
    O.ev_kind = ev_kind.data();
    O.ev_time = ev_time.data();
    O.ufc = ufc.data();
    O.rfc = rfc.data();
    O.counter = counter.data();
    O.completed = &completed;
    O.sim_end = &sim_end;
    O.counter_clamps = &clamps;
    O.status = &status;
    O.report = &rep;
    O.clients = cl.data();
    O.win = win.data();
    O.win_clients = win_clients.data();
    O.ev_i0 = ev_i0.data();
    O.ev_d0 = ev_d0.data();
    O.ev_d1 = ev_d1.data();
    O.ev_d2 = ev_d2.data();
    O.profile = prof_out.data();
    ctx.check(eqx_replay(ctx.p, &R, &O));
    if (status == 2)  // run_iteration's KV bound (engine.cpp:296-300)
      throw EngineError("KV memory bound violated: " + std::to_string(rep.max_resident_kv_tokens) +
                        " resident tokens exceed capacity");
    if (rep.n_windows <= win_cap) break;
    win_cap = rep.n_windows;
  }
  if (n_events > ev_cap) throw EngineError("B200 engine: event log overflow");

  // ---- device columns -> SimResult ----
  result.log.entries.resize(static_cast<std::size_t>(n_events));
  for (int64_t k = 0; k < n_events; ++k) {
    const Request& r = trace.requests[static_cast<std::size_t>(ev_id[k])];  // ids are trace positions
    LogEntry& e = result.log.entries[static_cast<std::size_t>(k)];
    e.time_s = ev_time[k];
    e.request_id = r.id;
    e.client_id = r.client_id;
    e.event = event_of(ev_kind[k]);
    switch (e.event) {
      case LogEvent::Arrived:
      case LogEvent::Rejected: e.input_tokens = ev_i0[k]; break;
      case LogEvent::Admitted:
        e.predicted_output_tokens = ev_i0[k];
        e.predicted_latency_ms = ev_d0[k];
        break;
      case LogEvent::Completed:
        e.input_tokens = r.input_tokens;
        e.output_tokens = ev_i0[k];
        e.latency_s = ev_d0[k];
        e.tps = ev_d1[k];
        e.gpu_util = ev_d2[k];
        break;
      case LogEvent::FirstToken: break;
    }
  }
  const int64_t nw = rep.n_windows;
  result.gpu_series.resize(static_cast<std::size_t>(nw));
  result.counter_series.resize(static_cast<std::size_t>(nw * C));
  for (int64_t w = 0; w < nw; ++w) {
    GpuWindowSample& g = result.gpu_series[static_cast<std::size_t>(w)];
    g.time_s = win[4 * w];
    g.busy_ms = win[4 * w + 1];
    g.overhead_ms = win[4 * w + 2];
    g.gpu_util = win[4 * w + 3];
    for (int32_t c = 0; c < C; ++c) {
      const double* x = &win_clients[4 * (w * C + c)];
      CounterSample& s = result.counter_series[static_cast<std::size_t>(w * C + c)];
      s.time_s = g.time_s;
      s.client_index = static_cast<std::size_t>(c);
      s.ufc = x[0];
      s.rfc = x[1];
      s.hf = x[2];
      s.service_cum = x[3];
    }
  }
  result.final_clients = roster;
  result.final_hf.resize(C);
  for (int32_t c = 0; c < C; ++c) {
    ClientState& s = result.final_clients[c];
    s.ufc = ufc[c];
    s.rfc = rfc[c];
    s.counter = counter[c];
    s.accumulated_service = cl[c].accumulated_service;
    s.backlogged = cl[c].backlogged != 0;
    result.final_hf[c] = cl[c].final_hf;
  }
  for (std::size_t e = 0; e < P; ++e) {
    result.profile.entries[e].latency_ms = prof_out[e];
    result.profile.entries[e].gpu_util = prof_out[P + e];
    result.profile.entries[e].tps = prof_out[2 * P + e];
  }
  result.sim_end_s = sim_end;
  result.busy_ms_total = rep.busy_ms_total;
  result.overhead_ms_total = rep.overhead_ms_total;
  result.max_resident_kv_tokens = rep.max_resident_kv_tokens;
  result.completed = completed;
  result.rejected = rep.rejected;
  result.counter_clamps = clamps;
  return result;
}

}  // namespace equinox
