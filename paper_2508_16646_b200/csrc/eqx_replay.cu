// eqx_replay.cu -- many independent engine replays per launch (SURVEY.md 8f row 3, config 5:
// the Holistic-Fairness alpha sweep, 1024 replays).
//
// One warp runs one whole replay: the reference's SimulationRun::run loop (engine.cpp:
// 119-146) with drain_arrivals (:171-197), admit_requests (:207-271), run_iteration
// (:273-325) and complete_finished (:327-375), and the SchedulerPolicy / GpuProfile
// operations they call, in the reference's order and FP64 operation order.  Replays are
// independent, so the GPU runs them side by side (148 SMs x many warps); each replay keeps its
// ledger, profile copy, per-client FIFO cursors and batch in its own slice of global scratch.
// The scalar engine logic runs uniformly on all 32 lanes (identical values, identical stores:
// no divergence between replays of a warp, as one-thread-per-replay had), and the loops over
// batch members (reservations, decode step, completion scan and erase) are split across lanes.
// Reporting windows (advance_clock's samples) do not change the schedule and are not produced.
#include <cstdint>

#include "eqx_device.cuh"
#include "eqx_kernels.h"

namespace eqx {

namespace {

__device__ __forceinline__ bool key_better(double k, double a, uint32_t o, double bk, double ba, uint32_t bo) {
  // select_next (scheduler.cpp:139-153): key, then head arrival, then client_id bytes
  if (k < bk) return true;
  if (bk < k) return false;
  if (a < ba) return true;
  if (ba < a) return false;
  return o < bo;
}

}  // namespace

__device__ __forceinline__ int64_t warp_sum64(int64_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(128) replay_kernel(const ReplayArgs A) {
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= A.n_replays) return;  // warp-uniform
  const ModelTables& M = *A.model;
  const Policy P = A.pol;
  const int32_t C = A.C;
  const int64_t t0 = A.row_off[r], n = A.row_off[r + 1] - t0;
  const int32_t* client = A.client + t0;
  const double* arrival = A.arrival + t0;
  const int32_t* in_tok = A.in_tok + t0;
  const int32_t* true_out = A.true_out + t0;
  const uint8_t* tag = A.tag + t0;
  const int64_t* id = A.id + t0;
  // per-replay scratch
  int32_t* crow = A.crow + t0;                          // rows grouped by client, FIFO order
  int32_t* f_pred = A.f_pred + t0;                      // frozen prediction records
  double* f_preds = A.f_preds + t0;
  double* f_rfc = A.f_rfc + t0;
  double* f_ttft = A.f_ttft + t0;
  for (int64_t i = lane; i < n; i += 32) f_ttft[i] = -1.0;
  int64_t completed_tokens = 0;
  // Ledger, FIFO cursors and profile are private per lane (identical copies, updated uniformly),
  // so the read-modify-write engine steps need no intra-warp synchronisation; the batch lives
  // in global scratch, split across lanes.
  ReplayClient cl[kMaxReplayClients];
  double prof[4 * kMaxProfile];  // lat | util | tps | pred_s
  ReplayMember* mb = A.mb + static_cast<int64_t>(r) * P.max_batch;
  const int np = M.n_prof;
  for (int e = 0; e < np; ++e) {
    prof[e] = M.prof_lat[e];
    prof[kMaxProfile + e] = M.prof_util[e];
    prof[2 * kMaxProfile + e] = M.prof_tps[e];
    prof[3 * kMaxProfile + e] = M.prof_pred_s[e];
  }
  struct {
    double alpha, beta;
  } const eq{A.alpha[r], __dsub_rn(1.0, A.alpha[r])};  // EquinoxParams::beta()
  // roster (engine.cpp:148-157): zero ledgers; client-grouped row lists
  for (int c = 0; c < C; ++c) {
    ReplayClient z{};
    z.weight = A.weight[c];
    z.order = A.order[c];
    cl[c] = z;
  }
  for (int64_t i = 0; i < n; ++i) cl[client[i]].qend += 1;  // counts -> offsets
  {
    int32_t run = 0;
    for (int c = 0; c < C; ++c) {
      const int32_t k = cl[c].qend;
      cl[c].qbase = run;
      cl[c].qhead = run;
      cl[c].qend = run;  // drained so far
      run += k;
    }
    for (int64_t i = 0; i < n; ++i) {  // stable placement through a per-client cursor
      ReplayClient& x = cl[client[i]];
      crow[x.qend++] = static_cast<int32_t>(i);
    }
    for (int c = 0; c < C; ++c) cl[c].qend = cl[c].qbase;
  }
  const double max_sim = A.max_sim_time_s > 0.0 ? A.max_sim_time_s : (n > 0 ? arrival[n - 1] : 0.0);
  double now = 0.0, busy_cum = 0.0, ovh_cum = 0.0;
  int64_t arrival_idx = 0, total_queued = 0, n_ev = 0, completed = 0, clamps = 0;
  int32_t members = 0;
  bool comp_changed = false;
  int32_t status = 0;
  int64_t* ev_id = A.ev_id + static_cast<int64_t>(r) * A.ev_cap;
  int32_t* ev_kind = A.ev_kind + static_cast<int64_t>(r) * A.ev_cap;
  double* ev_time = A.ev_time + static_cast<int64_t>(r) * A.ev_cap;
  auto log_ev = [&](int64_t rid, int32_t kind) {
    if (n_ev < A.ev_cap) {
      ev_id[n_ev] = rid;
      ev_kind[n_ev] = kind;
      ev_time[n_ev] = now;
    }
    ++n_ev;
  };
  auto entry_for = [&](int32_t out) {  // gpu_model.cpp:74-80
    int b = np - 1;
    for (int e = np - 1; e >= 0; --e)
      if (out <= M.prof_upper[e]) b = e;
    return b;
  };
  auto on_activated = [&](int c) {  // scheduler.cpp:235-253
    if (!A.counter_lift) return;
    double mu = INFINITY, mr = INFINITY, mc = INFINITY;
    bool any = false;
    for (int i = 0; i < C; ++i) {
      if (i == c || !cl[i].backlogged) continue;
      any = true;
      mu = fmin(mu, cl[i].ufc);
      mr = fmin(mr, cl[i].rfc);
      mc = fmin(mc, cl[i].counter);
    }
    if (!any) return;
    if (cl[c].ufc < mu) cl[c].ufc = mu;
    if (cl[c].rfc < mr) cl[c].rfc = mr;
    if (cl[c].counter < mc) cl[c].counter = mc;
  };
  auto drain = [&](double upto) {  // engine.cpp:171-197 (prediction_overhead_ms = 0)
    while (arrival_idx < n && __dadd_rn(arrival[arrival_idx], 0.0) <= upto) {
      const int64_t i = arrival_idx++;
      const int c = client[i];
      const double w = cl[c].weight;
      const Scored s = score_request(M, P, 0.0, in_tok[i], tag[i], true_out[i], id[i], 0.0, w);  // max(1, predict)
      const int b = entry_for(s.pred);  // map_metrics against the replay's current profile
      f_pred[i] = s.pred;
      f_preds[i] = prof[3 * kMaxProfile + b];
      f_rfc[i] = __dmul_rn(__dmul_rn(w, prof[2 * kMaxProfile + b]), prof[kMaxProfile + b]);
      if (cl[c].qend == cl[c].qhead && cl[c].running == 0) on_activated(c);
      cl[c].qend += 1;
      ++total_queued;
      cl[c].backlogged = 1;
    }
  };
  auto pop_head = [&](int c) {
    cl[c].qhead += 1;
    --total_queued;
    if (cl[c].qhead == cl[c].qend) cl[c].backlogged = 0;
  };
  auto admit = [&]() -> int64_t {  // engine.cpp:207-271
    int64_t new_prefill = 0;
    uint64_t skipped = 0;
    for (;;) {
      double mu = 0.0, mr = 0.0;  // backlogged_maxima (scheduler.cpp:40-48)
      const bool maxmode = P.kind == kEquinox && P.norm_mode == 0;
      if (maxmode)
        for (int i = 0; i < C; ++i)
          if (cl[i].backlogged) {
            if (mu < cl[i].ufc) mu = cl[i].ufc;
            if (mr < cl[i].rfc) mr = cl[i].rfc;
          }
      int best = -1;
      double bk = 0.0, ba = 0.0;
      uint32_t bo = 0;
      for (int i = 0; i < C; ++i) {
        if (cl[i].qhead == cl[i].qend || ((skipped >> (i & 63)) & 1u)) continue;
        double k;
        if (P.kind == kFcfs) k = 0.0;
        else if (P.kind == kVtc) k = cl[i].counter;
        else if (P.norm_mode == 1) k = __dadd_rn(__dmul_rn(eq.alpha, cl[i].ufc), __dmul_rn(eq.beta, cl[i].rfc));
        else {
          const double u = mu > 0.0 ? __ddiv_rn(cl[i].ufc, mu) : 0.0;
          const double v = mr > 0.0 ? __ddiv_rn(cl[i].rfc, mr) : 0.0;
          k = __dadd_rn(__dmul_rn(eq.alpha, u), __dmul_rn(eq.beta, v));
        }
        const double a = arrival[crow[cl[i].qhead]];
        if (best < 0 || key_better(k, a, cl[i].order, bk, ba, bo)) {
          best = i;
          bk = k;
          ba = a;
          bo = cl[i].order;
        }
      }
      if (best < 0) break;
      const int c = best;
      const int32_t row = crow[cl[c].qhead];
      const int32_t in = in_tok[row], pred = f_pred[row];
      // fits_alone (gpu_model.cpp:69-72): the can_fit test on an empty batch
      if (!((1 <= P.max_batch) && __dmul_rn(static_cast<double>(static_cast<int64_t>(in) + pred), P.m) <= P.M)) {
        log_ev(id[row], 2);
        pop_head(c);
        continue;
      }
      int64_t reserved = 0;  // BatchState::reserved_kv_tokens (gpu_model.cpp:40-46)
      for (int j = lane; j < members; j += 32)
        reserved += mb[j].in + (mb[j].reserved_out > mb[j].generated ? mb[j].reserved_out : mb[j].generated);
      reserved = warp_sum64(reserved);
      if (!((members + 1 <= P.max_batch) &&
            __dmul_rn(static_cast<double>(reserved + in + pred), P.m) <= P.M)) {  // can_fit
        if (P.backfill) {
          skipped |= 1ull << (c & 63);
          continue;
        }
        break;
      }
      pop_head(c);
      ReplayMember& m = mb[members++];
      m.row = row;
      m.client = c;
      m.in = in;
      m.generated = 0;
      m.reserved_out = pred;
      m.admit_s = now;
      m.busy_at = busy_cum;
      m.ovh_at = ovh_cum;
      comp_changed = true;
      cl[c].running += 1;
      new_prefill += in;
      // on_admit (scheduler.cpp:158-183) with ScheduleContext{now, now - arrival, prediction}
      const double w = cl[c].weight;
      const double tokens = __dadd_rn(static_cast<double>(in), __dmul_rn(P.ow, static_cast<double>(pred)));
      const double wait = __dsub_rn(now, arrival[row]);
      m.p_ufc = __ddiv_rn(__dmul_rn(w, tokens), __dadd_rn(1.0, __dmul_rn(P.delta, __dadd_rn(wait, f_preds[row]))));
      m.p_rfc = f_rfc[row];
      m.p_vtc = 0.0;
      cl[c].ufc = __dadd_rn(cl[c].ufc, m.p_ufc);
      cl[c].rfc = __dadd_rn(cl[c].rfc, m.p_rfc);
      if (P.kind == kVtc) {
        m.p_vtc = P.vtc_use_prediction ? __dmul_rn(w, tokens) : __dmul_rn(w, static_cast<double>(in));
        cl[c].counter = __dadd_rn(cl[c].counter, m.p_vtc);
      }
      log_ev(id[row], 1);
    }
    return new_prefill;
  };
  // ---- SimulationRun::run ----
  while (now < max_sim) {
    drain(now);
    if (members == 0 && total_queued == 0) {
      if (arrival_idx >= n) break;
      const double next_t = __dadd_rn(arrival[arrival_idx], 0.0);
      if (next_t >= max_sim) break;
      now = next_t;  // advance_clock(now, next_t, 0, 0)
      drain(now);
    }
    const int64_t new_prefill = admit();
    if (members == 0) continue;
    // ---- run_iteration (engine.cpp:273-325) ----
    int64_t resident = 0;
    for (int j = lane; j < members; j += 32) resident += mb[j].in + mb[j].generated;
    resident = warp_sum64(resident);
    const double p = static_cast<double>(new_prefill);
    double iter_ms = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(A.prefill_linear_ms, p), __dmul_rn(__dmul_rn(A.prefill_quad_ms, p), p)),
                                         A.decode_base_ms),
                               __dmul_rn(A.decode_per_ctx_ms, static_cast<double>(resident)));
    if (comp_changed) iter_ms = __dadd_rn(iter_ms, A.refresh_ms);
    const double overhead_ms = comp_changed ? A.refresh_ms : 0.0;
    const double busy_ms = __dsub_rn(iter_ms, overhead_ms);
    const double t_end = __dadd_rn(now, __ddiv_rn(iter_ms, 1000.0));
    busy_cum = __dadd_rn(busy_cum, busy_ms);
    ovh_cum = __dadd_rn(ovh_cum, overhead_ms);
    now = t_end;
    comp_changed = false;
    for (int j = lane; j < members; j += 32) {
      mb[j].generated += 1;
      if (mb[j].generated == 1) f_ttft[mb[j].row] = __dsub_rn(now, arrival[mb[j].row]);  // FirstToken
    }
    __syncwarp();
    if (P.kind == kVtc && !P.vtc_use_prediction) {  // on_tokens per client (scheduler.cpp:185-190)
      for (int c = 0; c < C; ++c) {
        int64_t t = 0;
        for (int j = lane; j < members; j += 32) t += mb[j].client == c ? 1 : 0;
        t = warp_sum64(t);
        if (t > 0) cl[c].counter = __dadd_rn(cl[c].counter, __dmul_rn(__dmul_rn(cl[c].weight, P.ow), static_cast<double>(t)));
      }
    }
    const int64_t res2 = resident + members;  // every resident request generated one token
    if (__dmul_rn(static_cast<double>(res2), P.m) > P.M) {  // KV memory bound violated
      status = 2;
      break;
    }
    drain(now);
    // ---- complete_finished (engine.cpp:327-375) ----
    // finished members are processed in batch order (ledger and update_map chains), then the
    // survivors are compacted in order (members.erase keeps the relative order)
    int32_t kept = 0;
    for (int base = 0; base < members; base += 32) {
      const int j = base + lane;
      ReplayMember mine{};
      bool fin = false;
      if (j < members) {
        mine = mb[j];
        fin = mine.generated >= true_out[mine.row];
      }
      unsigned fm = __ballot_sync(0xffffffffu, fin);
      while (fm) {
        const int src = __ffs(fm) - 1;
        fm &= fm - 1;
        const ReplayMember m = mb[base + src];
        const int c = m.client;
        const double w = cl[c].weight;
        const int32_t out = m.generated;
        const double latency_s = __dsub_rn(now, arrival[m.row]);
        const double exec_s = __dsub_rn(now, m.admit_s);
        const double tps = __ddiv_rn(__dadd_rn(static_cast<double>(m.in), static_cast<double>(out)), exec_s);
        const double busy_span = __dsub_rn(busy_cum, m.busy_at);
        const double ovh_span = __dsub_rn(ovh_cum, m.ovh_at);
        const double util = __ddiv_rn(busy_span, __dadd_rn(busy_span, ovh_span));
        ++completed;
        completed_tokens += static_cast<int64_t>(m.in) + out;
        // on_complete (scheduler.cpp:192-233)
        const double wt = __dadd_rn(static_cast<double>(m.in), __dmul_rn(P.ow, static_cast<double>(out)));
        const double wwt = __dmul_rn(w, wt);
        const double au = __ddiv_rn(wwt, __dadd_rn(1.0, __dmul_rn(P.delta, latency_s)));
        const double ar = __dmul_rn(__dmul_rn(w, tps), util);
        double u = __dadd_rn(cl[c].ufc, __dsub_rn(au, m.p_ufc));
        if (u < 0.0) {
          u = 0.0;
          ++clamps;
        }
        double v = __dadd_rn(cl[c].rfc, __dsub_rn(ar, m.p_rfc));
        if (v < 0.0) {
          v = 0.0;
          ++clamps;
        }
        cl[c].ufc = u;
        cl[c].rfc = v;
        if (P.kind == kVtc && P.vtc_use_prediction) {
          double k = __dadd_rn(cl[c].counter, __dsub_rn(wwt, m.p_vtc));
          if (k < 0.0) {
            k = 0.0;
            ++clamps;
          }
          cl[c].counter = k;
        }
        // update_map (predictor.cpp:372-383) with ObservedMetrics{out, latency_s * 1000, util, tps}
        const int e = entry_for(out);
        const double al = A.ema_alpha, bl = __dsub_rn(1.0, A.ema_alpha);
        const double nl = __dadd_rn(__dmul_rn(bl, prof[e]), __dmul_rn(al, __dmul_rn(latency_s, 1000.0)));
        const double nu = __dadd_rn(__dmul_rn(bl, prof[kMaxProfile + e]), __dmul_rn(al, util));
        const double nt = __dadd_rn(__dmul_rn(bl, prof[2 * kMaxProfile + e]), __dmul_rn(al, tps));
        prof[e] = nl;
        prof[kMaxProfile + e] = nu;
        prof[2 * kMaxProfile + e] = nt;
        prof[3 * kMaxProfile + e] = __ddiv_rn(nl, 1000.0);
        cl[c].running -= 1;
        comp_changed = true;
        __syncwarp();
      }
      // stable compaction of this chunk's survivors
      const unsigned keep = __ballot_sync(0xffffffffu, j < members && !fin);
      if (j < members && !fin) mb[kept + __popc(keep & ((1u << lane) - 1u))] = mine;
      kept += __popc(keep);
      __syncwarp();
    }
    members = kept;
  }
  // ---- build_report's sweep metrics (metrics.cpp:76-105,170-189) ----
  {
    // per-client p90 TTFT (percentile_stats: nearest rank ceil(0.9 n)), clients in client_id
    // order (the std::map of ttft_stats), Jain index over those with any first token
    double sum = 0.0, sum_sq = 0.0;
    int32_t m_clients = 0;
    for (uint32_t rank = 0; rank < static_cast<uint32_t>(C); ++rank) {
      int c = -1;
      for (int i = 0; i < C; ++i)
        if (cl[i].order == rank) c = i;
      if (c < 0) continue;
      // rows of client c: crow[qbase[c] .. qbase[c + 1])
      int64_t cnt = 0;
      const int32_t c_rows = (c + 1 < C ? cl[c + 1].qbase : static_cast<int32_t>(n)) - cl[c].qbase;
      for (int32_t j = lane; j < c_rows; j += 32) cnt += f_ttft[crow[cl[c].qbase + j]] >= 0.0 ? 1 : 0;
      cnt = warp_sum64(cnt);
      if (cnt == 0) continue;
      int64_t k = static_cast<int64_t>(ceil(__dmul_rn(__ddiv_rn(90.0, 100.0), static_cast<double>(cnt))));
      k = k < 1 ? 1 : (k > cnt ? cnt : k);
      uint64_t prefix = 0, mask = 0;  // k-th smallest by MSB-first radix select on the bits
      for (int bit = 63; bit >= 0; --bit) {
        const uint64_t b = 1ull << bit;
        int64_t zeros = 0;
        for (int32_t j = lane; j < c_rows; j += 32) {
          const double v = f_ttft[crow[cl[c].qbase + j]];
          if (v < 0.0) continue;
          const uint64_t u = static_cast<uint64_t>(__double_as_longlong(v));
          zeros += ((u & mask) == prefix && !(u & b)) ? 1 : 0;
        }
        zeros = warp_sum64(zeros);
        if (zeros < k) {
          k -= zeros;
          prefix |= b;
        }
        mask |= b;
      }
      const double p90 = __longlong_as_double(static_cast<long long>(prefix));
      sum = __dadd_rn(sum, p90);
      sum_sq = __dadd_rn(sum_sq, __dmul_rn(p90, p90));
      ++m_clients;
    }
    double jain = 1.0;  // no first tokens: 1.0 (metrics.cpp:176); jain_index: all-zero -> 1.0
    if (m_clients > 0 && sum_sq != 0.0)
      jain = __ddiv_rn(__dmul_rn(sum, sum), __dmul_rn(static_cast<double>(m_clients), sum_sq));
    A.jain_ttft_p90[r] = jain;
    A.throughput_tps[r] = now > 0.0 ? __ddiv_rn(static_cast<double>(completed_tokens), now) : 0.0;
  }
  A.n_events[r] = n_ev;
  A.completed[r] = completed;
  A.sim_end[r] = now;
  A.clamps[r] = clamps;
  A.status[r] = status;
  for (int c = 0; c < C; ++c) {
    A.out_ufc[static_cast<int64_t>(r) * C + c] = cl[c].ufc;
    A.out_rfc[static_cast<int64_t>(r) * C + c] = cl[c].rfc;
    A.out_counter[static_cast<int64_t>(r) * C + c] = cl[c].counter;
  }
}

}  // namespace eqx
