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
// The reporting side follows the run on the same warp: the engine's window samples
// (advance_clock / emit_window_samples, engine.cpp:379-430) at every clock advance, the
// service-difference samples and per-client service-rate windows of build_report (metrics.cpp:
// 21-69,199-226) online at each completion (the event log is in time order, so a sample at
// window end t sees exactly the completions logged at or before t), and the percentile /
// Jain reductions at the end by radix selection over the per-request TTFT and latency.
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

// k-th smallest (1-based) of the non-negative values get(j), j in [0, m) (negative = absent):
// MSB-first radix select on the FP64 bit patterns (monotone for values >= 0), one byte per
// pass through a warp-private 256-bin shared-memory histogram (8 passes over the values).
template <class Get>
__device__ double warp_kth(Get get, int64_t m, int64_t k, uint32_t* hist) {
  const int lane = threadIdx.x & 31;
  uint64_t prefix = 0;
  uint32_t kk = static_cast<uint32_t>(k);
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int b = lane; b < 256; b += 32) hist[b] = 0;
    __syncwarp();
    const uint64_t hmask = shift == 56 ? 0ull : (~0ull << (shift + 8));
    for (int64_t j = lane; j < m; j += 32) {
      const double v = get(j);
      if (v < 0.0) continue;
      const uint64_t u = static_cast<uint64_t>(__double_as_longlong(v));
      if ((u & hmask) == prefix) atomicAdd(&hist[(u >> shift) & 255u], 1u);
    }
    __syncwarp();
    uint32_t c[8], sum = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      c[t] = hist[8 * lane + t];
      sum += c[t];
    }
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t x = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += x;
    }
    const uint32_t excl = incl - sum;
    const bool mine = excl < kk && kk <= incl;
    uint32_t digit = 0, rest = 0;
    if (mine) {
      uint32_t acc = excl;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        if (acc + c[t] >= kk && digit == 0 && rest == 0) {
          digit = 8 * lane + t + 1;  // +1: found marker
          rest = kk - acc;
        }
        acc += c[t];
      }
    }
    const int src = __ffs(__ballot_sync(0xffffffffu, mine)) - 1;
    digit = __shfl_sync(0xffffffffu, digit, src) - 1;
    kk = __shfl_sync(0xffffffffu, rest, src);
    prefix |= static_cast<uint64_t>(digit) << shift;
    __syncwarp();
  }
  return __longlong_as_double(static_cast<long long>(prefix));
}

// percentile_stats (metrics.cpp:76-91): nearest rank ceil(pct / 100 * count), clamped to [1, count]
template <class Get>
__device__ void warp_percentiles(Get get, int64_t m, double* p50, double* p90, int64_t* count, uint32_t* hist) {
  int64_t cnt = 0;
  for (int64_t j = threadIdx.x & 31; j < m; j += 32) cnt += get(j) >= 0.0 ? 1 : 0;
  cnt = warp_sum64(cnt);
  *count = cnt;
  *p50 = 0.0;
  *p90 = 0.0;
  if (cnt == 0) return;
  auto rank = [&](double pct) {
    int64_t r = static_cast<int64_t>(ceil(__dmul_rn(__ddiv_rn(pct, 100.0), static_cast<double>(cnt))));
    return r < 1 ? int64_t(1) : (r > cnt ? cnt : r);
  };
  *p50 = warp_kth(get, m, rank(50.0), hist);
  *p90 = warp_kth(get, m, rank(90.0), hist);
}

// Reporting state of one replay (uniform across the warp's lanes, like the engine state).
struct Reporter {
  int r, C, norm_mode;
  double alpha, beta, ws;
  int64_t wcap;
  double *win, *win_clients, *diff, *rate;
  double window_start, win_busy, win_ovh;  // advance_clock's open window
  int64_t n_win;
  double sd_t, sd_sum, sd_sq, sd_max;      // service_difference
  int64_t n_diff;
  int64_t rate_w;                          // current service-rate window (-1: none yet)
};

__device__ __forceinline__ void all_maxima(const ReplayClient* cl, int C, double& mu, double& mr) {
  mu = 0.0;  // metric_hf's Normalizers over all clients (std::max keeps the first on ties)
  mr = 0.0;
  for (int i = 0; i < C; ++i) {
    if (mu < cl[i].ufc) mu = cl[i].ufc;
    if (mr < cl[i].rfc) mr = cl[i].rfc;
  }
}

// metric_hf (scheduler.cpp:68-81) for one client, combine() in the reference's order
__device__ __forceinline__ double metric_hf(const Reporter& R, const ReplayClient& c, double mu, double mr) {
  if (R.norm_mode == 1) return __dadd_rn(__dmul_rn(R.alpha, c.ufc), __dmul_rn(R.beta, c.rfc));
  const double u = mu > 0.0 ? __ddiv_rn(c.ufc, mu) : 0.0;
  const double v = mr > 0.0 ? __ddiv_rn(c.rfc, mr) : 0.0;
  return __dadd_rn(__dmul_rn(R.alpha, u), __dmul_rn(R.beta, v));
}

// emit_window_samples (engine.cpp:409-430): the GPU sample and one counter sample per client
__device__ __noinline__ void rep_emit(Reporter& R, const ReplayClient* cl, double time_s, double len_s) {
  const int lane = threadIdx.x & 31;
  if (R.n_win < R.wcap) {
    if (R.win && lane == 0) {
      double* w = R.win + (static_cast<int64_t>(R.r) * R.wcap + R.n_win) * 4;
      w[0] = time_s;
      w[1] = R.win_busy;
      w[2] = R.win_ovh;
      w[3] = len_s > 0.0 ? __ddiv_rn(R.win_busy, __dmul_rn(len_s, 1000.0)) : 0.0;
    }
    if (R.win_clients) {
      double mu, mr;
      all_maxima(cl, R.C, mu, mr);
      double* w = R.win_clients + (static_cast<int64_t>(R.r) * R.wcap + R.n_win) * R.C * 4;
      for (int c = lane; c < R.C; c += 32) {
        w[4 * c + 0] = cl[c].ufc;
        w[4 * c + 1] = cl[c].rfc;
        w[4 * c + 2] = metric_hf(R, cl[c], mu, mr);
        w[4 * c + 3] = cl[c].service;
      }
    }
  }
  ++R.n_win;
  R.win_busy = 0.0;
  R.win_ovh = 0.0;
}

// advance_clock's general path (engine.cpp:379-399): the span split pro rata over the windows
// it crosses, one sample per closed window
__device__ __noinline__ void rep_clock_cross(Reporter& R, const ReplayClient* cl, double t_from, double t_to,
                                             double busy_ms, double ovh_ms) {
  const double span = __dsub_rn(t_to, t_from);
  double t = t_from;
  while (t < t_to) {
    const double window_end = __dadd_rn(R.window_start, R.ws);
    const double cut = window_end < t_to ? window_end : t_to;
    const double frac = __ddiv_rn(__dsub_rn(cut, t), span);
    R.win_busy = __dadd_rn(R.win_busy, __dmul_rn(busy_ms, frac));
    R.win_ovh = __dadd_rn(R.win_ovh, __dmul_rn(ovh_ms, frac));
    if (cut == window_end) {
      rep_emit(R, cl, window_end, R.ws);
      R.window_start = window_end;
    }
    t = cut;
  }
}

// service_difference's sample_diff (metrics.cpp:39-46): max - min accumulated service
__device__ __noinline__ void rep_sample_diff(Reporter& R, const ReplayClient* cl, double t) {
  double lo = cl[0].service, hi = cl[0].service;
  for (int c = 1; c < R.C; ++c) {
    if (cl[c].service < lo) lo = cl[c].service;
    if (!(cl[c].service < hi)) hi = cl[c].service;
  }
  const double d = __dsub_rn(hi, lo);
  if (R.diff && R.n_diff < R.wcap && (threadIdx.x & 31) == 0) {
    R.diff[(static_cast<int64_t>(R.r) * R.wcap + R.n_diff) * 2] = t;
    R.diff[(static_cast<int64_t>(R.r) * R.wcap + R.n_diff) * 2 + 1] = d;
  }
  if (R.sd_max < d) R.sd_max = d;
  R.sd_sum = __dadd_rn(R.sd_sum, d);
  R.sd_sq = __dadd_rn(R.sd_sq, __dmul_rn(d, d));
  ++R.n_diff;
}

// the samples at window ends t < now (they precede a completion logged at now)
__device__ __noinline__ void rep_diff_until(Reporter& R, const ReplayClient* cl, double now) {
  while (R.sd_t < now) {
    rep_sample_diff(R, cl, R.sd_t);
    R.sd_t = __dadd_rn(R.sd_t, R.ws);
  }
}

// a completion opened service-rate window w > the current one: close the current window and
// restart the previous + current sums (the last window absorbs completions at the very end)
__device__ __noinline__ void rep_rate_advance(Reporter& R, ReplayClient* cl, int64_t w) {
  for (int k = 0; k < R.C; ++k) {
    if (R.rate && R.rate_w >= 0 && R.rate_w < R.wcap && (threadIdx.x & 31) == 0)
      R.rate[static_cast<int64_t>(k) * R.wcap + R.rate_w] = cl[k].bucket;
    cl[k].merged = (R.rate_w >= 0 && w == R.rate_w + 1) ? cl[k].bucket : 0.0;
    cl[k].bucket = 0.0;
  }
  R.rate_w = w;
}

// KIND: the policy kind, fixed per instantiation so a replay carries only its policy's code
// (the kernel is long scalar code; its instruction footprint is what its single warps stall on).
template <int KIND, bool kBig>
__global__ void __launch_bounds__(128) replay_kernel(const ReplayArgs A) {
  __shared__ uint32_t s_hist[4][256];  // radix-select histograms, one per warp
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= A.n_replays) return;  // warp-uniform
  uint32_t* hist = s_hist[threadIdx.x >> 5];
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
  double* f_lat = A.f_lat + t0;
  for (int64_t i = lane; i < n; i += 32) {
    f_ttft[i] = -1.0;
    f_lat[i] = -1.0;
  }
  int64_t completed_tokens = 0, rejected = 0;
  // Ledger, FIFO cursors and profile are private per lane (identical copies, updated uniformly),
  // so the read-modify-write engine steps need no intra-warp synchronisation; the batch lives
  // in global scratch, split across lanes.
  // kBig (rosters beyond kMaxReplayClients): one copy in global scratch, stored identically by
  // every lane (each lane reads back its own store, so no intra-warp synchronisation either)
  ReplayClient cl_local[kBig ? 1 : kMaxReplayClients];
  ReplayClient* const cl = kBig ? A.cl + static_cast<int64_t>(r) * C : cl_local;
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
    z.skip = -1;
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
  // run() (engine.cpp:120-121): max_sim_time_s, else Trace::duration_s
  const double max_sim = A.max_sim_time_s > 0.0 ? A.max_sim_time_s
                         : A.duration             ? A.duration[r]
                                                  : (n > 0 ? arrival[n - 1] : 0.0);
  // eligible_at (engine.cpp:165-168): arrival + prediction_overhead_ms / 1000
  auto eligible_at = [&](int64_t i) { return __dadd_rn(arrival[i], A.overhead_s); };
  double now = 0.0, busy_cum = 0.0, ovh_cum = 0.0;
  int64_t arrival_idx = 0, total_queued = 0, n_ev = 0, completed = 0, clamps = 0, max_resident = 0;
  int32_t admit_no = 0;  // admit_requests calls (the skipped stamps of large rosters)
  int32_t members = 0;
  bool comp_changed = false;
  int32_t status = 0;
  // ---- reporting state (the rare paths are out-of-line: the hot loop's code stays small) ----
  const double ws = A.window_s;
  const int64_t wcap = A.win_cap;
  Reporter R;
  R.r = r;
  R.C = C;
  R.norm_mode = P.norm_mode;
  R.alpha = eq.alpha;
  R.beta = eq.beta;
  R.ws = ws;
  R.wcap = wcap;
  R.win = A.win;
  R.win_clients = A.win_clients;
  R.diff = A.diff;
  R.rate = A.rate ? A.rate + static_cast<int64_t>(r) * C * wcap : nullptr;
  R.window_start = R.win_busy = R.win_ovh = 0.0;
  R.n_win = 0;
  R.sd_t = ws;
  R.sd_sum = R.sd_sq = R.sd_max = 0.0;
  R.n_diff = 0;
  R.rate_w = -1;
  // advance_clock (engine.cpp:379-399).  Within one window the single segment's fraction is
  // span / span = 1 exactly, so busy / overhead add as they are; crossings take the general
  // pro-rata loop with its window samples.
  double w_end = ws, w_busy = 0.0, w_ovh = 0.0;  // register copies of the open window
  auto advance_clock = [&](double t_from, double t_to, double busy_ms, double ovh_ms) {
    busy_cum = __dadd_rn(busy_cum, busy_ms);
    ovh_cum = __dadd_rn(ovh_cum, ovh_ms);
    if (t_to <= t_from) return;
    if (w_end > t_to) {
      w_busy = __dadd_rn(w_busy, busy_ms);
      w_ovh = __dadd_rn(w_ovh, ovh_ms);
      return;
    }
    R.win_busy = w_busy;
    R.win_ovh = w_ovh;
    rep_clock_cross(R, cl, t_from, t_to, busy_ms, ovh_ms);
    w_busy = R.win_busy;
    w_ovh = R.win_ovh;
    w_end = __dadd_rn(R.window_start, ws);
  };
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
  // the whole log (log_all): LogEntry payloads (engine.cpp:44-76)
  const int64_t evo = static_cast<int64_t>(r) * A.ev_cap;
  auto log_full = [&](int64_t rid, int32_t kind, double t, int32_t i0, double d0, double d1, double d2) {
    if (n_ev < A.ev_cap) {
      ev_id[n_ev] = rid;
      ev_kind[n_ev] = kind;
      ev_time[n_ev] = t;
      if (A.ev_i0) {
        A.ev_i0[evo + n_ev] = i0;
        A.ev_d0[evo + n_ev] = d0;
        A.ev_d1[evo + n_ev] = d1;
        A.ev_d2[evo + n_ev] = d2;
      }
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
  auto drain = [&](double upto) {  // engine.cpp:171-197
    while (arrival_idx < n && eligible_at(arrival_idx) <= upto) {
      const int64_t i = arrival_idx++;
      const int c = client[i];
      const double w = cl[c].weight;
      int32_t pred;  // max(1, predict(req)) (engine.cpp:179)
      if (A.given_pred) {
        pred = A.given_pred[t0 + i] > 1 ? A.given_pred[t0 + i] : 1;
      } else {
        pred = score_request(M, P, 0.0, in_tok[i], tag[i], true_out[i], id[i], 0.0, w).pred;
      }
      const int b = entry_for(pred);  // map_metrics against the replay's current profile
      f_pred[i] = pred;
      f_preds[i] = prof[3 * kMaxProfile + b];
      f_rfc[i] = __dmul_rn(__dmul_rn(w, prof[2 * kMaxProfile + b]), prof[kMaxProfile + b]);
      if (A.log_all) {
        A.f_plat[t0 + i] = prof[b];  // every lane stores the same value and reads back its own
        log_full(id[i], 3, arrival[i], in_tok[i], 0.0, 0.0, 0.0);  // Arrived at arrival_time_s
      }
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
    ++admit_no;
    for (;;) {
      double mu = 0.0, mr = 0.0;  // backlogged_maxima (scheduler.cpp:40-48)
      const bool maxmode = KIND == kEquinox && P.norm_mode == 0;
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
        if (cl[i].qhead == cl[i].qend || (kBig ? cl[i].skip == admit_no : ((skipped >> (i & 63)) & 1u))) continue;
        double k;
        if (KIND == kFcfs) k = 0.0;
        else if (KIND == kVtc) k = cl[i].counter;
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
        if (A.log_all) log_full(id[row], 2, now, in, 0.0, 0.0, 0.0);
        else log_ev(id[row], 2);
        ++rejected;
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
          if (kBig) cl[c].skip = admit_no;
          else skipped |= 1ull << (c & 63);
          continue;
        }
        break;
      }
      pop_head(c);
      ReplayMember& m = mb[members++];
      m.pad = 0;
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
      if (KIND == kVtc) {
        m.p_vtc = P.vtc_use_prediction ? __dmul_rn(w, tokens) : __dmul_rn(w, static_cast<double>(in));
        cl[c].counter = __dadd_rn(cl[c].counter, m.p_vtc);
      }
      if (A.log_all) {
        log_full(id[row], 1, now, pred, A.f_plat[t0 + row], 0.0, 0.0);
      } else {
        log_ev(id[row], 1);
      }
    }
    return new_prefill;
  };
  // ---- SimulationRun::run ----
  while (now < max_sim) {
    drain(now);
    if (members == 0 && total_queued == 0) {
      if (arrival_idx >= n) break;
      const double next_t = eligible_at(arrival_idx);
      if (next_t >= max_sim) break;
      advance_clock(now, next_t, 0.0, 0.0);
      now = next_t;
      drain(now);
    }
    const int32_t members0 = members;  // admissions of this round are members [members0, members)
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
    advance_clock(now, t_end, busy_ms, overhead_ms);
    now = t_end;
    comp_changed = false;
    for (int j = lane; j < members; j += 32) {
      mb[j].generated += 1;
      if (mb[j].generated == 1) f_ttft[mb[j].row] = __dsub_rn(now, arrival[mb[j].row]);  // FirstToken
    }
    __syncwarp();
    if (KIND == kVtc && !P.vtc_use_prediction) {  // on_tokens per client (scheduler.cpp:185-190)
      for (int c = 0; c < C; ++c) {
        int64_t t = 0;
        for (int j = lane; j < members; j += 32) t += mb[j].client == c ? 1 : 0;
        t = warp_sum64(t);
        if (t > 0) cl[c].counter = __dadd_rn(cl[c].counter, __dmul_rn(__dmul_rn(cl[c].weight, P.ow), static_cast<double>(t)));
      }
    }
    const int64_t res2 = resident + members;  // every resident request generated one token
    if (res2 > max_resident) max_resident = res2;
    if (__dmul_rn(static_cast<double>(res2), P.m) > P.M) {  // KV memory bound violated
      status = 2;
      break;
    }
    drain(now);
    // FirstToken of this round's admissions, in admission order, after the iteration's
    // arrivals (engine.cpp:305-318)
    if (A.log_all)
      for (int32_t j = members0; j < members; ++j)
        if (mb[j].generated == 1) log_full(id[mb[j].row], 4, now, 0, 0.0, 0.0, 0.0);
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
        if (A.log_all) log_full(id[m.row], 5, now, out, latency_s, tps, util);  // Completed
        if (lane == 0) f_lat[m.row] = latency_s;
        if (C >= 2 && R.sd_t < now) rep_diff_until(R, cl, now);  // windows closed before this completion
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
        cl[c].service = __dadd_rn(cl[c].service, wwt);  // accumulated_service (scheduler.cpp:232)
        {  // build_report's service-rate window of this completion: weight * (in + ow * out), same value
          const int64_t w = static_cast<int64_t>(__ddiv_rn(now, ws));
          if (w > R.rate_w) rep_rate_advance(R, cl, w);
          cl[c].bucket = __dadd_rn(cl[c].bucket, wwt);
          cl[c].merged = __dadd_rn(cl[c].merged, wwt);
        }
        if (KIND == kVtc && P.vtc_use_prediction) {
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
  // ---- end of run (engine.cpp:137-145): flush_window, then build_report (metrics.cpp:151-229) ----
  R.win_busy = w_busy;
  R.win_ovh = w_ovh;
  if (now > R.window_start) rep_emit(R, cl, now, __dsub_rn(now, R.window_start));  // flush_window
  __syncwarp();
  eqx_replay_report rep{};
  rep.sim_end_s = now;
  rep.busy_ms_total = busy_cum;
  rep.overhead_ms_total = ovh_cum;
  rep.completed = completed;
  rep.rejected = rejected;
  rep.total_completed_tokens = completed_tokens;
  rep.n_windows = R.n_win;
  rep.max_resident_kv_tokens = max_resident;
  rep.drained = arrival_idx;
  if (C >= 2) {  // service_difference: the remaining windows up to the end, then the moments
    const double lim = __dadd_rn(now, 1e-12);
    while (R.sd_t <= lim) {
      rep_sample_diff(R, cl, R.sd_t);
      R.sd_t = __dadd_rn(R.sd_t, ws);
    }
    if (R.n_diff == 0) rep_sample_diff(R, cl, now);
    const double nd = static_cast<double>(R.n_diff);
    rep.max_diff = R.sd_max;
    rep.avg_diff = __ddiv_rn(R.sd_sum, nd);
    rep.var_diff = __dsub_rn(__ddiv_rn(R.sd_sq, nd), __dmul_rn(rep.avg_diff, rep.avg_diff));
    if (rep.var_diff < 0.0) rep.var_diff = 0.0;
    rep.n_diff = R.n_diff;
  }
  {  // jain_hf over final_hf = metric_hf(final_clients), roster order
    double mu, mr, sum = 0.0, sum_sq = 0.0;
    all_maxima(cl, C, mu, mr);
    for (int c = 0; c < C; ++c) {
      const double h = metric_hf(R, cl[c], mu, mr);
      if (A.rclients && lane == 0) A.rclients[static_cast<int64_t>(r) * C + c].final_hf = h;
      sum = __dadd_rn(sum, h);
      sum_sq = __dadd_rn(sum_sq, __dmul_rn(h, h));
    }
    rep.jain_hf = sum_sq == 0.0 ? 1.0 : __ddiv_rn(__dmul_rn(sum, sum), __dmul_rn(static_cast<double>(C), sum_sq));
  }
  // per-client service-rate windows: n_windows = max(1, ceil(sim_end / ws - 1e-12))
  const int64_t n_rate = static_cast<int64_t>(fmax(1.0, ceil(__dsub_rn(__ddiv_rn(now, ws), 1e-12))));
  rep.n_rate = n_rate;
  if (double* rate = R.rate) {
    const int64_t rate_w = R.rate_w;
    if (rate_w >= 0 && lane == 0)
      for (int k = 0; k < C; ++k) {
        if (rate_w < n_rate) {
          if (rate_w < wcap) rate[static_cast<int64_t>(k) * wcap + rate_w] = cl[k].bucket;
        } else if (n_rate - 1 < wcap) {  // completions at the very end fell past the last window
          rate[static_cast<int64_t>(k) * wcap + n_rate - 1] = cl[k].merged;
          if (rate_w < wcap) rate[static_cast<int64_t>(k) * wcap + rate_w] = 0.0;
        }
      }
    __syncwarp();
    const int64_t kept = n_rate < wcap ? n_rate : wcap;
    for (int64_t j = lane; j < static_cast<int64_t>(C) * kept; j += 32) {
      double* x = rate + (j / kept) * wcap + (j % kept);
      *x = __ddiv_rn(*x, ws);
    }
  }
  {
    // per-client TTFT percentiles (ttft_stats' per_client map); jain_ttft_p90 over the clients
    // with any first token, in client_id order
    double sum = 0.0, sum_sq = 0.0;
    int32_t m_clients = 0;
    for (uint32_t rank = 0; rank < static_cast<uint32_t>(C); ++rank) {
      const int c = static_cast<int>(A.by_order[rank]);
      const int32_t c_rows = (c + 1 < C ? cl[c + 1].qbase : static_cast<int32_t>(n)) - cl[c].qbase;
      const int32_t* rows_c = crow + cl[c].qbase;
      double p50, p90;
      int64_t cnt;
      warp_percentiles([&](int64_t j) { return f_ttft[rows_c[j]]; }, c_rows, &p50, &p90, &cnt, hist);
      if (A.rclients && lane == 0) {
        eqx_replay_client& o = A.rclients[static_cast<int64_t>(r) * C + c];
        o.accumulated_service = cl[c].service;
        o.mean_service_rate = now > 0.0 ? __ddiv_rn(cl[c].service, now) : 0.0;
        o.ttft_p50 = p50;
        o.ttft_p90 = p90;
        o.ttft_count = cnt;
        o.backlogged = cl[c].backlogged;
      }
      if (cnt == 0) continue;
      sum = __dadd_rn(sum, p90);
      sum_sq = __dadd_rn(sum_sq, __dmul_rn(p90, p90));
      ++m_clients;
    }
    double jain = 1.0;  // no first tokens: 1.0 (metrics.cpp:176); jain_index: all-zero -> 1.0
    if (m_clients > 0 && sum_sq != 0.0)
      jain = __ddiv_rn(__dmul_rn(sum, sum), __dmul_rn(static_cast<double>(m_clients), sum_sq));
    rep.jain_ttft_p90 = jain;
    rep.throughput_tps = now > 0.0 ? __ddiv_rn(static_cast<double>(completed_tokens), now) : 0.0;
    rep.mean_gpu_util = now > 0.0 ? __ddiv_rn(busy_cum, __dmul_rn(now, 1000.0)) : 0.0;
    A.jain_ttft_p90[r] = jain;
    A.throughput_tps[r] = rep.throughput_tps;
  }
  if (A.report) {
    warp_percentiles([&](int64_t j) { return f_ttft[j]; }, n, &rep.ttft_p50, &rep.ttft_p90, &rep.ttft_count, hist);
    warp_percentiles([&](int64_t j) { return f_lat[j]; }, n, &rep.latency_p50, &rep.latency_p90, &rep.latency_count, hist);
    if (lane == 0) A.report[r] = rep;
  }
  if (lane == 0) {  // SimResult::profile (the feedback-updated map)
    double* po = A.prof + static_cast<int64_t>(r) * 3 * np;
    for (int e = 0; e < np; ++e) {
      po[e] = prof[e];
      po[np + e] = prof[kMaxProfile + e];
      po[2 * np + e] = prof[2 * kMaxProfile + e];
    }
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

template __global__ void replay_kernel<kFcfs, false>(ReplayArgs);
template __global__ void replay_kernel<kVtc, false>(ReplayArgs);
template __global__ void replay_kernel<kEquinox, false>(ReplayArgs);
template __global__ void replay_kernel<kFcfs, true>(ReplayArgs);
template __global__ void replay_kernel<kVtc, true>(ReplayArgs);
template __global__ void replay_kernel<kEquinox, true>(ReplayArgs);

}  // namespace eqx
