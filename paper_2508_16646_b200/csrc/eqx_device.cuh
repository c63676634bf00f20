// eqx_device.cuh -- device-side data layout and per-request arithmetic of the Equinox step.
//
// All FP64 arithmetic follows the reference's operation order exactly with explicit
// round-to-nearest intrinsics (no FMA contraction is possible through __dadd_rn/__dmul_rn/
// __ddiv_rn, and the library is additionally built with -fmad=false), so every value is
// bit-identical to the reference CPU path compiled without -march.
#pragma once

#include <cstddef>
#include <cstdint>

namespace eqx {

constexpr int kMaxProfile = 32;   // GpuProfile entries (default 8, gpu_model.cpp:128-130)
constexpr int kMaxCuts = 127;     // merged router thresholds + expert bin bounds
constexpr int kMaxTagStates = 256; // tag id 0 (untagged) .. 255
constexpr int kMaxLut = 8192;     // (n_cuts + 1) * n_tag_states

enum PredKind : int32_t { kPredOracle = 0, kPredMope = 1, kPredNoisy = 2, kPredSingle = 3 };
enum PolicyKindDev : int32_t { kFcfs = 0, kVtc = 1, kEquinox = 2 };

// Compiled predictor + profile tables (built on the host by the "model compiler" in
// eqx_capi.cu from MopeModel / GpuProfile; one copy per context in device memory).
struct ModelTables {
  int32_t pred_kind;
  int32_t n_cuts;        // sorted unique cut points (ints): interval = #cuts < input_tokens
  int32_t n_tag_states;  // LUT columns: tag id 0..n_tag_states-1
  int32_t n_prof;
  int32_t cuts[kMaxCuts + 1];
  int32_t prof_upper[kMaxProfile];
  double prof_pred_s[kMaxProfile];  // latency_ms / 1000.0 (scheduler.cpp:23), same IEEE op
  double prof_lat[kMaxProfile];
  double prof_util[kMaxProfile];
  double prof_tps[kMaxProfile];
  double noisy_l1;
  uint64_t noisy_key;    // mix_keys(seed, fnv1a("noisy_oracle")) (predictor.cpp:18)
  // lut[interval * n_tag_states + tag] = predicted output tokens after the engine's
  // max(1, .) clamp (engine.cpp:179); negative when route() took the length fallback.
  int32_t lut[kMaxLut];
};

// Scheduling knobs used on the device (PolicySpec, EquinoxParams, PerfParams, backfill).
struct Policy {
  int32_t kind;
  int32_t norm_mode;       // 0 = MaxOverClients, 1 = None
  int32_t vtc_use_prediction;
  int32_t backfill;
  int32_t max_batch;
  double alpha, beta, delta, ow;  // beta = 1.0 - alpha computed once, as beta() does
  double m, M;             // mem_per_token_bytes, mem_capacity_bytes
};

// Device-resident scalars of one context.
struct DevState {
  int32_t members;        // BatchState::members.size()
  int32_t pad0;
  int64_t reserved;       // BatchState::reserved_kv_tokens()
  int64_t n_events, n_admitted, n_rejected, new_prefill;
  unsigned long long fallbacks;   // MopePredictor::length_fallbacks_ over scored rows
  unsigned long long near_ties;   // noisy predictor near-.5 flags
  int32_t bad_client;     // drain saw a client index out of range
  int32_t underflow;      // client-sharded step: a gathered head window ran out (retry deeper)
  // phase timestamps (%globaltimer ns) of the last step, for profiling:
  // [0] selection start [1] windows filled [2] loop start [3] loop end
  // [4] first worker start (min) [5] last worker end (max) [6] #batches [7] #seq phases
  // [8..11] batch cycles: stream generation, sort, verify, commit
  unsigned long long t[16];
  int64_t n_queued;       // client-sharded step: queued requests over all ranks at step start
  // EQX_PROF builds: drain timeline (%globaltimer ns): hist start (min) / walk end (max) /
  // epilogue end, rank start (min) / walk end (max) / epilogue end
  unsigned long long dt[8];
  int64_t clamps;          // SchedulerPolicy::counter_clamps() (on_complete clamps at 0)
  unsigned long long tk[8];  // EQX_PROF builds: top-K selection sub-phase cycles / pass counts
};

// The host-visible copy of a step's DevState (mapped host memory) is written by the selection
// CTA's epilogue, with no copy kernel behind the step, once the concurrently running scoring
// kernel (fallbacks, near_ties, the t[4] / t[5] stamps) has signalled completion.
static_assert(sizeof(DevState) % 8 == 0, "DevState is copied in 8-byte words");

// Order-preserving map double -> uint64 (IEEE total order on non-NaN values, with -0.0 and
// +0.0 made equal as operator< / operator== treat them), so tuple comparisons in the
// selection loop are integer compares.
__device__ __forceinline__ uint64_t ordered_bits(double d) {
  const uint64_t b = static_cast<uint64_t>(__double_as_longlong(d == 0.0 ? 0.0 : d));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}
__device__ __forceinline__ double from_ordered_bits(uint64_t o) {
  const uint64_t b = (o >> 63) ? (o & 0x7fffffffffffffffULL) : ~o;
  return __longlong_as_double(static_cast<long long>(b));
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ---- rng.hpp:13-75 restated for the noisy oracle ----------------------------------------
__host__ __device__ __forceinline__ uint64_t splitmix_step(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t mix_keys(uint64_t a, uint64_t b) {
  return splitmix_step(a + 0x9e3779b97f4a7c15ULL * (b + 1));
}

struct Scored {
  int32_t pred;
  int32_t bucket;
  double ufc_inc;
  double rfc_inc;
  uint32_t fallback;
  uint32_t near_tie;
};

// Predict + map_metrics + ufc_increment + rfc_increment for one request.
//   MoPE:   route (predictor.cpp:36-60) + ExpertModel::predict (:62-71) through the LUT
//           (single-proxy uses the same LUT path, compiled from one expert)
//   oracle: true_output_tokens (predictor.hpp:36); noisy: predictor.cpp:17-23
//   map:    GpuProfile::entry_for (gpu_model.cpp:74-80), first bucket with pred <= upper
//   ufc:    w * (in + ow * pred) / (1 + delta * ((now - arrival) + lat_ms / 1000))
//           (scheduler.cpp:19-27 with wait = now - arrival, engine.cpp:257)
//   rfc:    (w * tps) * util (scheduler.cpp:29-31)
// KIND is the predictor family (kPredMope for MoPE and single-proxy tables).
template <int KIND>
__device__ __forceinline__ Scored score_request_t(const ModelTables& M, const Policy& P, double now, int32_t in,
                                                  uint32_t tag, int32_t true_out, int64_t id, double arrival,
                                                  double w) {
  Scored s;
  s.fallback = 0;
  s.near_tie = 0;
  int32_t pred;
  if constexpr (KIND == kPredMope) {
    int32_t iv = 0;
    for (int i = 0; i < M.n_cuts; ++i) iv += (M.cuts[i] < in) ? 1 : 0;
    const uint32_t t = tag < static_cast<uint32_t>(M.n_tag_states) ? tag : 0u;
    const int32_t e = M.lut[iv * M.n_tag_states + static_cast<int32_t>(t)];
    s.fallback = e < 0 ? 1u : 0u;
    pred = e < 0 ? -e : e;
  } else if constexpr (KIND == kPredOracle) {
    pred = true_out > 1 ? true_out : 1;
  } else {
    // NoisyOraclePredictor: Rng(mix_keys(mix_keys(seed, fnv1a("noisy_oracle")), id)).laplace(l1)
    uint64_t st = mix_keys(M.noisy_key, static_cast<uint64_t>(id));
    st += 0x9e3779b97f4a7c15ULL;
    const uint64_t z = splitmix_step(st);
    const double u = __dsub_rn(__dmul_rn(__dadd_rn(static_cast<double>(z >> 11), 0.5), 0x1.0p-53), 0.5);
    const double mag = -log1p(__dmul_rn(-2.0, fabs(u)));
    const double noise = u < 0 ? __dmul_rn(-M.noisy_l1, mag) : __dmul_rn(M.noisy_l1, mag);
    const double v = __dadd_rn(static_cast<double>(true_out), noise);
    // CUDA's log1p and glibc's may differ by an ulp; only a value on a .5 boundary can round
    // differently, so such requests are counted as flagged near-ties (north-star tolerance).
    const double frac = v - floor(v);
    s.near_tie = fabs(frac - 0.5) <= 1e-9 ? 1u : 0u;
    const double r = round(v);
    int32_t p = static_cast<int32_t>(1.0 < r ? r : 1.0);
    pred = p > 1 ? p : 1;
  }
  int32_t b = M.n_prof - 1;
  for (int e = M.n_prof - 1; e >= 0; --e)
    if (pred <= M.prof_upper[e]) b = e;
  const double tokens = __dadd_rn(static_cast<double>(in), __dmul_rn(P.ow, static_cast<double>(pred)));
  const double wait = __dsub_rn(now, arrival);
  const double denom = __dadd_rn(1.0, __dmul_rn(P.delta, __dadd_rn(wait, M.prof_pred_s[b])));
  s.pred = pred;
  s.bucket = b;
  s.ufc_inc = __ddiv_rn(__dmul_rn(w, tokens), denom);
  s.rfc_inc = __dmul_rn(__dmul_rn(w, M.prof_tps[b]), M.prof_util[b]);
  return s;
}

// Same result as score_request_t<KIND>, with the predict + map_metrics lookups served by the
// host-compiled direct table when the input is inside it (one read-only-cache load instead of
// the interval and bucket searches).
template <int KIND>
__device__ __forceinline__ Scored score_request_direct(const ModelTables& M, const Policy& P, const uint32_t* direct,
                                                       int32_t direct_n, double now, int32_t in, uint32_t tag,
                                                       int32_t true_out, int64_t id, double arrival, double w) {
  int32_t pred, b;
  Scored s;
  s.fallback = 0;
  s.near_tie = 0;
  if constexpr (KIND == kPredMope) {
    const uint32_t t = tag < static_cast<uint32_t>(M.n_tag_states) ? tag : 0u;
    if (static_cast<uint32_t>(in) < static_cast<uint32_t>(direct_n)) {
      const uint32_t e = direct[t * static_cast<uint32_t>(direct_n) + static_cast<uint32_t>(in)];
      pred = static_cast<int32_t>(e & 0xffffu);
      b = static_cast<int32_t>((e >> 16) & 0xffu);
      s.fallback = e >> 24;
    } else {
      return score_request_t<KIND>(M, P, now, in, tag, true_out, id, arrival, w);
    }
  } else if constexpr (KIND == kPredOracle) {
    pred = true_out > 1 ? true_out : 1;
    if (pred < direct_n) {
      b = static_cast<int32_t>(direct[pred]);
    } else {
      return score_request_t<KIND>(M, P, now, in, tag, true_out, id, arrival, w);
    }
  } else {
    return score_request_t<KIND>(M, P, now, in, tag, true_out, id, arrival, w);
  }
  const double tokens = __dadd_rn(static_cast<double>(in), __dmul_rn(P.ow, static_cast<double>(pred)));
  const double wait = __dsub_rn(now, arrival);
  const double denom = __dadd_rn(1.0, __dmul_rn(P.delta, __dadd_rn(wait, M.prof_pred_s[b])));
  s.pred = pred;
  s.bucket = b;
  s.ufc_inc = __ddiv_rn(__dmul_rn(w, tokens), denom);
  s.rfc_inc = __dmul_rn(__dmul_rn(w, M.prof_tps[b]), M.prof_util[b]);
  return s;
}

// Runtime-dispatched variant (cold paths: head windows, deep heads).
static __device__ __noinline__ Scored score_request(const ModelTables& M, const Policy& P, double now, int32_t in,
                                             uint32_t tag, int32_t true_out, int64_t id, double arrival, double w) {
  if (M.pred_kind == kPredOracle) return score_request_t<kPredOracle>(M, P, now, in, tag, true_out, id, arrival, w);
  if (M.pred_kind == kPredNoisy) return score_request_t<kPredNoisy>(M, P, now, in, tag, true_out, id, arrival, w);
  return score_request_t<kPredMope>(M, P, now, in, tag, true_out, id, arrival, w);
}

}  // namespace eqx
