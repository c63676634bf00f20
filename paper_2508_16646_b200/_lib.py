"""ctypes binding of libeqx_b200.so (include/eqx.h).  No fallback: importing the scheduler
without the built CUDA library, or creating a context without a B200, raises."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# EQX_LIB selects an instrumented build (csrc/Makefile `prof`: libeqx_b200_prof.so) for profiling
LIB_PATH = os.environ.get("EQX_LIB") or os.path.join(HERE, "libeqx_b200.so")

EQX_OK, EQX_ERR_CONFIG, EQX_ERR_PARSE, EQX_ERR_ENGINE, EQX_ERR_CUDA, EQX_ERR_ARG = range(6)
EQX_HOST, EQX_DEVICE = 0, 1

_dp = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_u8p = C.POINTER(C.c_uint8)


class Policy(C.Structure):
    _fields_ = [("kind", C.c_int32), ("alpha", C.c_double), ("delta", C.c_double),
                ("output_weight", C.c_double), ("norm_mode", C.c_int32),
                ("vtc_use_prediction", C.c_int32), ("counter_lift", C.c_int32),
                ("backfill", C.c_int32)]


class Perf(C.Structure):
    _fields_ = [("max_batch", C.c_int32), ("mem_per_token_bytes", C.c_double),
                ("mem_capacity_bytes", C.c_double)]


class Profile(C.Structure):
    _fields_ = [("n", C.c_int32), ("bucket_upper", _i32p), ("latency_ms", _dp),
                ("gpu_util", _dp), ("tps", _dp)]


class Mope(C.Structure):
    _fields_ = [("n_thresholds", C.c_int32), ("thresholds", _i32p), ("mix_weight", C.c_double),
                ("num_buckets", C.c_int32), ("n_rows", C.c_int32), ("rows", _dp),
                ("n_experts", C.c_int32), ("n_bins", C.c_int32), ("bin_upper", _i32p),
                ("bin_value", _i32p), ("out_min", _i32p), ("out_max", _i32p),
                ("n_tags", C.c_int32), ("tag_row", _i32p)]


class Predictor(C.Structure):
    _fields_ = [("kind", C.c_int32), ("mope", Mope), ("noisy_l1", C.c_double),
                ("noisy_seed", C.c_uint64)]


class Requests(C.Structure):
    _fields_ = [("n", C.c_int64), ("id", C.c_void_p), ("id_base", C.c_int64),
                ("client", C.c_void_p), ("arrival_s", C.c_void_p), ("input_tokens", C.c_void_p),
                ("true_output_tokens", C.c_void_p), ("tag", C.c_void_p), ("location", C.c_int32),
                ("narrow", C.c_int32)]


class StepSummary(C.Structure):
    _fields_ = [("n_events", C.c_int64), ("n_admitted", C.c_int64), ("n_rejected", C.c_int64),
                ("new_prefill_tokens", C.c_int64), ("length_fallbacks", C.c_int64),
                ("noisy_near_ties", C.c_int64), ("batch_members", C.c_int32),
                ("batch_reserved_kv_tokens", C.c_int64), ("queued", C.c_int64),
                ("window_underflow", C.c_int32)]


class Completions(C.Structure):
    _fields_ = [("n", C.c_int64), ("client", C.c_void_p), ("input_tokens", C.c_void_p),
                ("output_tokens", C.c_void_p), ("latency_s", C.c_void_p), ("tps", C.c_void_p),
                ("gpu_util", C.c_void_p), ("pending_ufc", C.c_void_p), ("pending_rfc", C.c_void_p),
                ("pending_vtc", C.c_void_p), ("location", C.c_int32)]


class Replays(C.Structure):
    _fields_ = [("n_replays", C.c_int32), ("row_off", C.c_void_p), ("client", C.c_void_p),
                ("arrival_s", C.c_void_p), ("input_tokens", C.c_void_p), ("true_output_tokens", C.c_void_p),
                ("tag", C.c_void_p), ("id", C.c_void_p), ("alpha", C.c_void_p), ("max_sim_time_s", C.c_double),
                ("ema_alpha", C.c_double), ("ev_cap", C.c_int64), ("report_window_s", C.c_double),
                ("win_cap", C.c_int64), ("duration_s", C.c_void_p), ("prediction_overhead_ms", C.c_double),
                ("predicted", C.c_void_p), ("log_all", C.c_int32)]


REPORT_FIELDS = ("max_diff", "avg_diff", "var_diff", "jain_hf", "jain_ttft_p90", "throughput_tps", "mean_gpu_util",
                 "ttft_p50", "ttft_p90", "latency_p50", "latency_p90", "ttft_count", "latency_count", "sim_end_s",
                 "busy_ms_total", "overhead_ms_total", "completed", "rejected", "total_completed_tokens",
                 "n_windows", "n_diff", "n_rate", "max_resident_kv_tokens", "drained")
REPORT_INT = {"ttft_count", "latency_count", "completed", "rejected", "total_completed_tokens", "n_windows", "n_diff",
              "n_rate", "max_resident_kv_tokens", "drained"}
REPORT_DTYPE = np.dtype([(f, np.int64 if f in REPORT_INT else np.float64) for f in REPORT_FIELDS])
CLIENT_FIELDS = ("final_hf", "accumulated_service", "mean_service_rate", "ttft_p50", "ttft_p90", "ttft_count",
                 "backlogged")
CLIENT_DTYPE = np.dtype([(f, np.int64 if f in ("ttft_count", "backlogged") else np.float64) for f in CLIENT_FIELDS])


class ReplayOut(C.Structure):
    _fields_ = [("n_events", C.c_void_p), ("ev_id", C.c_void_p), ("ev_kind", C.c_void_p), ("ev_time", C.c_void_p),
                ("ufc", C.c_void_p), ("rfc", C.c_void_p), ("counter", C.c_void_p), ("completed", C.c_void_p),
                ("sim_end", C.c_void_p), ("counter_clamps", C.c_void_p), ("status", C.c_void_p),
                ("jain_ttft_p90", C.c_void_p), ("throughput_tps", C.c_void_p), ("report", C.c_void_p),
                ("clients", C.c_void_p), ("win", C.c_void_p), ("win_clients", C.c_void_p), ("diff", C.c_void_p),
                ("rate", C.c_void_p), ("ev_i0", C.c_void_p), ("ev_d0", C.c_void_p), ("ev_d1", C.c_void_p),
                ("ev_d2", C.c_void_p), ("profile", C.c_void_p)]


class TraceView(C.Structure):
    _fields_ = [("n", C.c_int64), ("n_clients", C.c_int32), ("n_tags", C.c_int32), ("n_warnings", C.c_int32),
                ("pinned", C.c_int32), ("duration_s", C.c_double), ("client", C.c_void_p), ("arrival_s", C.c_void_p),
                ("input_tokens", C.c_void_p), ("output_tokens", C.c_void_p), ("tag", C.c_void_p),
                ("client_names", C.c_void_p), ("tag_names", C.c_void_p), ("warnings", C.c_void_p),
                ("stored_hash", C.c_char * 17)]


_SIGS = {
    "eqx_trace_load_csv": ([C.c_char_p, C.POINTER(C.c_void_p), C.c_char_p, C.c_int32], C.c_int),
    "eqx_trace_load_bin": ([C.c_char_p, C.POINTER(C.c_void_p), C.c_char_p, C.c_int32], C.c_int),
    "eqx_trace_create": ([C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                          C.c_char_p, C.c_int32, C.c_char_p, C.POINTER(C.c_void_p)], C.c_int),
    "eqx_trace_view_get": ([C.c_void_p, C.c_void_p], C.c_int),
    "eqx_trace_hash": ([C.c_void_p, C.c_char_p], C.c_int),
    "eqx_trace_save_csv": ([C.c_void_p, C.c_char_p], C.c_int),
    "eqx_trace_save_bin": ([C.c_void_p, C.c_char_p], C.c_int),
    "eqx_trace_free": ([C.c_void_p], None),
    "eqx_abi_version": ([], C.c_int32),
    "eqx_host_alloc": ([C.c_int64], C.c_void_p),
    "eqx_host_free": ([C.c_void_p], C.c_int),
    "eqx_ctx_create": ([C.c_int32, C.POINTER(C.c_void_p)], C.c_int),
    "eqx_ctx_destroy": ([C.c_void_p], None),
    "eqx_last_error": ([C.c_void_p], C.c_char_p),
    "eqx_ctx_stream": ([C.c_void_p], C.c_void_p),
    "eqx_ctx_copy_stream": ([C.c_void_p], C.c_void_p),
    "eqx_ctx_set_stream": ([C.c_void_p, C.c_void_p], C.c_int),
    "eqx_shard_record_bytes": ([C.c_int32, C.c_int32], C.c_int64),
    "eqx_shard_export_async": ([C.c_void_p, C.c_double, C.c_int32, C.c_int32, C.c_void_p], C.c_int),
    "eqx_shard_select_async": ([C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, _i32p, C.c_int32, C.c_int32,
                                C.c_double], C.c_int),
    "eqx_feedback": ([C.c_void_p, _i64p, C.POINTER(Completions), C.c_double], C.c_int),
    "eqx_set_timing": ([C.c_void_p, C.c_double, C.c_double, C.c_double, C.c_double, C.c_double], C.c_int),
    "eqx_replay": ([C.c_void_p, C.POINTER(Replays), C.POINTER(ReplayOut)], C.c_int),
    "eqx_get_service": ([C.c_void_p, C.c_int32, _dp, _i64p], C.c_int),
    "eqx_set_service": ([C.c_void_p, C.c_int32, _dp], C.c_int),
    "eqx_get_profile": ([C.c_void_p, C.c_int32, _dp, _dp, _dp], C.c_int),
    "eqx_set_policy": ([C.c_void_p, C.POINTER(Policy)], C.c_int),
    "eqx_set_perf": ([C.c_void_p, C.POINTER(Perf)], C.c_int),
    "eqx_set_profile": ([C.c_void_p, C.POINTER(Profile)], C.c_int),
    "eqx_set_predictor": ([C.c_void_p, C.POINTER(Predictor)], C.c_int),
    "eqx_set_clients": ([C.c_void_p, C.c_int32, C.c_char_p, _dp, _dp, _dp, _dp, _i32p], C.c_int),
    "eqx_get_clients": ([C.c_void_p, C.c_int32, _dp, _dp, _dp, _i32p, _i32p], C.c_int),
    "eqx_step_ledger": ([C.c_void_p, C.c_int32, _dp, _dp, _dp, _i32p, _i32p], C.c_int),
    "eqx_set_batch": ([C.c_void_p, C.c_int32, C.c_int64], C.c_int),
    "eqx_ledger_checkpoint": ([C.c_void_p], C.c_int),
    "eqx_ledger_restore_async": ([C.c_void_p], C.c_int),
    "eqx_drain": ([C.c_void_p, C.POINTER(Requests)], C.c_int),
    "eqx_stage_async": ([C.c_void_p, C.POINTER(Requests)], C.c_int),
    "eqx_append": ([C.c_void_p, C.POINTER(Requests)], C.c_int),
    "eqx_step_async": ([C.c_void_p, C.c_double], C.c_int),
    "eqx_drain_step_async": ([C.c_void_p, C.POINTER(Requests), C.c_double], C.c_int),
    "eqx_step_collect": ([C.c_void_p, C.POINTER(StepSummary)], C.c_int),
    "eqx_step": ([C.c_void_p, C.c_double, C.POINTER(StepSummary)], C.c_int),
    "eqx_copy_events": ([C.c_void_p, C.c_int64, _i64p, _i32p, _i32p, _i32p, _dp, _dp, _dp, _dp], C.c_int),
    "eqx_phase_times": ([C.c_void_p, _dp, C.c_int32], C.c_int),
    "eqx_kernel_times": ([C.c_void_p, C.POINTER(C.c_float)], C.c_int),
    "eqx_copy_scores": ([C.c_void_p, C.c_int64, _i32p, _u8p, _dp, _dp], C.c_int),
    "eqx_ufc_increment": ([C.c_double, C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_double, C.c_double], C.c_double),
    "eqx_rfc_increment": ([C.c_double, C.c_double, C.c_double], C.c_double),
    "eqx_pack_arrivals": ([C.c_void_p, C.c_int64, C.c_void_p, C.c_int64], C.c_int64),
}
EQX_NARROW_U16, EQX_PACKED_ARRIVALS = 1, 2

EXPORTED = sorted(_SIGS)

_lib = None


def load() -> C.CDLL:
    """Load libeqx_b200.so (built by __graft_entry__.build()); raises if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`. "
                "There is no CPU fallback for the scheduling step.")
        lib = C.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
    return _lib
