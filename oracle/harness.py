"""ctypes harness over the two CPU oracles -- TEST INFRASTRUCTURE ONLY.

Loads
  * ``oracle/liboracle.so``       -- the plain-C restatement (oracle/eqx_oracle.c), and
  * ``oracle/_ref/libeqx_ref.so`` -- the reference's own code compiled from
    /root/reference/proj/src plus the ref_step.cpp driver (oracle/Makefile ``ref``),
and runs one scheduling step (eqx_oracle.h) on numpy arrays.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs import this.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_ORACLE = os.path.join(HERE, "liboracle.so")
LIB_REF = os.path.join(HERE, "_ref", "libeqx_ref.so")

FCFS, VTC, EQUINOX = 0, 1, 2
NORM_MAX, NORM_NONE = 0, 1
PRED_ORACLE, PRED_MOPE, PRED_NOISY, PRED_SINGLE = 0, 1, 2, 3
EV_ADMIT, EV_REJECT = 1, 2

_dp = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)


class Mope(C.Structure):
    _fields_ = [
        ("n_thresholds", C.c_int32), ("thresholds", _i32p), ("mix_weight", C.c_double),
        ("num_buckets", C.c_int32), ("n_rows", C.c_int32), ("rows", _dp),
        ("n_experts", C.c_int32), ("n_bins", C.c_int32), ("bin_upper", _i32p),
        ("bin_value", _i32p), ("out_min", _i32p), ("out_max", _i32p),
    ]


class StepIn(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("alpha", C.c_double), ("delta", C.c_double),
        ("output_weight", C.c_double), ("norm_mode", C.c_int32),
        ("vtc_use_prediction", C.c_int32), ("counter_lift", C.c_int32), ("backfill", C.c_int32),
        ("max_batch", C.c_int32), ("mem_per_token_bytes", C.c_double),
        ("mem_capacity_bytes", C.c_double),
        ("n_profile", C.c_int32), ("prof_upper", _i32p), ("prof_lat", _dp), ("prof_util", _dp),
        ("prof_tps", _dp),
        ("pred_kind", C.c_int32), ("mope", Mope), ("noisy_l1", C.c_double),
        ("noisy_seed", C.c_uint64),
        ("n_clients", C.c_int32), ("client_names", C.c_char_p), ("weight", _dp), ("ufc0", _dp),
        ("rfc0", _dp), ("counter0", _dp), ("running", _i32p),
        ("n_members", C.c_int32), ("mem_in", _i32p), ("mem_generated", _i32p),
        ("mem_reserved", _i32p),
        ("n_req", C.c_int64), ("id", _i64p), ("client", _i32p), ("arrival", _dp),
        ("in_tokens", _i32p), ("true_out", _i32p), ("tag", _i32p), ("n_tags", C.c_int32),
        ("tag_names", C.c_char_p), ("tag_row", _i32p), ("now", C.c_double), ("duration_s", C.c_double),
        ("prediction_overhead_ms", C.c_double),
    ]


class StepOut(C.Structure):
    _fields_ = [
        ("pred", _i32p), ("bucket", _i32p), ("lat", _dp), ("util", _dp), ("tps", _dp),
        ("ufc_inc", _dp), ("rfc_inc", _dp),
        ("n_events", C.c_int64), ("ev_id", _i64p), ("ev_kind", _i32p), ("ev_client", _i32p),
        ("ev_ufc_inc", _dp), ("ev_rfc_inc", _dp), ("ev_vtc_inc", _dp), ("ev_wait", _dp),
        ("ufc", _dp), ("rfc", _dp), ("counter", _dp), ("backlogged", _i32p),
        ("n_admitted", C.c_int64), ("n_rejected", C.c_int64), ("new_prefill", C.c_int64),
        ("length_fallbacks", C.c_int64), ("ns_drain", C.c_double), ("ns_admit", C.c_double),
    ]


def _ptr(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


@dataclass
class StepCase:
    """Everything one scheduling step consumes (numpy arrays + scalars)."""

    # requests (arrival order)
    client: np.ndarray
    arrival: np.ndarray
    in_tokens: np.ndarray
    true_out: np.ndarray
    tag: np.ndarray                      # -1 = untagged, else index into tag_names
    id: np.ndarray | None = None
    # roster
    client_names: list = field(default_factory=list)
    weight: np.ndarray | None = None
    ufc0: np.ndarray | None = None
    rfc0: np.ndarray | None = None
    counter0: np.ndarray | None = None
    running: np.ndarray | None = None
    # batch
    mem_in: np.ndarray | None = None
    mem_generated: np.ndarray | None = None
    mem_reserved: np.ndarray | None = None
    # tags / model
    tag_names: list = field(default_factory=lambda: ["short", "medium", "long"])
    model: dict | None = None            # reference MopeModel JSON (predictor.cpp:408-430)
    pred_kind: int = PRED_MOPE
    noisy_l1: float = 33.0
    noisy_seed: int = 1
    # profile
    profile: dict | None = None          # {"upper","lat","util","tps"}
    # policy / perf
    kind: int = EQUINOX
    alpha: float = 0.7
    delta: float = 0.1
    output_weight: float = 4.0
    norm_mode: int = NORM_MAX
    vtc_use_prediction: bool = False
    counter_lift: bool = True
    backfill: bool = False
    max_batch: int = 64
    mem_per_token_bytes: float = 0.5 * 1024.0 * 1024.0
    mem_capacity_bytes: float = 60.0 * 1024.0 * 1024.0 * 1024.0
    now: float = 1.0
    duration_s: float = 0.0              # replays: Trace::duration_s (0: the last arrival)
    prediction_overhead_ms: float = 0.0  # replays: EngineConfig::prediction_overhead_ms

    def finalize(self):
        n = len(self.client)
        C_ = len(self.client_names)
        if self.id is None:
            self.id = np.arange(n, dtype=np.int64)
        z = np.zeros(C_, dtype=np.float64)
        self.weight = np.ones(C_) if self.weight is None else self.weight
        self.ufc0 = z.copy() if self.ufc0 is None else self.ufc0
        self.rfc0 = z.copy() if self.rfc0 is None else self.rfc0
        self.counter0 = z.copy() if self.counter0 is None else self.counter0
        self.running = np.zeros(C_, np.int32) if self.running is None else self.running
        e = np.zeros(0, np.int32)
        self.mem_in = e if self.mem_in is None else self.mem_in
        self.mem_generated = np.zeros_like(self.mem_in) if self.mem_generated is None else self.mem_generated
        self.mem_reserved = np.zeros_like(self.mem_in) if self.mem_reserved is None else self.mem_reserved
        return self


def mope_arrays(model: dict, tag_names: list):
    """Flatten a reference MopeModel JSON into the eqxo_mope arrays + per-tag row map."""
    r = model["router"]
    ks = r["keyword_scores"]
    row_names = sorted(ks.keys())  # std::map order (bytewise)
    nb = int(r["num_buckets"])
    rows = np.array([ks[k] for k in row_names], dtype=np.float64).reshape(len(row_names), nb)
    ex = model["experts"]
    nbins = len(ex[0]["bin_upper"])
    return dict(
        thresholds=np.array(r["input_len_thresholds"], np.int32),
        mix=float(r["mix_weight"]), num_buckets=nb, rows=rows,
        bin_upper=np.array([e["bin_upper"] for e in ex], np.int32).reshape(len(ex), nbins),
        bin_value=np.array([e["bin_value"] for e in ex], np.int32).reshape(len(ex), nbins),
        out_min=np.array([e["out_min"] for e in ex], np.int32),
        out_max=np.array([e["out_max"] for e in ex], np.int32),
        tag_row=np.array([row_names.index(t) if t in ks else -1 for t in tag_names], np.int32),
    )


def _build_in(case: StepCase, keep: list) -> StepIn:
    case.finalize()

    def arr(a, dt):
        a = np.ascontiguousarray(a, dtype=dt)
        keep.append(a)
        return a

    s = StepIn()
    s.kind, s.alpha, s.delta, s.output_weight = case.kind, case.alpha, case.delta, case.output_weight
    s.norm_mode = case.norm_mode
    s.vtc_use_prediction, s.counter_lift, s.backfill = int(case.vtc_use_prediction), int(case.counter_lift), int(case.backfill)
    s.max_batch = case.max_batch
    s.mem_per_token_bytes, s.mem_capacity_bytes = case.mem_per_token_bytes, case.mem_capacity_bytes
    p = case.profile
    s.n_profile = len(p["upper"])
    s.prof_upper = _ptr(arr(p["upper"], np.int32), C.c_int32)
    s.prof_lat = _ptr(arr(p["lat"], np.float64), C.c_double)
    s.prof_util = _ptr(arr(p["util"], np.float64), C.c_double)
    s.prof_tps = _ptr(arr(p["tps"], np.float64), C.c_double)
    s.pred_kind = case.pred_kind
    s.noisy_l1, s.noisy_seed = case.noisy_l1, case.noisy_seed
    if case.model is not None:
        m = mope_arrays(case.model, case.tag_names)
        s.mope.n_thresholds = len(m["thresholds"])
        s.mope.thresholds = _ptr(arr(m["thresholds"], np.int32), C.c_int32)
        s.mope.mix_weight = m["mix"]
        s.mope.num_buckets = m["num_buckets"]
        s.mope.n_rows = m["rows"].shape[0]
        s.mope.rows = _ptr(arr(m["rows"], np.float64), C.c_double)
        s.mope.n_experts, s.mope.n_bins = m["bin_upper"].shape
        s.mope.bin_upper = _ptr(arr(m["bin_upper"], np.int32), C.c_int32)
        s.mope.bin_value = _ptr(arr(m["bin_value"], np.int32), C.c_int32)
        s.mope.out_min = _ptr(arr(m["out_min"], np.int32), C.c_int32)
        s.mope.out_max = _ptr(arr(m["out_max"], np.int32), C.c_int32)
        tag_row = m["tag_row"]
    else:
        tag_row = -np.ones(len(case.tag_names), np.int32)
    s.n_clients = len(case.client_names)
    names = b"".join(n.encode() + b"\0" for n in case.client_names)
    keep.append(names)
    s.client_names = names
    s.weight = _ptr(arr(case.weight, np.float64), C.c_double)
    s.ufc0 = _ptr(arr(case.ufc0, np.float64), C.c_double)
    s.rfc0 = _ptr(arr(case.rfc0, np.float64), C.c_double)
    s.counter0 = _ptr(arr(case.counter0, np.float64), C.c_double)
    s.running = _ptr(arr(case.running, np.int32), C.c_int32)
    s.n_members = len(case.mem_in)
    s.mem_in = _ptr(arr(case.mem_in, np.int32), C.c_int32)
    s.mem_generated = _ptr(arr(case.mem_generated, np.int32), C.c_int32)
    s.mem_reserved = _ptr(arr(case.mem_reserved, np.int32), C.c_int32)
    s.n_req = len(case.client)
    s.id = _ptr(arr(case.id, np.int64), C.c_int64)
    s.client = _ptr(arr(case.client, np.int32), C.c_int32)
    s.arrival = _ptr(arr(case.arrival, np.float64), C.c_double)
    s.in_tokens = _ptr(arr(case.in_tokens, np.int32), C.c_int32)
    s.true_out = _ptr(arr(case.true_out, np.int32), C.c_int32)
    s.tag = _ptr(arr(case.tag, np.int32), C.c_int32)
    s.n_tags = len(case.tag_names)
    tn = b"".join(n.encode() + b"\0" for n in case.tag_names)
    keep.append(tn)
    s.tag_names = tn
    s.tag_row = _ptr(arr(tag_row, np.int32), C.c_int32)
    s.now = case.now
    s.duration_s = float(case.duration_s)
    s.prediction_overhead_ms = float(case.prediction_overhead_ms)
    return s


_libs: dict = {}


def _lib(which: str):
    if which not in _libs:
        path = LIB_REF if which == "ref" else LIB_ORACLE
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run __graft_entry__.build())")
        if which == "ref":
            # the reference objects use iostreams / locale state of the system libstdc++; load it
            # globally first so it is not resolved against a copy a wheel loaded privately
            C.CDLL("libstdc++.so.6", mode=C.RTLD_GLOBAL)
        lib = C.CDLL(path)
        fn = lib.ref_step if which == "ref" else lib.eqxo_step
        fn.argtypes = [C.POINTER(StepIn), C.POINTER(StepOut), C.c_char_p, C.c_int]
        fn.restype = C.c_int
        _libs[which] = (lib, fn)
    return _libs[which]


def available(which: str) -> bool:
    return os.path.exists(LIB_REF if which == "ref" else LIB_ORACLE)


def run_step(case: StepCase, which: str = "oracle") -> dict:
    """Run one step on the C restatement (``oracle``) or the reference build (``ref``)."""
    keep: list = []
    s = _build_in(case, keep)
    n, nc = int(s.n_req), int(s.n_clients)
    o = {
        "pred": np.zeros(n, np.int32), "bucket": np.zeros(n, np.int32),
        "lat": np.zeros(n), "util": np.zeros(n), "tps": np.zeros(n),
        "ufc_inc": np.zeros(n), "rfc_inc": np.zeros(n),
        "ev_id": np.zeros(max(n, 1), np.int64), "ev_kind": np.zeros(max(n, 1), np.int32),
        "ev_client": np.zeros(max(n, 1), np.int32), "ev_ufc_inc": np.zeros(max(n, 1)),
        "ev_rfc_inc": np.zeros(max(n, 1)), "ev_vtc_inc": np.zeros(max(n, 1)),
        "ev_wait": np.zeros(max(n, 1)),
        "ufc": np.zeros(nc), "rfc": np.zeros(nc), "counter": np.zeros(nc),
        "backlogged": np.zeros(nc, np.int32),
    }
    so = StepOut()
    for k, v in o.items():
        setattr(so, k, _ptr(v, np.ctypeslib.as_ctypes_type(v.dtype)))
    err = C.create_string_buffer(512)
    _, fn = _lib(which)
    rc = fn(C.byref(s), C.byref(so), err, 512)
    if rc != 0:
        raise ValueError(err.value.decode())
    ne = int(so.n_events)
    for k in list(o):
        if k.startswith("ev_"):
            o[k] = o[k][:ne]
    o.update(n_events=ne, n_admitted=int(so.n_admitted), n_rejected=int(so.n_rejected),
             new_prefill=int(so.new_prefill), length_fallbacks=int(so.length_fallbacks),
             ns_drain=float(so.ns_drain), ns_admit=float(so.ns_admit))
    return o


# ---- reference fixture helpers (ref build only) ----------------------------------------
def ref_train_mope_json(corpus_size=10000, seed=7, experts=3) -> str:
    lib, _ = _lib("ref")
    f = lib.ref_train_mope_json
    f.argtypes = [C.c_int, C.c_uint64, C.c_int, C.c_char_p, C.c_int64]
    f.restype = C.c_int64
    n = f(corpus_size, seed, experts, None, 0)
    buf = C.create_string_buffer(int(n))
    f(corpus_size, seed, experts, buf, n)
    return buf.value.decode()


def ref_build_profile(bounds=(32, 64, 128, 256, 512, 1024, 2048, 4096), ref_input=1) -> dict:
    lib, _ = _lib("ref")
    n = len(bounds)
    b = np.array(bounds, np.int32)
    up = np.zeros(n, np.int32)
    lat, util, tps = np.zeros(n), np.zeros(n), np.zeros(n)
    lib.ref_build_profile.restype = C.c_int
    rc = lib.ref_build_profile(_ptr(b, C.c_int32), C.c_int(n), C.c_int(ref_input),
                               _ptr(up, C.c_int32), _ptr(lat, C.c_double),
                               _ptr(util, C.c_double), _ptr(tps, C.c_double))
    if rc != 0:
        raise ValueError("build_profile rejected its arguments")
    return {"upper": up, "lat": lat, "util": util, "tps": tps}


def ref_noisy_predict(l1, seed, ids, true_out):
    lib, _ = _lib("ref")
    ids = np.ascontiguousarray(ids, np.int64)
    t = np.ascontiguousarray(true_out, np.int32)
    out = np.zeros(len(ids), np.int32)
    lib.ref_noisy_predict.argtypes = [C.c_double, C.c_uint64, C.c_int64, _i64p, _i32p, _i32p]
    lib.ref_noisy_predict(l1, seed, len(ids), _ptr(ids, C.c_int64), _ptr(t, C.c_int32),
                          _ptr(out, C.c_int32))
    return out


def ref_replay(case: StepCase, max_sim_time_s=3600.0, ema_alpha=0.2, cap=None):
    """Full run_simulation replay; returns (ev_id, ev_kind, ev_time, ufc, rfc, counter)."""
    lib, _ = _lib("ref")
    keep: list = []
    s = _build_in(case, keep)
    cap = cap or max(1, 2 * int(s.n_req))
    ev_id = np.zeros(cap, np.int64)
    ev_kind = np.zeros(cap, np.int32)
    ev_time = np.zeros(cap)
    nc = int(s.n_clients)
    u, r, c = np.zeros(nc), np.zeros(nc), np.zeros(nc)
    err = C.create_string_buffer(512)
    f = lib.ref_replay
    f.argtypes = [C.POINTER(StepIn), C.c_double, C.c_double, _i64p, _i32p, _dp, C.c_int64,
                  _dp, _dp, _dp, C.c_char_p, C.c_int]
    f.restype = C.c_int64
    n = f(C.byref(s), max_sim_time_s, ema_alpha, _ptr(ev_id, C.c_int64), _ptr(ev_kind, C.c_int32),
          _ptr(ev_time, C.c_double), cap, _ptr(u, C.c_double), _ptr(r, C.c_double),
          _ptr(c, C.c_double), err, 512)
    if n < 0:
        raise ValueError(err.value.decode())
    n = min(int(n), cap)
    return ev_id[:n], ev_kind[:n], ev_time[:n], u, r, c


# ---- completion / feedback path ---------------------------------------
class Feedback(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("alpha", C.c_double), ("delta", C.c_double), ("output_weight", C.c_double),
        ("vtc_use_prediction", C.c_int32), ("n_clients", C.c_int32), ("weight", _dp),
        ("ufc", _dp), ("rfc", _dp), ("counter", _dp), ("service", _dp), ("running", _i32p),
        ("n_profile", C.c_int32), ("prof_upper", _i32p), ("prof_lat", _dp), ("prof_util", _dp),
        ("prof_tps", _dp), ("ema_alpha", C.c_double), ("tokens", _i64p), ("n_done", C.c_int64),
        ("client", _i32p), ("in_tokens", _i32p), ("out_tokens", _i32p), ("latency_s", _dp), ("tps", _dp),
        ("util", _dp), ("pend_ufc", _dp), ("pend_rfc", _dp), ("pend_vtc", _dp), ("clamps", C.c_int64),
    ]


def _feedback_struct(fb: dict, ledger: dict, done_client, pend, keep: list) -> Feedback:
    def arr(x, dt):
        a = np.ascontiguousarray(x, dt)
        keep.append(a)
        return a
    f = Feedback()
    f.kind, f.alpha, f.delta, f.output_weight = fb["kind"], fb["alpha"], fb["delta"], fb["output_weight"]
    f.vtc_use_prediction = int(fb["vtc_use_prediction"])
    f.n_clients = len(fb["weight"])
    f.weight = _ptr(arr(fb["weight"], np.float64), C.c_double)
    for k in ("ufc", "rfc", "counter", "service"):
        setattr(f, k, _ptr(ledger[k], C.c_double))
    f.running = _ptr(ledger["running"], C.c_int32)
    prof = fb["profile"]
    f.n_profile = len(prof["upper"])
    f.prof_upper = _ptr(arr(prof["upper"], np.int32), C.c_int32)
    for k, src in (("prof_lat", "lat"), ("prof_util", "util"), ("prof_tps", "tps")):
        setattr(f, k, _ptr(ledger[k], C.c_double))
    f.ema_alpha = fb["ema_alpha"]
    f.tokens = _ptr(arr(fb["tokens"], np.int64), C.c_int64)
    d = fb["done"]
    f.n_done = len(d["adm"])
    f.client = _ptr(arr(done_client, np.int32), C.c_int32)
    f.in_tokens = _ptr(arr(np.asarray(fb["adm"]["in"])[np.asarray(d["adm"], np.int64)], np.int32), C.c_int32)
    f.out_tokens = _ptr(arr(d["out"], np.int32), C.c_int32)
    f.latency_s = _ptr(arr(d["latency_s"], np.float64), C.c_double)
    f.tps = _ptr(arr(d["tps"], np.float64), C.c_double)
    f.util = _ptr(arr(d["util"], np.float64), C.c_double)
    f.pend_ufc = _ptr(arr(pend[0], np.float64), C.c_double)
    f.pend_rfc = _ptr(arr(pend[1], np.float64), C.c_double)
    f.pend_vtc = _ptr(arr(pend[2], np.float64), C.c_double)
    return f


def run_feedback(fb: dict, which: str = "ref", pend=None, mid=None) -> dict:
    """One iteration's feedback (on_admit registrations, on_tokens, on_complete + update_map).

    ``ref``: through the reference objects (admissions included); returns the registered
    pending increments and the ledger after the admissions too.  ``oracle``: the C restatement,
    starting from ``mid`` (ledger after admissions) with the given ``pend`` increments."""
    keep: list = []
    nc = len(fb["weight"])
    done_adm = np.asarray(fb["done"]["adm"], np.int64)
    adm_client = np.asarray(fb["adm"]["client"], np.int32)
    done_client = adm_client[done_adm] if len(done_adm) else np.zeros(0, np.int32)
    led = {k: np.array(fb[k + "0"], np.float64) for k in ("ufc", "rfc", "counter", "service")}
    led["running"] = np.array(fb.get("running0", np.zeros(nc)), np.int32)
    for k, src in (("prof_lat", "lat"), ("prof_util", "util"), ("prof_tps", "tps")):
        led[k] = np.array(fb["profile"][src], np.float64)
    n_adm = len(adm_client)
    if which == "ref":
        pend_out = np.zeros(3 * max(n_adm, 1))
        mid_out = np.zeros(3 * max(nc, 1))
        pend_in = pend_out.reshape(3, -1)[:, done_adm] if n_adm else np.zeros((3, 0))
        f = _feedback_struct(fb, led, done_client, np.zeros((3, len(done_adm))), keep)
        lib, _ = _lib("ref")
        fn = lib.ref_feedback
        fn.restype = C.c_int
        names = b"".join(n.encode() + b"\0" for n in fb["names"])
        a = {k: np.ascontiguousarray(fb["adm"][k], dt) for k, dt in
             (("id", np.int64), ("client", np.int32), ("in", np.int32), ("pred", np.int32), ("wait", np.float64))}
        err = C.create_string_buffer(512)
        rc = fn(C.byref(f), C.c_char_p(names), C.c_double(fb["now"]), C.c_int64(n_adm),
                _ptr(a["id"], C.c_int64), _ptr(a["client"], C.c_int32), _ptr(a["in"], C.c_int32), _ptr(a["pred"], C.c_int32),
                _ptr(a["wait"], C.c_double), _ptr(np.ascontiguousarray(done_adm.astype(np.int32)), C.c_int32),
                _ptr(pend_out, C.c_double), _ptr(mid_out, C.c_double), err, 512)
        if rc:
            raise RuntimeError(err.value.decode())
        pend = pend_out[:3 * n_adm].reshape(3, n_adm) if n_adm else np.zeros((3, 0))
        mid = mid_out[:3 * nc].reshape(3, nc)
        del pend_in
    else:
        for i, k in enumerate(("ufc", "rfc", "counter")):
            led[k][:] = mid[i]
        f = _feedback_struct(fb, led, done_client, np.asarray(pend)[:, done_adm], keep)
        lib = _lib("oracle")[0]
        lib.eqxo_feedback_run.restype = C.c_int
        if lib.eqxo_feedback_run(C.byref(f)):
            raise ValueError("ema_alpha must lie in (0, 1]")
    out = {k: led[k].copy() for k in ("ufc", "rfc", "counter", "service", "running", "prof_lat", "prof_util",
                                        "prof_tps")}
    out["clamps"] = int(f.clamps)
    out["pend"] = pend
    out["mid"] = mid
    return out


def feedback_case(seed: int, kind: int = 2, vtc_use_prediction: int = 0, n_clients: int = 5, n_adm: int = 12,
                  n_done: int = 8, ledger_scale: float = 1.0, ema_alpha: float = 0.2, profile: dict | None = None,
                  weights=None) -> dict:
    """A seeded feedback scenario: n_adm admissions (registered through on_admit), one
    iteration's decode tokens, and n_done of the admitted requests completing in a random order."""
    rng = np.random.default_rng(seed)
    C = n_clients
    w = np.asarray(weights, np.float64) if weights is not None else rng.choice([0.5, 1.0, 2.0], C)
    return dict(kind=kind, alpha=0.7, delta=0.1, output_weight=4.0, vtc_use_prediction=vtc_use_prediction,
                names=[f"client{i}" for i in range(C)], weight=w,
                ufc0=rng.uniform(0, 1e4, C) * ledger_scale, rfc0=rng.uniform(0, 1e3, C) * ledger_scale,
                counter0=rng.uniform(0, 1e4, C) * ledger_scale, service0=rng.uniform(0, 1e5, C) * ledger_scale,
                profile={k: np.asarray(v) for k, v in profile.items()}, ema_alpha=ema_alpha, now=3.0,
                adm={"id": np.arange(100, 100 + n_adm, dtype=np.int64), "client": rng.integers(0, C, n_adm),
                     "in": rng.integers(8, 1000, n_adm), "pred": rng.integers(1, 1500, n_adm),
                     "wait": rng.uniform(0, 2, n_adm)},
                tokens=rng.integers(0, 5, C),
                done={"adm": rng.permutation(n_adm)[:n_done], "out": rng.integers(1, 5000, n_done),
                      "latency_s": rng.uniform(0.1, 30, n_done), "tps": rng.uniform(10, 5000, n_done),
                      "util": rng.uniform(0.2, 1, n_done)})


FEEDBACK_KEYS = ("ufc", "rfc", "counter", "service", "running", "prof_lat", "prof_util", "prof_tps")


def ref_multi(case: "StepCase", step_end, step_now, act_extra, act_tps, act_util, ema_alpha=0.2, complete_mod=3):
    """Several engine steps on live queues through the reference objects (oracle/ref_step.cpp
    ref_multi): events (id, kind, step, ufc_inc, rfc_inc), final ledger and profile."""
    lib, _ = _lib("ref")
    keep: list = []
    s = _build_in(case, keep)
    cap = max(1, 2 * int(s.n_req))
    out = {k: np.zeros(cap, dt) for k, dt in (("ev_id", np.int64), ("ev_kind", np.int32), ("ev_step", np.int32),
                                               ("ev_ufc", np.float64), ("ev_rfc", np.float64))}
    nc, npf = int(s.n_clients), int(s.n_profile)
    led = {k: np.zeros(nc) for k in ("ufc", "rfc", "counter")}
    prof = {k: np.zeros(npf) for k in ("lat", "util", "tps")}
    arr = {k: np.ascontiguousarray(v, np.float64) for k, v in (("now", step_now), ("extra", act_extra),
                                                                ("tps", act_tps), ("util", act_util))}
    end = np.ascontiguousarray(step_end, np.int64)
    err = C.create_string_buffer(512)
    f = lib.ref_multi
    f.restype = C.c_int64
    n = f(C.byref(s), C.c_int32(len(end)), _ptr(end, C.c_int64), _ptr(arr["now"], C.c_double),
          _ptr(arr["extra"], C.c_double), _ptr(arr["tps"], C.c_double), _ptr(arr["util"], C.c_double),
          C.c_double(ema_alpha), C.c_int32(complete_mod), _ptr(out["ev_id"], C.c_int64),
          _ptr(out["ev_kind"], C.c_int32), _ptr(out["ev_step"], C.c_int32), _ptr(out["ev_ufc"], C.c_double),
          _ptr(out["ev_rfc"], C.c_double), C.c_int64(cap), _ptr(led["ufc"], C.c_double), _ptr(led["rfc"], C.c_double),
          _ptr(led["counter"], C.c_double), _ptr(prof["lat"], C.c_double), _ptr(prof["util"], C.c_double),
          _ptr(prof["tps"], C.c_double), err, 512)
    if n < 0:
        raise ValueError(err.value.decode())
    n = min(int(n), cap)
    res = {k: v[:n] for k, v in out.items()}
    res.update(led)
    res.update({"prof_" + k: v for k, v in prof.items()})
    return res


REPORT_FIELDS = ("max_diff", "avg_diff", "var_diff", "jain_hf", "jain_ttft_p90", "throughput_tps", "mean_gpu_util",
                 "ttft_p50", "ttft_p90", "latency_p50", "latency_p90", "ttft_count", "latency_count", "sim_end_s",
                 "busy_ms_total", "overhead_ms_total", "completed", "rejected", "total_completed_tokens",
                 "n_windows", "n_diff", "n_rate")
CLIENT_FIELDS = ("final_hf", "accumulated_service", "mean_service_rate", "ttft_p50", "ttft_p90", "ttft_count")


def ref_replay_log(case: "StepCase", max_sim_time_s=0.0, ema_alpha=0.2, window_s=1.0) -> dict:
    """run_simulation's whole SimResult (oracle/_ref): the event log with its payloads (kind as
    EQX_EV_*, id, time, i0, d0..d2 -- include/eqx.h), the feedback-updated profile, the
    final ledger / accumulated service, max_resident_kv_tokens and the run totals."""
    lib, _ = _lib("ref")
    keep: list = []
    s = _build_in(case, keep)
    n, nc, npf = int(s.n_req), int(s.n_clients), int(s.n_profile)
    cap = 4 * n + 4
    o = {"id": np.zeros(cap, np.int64), "kind": np.zeros(cap, np.int32), "time": np.zeros(cap),
         "i0": np.zeros(cap, np.int32), "d0": np.zeros(cap), "d1": np.zeros(cap), "d2": np.zeros(cap),
         "profile": np.zeros((3, npf)), "clients": np.zeros((nc, 5)), "totals": np.zeros(8)}
    err = C.create_string_buffer(512)
    f = lib.ref_replay_log
    f.argtypes = [C.POINTER(StepIn), C.c_double, C.c_double, C.c_double, C.c_int64] + [C.c_void_p] * 10 + \
        [C.c_char_p, C.c_int]
    f.restype = C.c_int64
    ne = f(C.byref(s), max_sim_time_s, ema_alpha, window_s, cap,
           *[o[k].ctypes.data for k in ("id", "kind", "time", "i0", "d0", "d1", "d2", "profile", "clients", "totals")],
           err, 512)
    if ne < 0:
        raise ValueError(err.value.decode())
    for k in ("id", "kind", "time", "i0", "d0", "d1", "d2"):
        o[k] = o[k][:ne]
    t = o.pop("totals")
    o.update(sim_end=t[0], busy_ms_total=t[1], overhead_ms_total=t[2], max_resident_kv_tokens=int(t[3]),
             completed=int(t[4]), rejected=int(t[5]), counter_clamps=int(t[6]))
    return o


def ref_replay_full(case: "StepCase", max_sim_time_s=0.0, ema_alpha=0.2, window_s=1.0, win_cap=256) -> dict:
    """run_simulation + build_report through the reference objects (oracle/ref_step.cpp
    ref_replay_full): the SimReport summary, per-client reports (roster order) and the series
    (gpu_series, counter_series, diff_series, service_rate_series), cut at win_cap windows."""
    lib, _ = _lib("ref")
    keep: list = []
    s = _build_in(case, keep)
    nc = len(case.client_names)
    rep, cli = np.zeros(len(REPORT_FIELDS)), np.zeros((nc, len(CLIENT_FIELDS)))
    win, winc = np.zeros((win_cap, 4)), np.zeros((win_cap, nc, 4))
    diff, rate = np.zeros((win_cap, 2)), np.zeros((nc, win_cap))
    err = C.create_string_buffer(512)
    f = lib.ref_replay_full
    f.restype = C.c_int
    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
    if f(C.byref(s), C.c_double(max_sim_time_s), C.c_double(ema_alpha), C.c_double(window_s), C.c_int64(win_cap),
         dp(rep), dp(cli), dp(win), dp(winc), dp(diff), dp(rate), err, 512):
        raise ValueError(err.value.decode())
    return {"report": dict(zip(REPORT_FIELDS, rep)), "clients": {k: cli[:, i] for i, k in enumerate(CLIENT_FIELDS)},
            "win": win, "win_clients": winc, "diff": diff, "rate": rate}


def ref_replay_report(case: "StepCase", max_sim_time_s=0.0, ema_alpha=0.2) -> dict:
    """run_simulation + build_report: jain_ttft_p90, throughput_tps, completed, sim_end_s."""
    lib, _ = _lib("ref")
    keep: list = []
    s = _build_in(case, keep)
    j, t, e = C.c_double(), C.c_double(), C.c_double()
    n = C.c_int64()
    err = C.create_string_buffer(512)
    f = lib.ref_replay_report
    f.restype = C.c_int
    if f(C.byref(s), C.c_double(max_sim_time_s), C.c_double(ema_alpha), C.byref(j), C.byref(t), C.byref(n),
         C.byref(e), err, 512):
        raise ValueError(err.value.decode())
    return {"jain_ttft_p90": j.value, "throughput_tps": t.value, "completed": n.value, "sim_end": e.value}


# ---- traces -----------------------------------------------------------------
def ref_trace_load(path: str, cap: int = 1 << 18) -> dict:
    """The reference's load_trace + trace_hash (oracle/ref_step.cpp ref_trace_load); raises
    ValueError with the reference's ParseError message."""
    lib, _ = _lib("ref")
    n, nc, nw = C.c_int64(), C.c_int32(), C.c_int32()
    dur = C.c_double()
    client, arrival = np.zeros(cap, np.int32), np.zeros(cap)
    tin, tout = np.zeros(cap, np.int32), np.zeros(cap, np.int32)
    tags, names = C.create_string_buffer(32 * cap + 1), C.create_string_buffer(1 << 16)
    h, err = C.create_string_buffer(17), C.create_string_buffer(1024)
    f = lib.ref_trace_load
    f.restype = C.c_int
    vp = C.c_void_p
    f.argtypes = [C.c_char_p, C.c_int64, vp, vp, vp, vp, vp, C.c_char_p, C.c_int64, C.c_char_p, C.c_int64, vp, vp, vp,
                  C.c_char_p, C.c_char_p, C.c_int]
    if f(str(path).encode(), cap, C.addressof(n), client.ctypes.data, arrival.ctypes.data, tin.ctypes.data,
         tout.ctypes.data, tags, len(tags), names, len(names), C.addressof(nc), C.addressof(nw), C.addressof(dur), h,
         err, 1024):
        raise ValueError(err.value.decode())
    k = int(n.value)
    return {"n": k, "client": client[:k], "arrival": arrival[:k], "in_tokens": tin[:k], "out_tokens": tout[:k],
            "tags": tags.raw.split(b"\0")[:k] if k else [],
            "client_names": [x.decode() for x in names.raw.split(b"\0")[:nc.value]],
            "n_warnings": nw.value, "duration": dur.value, "hash": h.value.decode()}


def ref_scenario_csv(preset: str, seed: int, duration_s: float, path: str) -> str:
    """generate_scenario written by the reference's write_trace_csv; returns its trace_hash."""
    lib, _ = _lib("ref")
    h, err = C.create_string_buffer(17), C.create_string_buffer(1024)
    f = lib.ref_scenario_csv
    f.restype = C.c_int
    f.argtypes = [C.c_char_p, C.c_uint64, C.c_double, C.c_char_p, C.c_char_p, C.c_char_p, C.c_int]
    if f(preset.encode(), seed, duration_s, str(path).encode(), h, err, 1024):
        raise ValueError(err.value.decode())
    return h.value.decode()
