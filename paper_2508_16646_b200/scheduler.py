"""Host mirror of the reference scheduler interface over the C ABI (include/eqx.h).

Names, argument meaning and error behaviour follow the reference:
  * types      PolicySpec / EquinoxParams (scheduler.hpp:18-81), PerfParams (gpu_model.hpp:14-28),
               GpuProfile / ProfileEntry (gpu_model.hpp:61-77), ClientState (scheduler.hpp:35-43),
               MopeModel (predictor.hpp:85-92, JSON as predictor.cpp:408-454)
  * errors     ConfigError/ParseError -> ValueError, TrainingError/EngineError -> RuntimeError
               (bindings/module.cpp:53-56)
  * functions  ufc_increment / rfc_increment with the pybind signatures (module.cpp:144-172),
               default_bucket_bounds (gpu_model.cpp:128-130)
  * the path   GpuScheduler.drain() == SimulationRun::drain_arrivals (engine.cpp:171-197) for a
               batch of arrivals, GpuScheduler.step(now) == SimulationRun::admit_requests
               (engine.cpp:207-271) plus whole-queue scoring, both executed by sm_100a kernels.

Every scheduling decision runs on the GPU; nothing here computes a step on the CPU.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field
from typing import Iterable, Sequence

import numpy as np

from . import _lib as L


# ---- errors (errors.hpp:10-31; module.cpp:53-56) -------------------------------------------
class ConfigError(ValueError):
    pass


class ParseError(ValueError):
    pass


class TrainingError(RuntimeError):
    pass


class EngineError(RuntimeError):
    pass


_ERRORS = {L.EQX_ERR_CONFIG: ConfigError, L.EQX_ERR_PARSE: ParseError,
           L.EQX_ERR_ENGINE: EngineError, L.EQX_ERR_CUDA: EngineError, L.EQX_ERR_ARG: ValueError}

POLICY_KINDS = {"fcfs": 0, "vtc": 1, "equinox": 2}
NORM_MODES = {"max_over_clients": 0, "none": 1}
PREDICTORS = {"oracle": 0, "mope": 1, "noisy_oracle": 2, "single_proxy": 3}
EV_ADMITTED, EV_REJECTED = 1, 2


# ---- parameter blocks ------------------------------------------------------------------------
@dataclass
class EquinoxParams:
    alpha: float = 0.7
    delta: float = 0.1
    output_weight: float = 4.0
    norm_mode: str = "max_over_clients"

    def beta(self) -> float:
        return 1.0 - self.alpha

    def validate(self) -> None:  # scheduler.cpp:11-17
        if self.alpha < 0.0 or self.alpha > 1.0:
            raise ConfigError("alpha must lie in [0, 1]")
        if self.delta < 0.0:
            raise ConfigError("delta must be >= 0")
        if self.output_weight <= 0.0:
            raise ConfigError("output_weight must be > 0")


@dataclass
class PolicySpec:
    kind: str = "equinox"
    equinox: EquinoxParams = field(default_factory=EquinoxParams)
    vtc_use_prediction: bool = False
    counter_lift: bool = True

    def label(self) -> str:  # scheduler.cpp:86-90
        return self.kind + ("+pred" if self.kind == "vtc" and self.vtc_use_prediction else "")


@dataclass
class PerfParams:
    prefill_linear_ms: float = 0.05
    prefill_quad_ms: float = 1e-6
    decode_base_ms: float = 5.0
    decode_per_ctx_ms: float = 0.002
    refresh_ms: float = 15.0
    mem_per_token_bytes: float = 0.5 * 1024.0 * 1024.0
    mem_capacity_bytes: float = 60.0 * 1024.0 * 1024.0 * 1024.0
    max_batch: int = 64

    def token_capacity(self) -> float:
        return self.mem_capacity_bytes / self.mem_per_token_bytes


@dataclass
class ProfileEntry:
    bucket_upper: int
    latency_ms: float
    gpu_util: float
    tps: float


@dataclass
class GpuProfile:
    entries: list

    def empty(self) -> bool:
        return len(self.entries) == 0

    @staticmethod
    def from_arrays(upper, lat, util, tps) -> "GpuProfile":
        return GpuProfile([ProfileEntry(int(u), float(a), float(b), float(c))
                           for u, a, b, c in zip(upper, lat, util, tps)])

    @staticmethod
    def load_json(path: str) -> "GpuProfile":
        with open(path) as f:
            d = json.load(f)
        return GpuProfile.from_arrays(d["upper"], d["lat"], d["util"], d["tps"])


def default_bucket_bounds() -> list:
    """gpu_model.cpp:128-130."""
    return [32, 64, 128, 256, 512, 1024, 2048, 4096]


@dataclass
class ClientState:
    client_id: str
    weight: float = 1.0
    ufc: float = 0.0
    rfc: float = 0.0
    counter: float = 0.0
    accumulated_service: float = 0.0
    backlogged: bool = False


class MopeModel:
    """MopeModel JSON (predictor.cpp:408-454): bucket_bounds, router{input_len_thresholds,
    mix_weight, num_buckets, keyword_scores}, experts[{bucket, bin_upper, bin_value, out_min,
    out_max}]."""

    def __init__(self, doc: dict):
        try:
            self.bucket_bounds = [int(x) for x in doc["bucket_bounds"]]
            r = doc["router"]
            self.thresholds = [int(x) for x in r["input_len_thresholds"]]
            self.mix_weight = float(r["mix_weight"])
            self.num_buckets = int(r["num_buckets"])
            self.keyword_scores = {str(k): [float(v) for v in row] for k, row in r["keyword_scores"].items()}
            self.experts = [{"bucket": int(e["bucket"]), "bin_upper": [int(x) for x in e["bin_upper"]],
                             "bin_value": [int(x) for x in e["bin_value"]], "out_min": int(e["out_min"]),
                             "out_max": int(e["out_max"])} for e in doc["experts"]]
        except (KeyError, TypeError, ValueError) as exc:
            raise ParseError(f"malformed MoPE model JSON: {exc}") from exc
        if not self.experts:
            raise TrainingError("MoPE predictor constructed without trained experts")

    @staticmethod
    def from_json(doc) -> "MopeModel":
        return MopeModel(json.loads(doc) if isinstance(doc, str) else doc)

    @staticmethod
    def load(path: str) -> "MopeModel":
        with open(path) as f:
            return MopeModel(json.load(f))

    def to_json(self) -> dict:
        return {"bucket_bounds": self.bucket_bounds,
                "router": {"input_len_thresholds": self.thresholds, "mix_weight": self.mix_weight,
                           "num_buckets": self.num_buckets, "keyword_scores": self.keyword_scores},
                "experts": self.experts}


# ---- module.cpp:144-172 scalar helpers ---------------------------------------------------------
def ufc_increment(weight: float, input_tokens: int, predicted_output_tokens: int, wait_s: float = 0.0,
                  predicted_latency_ms: float = 0.0, delta: float = 0.1, output_weight: float = 4.0) -> float:
    return L.load().eqx_ufc_increment(weight, input_tokens, predicted_output_tokens, wait_s,
                                      predicted_latency_ms, delta, output_weight)


def rfc_increment(weight: float, tps: float, gpu_util: float) -> float:
    return L.load().eqx_rfc_increment(weight, tps, gpu_util)


# ---- the request batch -------------------------------------------------------------------------
def pinned_empty(shape, dtype) -> np.ndarray:
    """numpy array in the library's pinned host arena (eqx_host_alloc: 2 MiB-aligned, huge-page
    backed, driver-registered), for request columns a serving loop refills and stages every step.
    The arena is released when the array (and every view of it) is garbage."""
    import weakref
    dt = np.dtype(dtype)
    count = int(np.prod(shape, dtype=np.int64))
    nbytes = max(count * dt.itemsize, 1)
    lib = L.load()
    ptr = lib.eqx_host_alloc(nbytes)
    if not ptr:
        raise MemoryError(f"eqx_host_alloc({nbytes}) failed")
    buf = (C.c_uint8 * nbytes).from_address(ptr)
    weakref.finalize(buf, lib.eqx_host_free, C.c_void_p(ptr))
    return np.frombuffer(buf, dtype=dt, count=count).reshape(shape)


class PackedArrivals:
    """An arrival_s column packed by eqx_pack_arrivals (include/eqx.h): pass it as `arrival_s` of
    a host batch (drain / stage_async / drain_step_async) and about 6 instead of 8 bytes per
    request cross PCIe; the copy stream unpacks it on the device, bit-exact."""

    def __init__(self, data: np.ndarray, n: int):
        self.data = data  # uint8
        self.n = int(n)

    def __len__(self) -> int:
        return self.n


def pack_arrivals(arrival_s) -> PackedArrivals:
    """Lossless packing of an arrival column (pageable memory; pinned_copy() pins it): 256-row
    blocks of non-decreasing non-negative arrivals within 2^48 ulps of their first take 6 bytes
    per row, other blocks their 8-byte doubles (include/eqx.h: eqx_pack_arrivals)."""
    a = np.ascontiguousarray(arrival_s, dtype=np.float64)
    lib = L.load()
    ptr = a.ctypes.data if len(a) else None
    nbytes = int(lib.eqx_pack_arrivals(ptr, len(a), None, 0))
    if nbytes < 0:
        raise ValueError("eqx_pack_arrivals: bad arguments")
    out = np.empty(max(nbytes, 16), np.uint8)
    if int(lib.eqx_pack_arrivals(ptr, len(a), out.ctypes.data, out.nbytes)) != nbytes:
        raise RuntimeError("eqx_pack_arrivals: packing failed")
    return PackedArrivals(out, len(a))


def pinned_copy(x):
    if isinstance(x, PackedArrivals):
        return PackedArrivals(pinned_copy(x.data), x.n)
    a = np.ascontiguousarray(x)
    out = pinned_empty(a.shape, a.dtype)
    out[...] = a
    return out


def _as_col(x, dtype, keep: list):
    """numpy -> (host ptr, HOST); torch CUDA tensor -> (device ptr, DEVICE)."""
    if x is None:
        return None, None
    mod = type(x).__module__
    if mod.startswith("torch"):
        import torch
        want = {np.int32: torch.int32, np.int64: torch.int64, np.float64: torch.float64,
                np.uint8: torch.uint8}[dtype]
        if x.dtype != want:
            raise ValueError(f"column dtype {x.dtype} != {want}")
        x = x.contiguous()
        keep.append(x)
        return x.data_ptr(), (L.EQX_DEVICE if x.is_cuda else L.EQX_HOST)
    a = np.ascontiguousarray(x, dtype=dtype)
    keep.append(a)
    return a.ctypes.data, L.EQX_HOST


@dataclass
class StepResult:
    """Events of one step in log order (Admitted / Rejected, engine.cpp:223-268) with the
    PendingContribution of each admission (scheduler.hpp:131-138)."""
    ids: np.ndarray
    kinds: np.ndarray
    clients: np.ndarray
    preds: np.ndarray
    ufc_inc: np.ndarray
    rfc_inc: np.ndarray
    vtc_inc: np.ndarray
    wait_s: np.ndarray
    n_admitted: int
    n_rejected: int
    new_prefill_tokens: int
    length_fallbacks: int
    noisy_near_ties: int
    batch_members: int
    batch_reserved_kv_tokens: int
    queued: int = 0
    window_underflow: int = 0

    @property
    def admitted(self) -> np.ndarray:
        return self.ids[self.kinds == EV_ADMITTED]

    @property
    def rejected(self) -> np.ndarray:
        return self.ids[self.kinds == EV_REJECTED]


class GpuScheduler:
    """One engine instance's scheduler state on one B200 (one CUDA stream, not thread-safe,
    like SchedulerPolicy, scheduler.hpp:97-100)."""

    def __init__(self, clients: Sequence[ClientState], policy: PolicySpec | None = None,
                 perf: PerfParams | None = None, profile: GpuProfile | None = None,
                 predictor: str = "mope", model: MopeModel | None = None,
                 tag_names: Sequence[str] = (), noisy_l1: float = 33.0, noisy_seed: int = 1,
                 backfill: bool = False, running: Iterable[int] | None = None, device: int = 0):
        self._lib = L.load()
        h = C.c_void_p()
        self._check(self._lib.eqx_ctx_create(device, C.byref(h)), None)
        self._ctx = h
        self._keep: list = []
        self.policy = policy or PolicySpec()
        self.perf = perf or PerfParams()
        self.backfill = backfill
        self.tag_names = list(tag_names)
        self.client_ids = [c.client_id for c in clients]
        self._set_policy()
        p = L.Perf(int(self.perf.max_batch), float(self.perf.mem_per_token_bytes),
                   float(self.perf.mem_capacity_bytes))
        self._check(self._lib.eqx_set_perf(self._ctx, C.byref(p)))
        if profile is None or profile.empty():
            raise ConfigError("engine needs a non-empty GPU profile")
        self._set_profile(profile)
        self._set_predictor(predictor, model, noisy_l1, noisy_seed)
        self.set_clients(clients, running)

    # -- plumbing --
    def _check(self, rc: int, ctx="self") -> None:
        if rc != L.EQX_OK:
            msg = self._lib.eqx_last_error(self._ctx if ctx == "self" else None)
            raise _ERRORS.get(rc, EngineError)((msg or b"").decode())

    def close(self) -> None:
        if getattr(self, "_ctx", None):
            self._lib.eqx_ctx_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream_ptr(self) -> int:
        return self._lib.eqx_ctx_stream(self._ctx)

    def _set_policy(self) -> None:
        sp = self.policy
        if sp.kind not in POLICY_KINDS:
            raise ConfigError(f"unknown policy kind '{sp.kind}'")
        if sp.equinox.norm_mode not in NORM_MODES:
            raise ConfigError(f"unknown norm_mode '{sp.equinox.norm_mode}'")
        p = L.Policy(POLICY_KINDS[sp.kind], sp.equinox.alpha, sp.equinox.delta, sp.equinox.output_weight,
                     NORM_MODES[sp.equinox.norm_mode], int(sp.vtc_use_prediction), int(sp.counter_lift),
                     int(self.backfill))
        self._check(self._lib.eqx_set_policy(self._ctx, C.byref(p)))

    def _set_profile(self, profile: GpuProfile) -> None:
        e = profile.entries
        up = np.array([x.bucket_upper for x in e], np.int32)
        lat = np.array([x.latency_ms for x in e], np.float64)
        ut = np.array([x.gpu_util for x in e], np.float64)
        tp = np.array([x.tps for x in e], np.float64)
        self._n_profile = len(e)
        pr = L.Profile(len(e), up.ctypes.data_as(L._i32p), lat.ctypes.data_as(L._dp),
                       ut.ctypes.data_as(L._dp), tp.ctypes.data_as(L._dp))
        self._check(self._lib.eqx_set_profile(self._ctx, C.byref(pr)))

    def _set_predictor(self, kind: str, model: MopeModel | None, l1: float, seed: int) -> None:
        if kind not in PREDICTORS:
            raise ConfigError(f"unknown predictor kind '{kind}'")
        pd = L.Predictor()
        pd.kind = PREDICTORS[kind]
        pd.noisy_l1 = float(l1)
        pd.noisy_seed = int(seed)
        keep = []
        if kind in ("mope", "single_proxy"):
            if model is None:
                raise ConfigError(f"predictor '{kind}' needs a MopeModel")
            names = sorted(model.keyword_scores)  # std::map order
            nb = model.num_buckets
            rows = np.array([model.keyword_scores[k] for k in names], np.float64).reshape(len(names), nb)
            nbins = len(model.experts[0]["bin_upper"])
            if any(len(x["bin_upper"]) != nbins or len(x["bin_value"]) != nbins for x in model.experts):
                raise ParseError("malformed MoPE model: experts with different bin counts")
            arrs = dict(
                thr=np.array(model.thresholds, np.int32), rows=rows,
                bu=np.array([x["bin_upper"] for x in model.experts], np.int32),
                bv=np.array([x["bin_value"] for x in model.experts], np.int32),
                mn=np.array([x["out_min"] for x in model.experts], np.int32),
                mx=np.array([x["out_max"] for x in model.experts], np.int32),
                tr=np.array([names.index(t) if t in model.keyword_scores else -1 for t in self.tag_names] or [0],
                            np.int32))
            keep.append(arrs)
            m = pd.mope
            m.n_thresholds = len(model.thresholds)
            m.thresholds = arrs["thr"].ctypes.data_as(L._i32p)
            m.mix_weight = model.mix_weight
            m.num_buckets = nb
            m.n_rows = len(names)
            m.rows = arrs["rows"].ctypes.data_as(L._dp)
            m.n_experts = len(model.experts)
            m.n_bins = nbins
            m.bin_upper = arrs["bu"].ctypes.data_as(L._i32p)
            m.bin_value = arrs["bv"].ctypes.data_as(L._i32p)
            m.out_min = arrs["mn"].ctypes.data_as(L._i32p)
            m.out_max = arrs["mx"].ctypes.data_as(L._i32p)
            m.n_tags = len(self.tag_names)
            m.tag_row = arrs["tr"].ctypes.data_as(L._i32p)
        self.predictor = kind
        self._check(self._lib.eqx_set_predictor(self._ctx, C.byref(pd)))

    # -- ledger --
    def set_clients(self, clients: Sequence[ClientState], running: Iterable[int] | None = None) -> None:
        n = len(clients)
        self.client_ids = [c.client_id for c in clients]
        names = b"".join(c.client_id.encode() + b"\0" for c in clients)
        w = np.array([c.weight for c in clients], np.float64)
        u = np.array([c.ufc for c in clients], np.float64)
        r = np.array([c.rfc for c in clients], np.float64)
        k = np.array([c.counter for c in clients], np.float64)
        run = np.array(list(running) if running is not None else [0] * n, np.int32)
        self._check(self._lib.eqx_set_clients(self._ctx, n, names, w.ctypes.data_as(L._dp),
                                              u.ctypes.data_as(L._dp), r.ctypes.data_as(L._dp),
                                              k.ctypes.data_as(L._dp), run.ctypes.data_as(L._i32p)))

    def ledger(self) -> dict:
        n = len(self.client_ids)
        out = {k: np.zeros(n) for k in ("ufc", "rfc", "counter")}
        out["backlogged"] = np.zeros(n, np.int32)
        out["running"] = np.zeros(n, np.int32)
        self._check(self._lib.eqx_get_clients(self._ctx, n, out["ufc"].ctypes.data_as(L._dp),
                                              out["rfc"].ctypes.data_as(L._dp),
                                              out["counter"].ctypes.data_as(L._dp),
                                              out["backlogged"].ctypes.data_as(L._i32p),
                                              out["running"].ctypes.data_as(L._i32p)))
        return out

    def step_ledger(self) -> dict:
        """ledger() as the last collected step left it, from the mapped host copy its selection
        CTA wrote (eqx_step_ledger: no device copy); raises once the device ledger has changed."""
        n = len(self.client_ids)
        out = {k: np.zeros(n) for k in ("ufc", "rfc", "counter")}
        out["backlogged"] = np.zeros(n, np.int32)
        out["running"] = np.zeros(n, np.int32)
        self._check(self._lib.eqx_step_ledger(self._ctx, n, out["ufc"].ctypes.data_as(L._dp),
                                              out["rfc"].ctypes.data_as(L._dp),
                                              out["counter"].ctypes.data_as(L._dp),
                                              out["backlogged"].ctypes.data_as(L._i32p),
                                              out["running"].ctypes.data_as(L._i32p)))
        return out

    def clients(self) -> list:
        led = self.ledger()
        return [ClientState(cid, ufc=float(led["ufc"][i]), rfc=float(led["rfc"][i]),
                            counter=float(led["counter"][i]), backlogged=bool(led["backlogged"][i]))
                for i, cid in enumerate(self.client_ids)]

    def set_batch(self, members: int, reserved_kv_tokens: int) -> None:
        self._check(self._lib.eqx_set_batch(self._ctx, int(members), int(reserved_kv_tokens)))

    def checkpoint(self) -> None:
        """Device-side snapshot of ledger + batch state (restore() replays from it async)."""
        self._check(self._lib.eqx_ledger_checkpoint(self._ctx))

    def restore_async(self) -> None:
        self._check(self._lib.eqx_ledger_restore_async(self._ctx))

    # -- the hot path --
    def drain(self, client, arrival_s, input_tokens, tag=None, true_output_tokens=None, ids=None,
              id_base: int = 0) -> None:
        """Queue a batch of arrivals (arrival order).  numpy columns are copied host->device;
        torch CUDA tensors are used in place."""
        rq = self._requests(client, arrival_s, input_tokens, tag, true_output_tokens, ids, id_base)
        self._check(self._lib.eqx_drain(self._ctx, C.byref(rq)))

    def append(self, client, arrival_s, input_tokens, tag=None, true_output_tokens=None, ids=None,
               id_base: int = 0) -> None:
        """drain_arrivals for a batch that joins the requests still queued (live queue): the
        arrivals' prediction records are frozen against the current profile; step() then
        schedules from the whole live queue."""
        keep: list = []
        rq = self._requests(client, arrival_s, input_tokens, tag, true_output_tokens, ids, id_base, keep)
        self._check(self._lib.eqx_append(self._ctx, C.byref(rq)))

    def stage_async(self, client, arrival_s, input_tokens, tag=None, true_output_tokens=None, ids=None,
                    id_base: int = 0) -> None:
        """Prefetch a host batch (pinned numpy/torch CPU columns) into the context's next staging
        buffer on its copy stream; the drain of the same arrays then skips the copy.  The H2D
        overlaps the steps in flight (three staging buffers: up to two batches ahead)."""
        keep: list = []
        rq = self._requests(client, arrival_s, input_tokens, tag, true_output_tokens, ids, id_base, keep)
        if rq.location != L.EQX_HOST:
            raise ValueError("stage_async: host columns only")
        self._staged = getattr(self, "_staged", [])[-2:] + [keep]  # keep every staged batch alive (3 sets)
        self._check(self._lib.eqx_stage_async(self._ctx, C.byref(rq)))

    def drain_step_async(self, now: float, client, arrival_s, input_tokens, tag=None,
                         true_output_tokens=None, ids=None, id_base: int = 0) -> None:
        """drain + step_async in one call (CUDA-graph replay for a resident device queue)."""
        rq = self._requests(client, arrival_s, input_tokens, tag, true_output_tokens, ids, id_base)
        self._check(self._lib.eqx_drain_step_async(self._ctx, C.byref(rq), float(now)))

    def _requests(self, client, arrival_s, input_tokens, tag, true_output_tokens, ids, id_base, keep=None):
        staging = keep is not None
        keep = [] if keep is None else keep
        cols = {}
        loc = set()
        # uint16 host client + input_tokens columns travel narrow (13 instead of 17 bytes per
        # request over PCIe; eqx_requests::narrow) -- the caller chose them, so they are lossless
        narrow = (isinstance(client, np.ndarray) and client.dtype == np.uint16 and
                  isinstance(input_tokens, np.ndarray) and input_tokens.dtype == np.uint16)
        wide = np.uint16 if narrow else np.int32
        packed = isinstance(arrival_s, PackedArrivals)
        if packed:
            if arrival_s.n != len(client):
                raise ValueError("packed arrivals: row count differs from the client column")
            keep.append(arrival_s.data)
            cols["arrival_s"] = arrival_s.data.ctypes.data
            loc.add(L.EQX_HOST)
        for name, x, dt in (("client", client, wide), ("arrival_s", None if packed else arrival_s, np.float64),
                            ("input_tokens", input_tokens, wide), ("tag", tag, np.uint8),
                            ("true_output_tokens", true_output_tokens, np.int32), ("id", ids, np.int64)):
            if name == "arrival_s" and packed:
                continue
            ptr, where = _as_col(x, dt, keep)
            cols[name] = ptr
            if where is not None:
                loc.add(where)
        if len(loc) > 1:
            raise ValueError("drain: mix of host and device columns")
        n = len(client)
        rq = L.Requests(n, cols["id"], id_base, cols["client"], cols["arrival_s"], cols["input_tokens"],
                        cols["true_output_tokens"], cols["tag"], loc.pop() if loc else L.EQX_HOST,
                        (L.EQX_NARROW_U16 if narrow else 0) | (L.EQX_PACKED_ARRIVALS if packed else 0))
        if not staging:
            self._keep = keep  # device columns are used in place: keep them alive with the queue
            self.n_queued = n
        return rq

    def step_async(self, now: float) -> None:
        self._check(self._lib.eqx_step_async(self._ctx, float(now)))

    def collect(self, with_events: bool = True) -> StepResult:
        s = L.StepSummary()
        self._check(self._lib.eqx_step_collect(self._ctx, C.byref(s)))
        return self._result(s, with_events)

    def step(self, now: float, with_events: bool = True) -> StepResult:
        s = L.StepSummary()
        self._check(self._lib.eqx_step(self._ctx, float(now), C.byref(s)))
        return self._result(s, with_events)

    def _result(self, s: L.StepSummary, with_events: bool) -> StepResult:
        n = int(s.n_events) if with_events and not s.window_underflow else 0
        ids = np.zeros(n, np.int64)
        kinds, cl, pr = (np.zeros(n, np.int32) for _ in range(3))
        ui, ri, vi, wt = (np.zeros(n) for _ in range(4))
        if n:
            self._check(self._lib.eqx_copy_events(self._ctx, n, ids.ctypes.data_as(L._i64p),
                                                  kinds.ctypes.data_as(L._i32p), cl.ctypes.data_as(L._i32p),
                                                  pr.ctypes.data_as(L._i32p), ui.ctypes.data_as(L._dp),
                                                  ri.ctypes.data_as(L._dp), vi.ctypes.data_as(L._dp),
                                                  wt.ctypes.data_as(L._dp)))
        return StepResult(ids, kinds, cl, pr, ui, ri, vi, wt, int(s.n_admitted), int(s.n_rejected),
                          int(s.new_prefill_tokens), int(s.length_fallbacks), int(s.noisy_near_ties),
                          int(s.batch_members), int(s.batch_reserved_kv_tokens), int(s.queued),
                          int(s.window_underflow))

    # -- batched engine replays --
    def replay(self, row_off, client, arrival_s, input_tokens, true_output_tokens, alpha, tag=None, ids=None,
               max_sim_time_s: float = 0.0, ema_alpha: float = 0.2, ev_cap: int = 4096,
               report_window_s: float = 1.0, win_cap: int = 0, duration_s=None,
               prediction_overhead_ms: float = 0.0, predicted=None, log_all: bool = False) -> dict:
        """run_simulation (engine.cpp:119-146) for many traces at once on the GPU, one replay per
        warp: traces concatenated (row_off[r]..row_off[r+1]), per-replay alpha, the
        scheduler's policy / perf / profile / predictor / roster otherwise.  Returns the
        admitted/rejected event logs (id, kind, time), final ledgers and run statistics, and
        build_report's SimReport per replay ("report": a structured array with the fields of
        eqx_replay_report; "clients": [replay][client] ClientReport fields, roster order).
        With win_cap > 0 also the series, each cut at win_cap windows: "win" [r][w][4] (time,
        busy_ms, overhead_ms, gpu_util: SimResult::gpu_series), "win_clients" [r][w][C][4] (ufc,
        rfc, hf, service_cum: counter_series), "diff" [r][w][2] (diff_series) and "rate"
        [r][C][w] (service_rate_series values; window w ends at report_window_s * (w + 1)).

        ``duration_s`` [r]: each trace's Trace::duration_s, the horizon when max_sim_time_s is 0
        (engine.cpp:120-121; default: its last arrival).  ``prediction_overhead_ms`` delays
        eligibility (engine.cpp:165-168).  ``predicted`` [rows]: Predictor::predict of every row
        from a caller's predictor instead of the scheduler's.  ``log_all``: the events are the
        engine's whole log (EQX_EV_*: arrived 3, admitted 1, first_token 4, completed 5,
        rejected 2) with payloads "ev_i0", "ev_d0".."ev_d2" (include/eqx.h); "profile" [r][3][P]
        is the feedback-updated GPU profile (latency_ms, gpu_util, tps)."""
        n = len(alpha)
        nc = len(self.client_ids)
        cols = {"row_off": np.ascontiguousarray(row_off, np.int64), "client": np.ascontiguousarray(client, np.int32),
                "arrival_s": np.ascontiguousarray(arrival_s, np.float64),
                "input_tokens": np.ascontiguousarray(input_tokens, np.int32),
                "true_output_tokens": np.ascontiguousarray(true_output_tokens, np.int32),
                "alpha": np.ascontiguousarray(alpha, np.float64),
                "tag": None if tag is None else np.ascontiguousarray(tag, np.uint8),
                "id": None if ids is None else np.ascontiguousarray(ids, np.int64),
                "duration_s": None if duration_s is None else np.ascontiguousarray(duration_s, np.float64),
                "predicted": None if predicted is None else np.ascontiguousarray(predicted, np.int32)}
        ptr = {k: (v.ctypes.data if v is not None else None) for k, v in cols.items()}
        if report_window_s <= 0.0:
            raise ConfigError("'engine.report_window_s' must be > 0")
        wc = max(int(win_cap), 0)
        rq = L.Replays(n, ptr["row_off"], ptr["client"], ptr["arrival_s"], ptr["input_tokens"],
                       ptr["true_output_tokens"], ptr["tag"], ptr["id"], ptr["alpha"], float(max_sim_time_s),
                       float(ema_alpha), int(ev_cap), float(report_window_s), wc, ptr["duration_s"],
                       float(prediction_overhead_ms), ptr["predicted"], 1 if log_all else 0)
        out = {"n_events": np.zeros(n, np.int64), "ev_id": np.zeros((n, ev_cap), np.int64),
               "ev_kind": np.zeros((n, ev_cap), np.int32), "ev_time": np.zeros((n, ev_cap)),
               "ufc": np.zeros((n, nc)), "rfc": np.zeros((n, nc)), "counter": np.zeros((n, nc)),
               "completed": np.zeros(n, np.int64), "sim_end": np.zeros(n), "counter_clamps": np.zeros(n, np.int64),
               "status": np.zeros(n, np.int32), "jain_ttft_p90": np.zeros(n), "throughput_tps": np.zeros(n),
               "report": np.zeros(n, L.REPORT_DTYPE), "clients": np.zeros((n, nc), L.CLIENT_DTYPE),
               "profile": np.zeros((n, 3, self._n_profile))}
        if log_all:
            out.update(ev_i0=np.zeros((n, ev_cap), np.int32), ev_d0=np.zeros((n, ev_cap)),
                       ev_d1=np.zeros((n, ev_cap)), ev_d2=np.zeros((n, ev_cap)))
        if wc:
            out.update(win=np.zeros((n, wc, 4)), win_clients=np.zeros((n, wc, nc, 4)), diff=np.zeros((n, wc, 2)),
                       rate=np.zeros((n, nc, wc)))
        names = ("n_events", "ev_id", "ev_kind", "ev_time", "ufc", "rfc", "counter", "completed", "sim_end",
                 "counter_clamps", "status", "jain_ttft_p90", "throughput_tps", "report", "clients", "win",
                 "win_clients", "diff", "rate", "ev_i0", "ev_d0", "ev_d1", "ev_d2", "profile")
        ro = L.ReplayOut(*((out[k].ctypes.data if k in out else None) for k in names))
        self._check(self._lib.eqx_replay(self._ctx, C.byref(rq), C.byref(ro)))
        if np.any(out["status"] == 2):
            raise EngineError("KV memory bound violated in replay(s) " + str(np.nonzero(out["status"] == 2)[0][:8]))
        return out

    def sweep_alpha(self, alphas, traces: list, ema_alpha: float = 0.2) -> list:
        """run_sweep_alpha (experiments.cpp:331-373): every (alpha, trace) pair replayed on the
        GPU in one launch; per alpha the mean jain_ttft_p90 and throughput_tps over the traces
        and both normalised by their maximum over alphas (SweepPoint)."""
        alphas = list(alphas)
        pairs = [(a, t) for a in alphas for t in traces]
        row_off = np.concatenate([[0], np.cumsum([len(t["client"]) for _, t in pairs])]).astype(np.int64)
        cat = {k: np.concatenate([np.asarray(t[k]) for _, t in pairs]) for k in
               ("client", "arrival", "in_tokens", "true_out")}
        # every sweep point runs the Equinox policy (experiments.cpp:345-347), whatever this
        # scheduler was built with
        saved = self.policy
        if saved.kind != "equinox":
            import dataclasses
            self.policy = dataclasses.replace(saved, kind="equinox")
            self._set_policy()
        try:
            out = self.replay(row_off, cat["client"], cat["arrival"], cat["in_tokens"], cat["true_out"],
                              np.array([a for a, _ in pairs]), ema_alpha=ema_alpha, ev_cap=1,
                              duration_s=[t.get("duration_s", 0.0) or t["arrival"][-1] if len(t["arrival"]) else 0.0
                                          for _, t in pairs])
        finally:
            if self.policy is not saved:
                self.policy = saved
                self._set_policy()
        k = len(traces)
        points = []
        for i, a in enumerate(alphas):  # the reference's accumulation order (seeds in order)
            j = t = 0.0
            for s in range(k):
                j += out["jain_ttft_p90"][i * k + s]
                t += out["throughput_tps"][i * k + s]
            points.append({"alpha": a, "jain_ttft_p90": j / float(k), "throughput_tps": t / float(k)})
        mj = max([0.0] + [p["jain_ttft_p90"] for p in points])
        mt = max([0.0] + [p["throughput_tps"] for p in points])
        for p in points:
            p["jain_norm"] = p["jain_ttft_p90"] / mj if mj > 0.0 else 0.0
            p["throughput_norm"] = p["throughput_tps"] / mt if mt > 0.0 else 0.0
        return points

    # -- completion / feedback (engine.cpp:273-375) --
    def feedback(self, tokens=None, completions: dict | None = None, ema_alpha: float = 0.2) -> None:
        """One iteration's feedback in the engine's order: on_tokens(c, tokens[c]) for every
        client with tokens, then per completion (in order) on_complete + running-count
        decrement + update_map(profile, observed, ema_alpha).  ``completions`` holds columns
        client, input_tokens, output_tokens, latency_s, tps, gpu_util, pending_ufc, pending_rfc
        and (VTC with predictions) pending_vtc: the admission's PendingContribution, i.e. the
        StepResult fields ufc_inc / rfc_inc / vtc_inc of its event."""
        keep: list = []
        tok = None
        if tokens is not None:
            t = np.ascontiguousarray(tokens, np.int64)
            if t.shape != (len(self.client_ids),):
                raise ValueError("tokens must hold one count per client")
            keep.append(t)
            tok = t.ctypes.data_as(L._i64p)
        cp = None
        if completions is not None:
            cols = {}
            loc = set()
            n = len(completions["client"])
            for name, dt in (("client", np.int32), ("input_tokens", np.int32), ("output_tokens", np.int32),
                             ("latency_s", np.float64), ("tps", np.float64), ("gpu_util", np.float64),
                             ("pending_ufc", np.float64), ("pending_rfc", np.float64), ("pending_vtc", np.float64)):
                ptr, where = _as_col(completions.get(name), dt, keep)
                cols[name] = ptr
                if where is not None:
                    loc.add(where)
            if len(loc) > 1:
                raise ValueError("feedback: mix of host and device columns")
            cp = L.Completions(n, cols["client"], cols["input_tokens"], cols["output_tokens"], cols["latency_s"],
                               cols["tps"], cols["gpu_util"], cols["pending_ufc"], cols["pending_rfc"],
                               cols["pending_vtc"], loc.pop() if loc else L.EQX_HOST)
        self._check(self._lib.eqx_feedback(self._ctx, tok, C.byref(cp) if cp is not None else None,
                                           float(ema_alpha)))

    def service(self) -> tuple:
        """(ClientState::accumulated_service per client, SchedulerPolicy::counter_clamps())."""
        n = len(self.client_ids)
        out = np.zeros(n)
        cl = np.zeros(1, np.int64)
        self._check(self._lib.eqx_get_service(self._ctx, n, out.ctypes.data_as(L._dp), cl.ctypes.data_as(L._i64p)))
        return out, int(cl[0])

    def set_service(self, service) -> None:
        sv = np.ascontiguousarray(service, np.float64)
        self._check(self._lib.eqx_set_service(self._ctx, len(self.client_ids), sv.ctypes.data_as(L._dp)))

    def profile_metrics(self) -> dict:
        """The profile entries' latency_ms / gpu_util / tps as update_map left them."""
        n = self._n_profile
        out = {k: np.zeros(n) for k in ("lat", "util", "tps")}
        self._check(self._lib.eqx_get_profile(self._ctx, n, out["lat"].ctypes.data_as(L._dp),
                                              out["util"].ctypes.data_as(L._dp), out["tps"].ctypes.data_as(L._dp)))
        return out

    # -- client-sharded step (include/eqx.h; driven by sharded.ShardedScheduler) --
    def set_stream(self, stream_ptr: int) -> None:
        """Launch on the caller's CUDA stream (e.g. torch's current stream, where the NCCL
        all-gather of the sharded step is ordered)."""
        self._check(self._lib.eqx_ctx_set_stream(self._ctx, C.c_void_p(int(stream_ptr))))

    def shard_export_async(self, now: float, cmax: int, window: int, rec) -> None:
        """Score the local queue and write this rank's exchange record into ``rec`` (a CUDA
        uint8 tensor of at least eqx_shard_record_bytes(cmax, window) bytes)."""
        self._check(self._lib.eqx_shard_export_async(self._ctx, float(now), int(cmax), int(window),
                                                     C.c_void_p(rec.data_ptr())))

    def shard_select_async(self, recs, world: int, stride: int, client_off, cmax: int, window: int,
                           now: float) -> None:
        off = np.ascontiguousarray(client_off, np.int32)
        self._check(self._lib.eqx_shard_select_async(self._ctx, C.c_void_p(recs.data_ptr()), int(world),
                                                     int(stride), off.ctypes.data_as(L._i32p), int(cmax),
                                                     int(window), float(now)))

    def kernel_times_ms(self) -> dict:
        """CUDA-event durations of the last (non-graph) step's kernels."""
        out = (C.c_float * 3)()
        self._check(self._lib.eqx_kernel_times(self._ctx, out))
        return {"score_kernel": out[0], "select_kernel": out[1], "drain": out[2]}

    def scores(self) -> dict:
        """Per-request scores of the queue in drain order: pred, bucket, ufc_inc, rfc_inc."""
        n = self.n_queued
        out = {"pred": np.zeros(n, np.int32), "bucket": np.zeros(n, np.uint8),
               "ufc_inc": np.zeros(n), "rfc_inc": np.zeros(n)}
        self._check(self._lib.eqx_copy_scores(self._ctx, n, out["pred"].ctypes.data_as(L._i32p),
                                              out["bucket"].ctypes.data_as(L._u8p),
                                              out["ufc_inc"].ctypes.data_as(L._dp),
                                              out["rfc_inc"].ctypes.data_as(L._dp)))
        return out
