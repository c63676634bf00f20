"""Benchmark: requests scored + scheduled per second for one Equinox scheduling step.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg2|cfg3]

A "step" is one cold scheduling step over a resident queue: drain_arrivals of
the whole queue (client-grouped FIFO index + counter lift) followed by admit_requests with
whole-queue scoring (MoPE predict -> map_metrics -> ufc/rfc increments -> HF selection under
the slot/KV budget).  N=1 runs BASELINE configs[1] (1M LMSYS-shaped requests, 64 clients).
Under torchrun (N>1) the queue is client-sharded: each rank holds a
1M-request / 64-client shard of one global trace (weak scaling; --config cfg4: 2M / 1,250 per
rank = 16M / 10k clients at N=8), scores it locally, and the ranks all-gather their clients'
head-window records over NCCL before every rank runs the identical exact selection.

Timing: every timed step is bracketed by CUDA events on the context stream; the L2 (126 MB)
is flushed with a 256 MiB memset between steps, outside the events.  `e2e` repeats the step
through the public API with host (pinned) input buffers, the H2D copies and the D2H of the
step's events + ledger inside a wall-clock region.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ALGO_BYTES_K1 = 17 + 21       # per request: read client/arrival/in/tag, write pred/bucket/ufc/rfc
ALGO_BYTES_DRAIN = 4 + 4 + 4  # per request: histogram read, rank read, perm write


def load_inputs(cfg: str, rank: int):
    from paper_2508_16646_b200 import workload as W
    from paper_2508_16646_b200 import scheduler as S
    data = os.path.join(ROOT, "paper_2508_16646_b200", "data")
    model = S.MopeModel.load(os.path.join(data, "mope_builtin_c10000_s7_e3.json"))
    prof = S.GpuProfile.load_json(os.path.join(data, "profile_default.json"))
    if cfg == "cfg3":
        q = W.lmsys_queue(1_000_000, 1000, seed=3 + 100 * rank, heavy_frac=0.5)
        led = {k: np.zeros(1000) for k in ("ufc", "rfc", "counter")}
        perf = S.PerfParams(max_batch=4096)
        desc = "cfg3: 1M-request queue, 1000 clients (client0 = 50%), max_batch 4096 (KV budget cuts)"
    else:
        q = W.lmsys_queue(1_000_000, 64, seed=1 + 100 * rank)
        led = W.warm_ledger(64, seed=2 + 100 * rank)
        perf = S.PerfParams(max_batch=64)
        desc = "cfg2: LMSYS-shaped 1M-request queue, 64 clients, warm ledger, max_batch 64"
    return q, led, perf, model, prof, desc


def trace_hash(q) -> str:
    """trace_hash (workload.cpp:422-428) of the bench queue: FNV-1a of its canonical CSV
    (eqx_trace, host C++), recorded in `config` as the input's provenance."""
    from paper_2508_16646_b200.trace import Trace
    return Trace.from_columns(q["client"], q["arrival"], q["in_tokens"], q["true_out"], q["client_names"],
                              tag=q["tag"], tag_names=q["tag_names"]).hash()


def bench_config(desc: str, q, world: int = 1) -> dict:
    """`config` of the JSON line -- identical in both arms (--impl ours / reference)."""
    return {"workload": desc, "policy": "equinox (alpha 0.7, delta 0.1, max_over_clients)",
            "predictor": "mope(3) trained by the reference on its builtin corpus (seed 7)",
            "queue_per_gpu": int(len(q["client"])), "trace_hash": trace_hash(q),
            "inputs": "numpy PCG64 draws of the corpus mixture (paper_2508_16646_b200/workload.py)",
            "l2": "flushed between steps (256 MiB memset outside the events)",
            "parallelism": f"client-sharded x{world}" if world > 1 else "single GPU"}


def make_scheduler(q, led, perf, model, prof, device):
    from paper_2508_16646_b200 import scheduler as S
    clients = [S.ClientState(n, ufc=float(u), rfc=float(r), counter=float(c))
               for n, u, r, c in zip(q["client_names"], led["ufc"], led["rfc"], led["counter"])]
    return S.GpuScheduler(clients, policy=S.PolicySpec(), perf=perf, profile=prof, predictor="mope",
                          model=model, tag_names=q["tag_names"], device=device), clients


def tag_ids(q):
    return np.where(q["tag"] < 0, 0, q["tag"] + 1).astype(np.uint8)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def cpu_baseline(q, led, model, prof, reps: int, cores_note="1 (single-threaded reference engine)"):
    """The reference's own step (oracle/_ref, compiled from /root/reference sources) on the
    same queue: drain_arrivals + admit_requests through the reference objects."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import harness as H
    kind = "reference" if H.available("ref") else "port"
    case = H.StepCase(client=q["client"], arrival=q["arrival"], in_tokens=q["in_tokens"], true_out=q["true_out"],
                      tag=q["tag"], client_names=q["client_names"], model=model.to_json(),
                      profile={"upper": [e.bucket_upper for e in prof.entries],
                               "lat": [e.latency_ms for e in prof.entries],
                               "util": [e.gpu_util for e in prof.entries],
                               "tps": [e.tps for e in prof.entries]},
                      ufc0=led["ufc"], rfc0=led["rfc"], counter0=led["counter"])
    times = []
    out = None
    for _ in range(reps):
        t0 = time.perf_counter()
        out = H.run_step(case, "ref" if kind == "reference" else "oracle")
        wall = time.perf_counter() - t0
        # the reference build times drain + admission inside the driver; the C port by wall clock
        times.append((out["ns_drain"] + out["ns_admit"]) * 1e-9 if kind == "reference" else wall)
    return times, kind, out


def run_reference(args, rank, world):
    if rank != 0:
        return
    q, led, perf, model, prof, desc = load_inputs(args.config, 0)
    n = len(q["client"])
    times, kind, _ = cpu_baseline(q, led, model, prof, args.warmup + args.steps)
    t = np.array(times[args.warmup:])
    val = n / float(np.mean(t))
    line = {
        "impl": "reference", "metric": "requests scored+scheduled/sec", "value": val, "unit": "requests/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(np.mean(t) * 1e3),
        "p50_ms": float(np.median(t) * 1e3), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": bench_config(desc, q),
        "cpu_baseline": {"value": val, "unit": "requests/s", "cores": 1, "kind": kind,
                         "sample": f"full {n}-request step x {args.steps} (drain_arrivals + admit_requests "
                                   "via the reference objects, oracle/_ref)"},
        "e2e": {"value": val, "unit": "requests/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def shard_inputs(cfg: str, rank: int, world: int):
    """Rank `rank`'s shard of a client-sharded global trace: per GPU the cfg's
    queue shape (cfg2: 1M requests / 64 clients; cfg4: 2M / 1,250 = 16M / 10k over 8 GPUs).
    Global client g = rank * C_r + local, named client%06d so rank blocks are client_id-byte
    blocks; the rank's i-th request has trace position i * world + rank and arrival
    position / (n_r * world) s, so the union over ranks is one arrival-ordered trace."""
    from paper_2508_16646_b200 import workload as W
    from paper_2508_16646_b200 import scheduler as S
    data = os.path.join(ROOT, "paper_2508_16646_b200", "data")
    model = S.MopeModel.load(os.path.join(data, "mope_builtin_c10000_s7_e3.json"))
    prof = S.GpuProfile.load_json(os.path.join(data, "profile_default.json"))
    n_r, c_r = (2_000_000, 1250) if cfg == "cfg4" else (1_000_000, 64)
    q = W.lmsys_queue(n_r, c_r, seed=1 + 100 * rank)
    pos = np.arange(n_r, dtype=np.int64) * world + rank
    q["id"] = pos
    q["arrival"] = pos.astype(np.float64) / float(n_r * world)
    led = W.warm_ledger(c_r * world, seed=2)
    names = [f"client{g:06d}" for g in range(c_r * world)]
    desc = (f"{cfg} per GPU: {n_r} queued requests / {c_r} clients per rank, client-sharded over {world} "
            f"GPU(s) ({n_r * world} requests, {c_r * world} clients), warm ledger, max_batch 64")
    return q, led, names, c_r, S.PerfParams(max_batch=64), model, prof, desc


def run_sharded(args, rank, world):
    """N GPUs: one process per GPU, client-sharded queue, exact replicated selection after one
    NCCL all-gather of the ranks' head-window records per step."""
    import torch
    from paper_2508_16646_b200 import scheduler as S
    from paper_2508_16646_b200.sharded import ShardedScheduler
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # EQX_BENCH_SAME_DEVICE=1 + EQX_BENCH_BACKEND=gloo: every rank on cuda:0 with a CPU-staged
    # exchange, to exercise the multi-rank path on a one-GPU box (never for reported numbers)
    if os.environ.get("EQX_BENCH_SAME_DEVICE") == "1":
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("EQX_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    cfg = "cfg4" if args.config == "cfg4" else "cfg2"
    q, led, names, c_r, perf, model, prof, desc = shard_inputs(cfg, rank, world)
    n = len(q["client"])
    clients = [S.ClientState(nm, ufc=float(u), rfc=float(r), counter=float(c))
               for nm, u, r, c in zip(names, led["ufc"], led["rfc"], led["counter"])]
    owner = np.repeat(np.arange(world, dtype=np.int32), c_r)
    sch = ShardedScheduler(clients, rank, world, owner=owner, device=local, policy=S.PolicySpec(), perf=perf,
                           profile=prof, predictor="mope", model=model, tag_names=q["tag_names"])
    stream = sch.stream
    with torch.cuda.stream(stream):
        cols = dict(client=torch.from_numpy(q["client"]).to(dev), arrival_s=torch.from_numpy(q["arrival"]).to(dev),
                    input_tokens=torch.from_numpy(q["in_tokens"]).to(dev), tag=torch.from_numpy(tag_ids(q)).to(dev),
                    ids=torch.from_numpy(q["id"]).to(dev))
        flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()
    sch.set_batch(0, 0)
    sch.sel.checkpoint()
    # head-window depth: ShardedScheduler's adaptive default (8, grown 4x after an underflow and
    # kept), settled by one public step before the timed loop
    sch.drain(local=True, **cols)
    sch.step(1.0, with_events=False)
    window = sch.default_window()
    sch.sel.restore_async()

    def enqueue_step():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            sch.sel.restore_async()
            flush.zero_()
            e0.record(stream)
            sch.drain(local=True, **cols)
            sch.step_async(1.0, window)
            e1.record(stream)
        return e0, e1

    for _ in range(args.warmup):
        enqueue_step()
    res = sch.sel.collect(with_events=False)
    if res.window_underflow:
        raise RuntimeError("head windows underflowed on the bench workload")
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        recs = [enqueue_step() for _ in range(args.steps)]
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    res = sch.sel.collect(with_events=False)
    step_ms = np.array([a.elapsed_time(b) for a, b in recs])
    total_ms = float(step_ms.sum())
    p50 = float(np.median(step_ms))
    if dist:
        t = torch.tensor([total_ms, p50], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, p50 = float(t[0].item()), float(t[1].item())
    value = world * n * args.steps / (total_ms * 1e-3)

    # e2e: the public sharded API with this rank's pinned host columns (H2D inside), events D2H
    # narrow host columns as in the single-GPU e2e: local client indices and input tokens as
    # uint16 when they fit, arrivals packed (eqx_pack_arrivals), all lossless
    narrow = int(q["client"].max(initial=0)) < 65536 and int(q["in_tokens"].max(initial=0)) < 65536 and \
        int(q["in_tokens"].min(initial=0)) >= 0 and int(q["client"].min(initial=0)) >= 0
    cdt = np.uint16 if narrow else np.int32
    host = {k: S.pinned_copy(v) for k, v in
            dict(client=q["client"].astype(cdt), arrival_s=S.pack_arrivals(q["arrival"]),
                 input_tokens=q["in_tokens"].astype(cdt), tag=tag_ids(q), ids=q["id"]).items()}
    e2e_t, d2h = [], 0
    for i in range(args.warmup + max(3, args.steps // 4)):
        sch.sel.restore_async()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        sch.drain(local=True, **host)
        r = sch.step(1.0, window=window)
        t1 = time.perf_counter()
        if i >= args.warmup:
            e2e_t.append(t1 - t0)
        d2h = r.ids.nbytes + r.kinds.nbytes + r.clients.nbytes + r.preds.nbytes + 4 * r.ufc_inc.nbytes + 80
    e2e_med = float(np.median(e2e_t))
    if dist:
        t = torch.tensor([e2e_med], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_med = float(t.item())
    h2d = sum((v.data if isinstance(v, S.PackedArrivals) else v).nbytes for v in host.values())
    if rank == 0:
        from paper_2508_16646_b200.sharded import record_bytes
        rec = record_bytes(c_r, window)
        line = {
            "metric": "requests scored+scheduled/sec", "value": value, "unit": "requests/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "p50_ms": p50,
            "p99_ms": float(np.percentile(step_ms, 99)), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": desc, "policy": "equinox (alpha 0.7, delta 0.1, max_over_clients)",
                       "predictor": "mope(3) trained by the reference on its builtin corpus (seed 7)",
                       "queue_per_gpu": n, "l2": "flushed between steps (256 MiB memset outside the events)",
                       "parallelism": f"client-sharded x{world}: local drain+score+window export, NCCL all-gather "
                                      f"of {rec} B/rank, replicated exact selection"},
            "admitted": res.n_admitted,
            "exchange_bytes_per_rank": rec,
            "e2e": {"value": world * n / e2e_med, "unit": "requests/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "p50_ms": e2e_med * 1e3},
            # drain (3), score, shard_export, shard_ingest, shard_unpack, select (publishes the summary)
            "gpu_launches": 8 * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def run_cfg4_sim(args):
    """configs[3] at its global shape on ONE GPU: 16M queued requests over 10,000 clients as
    `--simulate-world` ranks (2M / 1,250 each, the layout an 8-GPU box runs).  Every rank's
    drain + scoring + exchange-record export runs on its own context, writing its slice of one
    gathered buffer (what the NCCL all-gather delivers); the selection context then runs the
    replicated exact selection over all 10k clients' heads.  Reported: the per-rank part (the
    max over the simulated ranks of drain + export, device time -- on the box the ranks run in
    parallel), the selection at 10k clients, and their sum as the simulated step (the
    all-gather itself is not on one GPU: exchange bytes per rank are reported beside it)."""
    import torch
    from paper_2508_16646_b200 import scheduler as S
    from paper_2508_16646_b200.sharded import record_bytes, _a16
    world = args.simulate_world
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    ranks = []
    for r in range(world):
        q, led, names, c_r, perf, model, prof, desc = shard_inputs("cfg4", r, world)
        ranks.append((q, names))
    clients = [S.ClientState(nm, ufc=float(u), rfc=float(v), counter=float(c))
               for nm, u, v, c in zip(names, led["ufc"], led["rfc"], led["counter"])]
    kw = dict(policy=S.PolicySpec(), perf=perf, profile=prof, predictor="mope", model=model, tag_names=q["tag_names"])
    sel = S.GpuScheduler(clients, device=0, **kw)
    stream = torch.cuda.Stream(dev)
    sel.set_stream(stream.cuda_stream)
    locs, cols = [], []
    for r, (q, _) in enumerate(ranks):
        loc = S.GpuScheduler(clients[r * c_r:(r + 1) * c_r], device=0, **kw)
        loc.set_stream(stream.cuda_stream)
        with torch.cuda.stream(stream):
            cols.append(dict(client=torch.from_numpy(q["client"]).to(dev),
                             arrival_s=torch.from_numpy(q["arrival"]).to(dev),
                             input_tokens=torch.from_numpy(q["in_tokens"]).to(dev),
                             tag=torch.from_numpy(tag_ids(q)).to(dev), ids=torch.from_numpy(q["id"]).to(dev)))
        locs.append(loc)
    off = np.arange(world + 1, dtype=np.int32) * c_r
    with torch.cuda.stream(stream):
        flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()
    sel.set_batch(0, 0)
    sel.checkpoint()
    W = 8  # ShardedScheduler's default head-window depth (grown 4x on an underflow)

    def step(W):
        stride = _a16(record_bytes(c_r, W))
        with torch.cuda.stream(stream):
            recv = torch.empty(world * stride, dtype=torch.uint8, device=dev)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * world + 2)]
        with torch.cuda.stream(stream):
            sel.restore_async()
            flush.zero_()
            for r, loc in enumerate(locs):
                ev[2 * r].record(stream)
                loc.drain(**cols[r])
                loc.shard_export_async(1.0, c_r, W, recv[r * stride:(r + 1) * stride])
                ev[2 * r + 1].record(stream)
            ev[2 * world].record(stream)
            sel.shard_select_async(recv, world, stride, off, c_r, W, 1.0)
            ev[2 * world + 1].record(stream)
        return ev, recv

    while True:
        step(W)
        res = sel.collect(with_events=False)
        if not res.window_underflow:
            break
        W *= 4
    for _ in range(args.warmup):
        step(W)
    torch.cuda.synchronize()
    recs = [step(W) for _ in range(args.steps)]
    torch.cuda.synchronize()
    res = sel.collect(with_events=False)
    assert not res.window_underflow
    if os.environ.get("EQX_TOPK_PROF"):  # instrumented library: the selection's round counters
        import ctypes as C
        from paper_2508_16646_b200 import _lib as L
        out = (C.c_double * 35)()
        L.load().eqx_phase_times(sel._ctx, out, 35)
        print("phase us (windows filled, loop start, loop end)", [round(x, 1) for x in out[1:4]], "rounds", out[7], "cycles heads/gather/chain/keys/select/rank/scan/seq", [int(x) for x in out[8:16]],
              "head loads, head radix, head passes, item passes, item selects, items", [int(x) for x in out[27:33]],
              flush=True)
    rank_ms = np.array([[e[2 * r].elapsed_time(e[2 * r + 1]) for r in range(world)] for e, _ in recs])
    sel_ms = np.array([e[2 * world].elapsed_time(e[2 * world + 1]) for e, _ in recs])
    per_rank = rank_ms.max(axis=1)
    step_ms = per_rank + sel_ms
    n = sum(len(q["client"]) for q, _ in ranks)
    rec = record_bytes(c_r, W)
    line = {
        "metric": "requests scored+scheduled/sec", "value": n / (float(np.median(step_ms)) * 1e-3), "unit": "requests/s",
        "n_gpus": 1, "simulated_world": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": float(np.mean(step_ms)), "p50_ms": float(np.median(step_ms)),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"cfg4 global shape simulated on one GPU: {n} queued requests, {c_r * world} clients, "
                               f"{world} ranks x ({n // world} requests / {c_r} clients), warm ledger, max_batch 64",
                   "policy": "equinox (alpha 0.7, delta 0.1, max_over_clients)",
                   "l2": "flushed between steps (256 MiB memset outside the events)"},
        "breakdown_ms": {"rank_drain_export_max_p50": float(np.median(per_rank)),
                         "rank_drain_export_mean_p50": float(np.median(rank_ms.mean(axis=1))),
                         "select_10k_p50": float(np.median(sel_ms))},
        "admitted": res.n_admitted, "window": W, "exchange_bytes_per_rank": rec,
        "allgather_bytes_total": rec * world,
        "note": "step = max over simulated ranks of (drain + score + export) + replicated selection; the NCCL "
                "all-gather of exchange_bytes_per_rank per rank is not part of a one-GPU simulation",
    }
    print(json.dumps(line), flush=True)


def preset_traces(n_replays: int, duration: float, seed0: int = 1):
    """The reference's poisson preset (workload.cpp:254-260: client1 Poisson 16/s, 512 in / 32
    out; client2 Poisson 3/s, 32 in / 512 out), one seeded trace per replay, concatenated."""
    traces = []
    for i in range(n_replays):
        rng = np.random.default_rng(seed0 + i)
        parts = []
        for c, (rate, tin, tout) in enumerate(((16.0, 512, 32), (3.0, 32, 512))):
            t = np.cumsum(rng.exponential(1.0 / rate, int(rate * duration * 2) + 16))
            t = t[t < duration]
            parts.append((t, np.full(len(t), c, np.int32), np.full(len(t), tin, np.int32),
                          np.full(len(t), tout, np.int32)))
        arr = np.concatenate([p[0] for p in parts])
        o = np.argsort(arr, kind="stable")
        traces.append({"arrival": arr[o], "client": np.concatenate([p[1] for p in parts])[o],
                       "in_tokens": np.concatenate([p[2] for p in parts])[o],
                       "true_out": np.concatenate([p[3] for p in parts])[o]})
    row_off = np.concatenate([[0], np.cumsum([len(t["client"]) for t in traces])]).astype(np.int64)
    cat = {k: np.concatenate([t[k] for t in traces]) for k in ("client", "arrival", "in_tokens", "true_out")}
    return traces, row_off, cat


CFG5_DURATION = 60.0  # Trace::duration_s of the generated scenarios: the replay horizon (engine.cpp:120-121)


def cfg5_setup(n_seeds: int):
    alphas = np.round(np.arange(0.5, 0.86, 0.05), 2)              # 8 values
    alpha = np.tile(alphas, n_seeds)                             # replay r: alpha[r % 8], seed r // 8
    traces, row_off, cat = preset_traces(len(alpha), CFG5_DURATION)
    return alpha, traces, row_off, cat


def ref_replay_one(args_):
    """One reference run_simulation (oracle/_ref) of a preset trace (the reference arm)."""
    q, a = args_
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import harness as H
    with open(os.path.join(ROOT, "paper_2508_16646_b200", "data", "profile_default.json")) as f:
        prof = {k: np.asarray(v) for k, v in json.load(f).items()}
    case = H.StepCase(client=q["client"], arrival=q["arrival"], in_tokens=q["in_tokens"], true_out=q["true_out"],
                      tag=np.full(len(q["client"]), -1, np.int32), client_names=["client1", "client2"],
                      alpha=float(a), pred_kind=0, profile=prof, duration_s=CFG5_DURATION)
    t0 = time.perf_counter()
    H.ref_replay(case, max_sim_time_s=0.0, ema_alpha=0.2, cap=1 << 20)
    return time.perf_counter() - t0


def run_cfg5(args, rank, world):
    """configs[4]: the Holistic-Fairness alpha sweep as 1024 independent engine replays (8 alpha
    values x 128 seeds of the poisson preset, 60 s each) in one eqx_replay launch per step; under
    torchrun the replays are partitioned round-robin over the ranks (replicas, no collective on
    the data path)."""
    if args.impl == "reference" and rank != 0:
        return
    alpha, traces, row_off, cat = cfg5_setup(128)
    n_total = len(alpha)
    if args.impl != "reference" and world > 1:  # this rank's share: replays rank, rank + world, ...
        mine = np.arange(rank, n_total, world)
        alpha = alpha[mine]
        traces = [traces[i] for i in mine]
        row_off = np.concatenate([[0], np.cumsum([len(t["client"]) for t in traces])]).astype(np.int64)
        cat = {k: np.concatenate([t[k] for t in traces]) for k in ("client", "arrival", "in_tokens", "true_out")}
    n = len(alpha)
    if args.impl == "reference":
        import multiprocessing as mp
        cores = os.cpu_count() or 1
        sample = min(n, 4 * cores)
        with mp.Pool(cores) as pool:
            pool.map(ref_replay_one, [(traces[i], alpha[i]) for i in range(cores)])  # warm
            t0 = time.perf_counter()
            pool.map(ref_replay_one, [(traces[i], alpha[i]) for i in range(sample)])
            dt = time.perf_counter() - t0
        val = sample / dt
        print(json.dumps({"impl": "reference", "metric": "engine replays/sec (alpha sweep)", "value": val,
                          "unit": "replays/s", "n_gpus": world, "higher_is_better": True,
                          "config": {"workload": "cfg5: 1024 replays = 8 alpha x 128 seeds, poisson preset, 60 s"},
                          "cpu_baseline": {"value": val, "unit": "replays/s", "cores": cores, "kind": "reference",
                                           "sample": f"{sample} replays (run_simulation, oracle/_ref) on a {cores}-process pool"},
                          "e2e": {"value": val, "unit": "replays/s", "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}), flush=True)
        return
    import torch
    from paper_2508_16646_b200 import scheduler as S
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    data = os.path.join(ROOT, "paper_2508_16646_b200", "data")
    prof = S.GpuProfile.load_json(os.path.join(data, "profile_default.json"))
    sch = S.GpuScheduler([S.ClientState("client1"), S.ClientState("client2")], policy=S.PolicySpec(),
                         perf=S.PerfParams(), profile=prof, predictor="oracle", device=local)
    cap = 1  # run_sweep_alpha reads the reports only: no event log comes back
    # the trace columns live in the library's pinned arena, as the other e2e legs' host batches do
    cat = {k: S.pinned_copy(v) for k, v in cat.items()}
    times, kms = [], []
    for i in range(args.warmup + args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = sch.replay(row_off, cat["client"], cat["arrival"], cat["in_tokens"], cat["true_out"], alpha,
                         ema_alpha=0.2, ev_cap=cap, duration_s=np.full(n, CFG5_DURATION))
        t1 = time.perf_counter()
        if i >= args.warmup:
            times.append(t1 - t0)
            kms.append(sch.kernel_times_ms()["select_kernel"])
    k = float(np.median(kms))
    e2e_s = float(np.median(times))
    if dist:  # slowest rank
        t = torch.tensor([k, e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        k, e2e_s = float(t[0].item()), float(t[1].item())
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    h2d = int(sum(v.nbytes for v in cat.values()) + row_off.nbytes + alpha.nbytes)
    n = n_total
    line = {"metric": "engine replays/sec (alpha sweep)", "value": n / (k * 1e-3), "unit": "replays/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": k, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "cfg5: 1024 replays = 8 alpha x 128 seeds of the poisson preset (60 s), "
                                   "one replay per GPU warp, build_report + window samples on the device", "requests": int(row_off[-1]),
                       "completed": int(out["completed"].sum()), "admissions": int(out["n_events"].sum())},
            "e2e": {"value": n / e2e_s, "unit": "replays/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": int(sum(v.nbytes for v in out.values())),
                    "ms_per_step": e2e_s * 1e3},
            "gpu_launches": args.steps}
    if world == 1:  # the sweep points run_sweep_alpha reports (per alpha, mean over seeds)
        pts = []
        for a in np.unique(alpha):
            sel = np.nonzero(alpha == a)[0]
            pts.append({"alpha": float(a), "jain_ttft_p90": float(np.mean(out["jain_ttft_p90"][sel])),
                        "throughput_tps": float(np.mean(out["throughput_tps"][sel]))})
        line["sweep"] = pts
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def e2e_live(args, q, led, perf, model, prof, device, steps: int = 40):
    """A serving loop over a live queue: the 1M-request queue stays resident and every step
    appends only that step's new arrivals (eqx_append: drain_arrivals into the non-empty queues,
    prediction records frozen at arrival, engine.cpp:171-197) from pinned host memory, then
    scores + schedules the whole queue (admit_requests at the step's `now`) and reads the
    step's events back.  The batch is reset to empty every step and the arrivals replace the
    admissions, so every step schedules over ~1M queued requests like the cold step.  Wall clock
    over consecutive steps, H2D of the arrivals and D2H of the events inside."""
    from paper_2508_16646_b200 import scheduler as S
    from paper_2508_16646_b200 import workload as W
    n = len(q["client"])
    C = len(q["client_names"])
    sch, _ = make_scheduler(q, led, perf, model, prof, device)
    sch.append(client=q["client"], arrival_s=q["arrival"], input_tokens=q["in_tokens"], tag=tag_ids(q))
    sch.set_batch(0, 0)
    sch.step(1.0, with_events=False)
    per = perf.max_batch  # arrivals per step = what a step admits
    total = per * (steps + args.warmup + 8)
    extra = W.lmsys_queue(total, C, seed=77)
    now0 = 1.0
    dt = 1e-3
    arr = now0 + dt * (1.0 + np.arange(total) // per) - dt * 0.5 / per * (per - np.arange(total) % per)
    batches = []
    for i in range(total // per):
        sl = slice(i * per, (i + 1) * per)
        batches.append({k: S.pinned_copy(v) for k, v in dict(client=extra["client"][sl], arrival_s=arr[sl],
                                                            input_tokens=extra["in_tokens"][sl],
                                                            tag=tag_ids(extra)[sl]).items()})
    times, adm = [], []
    for i, b in enumerate(batches[:steps + args.warmup]):
        t0 = time.perf_counter()
        sch.append(**b)
        sch.set_batch(0, 0)
        r = sch.step(now0 + dt * (i + 1))
        t1 = time.perf_counter()
        if i >= args.warmup:
            times.append(t1 - t0)
            adm.append(r.n_admitted)
    step_s = float(np.median(times))
    h2d = sum(v.nbytes for v in batches[0].values())
    queued = n  # arrivals replace the admissions: the queue stays at ~n
    sch.close()
    return {"value": queued / step_s, "unit": "requests/s", "ms_per_step": step_s * 1e3, "steps": len(times),
            "queue": queued, "arrivals_per_step": per, "h2d_bytes_per_step": int(h2d),
            "admitted_per_step": int(np.median(adm)),
            "note": "live queue: each step appends its new arrivals (eqx_append, pinned host columns) and "
                    "scores + schedules the whole resident queue; wall clock per step incl. the H2D of the "
                    "arrivals and the D2H of the step's events"}


def run_ours(args, rank, world):
    if args.config == "cfg5":
        return run_cfg5(args, rank, world)
    if args.config == "cfg4" and args.simulate_world > 1 and world == 1:
        return run_cfg4_sim(args)
    if world > 1 or args.sharded or args.config == "cfg4":
        return run_sharded(args, rank, world)
    import torch
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    q, led, perf, model, prof, desc = load_inputs(args.config, rank)
    n = len(q["client"])
    sch, clients = make_scheduler(q, led, perf, model, prof, local)
    dev = torch.device("cuda", local)
    cols = dict(client=torch.from_numpy(q["client"]).to(dev), arrival_s=torch.from_numpy(q["arrival"]).to(dev),
                input_tokens=torch.from_numpy(q["in_tokens"]).to(dev), tag=torch.from_numpy(tag_ids(q)).to(dev))
    stream = torch.cuda.ExternalStream(sch.stream_ptr, device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)

    sch.set_batch(0, 0)
    sch.checkpoint()  # device-side snapshot: every timed step restarts from the same cold state

    def enqueue_step(graph: bool):
        """All launches are asynchronous: the 256 MiB flush before each step lets the host run
        ahead, so the events time GPU work only."""
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        with torch.cuda.stream(stream):
            sch.restore_async()
            flush.zero_()
            e0.record(stream)
            if graph:
                sch.drain_step_async(1.0, **cols)
                e1.record(stream)
            else:
                sch.drain(**cols)
                e1.record(stream)
                sch.step_async(1.0)
            e2.record(stream)
        return e0, e1, e2

    def run_loop(graph: bool, steps: int, per_step_times: bool = False):
        for _ in range(args.warmup):
            enqueue_step(graph)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        recs, kts = [], []
        for _ in range(steps):
            recs.append(enqueue_step(graph))
            if per_step_times:  # host sync per step; the next step's 256 MiB flush keeps the GPU fed
                kts.append(sch.kernel_times_ms())
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        return recs, kts

    # split launches: per-phase breakdown + the HBM-bound scoring kernel's own duration
    split, kts = run_loop(False, args.steps, per_step_times=True)
    res = sch.collect(with_events=False)
    drain_ms = np.array([a.elapsed_time(b) for a, b, c in split])
    kern_ms = np.array([b.elapsed_time(c) for a, b, c in split])
    score_ms = np.array([k["score_kernel"] for k in kts])
    select_ms = np.array([k["select_kernel"] for k in kts])
    # headline: the public one-call path, replayed as a CUDA graph
    with ClockSampler(local) as clk:
        recs, _ = run_loop(True, args.steps)
    res_g = sch.collect(with_events=False)
    assert res_g.n_admitted == res.n_admitted
    step_ms = np.array([a.elapsed_time(c) for a, b, c in recs])
    total_ms = float(step_ms.sum())
    if dist:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    value = world * n * args.steps / (total_ms * 1e-3)

    # ---- the practical floor of a kernel moving the same bytes: a device copy of 19 MB (19 MB read
    # + 19 MB written = 38 B/request x 1M) after the same L2 flush, CUDA events around it ----
    cbytes = n * ALGO_BYTES_K1 // 2
    csrc = torch.empty(cbytes, dtype=torch.uint8, device=dev).random_(0, 255)
    cdst = torch.empty_like(csrc)
    copy_us = []
    for i in range(0 if args.profile else max(5, args.steps) + 3):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        cdst.copy_(csrc)
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            copy_us.append(e0.elapsed_time(e1) * 1e3)
    copy_floor_us = float(np.median(copy_us)) if copy_us else float("nan")
    del csrc, cdst

    # ---- e2e through the public API with pinned host buffers ----
    # Every step copies its batch H2D from pinned memory and reads its events + ledger back.
    # The batches of steps i+1 and i+2 are staged (eqx_stage_async, copy stream, three staging
    # buffers) while step i computes and is collected, so the steady-state step costs
    # max(H2D, compute) -- what a serving loop pays.  Three rotating pinned host batches (same
    # content, in the library's huge-page arena) keep the copies distinct.
    from paper_2508_16646_b200 import scheduler as S
    # client and input_tokens travel as uint16 when they fit (eqx_requests::narrow, checked here:
    # 64 / 1000 clients, inputs <= 1024 tokens): 13 B per request over PCIe instead of 17
    narrow = len(q["client_names"]) <= 65536 and int(q["in_tokens"].max()) < 65536 and int(q["in_tokens"].min()) >= 0
    cdt = np.uint16 if narrow else np.int32
    # arrivals travel packed (eqx_pack_arrivals: 6-byte offsets per 256-row block, raw blocks
    # near zero; lossless) -- prepared once per host batch, like the uint16 columns
    arr_host = S.pack_arrivals(q["arrival"])
    hosts = [{k: S.pinned_copy(v) for k, v in
              dict(client=q["client"].astype(cdt), arrival_s=arr_host, input_tokens=q["in_tokens"].astype(cdt),
                   tag=tag_ids(q)).items()} for _ in range(3)]
    e2e_steps = 0 if args.profile else max(8, args.steps)
    d2h = 0

    def e2e_loop(steps):
        nonlocal d2h
        adm = []
        for i in range(min(2, steps)):
            sch.stage_async(**hosts[i])
        for i in range(steps):
            if i + 2 < steps:
                sch.stage_async(**hosts[(i + 2) % 3])  # two batches ahead: the copy engine never idles
            sch.restore_async()
            sch.drain_step_async(1.0, **hosts[i % 3])  # staged batch -> one graph launch
            r = sch.collect(with_events=True)
            led_out = sch.step_ledger()  # written over PCIe by the step's selection CTA
            adm.append(r.n_admitted)
            d2h = r.ids.nbytes + r.kinds.nbytes + r.clients.nbytes + r.preds.nbytes + 4 * r.ufc_inc.nbytes + \
                sum(v.nbytes for v in led_out.values()) + 80
        return adm

    e2e_val, e2e_step_ms, single_ms = None, None, None
    if e2e_steps:
        e2e_loop(max(10, args.warmup))  # first touches of the pinned batches and staging graphs
        passes = []
        for _ in range(3):  # median of three timed passes
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            adm = e2e_loop(e2e_steps)
            t1 = time.perf_counter()
            assert all(a == res.n_admitted for a in adm)
            passes.append((t1 - t0) * 1e3 / e2e_steps)
        e2e_step_ms = float(np.median(passes))
        e2e_val = world * n / (e2e_step_ms * 1e-3)
        single = []
        for _ in range(5):  # unpipelined latency of one step through the same API
            sch.restore_async()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            sch.drain_step_async(1.0, **hosts[0])
            sch.collect(with_events=True)
            sch.ledger()
            single.append(time.perf_counter() - t0)
        single_ms = float(np.median(single) * 1e3)
    live = None if args.profile else e2e_live(args, q, led, perf, model, prof, local)
    h2d = sum((v.data if isinstance(v, S.PackedArrivals) else v).nbytes for v in hosts[0].values())

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peak, peak_src = 6449.4, "MEASURED_PEAKS.json hbm_gbs (measured)"
    if os.path.exists(peaks_path):
        with open(peaks_path) as f:
            peak = float(json.load(f).get("hbm_gbs", peak))
    else:
        peak_src = "fallback 6650 GB/s (B200_PROFILING.md)"
        peak = 6650.0
    k_ms = float(np.mean(score_ms))
    achieved = n * ALGO_BYTES_K1 / (k_ms * 1e-3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "step_kernel_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    line = {
        "metric": "requests scored+scheduled/sec", "value": value, "unit": "requests/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "p50_ms": float(np.median(step_ms)), "p99_ms": float(np.percentile(step_ms, 99)),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(desc, q, world),
        "breakdown_ms": {"drain_p50": float(np.median(drain_ms)), "step_p50": float(np.median(kern_ms)),
                         "score_kernel_p50": float(np.median(score_ms)),
                         "select_kernel_p50": float(np.median(select_ms)),
                         "split_launch_step_p50": float(np.median(drain_ms + kern_ms)),
                         "graph_step_p50": float(np.median(step_ms))},
        "admitted": res.n_admitted,
        "roofline": {"bound": "hbm", "kernel": "score_kernel (whole-queue predict/map/increments, HBM stream)",
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "algo_bytes_per_request": ALGO_BYTES_K1, "peak_source": peak_src,
                     "kernel_us_mean": k_ms * 1e3,
                     "copy_floor": {"what": f"torch device copy of {2 * cbytes / 1e6:.0f} MB (read + write) after "
                                            "the same L2 flush, CUDA events, median",
                                    "us": copy_floor_us, "gbs": 2 * cbytes / (copy_floor_us * 1e-6) / 1e9,
                                    "kernel_over_copy": k_ms * 1e3 / copy_floor_us}},
        "e2e": {"value": e2e_val, "unit": "requests/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_step_ms, "steps": e2e_steps,
                "passes": 3,
                "single_step_latency_ms": single_ms,
                "h2d_gbs": (h2d / (e2e_step_ms * 1e-3) / 1e9) if e2e_step_ms else None,
                "bound": f"pcie h2d ({h2d / n:.2f} B/request: packed arrivals"
                         f"{', uint16 client + input_tokens columns' if narrow else ''}; "
                         "~54.5 GB/s measured pinned H2D on the box, tools/pin_probe.py)",
                "note": "wall clock over consecutive steps; the H2D of steps i+1, i+2 (copy stream) "
                        "overlaps step i"},
        "e2e_live": live,
        # per step: drain (sort / hist, scan, scatter / rank), window, score, select, and the
        # selection's code warm-up on its scratch problem (the selection publishes the summary:
        # no state-copy kernel)
        "gpu_launches": 7 * args.steps,
        "clocks": clk.summary(),
    }
    if not (args.no_cpu_baseline or args.profile):
        times, kind, _ = cpu_baseline(q, led, model, prof, args.cpu_reps)
        if times:
            t = np.array(times[1:] if len(times) > 1 else times)
            what = ("the reference objects (oracle/_ref)" if kind == "reference"
                    else "the C restatement of the reference (oracle/eqx_oracle.c)")
            line["cpu_baseline"] = {"value": n / float(np.mean(t)), "unit": "requests/s", "cores": 1, "kind": kind,
                                    "sample": f"the same {n}-request cold step x {len(t)} through {what}, "
                                              "1 host thread"}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=["cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--sharded", action="store_true", help="client-sharded pipeline even at N=1")
    ap.add_argument("--simulate-world", type=int, default=0,
                    help="cfg4 on one GPU: simulate this many ranks of the global 16M / 10k-client step")
    ap.add_argument("--cpu-reps", type=int, default=6)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile", action="store_true", help="short run for ncu: no e2e / cpu legs")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference" and args.config == "cfg5":
        run_cfg5(args, rank, world)
    elif args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world)


if __name__ == "__main__":
    main()
