"""Batched engine replays (BASELINE configs[0] and configs[4]).

eqx_replay runs run_simulation (engine.cpp:119-146) for many traces in one launch, one replay
per GPU thread.  Oracle: the reference's own run_simulation through oracle/_ref (ref_replay),
replay by replay.  Bit-exact: the admitted / rejected event sequence with its simulated times
and the final FP64 ledgers.
"""
import numpy as np
import pytest

import harness as H
from helpers import case_clients, case_kwargs, default_model, default_profile
from paper_2508_16646_b200 import workload as W

pytestmark = pytest.mark.gpu
needs_ref = pytest.mark.skipif(not H.available("ref"), reason="reference build not present")


def poisson_trace(seed, n_clients=8, rate=400.0, duration=6.0):
    """cfg1-shaped: Poisson arrivals over n_clients, corpus-mixture lengths (workload.lmsys_queue)."""
    rng = np.random.default_rng(seed)
    n = int(rng.poisson(rate * duration))
    q = W.lmsys_queue(n, n_clients, seed=seed, tag_noise=0.2)
    q["arrival"] = np.sort(rng.uniform(0.0, duration, n))
    return q


def preset_trace(seed, duration=20.0):
    """The reference's poisson preset shape (workload.cpp:254-260): client1 16 req/s 512 in /
    32 out, client2 3 req/s 32 in / 512 out (configs/sweep_alpha.json)."""
    rng = np.random.default_rng(seed)
    parts = []
    for c, (rate, tin, tout) in enumerate(((16.0, 512, 32), (3.0, 32, 512))):
        t = np.cumsum(rng.exponential(1.0 / rate, int(rate * duration * 2)))
        t = t[t < duration]
        parts.append((t, np.full(len(t), c), np.full(len(t), tin), np.full(len(t), tout)))
    arr = np.concatenate([p[0] for p in parts])
    order = np.argsort(arr, kind="stable")
    q = {"arrival": arr[order], "client": np.concatenate([p[1] for p in parts])[order].astype(np.int32),
         "in_tokens": np.concatenate([p[2] for p in parts])[order].astype(np.int32),
         "true_out": np.concatenate([p[3] for p in parts])[order].astype(np.int32)}
    q["tag"] = np.full(len(arr), -1, np.int32)
    q["client_names"] = ["client1", "client2"]
    q["tag_names"] = list(W.TAG_NAMES)
    return q


def run_both(traces, alphas, **kw):
    from paper_2508_16646_b200 import scheduler as S
    base = dict(model=default_model(), profile=default_profile())
    base.update(kw)
    ref = []
    for q, a in zip(traces, alphas):
        case = H.StepCase(client=q["client"], arrival=q["arrival"], in_tokens=q["in_tokens"], true_out=q["true_out"],
                          tag=q["tag"], client_names=q["client_names"], alpha=float(a), **base)
        ref.append(H.ref_replay(case, max_sim_time_s=0.0, ema_alpha=0.2, cap=1 << 20))
    case0 = H.StepCase(client=traces[0]["client"], arrival=traces[0]["arrival"], in_tokens=traces[0]["in_tokens"],
                       true_out=traces[0]["true_out"], tag=traces[0]["tag"], client_names=traces[0]["client_names"],
                       alpha=float(alphas[0]), **base)
    sch = S.GpuScheduler(case_clients(case0), running=np.zeros(len(case0.client_names), np.int32), **case_kwargs(case0))
    row_off = np.concatenate([[0], np.cumsum([len(q["client"]) for q in traces])])
    cat = {k: np.concatenate([np.asarray(q[k]) for q in traces]) for k in ("client", "arrival", "in_tokens", "true_out")}
    tag = np.concatenate([np.where(np.asarray(q["tag"]) < 0, 0, np.asarray(q["tag"]) + 1) for q in traces])
    cap = max(len(r[0]) for r in ref) + 1
    got = sch.replay(row_off, cat["client"], cat["arrival"], cat["in_tokens"], cat["true_out"], alphas,
                     tag=tag.astype(np.uint8), ema_alpha=0.2, ev_cap=cap)
    return ref, got


def check(ref, got):
    for i, (ev_id, ev_kind, ev_time, u, r, c) in enumerate(ref):
        n = int(got["n_events"][i])
        assert n == len(ev_id), f"replay {i}: {n} events vs {len(ev_id)}"
        np.testing.assert_array_equal(got["ev_id"][i, :n], ev_id, err_msg=f"replay {i} ids")
        np.testing.assert_array_equal(got["ev_kind"][i, :n], ev_kind, err_msg=f"replay {i} kinds")
        np.testing.assert_array_equal(got["ev_time"][i, :n], ev_time, err_msg=f"replay {i} times")
        np.testing.assert_array_equal(got["ufc"][i], u, err_msg=f"replay {i} ufc")
        np.testing.assert_array_equal(got["rfc"][i], r, err_msg=f"replay {i} rfc")
        np.testing.assert_array_equal(got["counter"][i], c, err_msg=f"replay {i} counter")


@needs_ref
@pytest.mark.parametrize("pred_kind", [0, 1])
def test_cfg1_shaped_replays_match_reference(pred_kind):
    traces = [poisson_trace(s) for s in range(4)]
    ref, got = run_both(traces, [0.5, 0.6, 0.7, 0.85], pred_kind=pred_kind)
    check(ref, got)
    assert all(len(r[0]) > 30 for r in ref), [len(r[0]) for r in ref]


@needs_ref
@pytest.mark.parametrize("over", [{"kind": 1}, {"kind": 1, "vtc_use_prediction": True}, {"kind": 0},
                                  {"backfill": True, "max_batch": 8}, {"norm_mode": 1},
                                  {"mem_per_token_bytes": 1.0, "mem_capacity_bytes": 40000.0}])
def test_replay_policies_match_reference(over):
    traces = [poisson_trace(10 + s, rate=300.0, duration=4.0) for s in range(3)]
    ref, got = run_both(traces, [0.3, 0.7, 1.0], pred_kind=0, **over)
    check(ref, got)


@needs_ref
def test_alpha_sweep_preset_replays_match_reference():
    """configs[4]'s shape: the poisson preset under an alpha grid, many replays in one launch."""
    alphas = np.repeat(np.arange(0.5, 0.86, 0.05), 4)
    traces = [preset_trace(100 + i) for i in range(len(alphas))]
    ref, got = run_both(traces, alphas, pred_kind=0)
    check(ref, got)


@needs_ref
def test_sweep_metrics_match_reference_build_report():
    """build_report's jain_ttft_p90 and throughput_tps per replay (what run_sweep_alpha averages)."""
    alphas = [0.5, 0.7, 0.85]
    traces = [preset_trace(200 + i) for i in range(3)] + [poisson_trace(300, n_clients=5, rate=200.0, duration=5.0)]
    want = []
    for a in alphas:
        for q in traces[:3]:
            case = H.StepCase(client=q["client"], arrival=q["arrival"], in_tokens=q["in_tokens"],
                              true_out=q["true_out"], tag=q["tag"], client_names=q["client_names"], alpha=a,
                              pred_kind=0, profile=default_profile())
            want.append(H.ref_replay_report(case))
    ref, got = run_both(traces[:3] * 3, np.repeat(alphas, 3), pred_kind=0)
    check(ref, got)
    np.testing.assert_array_equal(got["jain_ttft_p90"], [w["jain_ttft_p90"] for w in want])
    np.testing.assert_array_equal(got["throughput_tps"], [w["throughput_tps"] for w in want])
    np.testing.assert_array_equal(got["completed"], [w["completed"] for w in want])
    np.testing.assert_array_equal(got["sim_end"], [w["sim_end"] for w in want])
    # the 5-client trace exercises the client_id-ordered Jain sum
    q = traces[3]
    case = H.StepCase(client=q["client"], arrival=q["arrival"], in_tokens=q["in_tokens"], true_out=q["true_out"],
                      tag=q["tag"], client_names=q["client_names"], alpha=0.6, pred_kind=0, profile=default_profile())
    w5 = H.ref_replay_report(case)
    _, g5 = run_both([q], [0.6], pred_kind=0)
    assert g5["jain_ttft_p90"][0] == w5["jain_ttft_p90"] and g5["throughput_tps"][0] == w5["throughput_tps"]


def run_full(traces, alphas, window_s=1.0, win_cap=128, max_sim=0.0, **kw):
    from paper_2508_16646_b200 import scheduler as S
    base = dict(model=default_model(), profile=default_profile())
    base.update(kw)
    cases = [H.StepCase(client=q["client"], arrival=q["arrival"], in_tokens=q["in_tokens"], true_out=q["true_out"],
                        tag=q["tag"], client_names=q["client_names"], alpha=float(a), **base)
             for q, a in zip(traces, alphas)]
    want = [H.ref_replay_full(c, max_sim_time_s=max_sim, window_s=window_s, win_cap=win_cap) for c in cases]
    sch = S.GpuScheduler(case_clients(cases[0]), running=np.zeros(len(cases[0].client_names), np.int32),
                         **case_kwargs(cases[0]))
    row_off = np.concatenate([[0], np.cumsum([len(q["client"]) for q in traces])])
    cat = {k: np.concatenate([np.asarray(q[k]) for q in traces]) for k in ("client", "arrival", "in_tokens", "true_out")}
    tag = np.concatenate([np.where(np.asarray(q["tag"]) < 0, 0, np.asarray(q["tag"]) + 1) for q in traces])
    got = sch.replay(row_off, cat["client"], cat["arrival"], cat["in_tokens"], cat["true_out"], alphas,
                     tag=tag.astype(np.uint8), ema_alpha=0.2, ev_cap=1, max_sim_time_s=max_sim,
                     report_window_s=window_s, win_cap=win_cap)
    return want, got


def check_full(want, got, win_cap):
    for i, w in enumerate(want):
        rep = got["report"][i]
        for k, v in w["report"].items():
            assert rep[k] == v, f"replay {i} report.{k}: {rep[k]!r} vs {v!r}"
        for k, v in w["clients"].items():
            np.testing.assert_array_equal(got["clients"][k][i], v, err_msg=f"replay {i} clients.{k}")
        nw, nd, nr = (min(int(rep[k]), win_cap) for k in ("n_windows", "n_diff", "n_rate"))
        np.testing.assert_array_equal(got["win"][i, :nw], w["win"][:nw], err_msg=f"replay {i} gpu_series")
        np.testing.assert_array_equal(got["win_clients"][i, :nw], w["win_clients"][:nw],
                                      err_msg=f"replay {i} counter_series")
        np.testing.assert_array_equal(got["diff"][i, :nd], w["diff"][:nd], err_msg=f"replay {i} diff_series")
        np.testing.assert_array_equal(got["rate"][i, :, :nr], w["rate"][:, :nr], err_msg=f"replay {i} service rates")


@needs_ref
@pytest.mark.parametrize("window_s", [1.0, 0.25, 0.7])
def test_full_report_preset_sweep(window_s):
    """build_report (metrics.cpp:151-229) and the engine's window samples (engine.cpp:379-430),
    every field and series bit-exact against the reference objects, over an alpha grid."""
    alphas = [0.5, 0.65, 0.85]
    traces = [preset_trace(400 + i, duration=12.0) for i in range(3)]
    want, got = run_full(traces, alphas, window_s=window_s, win_cap=128, pred_kind=0)
    check_full(want, got, 128)
    assert all(w["report"]["n_diff"] >= 10 for w in want)


@needs_ref
@pytest.mark.parametrize("over", [{}, {"kind": 1}, {"kind": 0, "max_batch": 8}, {"norm_mode": 1},
                                  {"pred_kind": 1}, {"backfill": True, "max_batch": 6}])
def test_full_report_policies(over):
    kw = dict(pred_kind=0)
    kw.update(over)
    traces = [poisson_trace(500 + s, n_clients=5, rate=250.0, duration=4.0) for s in range(2)]
    want, got = run_full(traces, [0.4, 0.8], window_s=0.5, win_cap=64, **kw)
    check_full(want, got, 64)


@needs_ref
def test_full_report_cutoff_caps_and_single_client():
    # max_sim_time_s cuts the run mid-window; a small win_cap truncates the series only
    traces = [poisson_trace(600, n_clients=4, rate=300.0, duration=5.0)]
    want, got = run_full(traces, [0.7], window_s=0.3, win_cap=5, max_sim=3.3, pred_kind=0)
    check_full(want, got, 5)
    assert want[0]["report"]["n_windows"] > 5
    # one client: service_difference is undefined, the report keeps zeros there
    q = preset_trace(601, duration=8.0)
    keep = q["client"] == 0
    one = {k: (np.asarray(v)[keep] if isinstance(v, np.ndarray) else v) for k, v in q.items()}
    one["client_names"] = ["client1"]
    want, got = run_full([one], [0.7], window_s=1.0, win_cap=32, pred_kind=0)
    check_full(want, got, 32)
    assert got["report"]["n_diff"][0] == 0 and got["report"]["max_diff"][0] == 0.0


# ---- the engine's whole log, horizons, eligibility, large rosters, caller predictions ----------
def run_log(traces, alphas, duration=None, overhead_ms=0.0, max_sim=0.0, predicted=None, window_s=1.0, **kw):
    """GPU replays with log_all against the reference's run_simulation SimResult (ref_replay_log)."""
    from paper_2508_16646_b200 import scheduler as S
    base = dict(model=default_model(), profile=default_profile())
    base.update(kw)
    cases = [H.StepCase(client=q["client"], arrival=q["arrival"], in_tokens=q["in_tokens"], true_out=q["true_out"],
                        tag=q["tag"], client_names=q["client_names"], alpha=float(a),
                        duration_s=float(duration[i]) if duration is not None else 0.0,
                        prediction_overhead_ms=overhead_ms, **base)
             for i, (q, a) in enumerate(zip(traces, alphas))]
    want = [H.ref_replay_log(c, max_sim_time_s=max_sim, window_s=window_s) for c in cases]
    gkw = case_kwargs(cases[0])
    if predicted is not None:  # the caller's predictor made the predictions; the device maps them
        gkw["predictor"] = "oracle"
    sch = S.GpuScheduler(case_clients(cases[0]), running=np.zeros(len(cases[0].client_names), np.int32), **gkw)
    row_off = np.concatenate([[0], np.cumsum([len(q["client"]) for q in traces])])
    cat = {k: np.concatenate([np.asarray(q[k]) for q in traces]) for k in ("client", "arrival", "in_tokens", "true_out")}
    tag = np.concatenate([np.where(np.asarray(q["tag"]) < 0, 0, np.asarray(q["tag"]) + 1) for q in traces])
    cap = max(len(w["id"]) for w in want) + 1
    got = sch.replay(row_off, cat["client"], cat["arrival"], cat["in_tokens"], cat["true_out"], alphas,
                     tag=tag.astype(np.uint8), ema_alpha=0.2, ev_cap=cap, max_sim_time_s=max_sim,
                     report_window_s=window_s, duration_s=duration, prediction_overhead_ms=overhead_ms,
                     predicted=None if predicted is None else np.concatenate(predicted), log_all=True)
    return want, got


def check_log(want, got):
    for i, w in enumerate(want):
        n = int(got["n_events"][i])
        assert n == len(w["id"]), f"replay {i}: {n} log entries vs {len(w['id'])}"
        for k, g in (("id", "ev_id"), ("kind", "ev_kind"), ("time", "ev_time"), ("i0", "ev_i0"), ("d0", "ev_d0"),
                     ("d1", "ev_d1"), ("d2", "ev_d2")):
            np.testing.assert_array_equal(got[g][i, :n], w[k], err_msg=f"replay {i} log {k}")
        np.testing.assert_array_equal(got["profile"][i], w["profile"], err_msg=f"replay {i} profile")
        np.testing.assert_array_equal(got["ufc"][i], w["clients"][:, 0])
        np.testing.assert_array_equal(got["rfc"][i], w["clients"][:, 1])
        np.testing.assert_array_equal(got["counter"][i], w["clients"][:, 2])
        np.testing.assert_array_equal(got["clients"]["accumulated_service"][i], w["clients"][:, 3])
        np.testing.assert_array_equal(got["clients"]["backlogged"][i], w["clients"][:, 4])
        rep = got["report"][i]
        assert rep["sim_end_s"] == w["sim_end"] and rep["busy_ms_total"] == w["busy_ms_total"]
        assert rep["overhead_ms_total"] == w["overhead_ms_total"]
        assert rep["max_resident_kv_tokens"] == w["max_resident_kv_tokens"]
        assert rep["completed"] == w["completed"] and rep["rejected"] == w["rejected"]
        assert got["counter_clamps"][i] == w["counter_clamps"]


@needs_ref
@pytest.mark.parametrize("over", [{}, {"kind": 1}, {"kind": 1, "vtc_use_prediction": True}, {"kind": 0},
                                  {"backfill": True, "max_batch": 6}, {"norm_mode": 1}, {"pred_kind": 1},
                                  {"mem_per_token_bytes": 1.0, "mem_capacity_bytes": 40000.0}])
def test_full_event_log_matches_reference(over):
    """log_all: arrived / admitted / first_token / completed / rejected entries with every
    payload field, in the reference's log order, bit-exact (engine.cpp:44-76,171-375)."""
    kw = dict(pred_kind=0)
    kw.update(over)
    traces = [poisson_trace(700 + s, n_clients=6, rate=250.0, duration=4.0) for s in range(3)]
    # a 30 s horizon (Trace::duration_s) past the 4 s of arrivals: most requests complete
    want, got = run_log(traces, [0.3, 0.7, 0.9], duration=[30.0] * 3, **kw)
    check_log(want, got)
    assert all((w["kind"] == 5).sum() > 25 for w in want), [(w["kind"] == 5).sum() for w in want]


@needs_ref
def test_duration_horizon_and_prediction_overhead():
    """Trace::duration_s beyond the last arrival (generated scenarios, workload.cpp:213) keeps
    the run going until then (engine.cpp:120-121); prediction_overhead_ms delays eligibility
    (engine.cpp:165-168)."""
    traces = [poisson_trace(800 + s, n_clients=4, rate=200.0, duration=3.0) for s in range(2)]
    for overhead in (0.0, 7.5):
        want, got = run_log(traces, [0.5, 0.8], duration=[6.0, 4.5], overhead_ms=overhead, pred_kind=0)
        check_log(want, got)
        assert all(w["sim_end"] > 3.0 for w in want)


@needs_ref
@pytest.mark.parametrize("n_clients", [17, 40, 300])
def test_large_roster_replays_match_reference(n_clients):
    """Rosters beyond 16 clients (ledger in global scratch, per-client skipped stamps) --
    run_simulation accepts any roster (engine.cpp:154-164)."""
    traces = [poisson_trace(900 + n_clients + s, n_clients=n_clients, rate=400.0, duration=3.0) for s in range(2)]
    for over in ({}, {"backfill": True, "max_batch": 8}, {"kind": 1}):
        kw = dict(pred_kind=1)
        kw.update(over)
        want, got = run_log(traces, [0.6, 0.75], **kw)
        check_log(want, got)


@needs_ref
def test_caller_predictions_column():
    """Predictions made by a caller's Predictor (here the reference's NoisyOraclePredictor),
    handed over per row: the device applies max(1, .) and maps them against the evolving
    profile, exactly as drain_arrivals does with predictor.predict (engine.cpp:177-180)."""
    traces = [poisson_trace(1000 + s, n_clients=5, rate=250.0, duration=4.0) for s in range(2)]
    preds = [H.ref_noisy_predict(33.0, 1, np.arange(len(q["client"]), dtype=np.int64), q["true_out"]) for q in traces]
    want, got = run_log(traces, [0.5, 0.7], predicted=preds, pred_kind=2, noisy_l1=33.0, noisy_seed=1)
    check_log(want, got)


def test_committed_cfg1_replay_golden():
    """tests/golden/replay_cfg1.npz: BASELINE configs[0] at its stated size through
    run_simulation (8 clients, Poisson arrivals at 400 req/s for 25 s = 10,218 requests,
    uniform(4, 1024) lengths, MoPE, max_sim_time_s 25) recorded from the reference build by
    `oracle/gen_golden.py --replay-cfg1` -- checked without the reference present: admitted /
    rejected sequence with its times and the final ledgers, bit-exact.  400 req/s overloads the
    64-slot batch, so the log is short (81 events) while the ledgers see every arrival."""
    import os
    from paper_2508_16646_b200 import scheduler as S
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "replay_cfg1.npz"))
    n = len(z["client"])
    case = H.StepCase(client=z["client"], arrival=z["arrival"], in_tokens=z["in_tokens"], true_out=z["true_out"],
                      tag=z["tag"], client_names=[f"client{i}" for i in range(8)], model=default_model(),
                      profile=default_profile())
    sch = S.GpuScheduler(case_clients(case), running=np.zeros(8, np.int32), **case_kwargs(case))
    tag = np.where(z["tag"] < 0, 0, z["tag"] + 1).astype(np.uint8)
    got = sch.replay(np.array([0, n]), z["client"], z["arrival"], z["in_tokens"], z["true_out"], [case.alpha],
                     tag=tag, ema_alpha=0.2, ev_cap=len(z["ev_id"]) + 1, max_sim_time_s=25.0)
    ne = int(got["n_events"][0])
    assert n > 10000 and ne == len(z["ev_id"]) > 50
    np.testing.assert_array_equal(got["ev_id"][0, :ne], z["ev_id"])
    np.testing.assert_array_equal(got["ev_kind"][0, :ne], z["ev_kind"])
    np.testing.assert_array_equal(got["ev_time"][0, :ne], z["ev_time"])
    for k in ("ufc", "rfc", "counter"):
        np.testing.assert_array_equal(got[k][0], z[k], err_msg=k)
