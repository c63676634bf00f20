"""The drop-in: the reference's C++ API and Python bindings with the engine's
translation unit replaced by the B200 one (paper_2508_16646_b200/dropin: engine_b200.cpp ->
eqx_replay on the GPU), against the reference's own unmodified build (oracle/_ref/py, CPU engine).

Both are the package ``equinox_sim`` (the reference's bindings/module.cpp over its core), so each
runs in its own interpreter (tests/dropin_driver.py).  The bar is the reference's own
determinism check (test_engine.cpp:83-94, acceptance C8 at acceptance_main.cpp:381-404): the
event log as NDJSON byte-identical, and every report of run / run_sweep_alpha / run_ablation
equal, through the public runners with run configs (run_config.cpp) -- scenario presets, a
cfg1-sized trace file (BASELINE configs[0]: 8 clients, ~10k requests, MoPE), every policy,
predictor and engine option.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DROPIN = os.path.join(ROOT, "paper_2508_16646_b200", "dropin")
REFPY = os.path.join(ROOT, "oracle", "_ref", "py")
DRIVER = os.path.join(ROOT, "tests", "dropin_driver.py")


def _have(d):
    return os.path.isdir(os.path.join(d, "equinox_sim")) and any(
        f.startswith("_core") for f in os.listdir(os.path.join(d, "equinox_sim")))


pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not (_have(DROPIN) and _have(REFPY)),
                                 reason="drop-in / reference Python modules not built (build() in the container)")]


def run_jobs(where: str, jobs: list) -> list:
    p = subprocess.run([sys.executable, DRIVER, where], input=json.dumps(jobs), capture_output=True, text=True,
                       timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    out = json.loads(p.stdout)
    assert out["engine"] == ("b200" if where == DROPIN else "reference-cpu")
    return out["results"]


def both(jobs: list):
    return run_jobs(DROPIN, jobs), run_jobs(REFPY, jobs)


def cfg1_trace(path: str, seed: int = 1) -> str:
    """BASELINE configs[0] / SURVEY.md 8(d) cfg1: 8 clients (client0..7), Poisson arrivals at
    400 req/s in total for 25 s, LengthDist::uniform(4, 1024) inputs and outputs, category tags
    by output tercile with noise 0.2 -- as a trace file in load_trace's format."""
    from paper_2508_16646_b200 import workload as W
    rng = np.random.default_rng(seed)
    t = np.cumsum(rng.exponential(1.0 / 400.0, 12000))
    t = t[t < 25.0]
    n = len(t)
    client = rng.integers(0, 8, n)
    tin = rng.integers(4, 1025, n)
    tout = rng.integers(4, 1025, n).astype(np.int32)
    tag = W.assign_category_tags(tout, rng, 0.2)
    names = ["short", "medium", "long"]
    with open(path, "w") as f:
        f.write("client_id,arrival_time_s,input_tokens,output_tokens,category_tag\n")
        for i in range(n):
            f.write(f"client{client[i]},{t[i]:.9f},{tin[i]},{tout[i]},{names[tag[i]]}\n")
    return path


MOPE = {"kind": "mope", "experts": 3, "corpus": "builtin", "corpus_size": 10000, "corpus_seed": 7}


def test_cfg1_event_log_ndjson_byte_identical(tmp_path):
    """cfg1 at its stated size through run_events: the whole NDJSON event log of the B200 engine
    equals the reference engine's byte for byte (MoPE predictor, Equinox alpha 0.7)."""
    trace = cfg1_trace(str(tmp_path / "cfg1.csv"))
    cfg = {"scenario": {"trace": trace}, "policy": {"kind": "equinox", "alpha": 0.7, "delta": 0.1,
                                                    "output_weight": 4.0},
           "predictor": MOPE, "seeds": [1]}
    (got,), (want,) = both([{"fn": "run_events", "config": cfg}])
    assert "ok" in want, want
    assert got == want
    lines = want["ok"].splitlines()
    assert len(lines) > 10000  # ~10k arrivals (400 req/s overloads a 64-slot batch: few complete)
    kinds = {json.loads(x)["event"] for x in lines}
    assert {"arrived", "admitted", "first_token", "completed"} <= kinds


@pytest.mark.parametrize("preset", ["balanced", "poisson", "overload", "dynamic_increase"])
def test_preset_event_logs_byte_identical(preset):
    """The reference's scenario presets (workload.cpp:243-297) under every policy and predictor."""
    jobs = []
    for pol in ({"kind": "equinox"}, {"kind": "equinox", "norm_mode": "none"}, {"kind": "vtc"},
                {"kind": "vtc", "use_prediction": True}, {"kind": "fcfs"}):
        for pred in ({"kind": "oracle"}, {"kind": "noisy_oracle", "target_l1": 33}):
            jobs.append({"fn": "run_events", "config": {"scenario": {"preset": preset, "duration_s": 20.0},
                                                        "policy": pol, "predictor": pred, "seeds": [3]}})
    got, want = both(jobs)
    for g, w, j in zip(got, want, jobs):
        assert "ok" in w, (j, w)
        assert g == w, j


def test_engine_options_byte_identical():
    """EngineConfig fields through the run config's engine block (run_config.cpp:222-244):
    horizon, report window, EMA rate, backfill, prediction overhead; and the perf block's KV
    budget (adaptive batching) and timing constants."""
    base = {"scenario": {"preset": "overload", "duration_s": 15.0}, "policy": {"kind": "equinox"},
            "predictor": {"kind": "oracle"}, "seeds": [5]}
    variants = [
        {"engine": {"max_sim_time_s": 9.5}},
        {"engine": {"report_window_s": 0.25, "ema_alpha": 0.5}},
        {"engine": {"backfill": True}, "perf": {"max_batch": 8}},
        {"engine": {"prediction_overhead_ms": 12.5}},
        {"perf": {"mem_capacity_bytes": 4.0e9, "max_batch": 4096}},
        {"perf": {"prefill_linear": 0.1, "decode_base": 3.0, "refresh_overhead": 5.0}},
    ]
    jobs = [{"fn": "run_events", "config": dict(base, **v)} for v in variants]
    got, want = both(jobs)
    for g, w, j in zip(got, want, jobs):
        assert "ok" in w, (j, w)
        assert g == w, j


def test_runner_reports_equal(tmp_path):
    """run (run_batch's aggregate over seeds, jobs=4 threads each calling run_simulation),
    run_sweep_alpha (experiments.cpp:331-373) and run_ablation: every reported number equal."""
    trace = cfg1_trace(str(tmp_path / "t.csv"), seed=2)
    jobs = [
        {"fn": "run", "config": {"scenario": {"preset": "balanced", "duration_s": 20.0},
                                 "policy": {"kind": "equinox"}, "predictor": {"kind": "oracle"},
                                 "seeds": [1, 2, 3]}, "jobs": 4},
        {"fn": "run", "config": {"scenario": {"trace": trace}, "policy": {"kind": "equinox"}, "predictor": MOPE,
                                 "seeds": [1]}, "jobs": 1},
        {"fn": "run_sweep_alpha", "config": {"scenario": {"preset": "poisson", "duration_s": 20.0},
                                             "policy": {"kind": "equinox"}, "predictor": {"kind": "oracle"},
                                             "seeds": [1, 2], "alphas": [0.5, 0.6, 0.7, 0.8, 0.9]}, "jobs": 4},
        {"fn": "run_ablation", "config": {
            "scenario": {"preset": "poisson", "duration_s": 20.0}, "policy": {"kind": "equinox"},
            "predictor": {"kind": "oracle"}, "seeds": [1, 2],
            "grid": [{"name": "FCFS", "policy": {"kind": "fcfs"}, "predictor": {"kind": "oracle"}},
                     {"name": "VTC", "policy": {"kind": "vtc", "use_prediction": False}},
                     {"name": "Equinox+noise", "policy": {"kind": "equinox"},
                      "predictor": {"kind": "noisy_oracle", "target_l1": 33}}]}, "jobs": 3},
    ]
    got, want = both(jobs)
    for g, w, j in zip(got, want, jobs):
        assert "ok" in w, (j, w)
        assert g == w, j["fn"]


def test_errors_match_reference():
    """ConfigError / EngineError types and messages through the same entry points."""
    jobs = [
        {"fn": "run_events", "config": {"scenario": {"preset": "balanced", "duration_s": 5.0},
                                        "policy": {"kind": "equinox", "alpha": 1.2}, "seeds": [1]}},
        {"fn": "run_events", "config": {"scenario": {"preset": "balanced", "duration_s": 5.0},
                                        "engine": {"ema_alpha": 0.0}, "seeds": [1]}},
        {"fn": "run_events", "config": {"scenario": {"preset": "overload", "duration_s": 10.0},
                                        "perf": {"mem_capacity_bytes": 3.0e8, "max_batch": 4096},
                                        "seeds": [1]}},
    ]
    got, want = both(jobs)
    assert got == want
    assert all("error" in w for w in want[:2])
