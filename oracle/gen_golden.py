"""Generate tests/golden/ fixtures and the model/profile data files -- TEST INFRASTRUCTURE.

Every output number here is produced by the *reference's own code* (oracle/_ref/libeqx_ref.so,
compiled from /root/reference/proj/src by ``make -C oracle ref``); nothing is produced by the
restatement or by the GPU path.  Run from the repo root:

    python oracle/gen_golden.py

Writes
  paper_2508_16646_b200/data/mope_builtin_c10000_s7_e3.json  train_mope on the builtin corpus
      (experiments.cpp:58-73 with PredictorConfig{experts=3}.bucket_percentiles())
  paper_2508_16646_b200/data/profile_default.json            build_profile(PerfParams{},
      default_bucket_bounds(), 1) (gpu_model.cpp:87-130)
  tests/golden/step_<name>.npz                               one scheduling step per case
  tests/golden/noisy_predict.npz                             NoisyOraclePredictor samples
  tests/golden/replay_cfg1.npz                               full run_simulation replay
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, HERE)
sys.path.insert(0, ROOT)

import harness as H  # noqa: E402
from paper_2508_16646_b200 import workload as W  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
DATA = os.path.join(ROOT, "paper_2508_16646_b200", "data")

PARAM_KEYS = ["kind", "alpha", "delta", "output_weight", "norm_mode", "vtc_use_prediction",
              "counter_lift", "backfill", "max_batch", "mem_per_token_bytes",
              "mem_capacity_bytes", "now", "pred_kind", "noisy_l1", "noisy_seed"]
ARRAY_KEYS = ["client", "arrival", "in_tokens", "true_out", "tag", "id", "weight", "ufc0",
              "rfc0", "counter0", "running", "mem_in", "mem_generated", "mem_reserved"]
OUT_KEYS = ["pred", "bucket", "lat", "util", "tps", "ufc_inc", "rfc_inc", "ev_id", "ev_kind",
            "ev_client", "ev_ufc_inc", "ev_rfc_inc", "ev_vtc_inc", "ev_wait", "ufc", "rfc",
            "counter", "backlogged"]


def save_case(name: str, case: H.StepCase, out: dict, note: str) -> None:
    case.finalize()
    d = {f"in_{k}": np.asarray(getattr(case, k)) for k in ARRAY_KEYS}
    d.update({f"out_{k}": out[k] for k in OUT_KEYS})
    meta = {k: getattr(case, k) for k in PARAM_KEYS}
    meta.update(client_names=case.client_names, tag_names=case.tag_names, note=note,
                n_admitted=out["n_admitted"], n_rejected=out["n_rejected"],
                new_prefill=out["new_prefill"], length_fallbacks=out["length_fallbacks"],
                model=case.model, profile={k: np.asarray(v).tolist() for k, v in case.profile.items()})
    d["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(GOLDEN, f"step_{name}.npz"), **d)


def base_case(q: dict, model: dict, profile: dict, **kw) -> H.StepCase:
    return H.StepCase(client=q["client"], arrival=q["arrival"], in_tokens=q["in_tokens"],
                      true_out=q["true_out"], tag=q["tag"], id=q["id"],
                      client_names=q["client_names"], tag_names=q["tag_names"], model=model,
                      profile=profile, **kw)


def main() -> None:
    os.makedirs(GOLDEN, exist_ok=True)
    os.makedirs(DATA, exist_ok=True)
    model = json.loads(H.ref_train_mope_json(10000, 7, 3))
    with open(os.path.join(DATA, "mope_builtin_c10000_s7_e3.json"), "w") as f:
        json.dump(model, f, indent=1, sort_keys=True)
    prof = H.ref_build_profile()
    with open(os.path.join(DATA, "profile_default.json"), "w") as f:
        json.dump({k: v.tolist() for k, v in prof.items()}, f, indent=1)

    cases = []
    q8 = W.lmsys_queue(1500, 8, seed=11)
    led8 = W.warm_ledger(8, seed=12)
    warm8 = dict(ufc0=led8["ufc"], rfc0=led8["rfc"], counter0=led8["counter"])
    cases.append(("eqx_max_warm", base_case(q8, model, prof, **warm8),
                  "equinox, max_over_clients (default), MoPE, warm ledger, C=8"))
    cases.append(("eqx_max_cold", base_case(q8, model, prof, max_batch=256),
                  "equinox default, cold (all-zero) ledger: maxima change every few picks"))
    cases.append(("eqx_none", base_case(q8, model, prof, norm_mode=H.NORM_NONE, max_batch=128, **warm8),
                  "equinox norm_mode=none"))
    cases.append(("vtc_bare", base_case(q8, model, prof, kind=H.VTC, **warm8), "VTC bare"))
    cases.append(("vtc_pred", base_case(q8, model, prof, kind=H.VTC, vtc_use_prediction=True, **warm8),
                  "VTC use_prediction"))
    cases.append(("fcfs", base_case(q8, model, prof, kind=H.FCFS, **warm8), "FCFS"))
    # tight KV budget: in+pred > 1500 tokens never fits -> rejections; no backfill -> prefix cut
    tight = dict(mem_per_token_bytes=1.0, mem_capacity_bytes=1500.0, max_batch=512)
    q8o = W.lmsys_queue(1500, 8, seed=13)
    cases.append(("tight_kv", base_case(q8o, model, prof, pred_kind=H.PRED_ORACLE, **tight, **warm8),
                  "oracle predictor, 1500-token KV budget: never-fit rejections + budget cut"))
    cases.append(("tight_kv_backfill", base_case(q8o, model, prof, pred_kind=H.PRED_ORACLE, backfill=True,
                                                 **tight, **warm8),
                  "same with backfill (skip clients that do not fit)"))
    rej = dict(mem_per_token_bytes=1.0, mem_capacity_bytes=700.0, max_batch=512)
    cases.append(("rejects", base_case(q8o, model, prof, pred_kind=H.PRED_ORACLE, **rej, **warm8),
                  "700-token budget: most long requests never fit -> streams of rejections"))
    cases.append(("rejects_backfill", base_case(q8o, model, prof, pred_kind=H.PRED_ORACLE, backfill=True,
                                                **rej, **warm8), "same with backfill"))
    q8s = dict(q8o)
    q8s["in_tokens"] = np.where(q8o["client"] == 0, 1000, q8o["in_tokens"]).astype(np.int32)
    cases.append(("reject_stream", base_case(q8s, model, prof, pred_kind=H.PRED_ORACLE, **rej),
                  "client 0 never fits and keeps the lowest key: long rejection streams (cold ledger)"))
    cases.append(("reject_stream_backfill", base_case(q8s, model, prof, pred_kind=H.PRED_ORACLE,
                                                      backfill=True, **rej), "same with backfill"))
    # existing batch + running clients + weights
    rng = np.random.default_rng(5)
    w = rng.choice([0.5, 1.0, 2.0, 3.0], 8)
    running = np.array([0, 2, 0, 1, 0, 0, 3, 0], np.int32)
    mem_in = rng.integers(10, 500, 6).astype(np.int32)
    cases.append(("batch_running", base_case(q8, model, prof, weight=w, running=running, mem_in=mem_in,
                                             mem_generated=rng.integers(0, 50, 6).astype(np.int32),
                                             mem_reserved=rng.integers(1, 300, 6).astype(np.int32),
                                             max_batch=40, **warm8),
                  "pre-existing batch of 6, running clients skip the lift, weights != 1"))
    cases.append(("no_lift", base_case(q8, model, prof, counter_lift=False, running=running, **warm8),
                  "counter_lift off"))
    # ties: quantised arrivals + FCFS and equal ledgers; untagged + unseen tags
    q16 = W.lmsys_queue(2000, 16, seed=17, untagged_frac=0.1)
    q16["arrival"] = np.floor(q16["arrival"] * 40) / 40.0
    q16["tag_names"] = ["short", "medium", "long", "mystery"]
    q16["tag"] = np.where(np.random.default_rng(3).random(2000) < 0.05, 3, q16["tag"]).astype(np.int32)
    q16["client_names"] = [f"c{(i * 7) % 16}x" for i in range(16)]
    cases.append(("ties_fcfs", base_case(q16, model, prof, kind=H.FCFS, max_batch=200),
                  "quantised arrivals: ties broken by client_id bytes"))
    cases.append(("ties_eqx", base_case(q16, model, prof, max_batch=200),
                  "equinox cold with quantised arrivals, untagged (-1) and unseen ('mystery') tags"))
    # predictors
    cases.append(("oracle_pred", base_case(q8, model, prof, pred_kind=H.PRED_ORACLE, **warm8), "oracle predictor"))
    cases.append(("single_proxy", base_case(q8, model, prof, pred_kind=H.PRED_SINGLE, **warm8),
                  "single-proxy table (expert 0 of the model stands in)"))
    cases.append(("noisy", base_case(q8, model, prof, pred_kind=H.PRED_NOISY, noisy_l1=33.0, noisy_seed=9,
                                     **warm8), "noisy oracle (Laplace via log1p)"))
    # heavy hitter, KV-budget-bound, large max_batch
    qh = W.lmsys_queue(6000, 200, seed=19, heavy_frac=0.5)
    ledh = W.warm_ledger(200, seed=20)
    cases.append(("heavy_kv", base_case(qh, model, prof, max_batch=4096, ufc0=ledh["ufc"], rfc0=ledh["rfc"],
                                        counter0=ledh["counter"]),
                  "cfg3 shape: heavy hitter, max_batch 4096, 122880-token KV budget binds"))
    cases.append(("heavy_kv_backfill", base_case(qh, model, prof, max_batch=4096, backfill=True),
                  "cfg3 shape with backfill, cold ledger"))
    # degenerate
    qe = W.lmsys_queue(0, 4, seed=1)
    cases.append(("empty", base_case(qe, model, prof), "empty queue"))
    q1 = W.lmsys_queue(300, 1, seed=23)
    cases.append(("one_client", base_case(q1, model, prof, max_batch=1000), "single client drains"))

    for name, case, note in cases:
        out = H.run_step(case, "ref")
        save_case(name, case, out, note)
        print(f"{name:20s} adm={out['n_admitted']:5d} rej={out['n_rejected']:4d} fb={out['length_fallbacks']}")

    # NoisyOraclePredictor samples (predictor.cpp:17-23) incl. small outputs that hit max(1, .)
    rng = np.random.default_rng(31)
    ids = rng.integers(0, 2**40, 20000).astype(np.int64)
    tout = rng.integers(1, 1500, 20000).astype(np.int32)
    np.savez_compressed(os.path.join(GOLDEN, "noisy_predict.npz"), id=ids, true_out=tout,
                        pred33=H.ref_noisy_predict(33.0, 17, ids, tout),
                        pred80=H.ref_noisy_predict(80.0, 17, ids, tout))

    gen_replay_cfg1(model, prof)
    gen_feedback(prof)


def gen_replay_cfg1(model: dict, prof: dict) -> None:
    """BASELINE configs[0] at its stated size through the reference's run_simulation: 8 clients,
    Poisson arrivals at 400 req/s for 25 s (~10k requests), LengthDist::uniform(4, 1024) inputs
    and outputs, category tags by output tercile with noise 0.2 (the shape of
    tests/test_dropin.py::cfg1_trace), MoPE, max_sim_time_s 25."""
    rng = np.random.default_rng(29)
    t = np.cumsum(rng.exponential(1.0 / 400.0, 12000))
    t = t[t < 25.0]
    n = len(t)
    tout = rng.integers(4, 1025, n).astype(np.int32)
    qr = {"client": rng.integers(0, 8, n).astype(np.int32), "arrival": t,
          "in_tokens": rng.integers(4, 1025, n).astype(np.int32), "true_out": tout,
          "tag": W.assign_category_tags(tout, rng, 0.2).astype(np.int32),
          "id": np.arange(n, dtype=np.int64), "client_names": [f"client{i}" for i in range(8)],
          "tag_names": ["short", "medium", "long"]}
    case = base_case(qr, model, prof)
    ev_id, ev_kind, ev_time, u, r, c = H.ref_replay(case, max_sim_time_s=25.0)
    np.savez_compressed(os.path.join(GOLDEN, "replay_cfg1.npz"), ev_id=ev_id, ev_kind=ev_kind,
                        ev_time=ev_time, ufc=u, rfc=r, counter=c, client=qr["client"],
                        arrival=qr["arrival"], in_tokens=qr["in_tokens"], true_out=qr["true_out"],
                        tag=qr["tag"])
    print("replay_cfg1: requests", n, "events", len(ev_id))


def gen_feedback(profile: dict) -> None:
    """Feedback goldens from the reference objects: the scenario, the
    pending increments on_admit registered, the ledger after the admissions, and the ledger,
    accumulated service, clamp count and profile after on_tokens + on_complete + update_map."""
    cases = {"fb_equinox": dict(seed=1), "fb_vtc_bare": dict(seed=2, kind=1),
             "fb_vtc_pred": dict(seed=3, kind=1, vtc_use_prediction=1), "fb_fcfs": dict(seed=4, kind=0),
             "fb_cold_many": dict(seed=5, n_clients=40, n_adm=300, n_done=250, ledger_scale=0.0),
             "fb_alpha1": dict(seed=6, ema_alpha=1.0)}
    for name, kw in cases.items():
        fb = H.feedback_case(profile=profile, **kw)
        r = H.run_feedback(fb, "ref")
        flat = {"meta": json.dumps({k: fb[k] for k in ("kind", "alpha", "delta", "output_weight",
                                                        "vtc_use_prediction", "ema_alpha", "now", "names")})}
        for k in ("weight", "ufc0", "rfc0", "counter0", "service0", "tokens"):
            flat["in_" + k] = np.asarray(fb[k])
        for k, v in fb["profile"].items():
            flat["prof_" + k] = np.asarray(v)
        for k, v in fb["adm"].items():
            flat["adm_" + k] = np.asarray(v)
        for k, v in fb["done"].items():
            flat["done_" + k] = np.asarray(v)
        flat["out_pend"] = r["pend"]
        flat["out_mid"] = r["mid"]
        for k in H.FEEDBACK_KEYS:
            flat["out_" + k] = r[k]
        flat["out_clamps"] = np.asarray(r["clamps"])
        np.savez_compressed(os.path.join(GOLDEN, f"{name}.npz"), **flat)
        print(name, "clamps", r["clamps"])


if __name__ == "__main__":
    if "--replay-cfg1" in sys.argv:  # only the cfg1 replay golden, with the committed model / profile
        with open(os.path.join(DATA, "mope_builtin_c10000_s7_e3.json")) as f:
            mdl = json.load(f)
        with open(os.path.join(DATA, "profile_default.json")) as f:
            gen_replay_cfg1(mdl, {k: np.asarray(v) for k, v in json.load(f).items()})
    elif "--feedback" in sys.argv:  # only the feedback goldens, with the committed profile
        with open(os.path.join(DATA, "profile_default.json")) as f:
            gen_feedback({k: np.asarray(v) for k, v in json.load(f).items()})
    else:
        main()
