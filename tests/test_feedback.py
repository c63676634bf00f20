"""Completion / feedback path: on_tokens, on_complete and update_map.

CPU: the C restatement (oracle/eqx_oracle.c eqxo_feedback_run) against the reference-generated
goldens (tests/golden/fb_*.npz, oracle/gen_golden.py --feedback) and, where the reference build
is present, against the reference objects on fresh seeds.

GPU: eqx_feedback through the C ABI, bit-exact against the goldens (ledger, accumulated
service, clamp count, running counts, EMA'd profile), the clamp branch against the
restatement, and the next step's scoring against the oracle run with the EMA'd profile.
"""
import glob
import json
import os

import numpy as np
import pytest

import harness as H
from helpers import GOLDEN, case_columns, default_model, default_profile

FB_NAMES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "fb_*.npz")))


def load_feedback(name: str):
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    meta = json.loads(str(z["meta"]))
    fb = dict(meta)
    for k in ("weight", "ufc0", "rfc0", "counter0", "service0", "tokens"):
        fb[k] = z["in_" + k]
    fb["profile"] = {k[5:]: z[k] for k in z.files if k.startswith("prof_")}
    fb["adm"] = {k[4:]: z[k] for k in z.files if k.startswith("adm_")}
    fb["done"] = {k[5:]: z[k] for k in z.files if k.startswith("done_")}
    out = {k[4:]: z[k] for k in z.files if k.startswith("out_")}
    out["clamps"] = int(out["clamps"])
    return fb, out


def running_counts(fb):
    C = len(fb["weight"])
    adm_client = np.asarray(fb["adm"]["client"])
    run0 = np.bincount(adm_client, minlength=C).astype(np.int32)
    done_client = adm_client[np.asarray(fb["done"]["adm"], np.int64)]
    return run0, run0 - np.bincount(done_client, minlength=C).astype(np.int32)


def compare(got: dict, want: dict, keys=("ufc", "rfc", "counter", "service", "prof_lat", "prof_util", "prof_tps")):
    for k in keys:
        np.testing.assert_array_equal(got[k], want[k], err_msg=k)
    assert got["clamps"] == want["clamps"]


# ---------------------------------------------------------------------------------- CPU ----
@pytest.mark.parametrize("name", FB_NAMES)
def test_restatement_matches_feedback_golden(name):
    fb, want = load_feedback(name)
    got = H.run_feedback(fb, "oracle", pend=want["pend"], mid=want["mid"])
    compare(got, want)


@pytest.mark.skipif(not H.available("ref"), reason="reference build not present")
@pytest.mark.parametrize("seed", range(6))
def test_restatement_matches_reference_fresh_seeds(seed):
    fb = H.feedback_case(seed=100 + seed, kind=seed % 3, vtc_use_prediction=seed % 2, n_clients=3 + 7 * seed,
                         n_adm=20 + 30 * seed, n_done=15 + 20 * seed, ledger_scale=float(seed % 2),
                         ema_alpha=[0.05, 0.2, 0.5, 1.0, 0.3, 0.9][seed], profile=default_profile())
    ref = H.run_feedback(fb, "ref")
    got = H.run_feedback(fb, "oracle", pend=ref["pend"], mid=ref["mid"])
    compare(got, ref)


def test_restatement_clamps_and_alpha_validation():
    fb = H.feedback_case(seed=9, kind=1, vtc_use_prediction=1, profile=default_profile())
    C, n = len(fb["weight"]), len(fb["adm"]["client"])
    pend = np.full((3, n), 1e9)  # far above any actual: every corrected counter goes negative
    got = H.run_feedback(fb, "oracle", pend=pend, mid=np.zeros((3, C)))
    assert got["clamps"] == 3 * len(fb["done"]["adm"])
    assert np.all(got["ufc"] == 0.0) and np.all(got["rfc"] == 0.0) and np.all(got["counter"] == 0.0)
    fb["ema_alpha"] = 0.0
    with pytest.raises(ValueError, match="ema_alpha"):
        H.run_feedback(fb, "oracle", pend=pend, mid=np.zeros((3, C)))


# ---------------------------------------------------------------------------------- GPU ----
def gpu_feedback(fb, pend, mid, model=None, tag_names=()):
    from paper_2508_16646_b200 import scheduler as S
    kind = {0: "fcfs", 1: "vtc", 2: "equinox"}[fb["kind"]]
    clients = [S.ClientState(nm, weight=float(w), ufc=float(u), rfc=float(r), counter=float(k))
               for nm, w, u, r, k in zip(fb["names"], fb["weight"], mid[0], mid[1], mid[2])]
    p = fb["profile"]
    run0, _ = running_counts(fb)
    sch = S.GpuScheduler(clients, policy=S.PolicySpec(kind=kind, equinox=S.EquinoxParams(fb["alpha"], fb["delta"],
                                                                                          fb["output_weight"]),
                                                      vtc_use_prediction=bool(fb["vtc_use_prediction"])),
                         profile=S.GpuProfile.from_arrays(p["upper"], p["lat"], p["util"], p["tps"]),
                         predictor="mope" if model else "oracle", model=S.MopeModel.from_json(model) if model else None,
                         tag_names=tag_names, running=run0)
    sch.set_service(fb["service0"])
    d = fb["done"]
    idx = np.asarray(d["adm"], np.int64)
    comp = dict(client=np.asarray(fb["adm"]["client"])[idx], input_tokens=np.asarray(fb["adm"]["in"])[idx],
                output_tokens=d["out"], latency_s=d["latency_s"], tps=d["tps"], gpu_util=d["util"],
                pending_ufc=pend[0][idx], pending_rfc=pend[1][idx], pending_vtc=pend[2][idx])
    sch.feedback(tokens=fb["tokens"], completions=comp, ema_alpha=fb["ema_alpha"])
    led = sch.ledger()
    sv, clamps = sch.service()
    pm = sch.profile_metrics()
    got = {"ufc": led["ufc"], "rfc": led["rfc"], "counter": led["counter"], "running": led["running"],
           "service": sv, "clamps": clamps, "prof_lat": pm["lat"], "prof_util": pm["util"], "prof_tps": pm["tps"]}
    return sch, got


@pytest.mark.gpu
@pytest.mark.parametrize("name", FB_NAMES)
def test_gpu_feedback_matches_golden(name):
    fb, want = load_feedback(name)
    _, got = gpu_feedback(fb, want["pend"], want["mid"])
    compare(got, want)
    np.testing.assert_array_equal(got["running"], running_counts(fb)[1])


@pytest.mark.gpu
def test_gpu_feedback_clamps_match_restatement():
    fb = H.feedback_case(seed=9, kind=1, vtc_use_prediction=1, profile=default_profile())
    C, n = len(fb["weight"]), len(fb["adm"]["client"])
    rng = np.random.default_rng(3)
    pend = rng.uniform(0, 3e4, (3, n))  # a mix of corrections that do and do not go negative
    mid = np.zeros((3, C))
    want = H.run_feedback(fb, "oracle", pend=pend, mid=mid)
    _, got = gpu_feedback(fb, pend, mid)
    assert want["clamps"] > 0
    compare(got, want)


@pytest.mark.gpu
def test_gpu_feedback_profile_feeds_the_next_step():
    """update_map's EMA is the profile the next drain maps against (engine order)."""
    from paper_2508_16646_b200 import workload as W
    fb, want = load_feedback("fb_cold_many")
    model = default_model()
    sch, got = gpu_feedback(fb, want["pend"], want["mid"], model=model, tag_names=W.TAG_NAMES)
    compare(got, want)
    C = len(fb["weight"])
    q = W.lmsys_queue(5000, C, seed=21)
    prof = {"upper": fb["profile"]["upper"], "lat": want["prof_lat"], "util": want["prof_util"],
            "tps": want["prof_tps"]}
    case = H.StepCase(client=q["client"], arrival=q["arrival"], in_tokens=q["in_tokens"], true_out=q["true_out"],
                      tag=q["tag"], client_names=list(fb["names"]), model=model, profile=prof,
                      weight=np.asarray(fb["weight"]), ufc0=want["ufc"], rfc0=want["rfc"], counter0=want["counter"],
                      running=running_counts(fb)[1])
    ref = H.run_step(case, "oracle")
    cols = case_columns(case)
    sch.drain(**cols)
    res = sch.step(case.now)
    np.testing.assert_array_equal(res.ids, ref["ev_id"])
    sc = sch.scores()
    np.testing.assert_array_equal(sc["ufc_inc"], ref["ufc_inc"])
    np.testing.assert_array_equal(sc["rfc_inc"], ref["rfc_inc"])
