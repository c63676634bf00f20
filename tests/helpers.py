"""Shared test helpers: golden fixtures <-> oracle StepCase <-> GpuScheduler."""
from __future__ import annotations

import glob
import json
import os

import numpy as np

import harness as H
from paper_2508_16646_b200 import scheduler as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
DATA = os.path.join(ROOT, "paper_2508_16646_b200", "data")
KIND_NAMES = {0: "fcfs", 1: "vtc", 2: "equinox"}
PRED_NAMES = {0: "oracle", 1: "mope", 2: "noisy_oracle", 3: "single_proxy"}


def golden_names():
    return sorted(os.path.basename(p)[5:-4] for p in glob.glob(os.path.join(GOLDEN, "step_*.npz")))


def load_golden(name: str):
    z = np.load(os.path.join(GOLDEN, f"step_{name}.npz"))
    meta = json.loads(str(z["meta"]))
    ins = {k[3:]: z[k] for k in z.files if k.startswith("in_")}
    outs = {k[4:]: z[k] for k in z.files if k.startswith("out_")}
    outs.update({k: meta[k] for k in ("n_admitted", "n_rejected", "new_prefill", "length_fallbacks")})
    return meta, ins, outs


def case_from_golden(meta: dict, ins: dict) -> H.StepCase:
    kw = {k: meta[k] for k in H.StepCase.__dataclass_fields__ if k in meta and k not in ("model", "profile")}
    prof = {k: np.asarray(v) for k, v in meta["profile"].items()}
    return H.StepCase(client=ins["client"], arrival=ins["arrival"], in_tokens=ins["in_tokens"],
                      true_out=ins["true_out"], tag=ins["tag"], id=ins["id"], weight=ins["weight"],
                      ufc0=ins["ufc0"], rfc0=ins["rfc0"], counter0=ins["counter0"], running=ins["running"],
                      mem_in=ins["mem_in"], mem_generated=ins["mem_generated"],
                      mem_reserved=ins["mem_reserved"], model=meta["model"], profile=prof, **kw)


def default_model() -> dict:
    with open(os.path.join(DATA, "mope_builtin_c10000_s7_e3.json")) as f:
        return json.load(f)


def default_profile() -> dict:
    with open(os.path.join(DATA, "profile_default.json")) as f:
        return {k: np.asarray(v) for k, v in json.load(f).items()}


def case_clients(case: H.StepCase) -> list:
    case.finalize()
    return [S.ClientState(n, weight=float(w), ufc=float(u), rfc=float(r), counter=float(k))
            for n, w, u, r, k in zip(case.client_names, case.weight, case.ufc0, case.rfc0, case.counter0)]


def case_kwargs(case: H.StepCase) -> dict:
    """GpuScheduler keyword arguments (policy, perf, profile, predictor) of a StepCase."""
    case.finalize()
    pol = S.PolicySpec(kind=KIND_NAMES[case.kind],
                       equinox=S.EquinoxParams(case.alpha, case.delta, case.output_weight,
                                               "none" if case.norm_mode == H.NORM_NONE else "max_over_clients"),
                       vtc_use_prediction=bool(case.vtc_use_prediction), counter_lift=bool(case.counter_lift))
    perf = S.PerfParams(max_batch=case.max_batch, mem_per_token_bytes=case.mem_per_token_bytes,
                        mem_capacity_bytes=case.mem_capacity_bytes)
    p = case.profile
    prof = S.GpuProfile.from_arrays(p["upper"], p["lat"], p["util"], p["tps"])
    model = S.MopeModel.from_json(case.model) if case.model is not None else None
    return dict(policy=pol, perf=perf, profile=prof, predictor=PRED_NAMES[case.pred_kind], model=model,
                tag_names=case.tag_names, noisy_l1=case.noisy_l1, noisy_seed=case.noisy_seed,
                backfill=bool(case.backfill))


def case_batch(case: H.StepCase) -> tuple:
    reserved = int(np.sum(case.mem_in.astype(np.int64) +
                          np.maximum(case.mem_reserved, case.mem_generated).astype(np.int64)))
    return len(case.mem_in), reserved


def case_columns(case: H.StepCase) -> dict:
    tag = np.where(np.asarray(case.tag) < 0, 0, np.asarray(case.tag) + 1).astype(np.uint8)
    return dict(client=np.asarray(case.client, np.int32), arrival_s=np.asarray(case.arrival, np.float64),
                input_tokens=np.asarray(case.in_tokens, np.int32), tag=tag,
                true_output_tokens=np.asarray(case.true_out, np.int32), ids=np.asarray(case.id, np.int64))


def gpu_run(case: H.StepCase, device_columns: bool = False):
    """Run one StepCase through the product (GpuScheduler over libeqx_b200.so)."""
    sch = S.GpuScheduler(case_clients(case), running=case.running, **case_kwargs(case))
    sch.set_batch(*case_batch(case))
    cols = case_columns(case)
    if device_columns:
        import torch
        cols = {k: torch.from_numpy(v).cuda() for k, v in cols.items()}
    sch.drain(**cols)
    res = sch.step(case.now)
    return sch, res


def compare_step(res, sch, want: dict, flagged_near_ties: int = 0, row_ids=None) -> None:
    """Bit-exact parity of events, ledger and per-request scores against an oracle output.

    ``flagged_near_ties`` > 0 (noisy-oracle predictions within 1e-9 of a .5 rounding boundary,
    where the device's log1p and glibc's may round apart -- the only differences the north
    star allows): every unflagged row must still match bit-exactly; a flagged row may differ
    by one token.  The schedule is compared in full when no prediction differs, else only up to
    the first event that a differing prediction could have influenced."""
    if flagged_near_ties and compare_flagged(res, sch.scores(), want, flagged_near_ties, row_ids):
        return
    np.testing.assert_array_equal(res.ids, want["ev_id"], err_msg="event ids / order")
    np.testing.assert_array_equal(res.kinds, want["ev_kind"], err_msg="event kinds")
    np.testing.assert_array_equal(res.clients, want["ev_client"])
    adm = want["ev_kind"] == H.EV_ADMIT
    np.testing.assert_array_equal(res.ufc_inc[adm], want["ev_ufc_inc"][adm])
    np.testing.assert_array_equal(res.rfc_inc[adm], want["ev_rfc_inc"][adm])
    np.testing.assert_array_equal(res.vtc_inc[adm], want["ev_vtc_inc"][adm])
    np.testing.assert_array_equal(res.wait_s[adm], want["ev_wait"][adm])
    assert res.n_admitted == want["n_admitted"] and res.n_rejected == want["n_rejected"]
    assert res.new_prefill_tokens == want["new_prefill"]
    led = sch.ledger()
    np.testing.assert_array_equal(led["ufc"], want["ufc"], err_msg="ledger ufc")
    np.testing.assert_array_equal(led["rfc"], want["rfc"], err_msg="ledger rfc")
    np.testing.assert_array_equal(led["counter"], want["counter"], err_msg="ledger counter")
    np.testing.assert_array_equal(led["backlogged"], want["backlogged"], err_msg="backlogged")
    sc = sch.scores()
    np.testing.assert_array_equal(sc["pred"], want["pred"], err_msg="pred")
    np.testing.assert_array_equal(sc["bucket"].astype(np.int32), want["bucket"], err_msg="bucket")
    np.testing.assert_array_equal(sc["ufc_inc"], want["ufc_inc"], err_msg="ufc_inc")
    np.testing.assert_array_equal(sc["rfc_inc"], want["rfc_inc"], err_msg="rfc_inc")
    assert res.length_fallbacks == want["length_fallbacks"]


def compare_flagged(res, sc: dict, want: dict, flagged: int, row_ids=None) -> bool:
    """Noisy-oracle near-ties (see compare_step): unflagged rows bit-exact, flagged rows within
    one token.  Returns True when a prediction differs -- the event prefix before the first
    event of a differing row was compared and the rest of the step may legitimately differ."""
    diff = np.nonzero(sc["pred"] != want["pred"])[0]
    assert len(diff) <= flagged, f"{len(diff)} predictions differ, {flagged} flagged"
    assert np.all(np.abs(sc["pred"][diff].astype(np.int64) - want["pred"][diff]) == 1)
    ok = np.ones(len(sc["pred"]), bool)
    ok[diff] = False
    for k in ("pred", "ufc_inc", "rfc_inc"):
        np.testing.assert_array_equal(sc[k][ok], want[k][ok], err_msg=k + " (unflagged rows)")
    np.testing.assert_array_equal(np.asarray(sc["bucket"]).astype(np.int32)[ok], want["bucket"][ok])
    if not len(diff):
        return False
    # the schedule agrees up to the first event of a request whose prediction differs (its
    # increments enter the ledger there); compare that prefix
    bad = set((np.arange(len(sc["pred"])) if row_ids is None else np.asarray(row_ids))[diff].tolist())
    n = min(len(res.ids), len(want["ev_id"]))
    stop = next((i for i in range(n) if int(want["ev_id"][i]) in bad or int(res.ids[i]) in bad), n)
    np.testing.assert_array_equal(res.ids[:stop], want["ev_id"][:stop], err_msg="event prefix")
    return True
