"""Live queues: several scheduling steps over one queue that arrivals are
appended to, with completions (on_complete + update_map) between the steps.

The oracle is the reference itself (oracle/ref_step.cpp ref_multi): drain_arrivals with the
prediction records frozen against the profile of the moment, admit_requests on the queues left
by earlier steps, completions in batch order.  The GPU side drives eqx_append / eqx_step /
eqx_feedback through the C ABI with the same host bookkeeping of the batch the reference
engine keeps (members in admission order, reserved KV tokens).  Bit-exact: every step's event
ids, kinds and pending increments, the final FP64 ledger and the EMA'd profile.
"""
import numpy as np
import pytest

import harness as H
from helpers import case_clients, case_columns, case_kwargs, default_model, default_profile
from paper_2508_16646_b200 import workload as W

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not H.available("ref"), reason="reference build not present")]


def scenario(seed, n=6000, C=16, **over):
    rng = np.random.default_rng(seed)
    q = W.lmsys_queue(n, C, seed=seed, heavy_frac=0.5 if seed % 2 else None, untagged_frac=0.02)
    kw = dict(max_batch=int(rng.choice([16, 64, 300])), kind=2, norm_mode=int(rng.integers(0, 2)))
    kw.update(over)
    case = H.StepCase(client=q["client"], arrival=q["arrival"] * 10.0, in_tokens=q["in_tokens"],
                      true_out=q["true_out"], tag=q["tag"], client_names=q["client_names"], model=default_model(),
                      profile=default_profile(), weight=rng.choice([0.5, 1.0, 2.0], C), **kw)
    cuts = np.sort(rng.choice(np.arange(1, n), 5, replace=False))
    step_end = np.concatenate([cuts, [n, n, n]])
    step_now = np.sort(rng.uniform(0.0, 10.0, len(step_end)))
    step_now = np.maximum(step_now, case.arrival[np.minimum(step_end, n) - 1])  # arrivals <= now
    act = dict(extra=rng.uniform(0, 2, n), tps=rng.uniform(10, 5000, n), util=rng.uniform(0.2, 1, n))
    return case, step_end, step_now, act


def gpu_multi(case, step_end, step_now, act, ema_alpha, complete_mod):
    from paper_2508_16646_b200 import scheduler as S
    case.finalize()
    sch = S.GpuScheduler(case_clients(case), running=np.zeros(len(case.client_names), np.int32), **case_kwargs(case))
    cols = case_columns(case)
    arrival, in_tok, true_out = cols["arrival_s"], cols["input_tokens"], cols["true_output_tokens"]
    members = []  # (id, client, need, pend_ufc, pend_rfc, pend_vtc) in admission order
    ev = {k: [] for k in ("ev_id", "ev_kind", "ev_step", "ev_ufc", "ev_rfc")}
    row = 0
    for k, (end, now) in enumerate(zip(step_end, step_now)):
        if end > row:
            sch.append(**{name: v[row:end] for name, v in cols.items()})
            row = end
        sch.set_batch(len(members), int(sum(m[2] for m in members)))
        res = sch.step(float(now))
        for i in range(len(res.ids)):
            ev["ev_id"].append(res.ids[i])
            ev["ev_kind"].append(res.kinds[i])
            ev["ev_step"].append(k)
            ev["ev_ufc"].append(res.ufc_inc[i])
            ev["ev_rfc"].append(res.rfc_inc[i])
            if res.kinds[i] == S.EV_ADMITTED:
                rid = int(res.ids[i])
                members.append((rid, int(res.clients[i]), int(in_tok[rid]) + int(res.preds[i]), res.ufc_inc[i],
                                res.rfc_inc[i], res.vtc_inc[i]))
        done = [m for m in members if (m[0] * 7 + k) % complete_mod == 0]
        members = [m for m in members if (m[0] * 7 + k) % complete_mod != 0]
        if done:
            ids = np.array([m[0] for m in done])
            sch.feedback(completions=dict(
                client=np.array([m[1] for m in done], np.int32), input_tokens=in_tok[ids], output_tokens=true_out[ids],
                latency_s=(float(now) - arrival[ids]) + act["extra"][ids], tps=act["tps"][ids],
                gpu_util=act["util"][ids], pending_ufc=np.array([m[3] for m in done]),
                pending_rfc=np.array([m[4] for m in done]), pending_vtc=np.array([m[5] for m in done])),
                ema_alpha=ema_alpha)
    out = {k: np.asarray(v) for k, v in ev.items()}
    out.update({k: v for k, v in sch.ledger().items() if k in ("ufc", "rfc", "counter")})
    pm = sch.profile_metrics()
    out.update({"prof_" + k: v for k, v in pm.items()})
    return out


@pytest.mark.parametrize("seed", range(8))
def test_live_queue_multi_step_vs_reference(seed):
    over = [{}, {"kind": 1}, {"kind": 1, "vtc_use_prediction": True}, {"kind": 0}, {"backfill": True},
            {"pred_kind": 0}, {"mem_per_token_bytes": 1.0, "mem_capacity_bytes": 6000.0}, {"counter_lift": False}][seed]
    case, step_end, step_now, act = scenario(seed, **over)
    mod = [2, 3, 5, 2, 3, 4, 2, 3][seed]
    want = H.ref_multi(case, step_end, step_now, act["extra"], act["tps"], act["util"], 0.2, mod)
    got = gpu_multi(case, step_end, step_now, act, 0.2, mod)
    for k in ("ev_id", "ev_kind", "ev_step"):
        np.testing.assert_array_equal(got[k], want[k], err_msg=k)
    adm = want["ev_kind"] == H.EV_ADMIT
    np.testing.assert_array_equal(got["ev_ufc"][adm], want["ev_ufc"][adm])
    np.testing.assert_array_equal(got["ev_rfc"][adm], want["ev_rfc"][adm])
    for k in ("ufc", "rfc", "counter", "prof_lat", "prof_util", "prof_tps"):
        np.testing.assert_array_equal(got[k], want[k], err_msg=k)
    assert want["ev_step"].max() >= 3  # several steps saw events
