"""CPU: pin the C restatement (oracle/eqx_oracle.c) to the reference.

1. every committed golden step (produced by the reference's own code, oracle/gen_golden.py)
   is reproduced bit-for-bit by the restatement;
2. the reference's unit-test known answers (test_scheduler.cpp, test_predictor.cpp,
   test_gpu_model.cpp, acceptance C1) hold for the restatement;
3. when the reference build (oracle/_ref) is present, restatement == reference on fresh seeds.
"""
import ctypes as C

import numpy as np
import pytest

import harness as H
from helpers import case_from_golden, default_model, default_profile, golden_names, load_golden
from paper_2508_16646_b200 import workload as W

OUT_KEYS = ["pred", "bucket", "lat", "util", "tps", "ufc_inc", "rfc_inc", "ev_id", "ev_kind", "ev_client",
            "ev_ufc_inc", "ev_rfc_inc", "ev_vtc_inc", "ev_wait", "ufc", "rfc", "counter", "backlogged"]


def assert_same(a, b):
    for k in OUT_KEYS:
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)
    for k in ("n_admitted", "n_rejected", "new_prefill", "length_fallbacks"):
        assert a[k] == b[k], k


@pytest.mark.parametrize("name", golden_names())
def test_restatement_matches_golden(name):
    meta, ins, outs = load_golden(name)
    got = H.run_step(case_from_golden(meta, ins), "oracle")
    assert_same(got, outs)


def test_golden_set_covers_edge_cases():
    names = set(golden_names())
    for must in ("eqx_max_warm", "eqx_max_cold", "eqx_none", "vtc_bare", "vtc_pred", "fcfs", "rejects",
                 "reject_stream_backfill", "tight_kv_backfill", "batch_running", "no_lift", "ties_fcfs",
                 "ties_eqx", "heavy_kv", "empty", "one_client", "noisy", "single_proxy", "oracle_pred"):
        assert must in names
    meta, _, outs = load_golden("reject_stream_backfill")
    assert outs["n_rejected"] > 100  # long rejection streams are exercised
    meta, _, outs = load_golden("ties_eqx")
    assert outs["length_fallbacks"] > 0  # untagged + unseen tags


def _lib():
    lib = C.CDLL(H.LIB_ORACLE)
    lib.eqxo_ufc_increment.restype = C.c_double
    lib.eqxo_ufc_increment.argtypes = [C.c_double, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_double]
    lib.eqxo_rfc_increment.restype = C.c_double
    lib.eqxo_rfc_increment.argtypes = [C.c_double, C.c_double, C.c_double]
    return lib


def test_unit_known_answers_ufc_rfc():
    lib = _lib()
    # test_scheduler.cpp:50-67, acceptance_main.cpp:119-137
    assert lib.eqxo_ufc_increment(1.0, 100, 400, 0.0, 0.0, 0.1, 4.0) == pytest.approx(1700.0, rel=1e-12)
    assert lib.eqxo_ufc_increment(1.0, 100, 400, 5.0, 5000.0, 0.1, 4.0) == pytest.approx(850.0, rel=1e-12)
    for wait in (0.0, 3.0, 60.0):
        assert lib.eqxo_ufc_increment(1.0, 100, 400, wait, 1000.0, 0.0, 4.0) == pytest.approx(1700.0, rel=1e-12)
    prev = 1e300
    for i in range(21):  # monotone in wait (test_scheduler.cpp:69-78)
        v = lib.eqxo_ufc_increment(1.0, 100, 400, 2.5 * i, 250.0, 0.1, 4.0)
        assert v <= prev
        prev = v
    # test_scheduler.cpp:80-87
    assert lib.eqxo_rfc_increment(1.0, 1000.0, 0.9) == pytest.approx(900.0, rel=1e-12)
    assert lib.eqxo_rfc_increment(1.0, 1000.0, 0.0) == 0.0
    assert lib.eqxo_rfc_increment(2.0, 750.0, 0.5) == pytest.approx(2 * lib.eqxo_rfc_increment(1.0, 750.0, 0.5))


def _two_client_case(kind, ufc, rfc, arrivals, names=("c1", "c2"), **kw):
    prof = default_profile()
    return H.StepCase(client=np.array([0, 1], np.int32), arrival=np.array(arrivals, np.float64),
                      in_tokens=np.array([10, 10], np.int32), true_out=np.array([5, 5], np.int32),
                      tag=np.array([-1, -1], np.int32), client_names=list(names), ufc0=np.array(ufc, np.float64),
                      rfc0=np.array(rfc, np.float64), profile=prof, pred_kind=H.PRED_ORACLE, kind=kind,
                      counter_lift=False, **{"max_batch": 1, **kw})


def test_holistic_selection_known_answers():
    # test_scheduler.cpp:89-110: HF(c1)=1.0 > HF(c2)=0.65 -> c2 admitted first
    out = H.run_step(_two_client_case(H.EQUINOX, [1000.0, 500.0], [100.0, 100.0], [0.0, 0.0]), "oracle")
    assert list(out["ev_client"]) == [1]
    # scale invariance (test_scheduler.cpp:112-133)
    a = H.run_step(_two_client_case(H.EQUINOX, [1200.0, 900.0], [40.0, 90.0], [0.0, 0.0]), "oracle")
    b = H.run_step(_two_client_case(H.EQUINOX, [1200 * 37.5, 900 * 37.5], [40 * 37.5, 90 * 37.5], [0.0, 0.0]), "oracle")
    assert list(a["ev_client"]) == list(b["ev_client"])


def test_tie_break_arrival_then_client_id():
    # test_scheduler.cpp:135-142 (FCFS): earlier head wins; equal arrival -> "c1" < "c2"
    out = H.run_step(_two_client_case(H.FCFS, [0, 0], [0, 0], [2.0, 1.0], max_batch=2), "oracle")
    assert list(out["ev_client"]) == [1, 0]
    out = H.run_step(_two_client_case(H.FCFS, [0, 0], [0, 0], [2.0, 2.0], max_batch=2), "oracle")
    assert list(out["ev_client"]) == [0, 1]
    out = H.run_step(_two_client_case(H.FCFS, [0, 0], [0, 0], [2.0, 2.0], names=("c2", "c10"), max_batch=2), "oracle")
    assert list(out["ev_client"]) == [1, 0]  # bytewise: "c10" < "c2"


def test_counter_lift_known_answers():
    # test_scheduler.cpp:191-217: an idle client activated behind a backlogged one is lifted
    prof = default_profile()
    case = H.StepCase(client=np.array([0, 1], np.int32), arrival=np.array([0.0, 0.1]),
                      in_tokens=np.array([10, 10], np.int32), true_out=np.array([5, 5], np.int32),
                      tag=np.array([-1, -1], np.int32), client_names=["c1", "c2"],
                      counter0=np.array([5000.0, 100.0]), profile=prof, pred_kind=H.PRED_ORACLE, kind=H.VTC,
                      max_batch=1)
    out = H.run_step(case, "oracle")
    assert out["counter"][1] == 5000.0  # c2 lifted to c1's counter before admission
    case.counter0 = np.array([100.0, 900.0])
    out = H.run_step(case, "oracle")
    assert out["counter"][1] == 900.0  # already above the minimum: kept
    case.counter0 = np.array([5000.0, 100.0])
    case.counter_lift = False
    out = H.run_step(case, "oracle")
    assert list(out["ev_client"]) == [1] and out["counter"][1] == 110.0  # not lifted: c2 wins, +in


def test_can_fit_and_rejection_known_answers():
    # test_gpu_model.cpp:28-44: 11 > 10 never fits, 10 <= 10 fits (m=1, M=10)
    prof = default_profile()
    case = H.StepCase(client=np.array([0, 0], np.int32), arrival=np.array([0.0, 0.1]),
                      in_tokens=np.array([5, 5], np.int32), true_out=np.array([6, 5], np.int32),
                      tag=np.array([-1, -1], np.int32), client_names=["a"], profile=prof,
                      pred_kind=H.PRED_ORACLE, mem_per_token_bytes=1.0, mem_capacity_bytes=10.0)
    out = H.run_step(case, "oracle")
    assert list(out["ev_kind"]) == [H.EV_REJECT, H.EV_ADMIT]  # test_engine.cpp:159-176 shape
    assert out["n_rejected"] == 1 and out["n_admitted"] == 1


def test_profile_lookup_and_route_known_answers():
    prof = default_profile()
    # entry_for: 1 -> 32, 33 -> 64, 1e5 -> 4096 (test_gpu_model.cpp:95-101)
    case = H.StepCase(client=np.zeros(3, np.int32), arrival=np.zeros(3), in_tokens=np.full(3, 1, np.int32),
                      true_out=np.array([1, 33, 100000], np.int32), tag=-np.ones(3, np.int32),
                      client_names=["a"], profile=prof, pred_kind=H.PRED_ORACLE)
    out = H.run_step(case, "oracle")
    assert [int(prof["upper"][b]) for b in out["bucket"]] == [32, 64, 4096]
    # route golden cases (test_predictor.cpp:83-115)
    lib = C.CDLL(H.LIB_ORACLE)
    thr = np.array([50, 200], np.int32)
    rows = np.array([[0.0, 0.1, 0.9], [0.4, 0.4, 0.2]], np.float64)
    m = H.Mope(n_thresholds=2, thresholds=thr.ctypes.data_as(C.POINTER(C.c_int32)), mix_weight=0.5,
               num_buckets=3, n_rows=2, rows=rows.ctypes.data_as(C.POINTER(C.c_double)))
    fb = C.c_int(0)
    lib.eqxo_route.argtypes = [C.POINTER(H.Mope), C.c_int, C.c_int, C.POINTER(C.c_int)]
    assert lib.eqxo_route(C.byref(m), 10, -1, C.byref(fb)) == 0 and fb.value == 1
    assert lib.eqxo_route(C.byref(m), 120, -1, C.byref(fb)) == 1 and fb.value == 1
    m.mix_weight = 0.0
    assert lib.eqxo_route(C.byref(m), 10, 0, C.byref(fb)) == 2 and fb.value == 0
    assert lib.eqxo_route(C.byref(m), 10000, 1, C.byref(fb)) == 0  # ties -> shorter bucket


def test_noisy_predictor_matches_reference_samples():
    z = np.load(f"{H.HERE}/../tests/golden/noisy_predict.npz")
    lib = C.CDLL(H.LIB_ORACLE)
    lib.eqxo_noisy_predict.argtypes = [C.c_double, C.c_uint64, C.c_int64, C.c_int]
    got33 = [lib.eqxo_noisy_predict(33.0, 17, int(i), int(t)) for i, t in zip(z["id"][:5000], z["true_out"][:5000])]
    np.testing.assert_array_equal(np.maximum(1, got33), z["pred33"][:5000])
    l1 = np.abs(z["pred80"].astype(float) - z["true_out"]).mean()
    assert 60 < l1 < 90  # C6 shape: the max(1, .) clamp pulls noisy-80 below 80


@pytest.mark.skipif(not H.available("ref"), reason="reference build (oracle/_ref) not present")
@pytest.mark.parametrize("seed", [101, 102, 103])
def test_restatement_matches_reference_fresh_seeds(seed):
    rng = np.random.default_rng(seed)
    C_ = int(rng.choice([3, 17, 64, 250]))
    q = W.lmsys_queue(int(rng.integers(200, 4000)), C_, seed=seed, untagged_frac=0.05,
                      heavy_frac=0.5 if seed % 2 else None)
    led = W.warm_ledger(C_, seed=seed)
    kw = dict(kind=int(rng.integers(0, 3)), norm_mode=int(rng.integers(0, 2)),
              vtc_use_prediction=bool(rng.integers(0, 2)), backfill=bool(rng.integers(0, 2)),
              max_batch=int(rng.choice([16, 64, 512])), mem_per_token_bytes=1.0,
              mem_capacity_bytes=float(rng.choice([900.0, 5000.0, 122880.0])),
              pred_kind=int(rng.choice([0, 1, 3])))
    case = H.StepCase(client=q["client"], arrival=q["arrival"], in_tokens=q["in_tokens"], true_out=q["true_out"],
                      tag=q["tag"], client_names=q["client_names"], model=default_model(),
                      profile=default_profile(), ufc0=led["ufc"] * rng.integers(0, 2), rfc0=led["rfc"],
                      counter0=led["counter"], **kw)
    assert_same(H.run_step(case, "oracle"), H.run_step(case, "ref"))
