"""Trace formats: the reference's CSV trace format (load_trace /
write_trace_csv / trace_hash, workload.cpp:300-428) and the binary struct-of-arrays format,
parsed by libeqx_b200.so (csrc/eqx_trace.cpp).

Oracle: the reference itself (oracle/_ref, ref_trace_load / ref_scenario_csv): columns, roster,
tags, warnings, trace_hash and every ParseError message must match exactly.  Host-only work, so
these run in the CPU suite (no GPU compute is involved).
"""
import os

import numpy as np
import pytest

import harness as H
from paper_2508_16646_b200.scheduler import ParseError
from paper_2508_16646_b200.trace import Trace

pytestmark = pytest.mark.skipif(not H.available("ref"), reason="reference build not present")

HEADER = "client_id,arrival_time_s,input_tokens,output_tokens,category_tag\n"


def same_as_reference(path):
    want = H.ref_trace_load(path)
    got = Trace.load_csv(path)
    assert len(got) == want["n"]
    np.testing.assert_array_equal(got.client, want["client"])
    np.testing.assert_array_equal(got.arrival_s, want["arrival"])
    np.testing.assert_array_equal(got.input_tokens, want["in_tokens"])
    np.testing.assert_array_equal(got.output_tokens, want["out_tokens"])
    tags = [got.tag_names[t].encode() if t >= 0 else b"" for t in got.tag]
    assert tags == want["tags"]
    assert got.client_names == want["client_names"]
    assert len(got.warnings) == want["n_warnings"]
    assert got.duration_s == want["duration"]
    assert got.hash() == want["hash"]
    return got, want


@pytest.mark.parametrize("preset,seed,duration", [("balanced", 2, 20.0), ("poisson", 42, 60.0),
                                                  ("overload", 7, 30.0), ("dynamic_increase", 3, 40.0)])
def test_reference_scenarios_load_and_hash(tmp_path, preset, seed, duration):
    """generate_scenario written by the reference -> our parser: same rows, roster and hash; the
    hash also equals trace_hash of the generated trace (the CSV round trip of test_workload.cpp)."""
    path = tmp_path / f"{preset}.csv"
    h0 = H.ref_scenario_csv(preset, seed, duration, str(path))
    got, want = same_as_reference(str(path))
    assert got.hash() == h0 and len(got) > 10
    # canonical re-serialisation is byte-identical to the reference's write_trace_csv
    out = tmp_path / "again.csv"
    got.save_csv(str(out))
    assert out.read_bytes() == path.read_bytes()


def test_unsorted_blank_crlf_and_lenient_numbers(tmp_path):
    p = tmp_path / "mixed.csv"
    p.write_bytes((HEADER.replace("\n", "\r\n") +
                   "b,2.0,10,20,coding\r\n\r\n"
                   "a,1.0,11,21,\n"
                   "c, 1.5,12abc,22,chat \n"
                   "a,1e0,13,+23,coding\n"
                   "d,1.0,14,24,x,\n"[:-3] + "\n").encode())
    got, want = same_as_reference(str(p))
    assert got.warnings == ["arrival times out of order; rows were re-sorted"]
    assert got.client_names == ["a", "d", "c", "b"] and len(got) == 5  # stable re-sort, first appearance


@pytest.mark.parametrize("body,needle", [
    ("a,0.5,100,400,\na,0.6,0,400,\n", "line 3"),
    ("a,0.5,100\n", "expected 5 fields, got 3"),
    ("a,0.5,100,400,x,\n", "expected 5 fields, got 6"),
    (",0.5,100,400,\n", "empty client_id"),
    ("a,abc,100,400,\n", "malformed numeric field"),
    ("a,0.5,99999999999,400,\n", "malformed numeric field"),
    ("a,1e999,100,400,\n", "malformed numeric field"),
    ("a,-0.5,100,400,\n", "negative arrival time"),
    ("a,0.5,100,0,\n", "token counts must be >= 1"),
])
def test_malformed_rows_raise_the_reference_message(tmp_path, body, needle):
    p = tmp_path / "bad.csv"
    p.write_text(HEADER + body)
    with pytest.raises(ValueError) as ref_err:
        H.ref_trace_load(str(p))
    with pytest.raises(ParseError) as our_err:
        Trace.load_csv(str(p))
    assert str(our_err.value) == str(ref_err.value)
    assert needle in str(our_err.value)


def test_header_empty_and_missing_files(tmp_path):
    cases = {"empty.csv": "", "hdr.csv": "client,arrival\n", "ok_empty.csv": HEADER}
    for name, text in cases.items():
        (tmp_path / name).write_text(text)
    for name in ("empty.csv", "hdr.csv"):
        with pytest.raises(ValueError) as ref_err:
            H.ref_trace_load(str(tmp_path / name))
        with pytest.raises(ParseError) as our_err:
            Trace.load_csv(str(tmp_path / name))
        assert str(our_err.value) == str(ref_err.value)
    t, _ = same_as_reference(str(tmp_path / "ok_empty.csv"))
    assert len(t) == 0 and t.duration_s == 0.0
    with pytest.raises(ParseError) as our_err:
        Trace.load_csv("/nonexistent/trace.csv")
    assert str(our_err.value) == "cannot open trace file '/nonexistent/trace.csv'"


def test_binary_round_trip_keeps_columns_and_hash(tmp_path):
    csv = tmp_path / "p.csv"
    H.ref_scenario_csv("poisson", 11, 30.0, str(csv))
    a = Trace.load_csv(str(csv))
    a.save_bin(str(tmp_path / "p.eqxt"))
    b = Trace.load(str(tmp_path / "p.eqxt"))
    for k in ("client", "arrival_s", "input_tokens", "output_tokens", "tag"):
        np.testing.assert_array_equal(getattr(a, k), getattr(b, k), err_msg=k)
    assert b.client_names == a.client_names and b.tag_names == a.tag_names
    assert b.stored_hash == a.hash() == b.hash()
    (tmp_path / "junk.eqxt").write_bytes(b"not a trace")
    with pytest.raises(ParseError):
        Trace.load(str(tmp_path / "junk.eqxt"))


def test_from_columns_matches_reference_reader(tmp_path):
    rng = np.random.default_rng(5)
    n = 5000
    arr = np.sort(rng.uniform(0, 100, n))
    cl = rng.integers(0, 3, n)
    tg = rng.integers(-1, 2, n)
    t = Trace.from_columns(cl, arr, rng.integers(1, 900, n), rng.integers(1, 900, n), ["u1", "u2", "u3"], tag=tg,
                           tag_names=["coding", "chat"])
    t.save_csv(str(tmp_path / "c.csv"))
    got, want = same_as_reference(str(tmp_path / "c.csv"))
    assert got.hash() == t.hash()
    # roster order is first appearance in the file, which the loader re-derives
    assert got.client_names == [["u1", "u2", "u3"][c] for c in dict.fromkeys(cl.tolist())]
    ids = t.tag_ids()
    assert ids.dtype == np.uint8 and ((ids == 0) == (tg < 0)).all()


@pytest.mark.gpu
@pytest.mark.parametrize("preset,seed", [("overload", 21), ("dynamic_increase", 22)])
def test_trace_file_to_device_step_matches_reference(tmp_path, preset, seed):
    """A trace file -> pinned columns (Trace) -> eqx_drain + eqx_step, bit-exact against the
    reference step on the same requests (roster / tags as the file defines them)."""
    from helpers import case_clients, case_kwargs, compare_step, default_model, default_profile
    from paper_2508_16646_b200 import scheduler as S
    path = tmp_path / "t.csv"
    H.ref_scenario_csv(preset, seed, 60.0, str(path))
    tr = Trace.load(str(path))
    assert tr.pinned  # the columns sit in the pinned host arena on a GPU box
    case = H.StepCase(client=tr.client, arrival=tr.arrival_s, in_tokens=tr.input_tokens, true_out=tr.output_tokens,
                      tag=tr.tag, id=np.arange(len(tr)), client_names=tr.client_names, tag_names=tr.tag_names,
                      model=default_model(), profile=default_profile(), now=float(tr.duration_s), max_batch=48)
    want = H.run_step(case, "ref")
    sch = S.GpuScheduler(case_clients(case), **case_kwargs(case))
    sch.drain(**tr.requests())
    res = sch.step(case.now)
    compare_step(res, sch, want)
    assert res.n_admitted > 0
