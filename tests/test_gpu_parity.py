"""GPU parity: the sm_100a path (through the C ABI) against the reference-generated goldens
and the C restatement, bit-exact (ids/order/kinds exact; FP64 ledger and increments exact,
which is stricter than the north star's 1e-5 relative)."""
import numpy as np
import pytest

import harness as H
from helpers import (case_columns, case_from_golden, compare_step, default_model, default_profile, golden_names,
                     gpu_run, load_golden)
from paper_2508_16646_b200 import workload as W

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", golden_names())
def test_golden_step(name):
    meta, ins, outs = load_golden(name)
    case = case_from_golden(meta, ins)
    sch, res = gpu_run(case)
    compare_step(res, sch, outs, flagged_near_ties=res.noisy_near_ties, row_ids=case.id)


def test_golden_step_device_columns():
    """Zero-copy drain of torch CUDA tensors (the resident-queue path the bench times)."""
    meta, ins, outs = load_golden("eqx_max_warm")
    sch, res = gpu_run(case_from_golden(meta, ins), device_columns=True)
    compare_step(res, sch, outs)


def _random_case(seed, n, C, **over):
    rng = np.random.default_rng(seed)
    q = W.lmsys_queue(n, C, seed=seed, untagged_frac=0.02, heavy_frac=0.5 if seed % 3 == 0 else None)
    led = W.warm_ledger(C, seed=seed + 1)
    kw = dict(kind=int(rng.integers(0, 3)), norm_mode=int(rng.integers(0, 2)),
              vtc_use_prediction=bool(rng.integers(0, 2)), backfill=bool(rng.integers(0, 2)),
              max_batch=int(rng.choice([8, 64, 300, 4096])), pred_kind=int(rng.choice([0, 1, 1, 3])),
              mem_per_token_bytes=float(rng.choice([1.0, 0.5 * 1024 * 1024])),
              alpha=float(rng.choice([0.0, 0.3, 0.7, 1.0])), delta=float(rng.choice([0.0, 0.1, 2.0])))
    kw["mem_capacity_bytes"] = (float(rng.choice([800.0, 4000.0, 30000.0])) if kw["mem_per_token_bytes"] == 1.0
                                else 60.0 * 1024 ** 3)
    kw.update(over)
    warm = rng.integers(0, 2)
    return H.StepCase(client=q["client"], arrival=q["arrival"], in_tokens=q["in_tokens"], true_out=q["true_out"],
                      tag=q["tag"], client_names=q["client_names"], model=default_model(), profile=default_profile(),
                      ufc0=led["ufc"] * warm, rfc0=led["rfc"] * warm, counter0=led["counter"] * warm,
                      weight=rng.choice([0.5, 1.0, 2.0], C), **kw)


@pytest.mark.parametrize("seed", range(24))
def test_random_steps_vs_oracle(seed):
    rng = np.random.default_rng(1000 + seed)
    C = int(rng.choice([1, 5, 31, 64, 200, 777, 1500, 3000]))
    n = int(rng.integers(0, 60000))
    case = _random_case(seed, n, C)
    want = H.run_step(case, "oracle")
    sch, res = gpu_run(case)
    compare_step(res, sch, want)


@pytest.mark.parametrize("C", [33, 48, 64, 65, 100, 128])
@pytest.mark.parametrize("seed", range(3))
def test_multiwarp_selection_rosters_vs_oracle(C, seed):
    """Rosters of 33..128 clients take the multi-warp selection (one client per lane, warp winners
    exchanged through shared memory); every policy mix of _random_case, bit-exact."""
    rng = np.random.default_rng(5000 + 10 * C + seed)
    case = _random_case(7000 + 10 * C + seed, int(rng.integers(2000, 40000)), C)
    want = H.run_step(case, "oracle")
    sch, res = gpu_run(case)
    compare_step(res, sch, want)


def _full_size_oracles():
    """Full-size checks are pinned to the reference itself (oracle/_ref, the reference's own
    sources compiled here, drain_arrivals + admit_requests through its objects) and to the C
    restatement."""
    return ["ref", "oracle"] if H.available("ref") else ["oracle"]


@pytest.mark.slow
def test_cfg2_full_size_vs_oracle():
    """BASELINE configs[1]: 1M queued requests, 64 clients, MoPE, warm ledger, max_batch 64."""
    q = W.lmsys_queue(1_000_000, 64, seed=1)
    led = W.warm_ledger(64, seed=2)
    case = H.StepCase(client=q["client"], arrival=q["arrival"], in_tokens=q["in_tokens"], true_out=q["true_out"],
                      tag=q["tag"], client_names=q["client_names"], model=default_model(),
                      profile=default_profile(), ufc0=led["ufc"], rfc0=led["rfc"], counter0=led["counter"])
    sch, res = gpu_run(case, device_columns=True)
    for which in _full_size_oracles():
        compare_step(res, sch, H.run_step(case, which))
    assert res.n_admitted == 64


@pytest.mark.slow
@pytest.mark.parametrize("backfill", [False, True])
def test_cfg3_heavy_hitter_vs_oracle(backfill):
    """configs[2]: 1k clients, client 0 sends 50%, max_batch 4096 -> the KV budget cuts."""
    q = W.lmsys_queue(1_000_000, 1000, seed=3, heavy_frac=0.5)
    case = H.StepCase(client=q["client"], arrival=q["arrival"], in_tokens=q["in_tokens"], true_out=q["true_out"],
                      tag=q["tag"], client_names=q["client_names"], model=default_model(),
                      profile=default_profile(), max_batch=4096, backfill=backfill)
    sch, res = gpu_run(case, device_columns=True)
    for which in _full_size_oracles():
        compare_step(res, sch, H.run_step(case, which))
    # size-independent properties: the KV reservation never exceeds the budget
    assert res.batch_reserved_kv_tokens * case.mem_per_token_bytes <= case.mem_capacity_bytes


def test_scalar_helpers_and_errors():
    from paper_2508_16646_b200 import scheduler as S
    assert S.ufc_increment(1.0, 100, 400) == 1700.0
    assert S.ufc_increment(1.0, 100, 400, 5.0, 5000.0) == 850.0
    assert S.rfc_increment(1.0, 1000.0, 0.9) == 900.0
    prof = S.GpuProfile([S.ProfileEntry(32, 1.0, 0.5, 100.0)])
    with pytest.raises(S.ConfigError, match="alpha"):
        S.GpuScheduler([S.ClientState("a")], policy=S.PolicySpec(equinox=S.EquinoxParams(alpha=1.2)),
                       profile=prof, predictor="oracle")
    with pytest.raises(S.ConfigError, match="non-positive weight"):
        S.GpuScheduler([S.ClientState("a", weight=0.0)], profile=prof, predictor="oracle")
    with pytest.raises(S.ConfigError, match="non-empty GPU profile"):
        S.GpuScheduler([S.ClientState("a")], profile=S.GpuProfile([]), predictor="oracle")


def test_staged_host_batches_in_order():
    """eqx_stage_async: two host batches staged ahead on the copy stream are consumed by the
    drains of the same arrays, oldest first, with results identical to unstaged drains."""
    import torch
    from helpers import case_batch, case_clients, case_columns, case_kwargs
    from paper_2508_16646_b200 import scheduler as S
    c0 = _random_case(41, 20000, 64, kind=2, norm_mode=0, backfill=False)
    same = {k: getattr(c0, k) for k in ("vtc_use_prediction", "max_batch", "pred_kind", "mem_per_token_bytes",
                                        "mem_capacity_bytes", "alpha", "delta")}
    cases = [c0, _random_case(42, 20000, 64, kind=2, norm_mode=0, backfill=False, **same)]
    wants = [H.run_step(c, "oracle") for c in cases]
    sch = S.GpuScheduler(case_clients(cases[0]), running=cases[0].running, **case_kwargs(cases[0]))
    cols = [{k: torch.from_numpy(v).pin_memory() for k, v in case_columns(c).items()} for c in cases]
    for rnd in range(2):
        for c in cols:
            sch.stage_async(**c)
        for c, case, want in zip(cols, cases, wants):
            sch.set_clients(case_clients(case), case.running)
            sch.set_batch(*case_batch(case))
            sch.drain(**c)
            res = sch.step(case.now)
            compare_step(res, sch, want)


def test_narrow_host_columns_staged_and_unstaged():
    """uint16 client / input_tokens host columns (eqx_requests::narrow: 13 B per request over
    PCIe, widened on the copy stream) give the same step as the i32 columns, staged ahead, staged
    by the drain itself, and through the graph path."""
    from helpers import case_batch, case_clients, case_kwargs
    from paper_2508_16646_b200 import scheduler as S
    for seed, C in ((51, 64), (52, 1000), (53, 5)):
        case = _random_case(seed, 30011, C)
        want = H.run_step(case, "oracle")
        cols = case_columns(case)
        cols["client"] = cols["client"].astype(np.uint16)
        cols["input_tokens"] = cols["input_tokens"].astype(np.uint16)
        pinned = {k: S.pinned_copy(v) for k, v in cols.items()}
        for mode in ("plain", "staged", "graph"):
            sch = S.GpuScheduler(case_clients(case), running=case.running, **case_kwargs(case))
            sch.set_batch(*case_batch(case))
            src = cols if mode == "plain" else pinned
            if mode == "staged":
                sch.stage_async(**src)
            if mode == "graph":
                sch.checkpoint()
                for _ in range(2):
                    sch.restore_async()
                    sch.stage_async(**src)
                    sch.drain_step_async(case.now, **src)
                    res = sch.collect(with_events=True)
            else:
                sch.drain(**src)
                res = sch.step(case.now)
            compare_step(res, sch, want)


@pytest.mark.parametrize("narrow", [False, True])
def test_packed_arrival_host_columns(narrow):
    """Packed arrivals (eqx_pack_arrivals, eqx_requests::narrow & EQX_PACKED_ARRIVALS: ~6 B per
    request over PCIe, unpacked on the copy stream) give the same step as the doubles, with and
    without the uint16 columns, unstaged, staged and through the graph path.  The random queues
    start near zero, so their first blocks are stored raw and the rest packed; one case shifts
    the arrivals far from zero (every block packed), one draws them sparse (every block raw)."""
    from helpers import case_batch, case_clients, case_kwargs
    from paper_2508_16646_b200 import scheduler as S
    for seed, C, shift, sparse in ((61, 64, 0.0, False), (62, 1000, 1000.0, False), (63, 5, 0.0, True)):
        case = _random_case(seed, 30011, C)
        if sparse:
            case.arrival = np.sort(np.random.default_rng(seed).uniform(0.0, 1e6, len(case.arrival)))
        case.arrival = case.arrival + shift
        want = H.run_step(case, "oracle")
        cols = case_columns(case)
        if narrow:
            cols["client"] = cols["client"].astype(np.uint16)
            cols["input_tokens"] = cols["input_tokens"].astype(np.uint16)
        cols["arrival_s"] = S.pack_arrivals(cols["arrival_s"])
        pinned = {k: S.pinned_copy(v) for k, v in cols.items()}
        for mode in ("plain", "staged", "graph"):
            sch = S.GpuScheduler(case_clients(case), running=case.running, **case_kwargs(case))
            sch.set_batch(*case_batch(case))
            src = cols if mode == "plain" else pinned
            if mode == "staged":
                sch.stage_async(**src)
            if mode == "graph":
                sch.checkpoint()
                for _ in range(2):
                    sch.restore_async()
                    sch.stage_async(**src)
                    sch.drain_step_async(case.now, **src)
                    res = sch.collect(with_events=True)
            else:
                sch.drain(**src)
                res = sch.step(case.now)
            compare_step(res, sch, want)


def test_packed_arrivals_rejects_corrupt_header():
    """A packed column whose header points outside itself is refused before any device read."""
    from helpers import case_batch, case_clients, case_kwargs
    from paper_2508_16646_b200 import scheduler as S
    case = _random_case(64, 5000, 8)
    H.run_step(case, "oracle")  # finalizes the case
    cols = case_columns(case)
    pk = S.pack_arrivals(cols["arrival_s"])
    nb = (len(cols["arrival_s"]) + 255) // 256
    bad = pk.data.copy()
    bad[8 + 8 * nb:16 + 8 * nb] = np.frombuffer(np.int64(1 << 40).tobytes(), np.uint8)  # block 0 offset
    cols["arrival_s"] = S.PackedArrivals(bad, pk.n)
    sch = S.GpuScheduler(case_clients(case), running=case.running, **case_kwargs(case))
    sch.set_batch(*case_batch(case))
    with pytest.raises(ValueError):
        sch.drain(**cols)


def _graph_step(case, device_columns: bool, staged: bool = False, reps: int = 2):
    """The path bench.py times: eqx_drain_step_async (one CUDA-graph replay of drain, windows
    with the counter lift, scoring and selection), repeated on the restored ledger so the cached
    graph is replayed, then eqx_step_collect."""
    import torch
    from helpers import case_batch, case_clients, case_columns, case_kwargs
    from paper_2508_16646_b200 import scheduler as S
    sch = S.GpuScheduler(case_clients(case), running=case.running, **case_kwargs(case))
    sch.set_batch(*case_batch(case))
    sch.checkpoint()
    cols = case_columns(case)
    if device_columns:
        cols = {k: torch.from_numpy(v).cuda() for k, v in cols.items()}
    elif staged:
        cols = {k: S.pinned_copy(v) for k, v in cols.items()}
    res = None
    for _ in range(reps):
        sch.restore_async()
        if staged:
            sch.stage_async(**cols)
        sch.drain_step_async(case.now, **cols)
        res = sch.collect(with_events=True)
    return sch, res


@pytest.mark.parametrize("name", golden_names())
def test_golden_graph_step(name):
    """Every golden through the graph path with resident device columns."""
    meta, ins, outs = load_golden(name)
    case = case_from_golden(meta, ins)
    sch, res = _graph_step(case, device_columns=True)
    compare_step(res, sch, outs, flagged_near_ties=res.noisy_near_ties, row_ids=case.id)


@pytest.mark.parametrize("seed", range(8))
def test_random_graph_steps_vs_oracle(seed):
    """Random policies / rosters (with running clients and warm ledgers, so the counter lift in
    the window kernel's extra CTA has work) through the graph path, host columns staged from the
    pinned arena on even seeds, device columns on odd ones."""
    rng = np.random.default_rng(9000 + seed)
    C = int(rng.choice([5, 31, 64, 100, 200, 777]))
    case = _random_case(9100 + seed, int(rng.integers(1000, 50000)), C)
    case.finalize()
    case.running = (rng.random(C) < 0.3).astype(np.int32) * rng.integers(0, 3, C).astype(np.int32)
    want = H.run_step(case, "oracle")
    sch, res = _graph_step(case, device_columns=bool(seed % 2), staged=not seed % 2)
    compare_step(res, sch, want)
