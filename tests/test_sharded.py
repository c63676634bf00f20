"""Client-sharded step.

CPU (no GPU): the record layout mirror agrees with the C ABI, the roster partition, and a
world-size-2 gloo run of the exchange -- each rank encodes its clients' records (test-side
numpy encoder over the oracle's per-request scores), all-gathers them, and every rank decodes
the same global head view that the unsharded queue has.

GPU: `world` ranks simulated on one B200 -- one local context per shard drains and exports its
clients' records into its slice of the gathered buffer (exactly what the all-gather produces),
one selection context runs the exact step over the gathered heads -- bit-exact against the
oracle of the *unsharded* queue: ids/order/kinds, FP64 ledger (counter lift in global arrival
order) and every per-request score.
"""
import os
import socket

import numpy as np
import pytest

import harness as H
from helpers import (case_batch, compare_flagged, case_clients, case_columns, case_from_golden, case_kwargs, default_model,
                     default_profile, golden_names, load_golden)
from paper_2508_16646_b200 import sharded as SH
from paper_2508_16646_b200 import workload as W


# ---------------------------------------------------------------------------------- CPU ----
def test_record_layout_matches_c_abi():
    for cmax, w in [(0, 1), (1, 1), (3, 5), (64, 65), (1250, 65), (7, 4097)]:
        assert SH.record_bytes(cmax, w) == SH.rec_layout(cmax, w)["bytes"]
        assert SH.rec_layout(cmax, w)["bytes"] % 16 == 0
    assert SH.record_bytes(4, 0) == -1


def test_shard_owners_are_contiguous_name_blocks():
    names = [f"client{i}" for i in range(37)]  # bytewise order: client0, client1, client10, ...
    for world in (1, 2, 3, 8):
        owner = SH.shard_owners(names, world)
        order = sorted(range(len(names)), key=lambda i: names[i].encode())
        assert list(owner[order]) == sorted(owner[order])  # blocks follow the byte order
        sizes = np.bincount(owner, minlength=world)
        assert sizes.max() - sizes.min() <= 1
        lay = SH.ShardLayout(owner, world)
        assert lay.off[-1] == len(names) and lay.cmax == sizes.max()
        for r in range(world):
            blk = lay.perm[lay.off[r]:lay.off[r + 1]]
            assert np.all(owner[blk] == r)
            np.testing.assert_array_equal(lay.local_index(r, blk), np.arange(len(blk)))
    with pytest.raises(SH.ConfigError):
        SH.ShardLayout(SH.shard_owners(names, 2), 2).local_index(0, np.array([order[-1]]))


def test_ordered_bits_roundtrip():
    x = np.array([0.0, -0.0, 1.0, -1.0, 1e-300, 3.5, np.inf, -np.inf])
    b = SH.double_to_ordered_bits(x)
    back = SH.ordered_bits_to_double(b)
    np.testing.assert_array_equal(back, np.where(x == 0.0, 0.0, x))
    assert np.all(np.diff(SH.double_to_ordered_bits(np.sort(x[2:]))).astype(np.int64) != 0)


def encode_record(case, want, lay, rank, window):
    """Test-side numpy encoder of one rank's exchange record (the device's shard_export_kernel
    restated over the oracle's per-request scores)."""
    cmax = lay.cmax
    L = SH.rec_layout(cmax, window)
    buf = np.zeros(_stride(cmax, window), np.uint8)
    count = buf[L["count"]:L["count"] + 4 * cmax].view(np.int32)
    first = buf[L["first"]:L["first"] + 8 * cmax].view(np.int64)
    win = buf[L["win"]:L["win"] + 40 * cmax * window].view(SH.WIN_DTYPE).reshape(cmax, window)
    ids = buf[L["id"]:L["id"] + 8 * cmax * window].view(np.int64).reshape(cmax, window)
    first[:] = np.iinfo(np.int64).max
    client = np.asarray(case.client)
    tmax_ok = lambda t: float(t) * case.mem_per_token_bytes <= case.mem_capacity_bytes  # noqa: E731
    for l, g in enumerate(range(lay.off[rank], lay.off[rank + 1])):
        rows = np.nonzero(client == lay.perm[g])[0]
        count[l] = len(rows)
        if len(rows):
            first[l] = case.id[rows[0]]
        for k, row in enumerate(rows[:window]):
            win[l, k] = (want["ufc_inc"][row], want["rfc_inc"][row],
                         SH.double_to_ordered_bits(np.array([case.arrival[row]]))[0], case.in_tokens[row],
                         want["pred"][row], -1, int(case.max_batch >= 1 and tmax_ok(case.in_tokens[row] +
                                                                                      want["pred"][row])))
            ids[l, k] = case.id[row]
    return buf


def _stride(cmax, window):
    return (SH.rec_layout(cmax, window)["bytes"] + 15) & ~15


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        case = _exchange_case()
        want = H.run_step(case, "oracle")
        lay = SH.ShardLayout(SH.shard_owners(case.client_names, world), world)
        window = 5
        send = torch.from_numpy(encode_record(case, want, lay, rank, window))
        recv = SH.all_gather_records(send, world)
        q.put((rank, recv.numpy().tobytes()))
    finally:
        dist.destroy_process_group()


def _exchange_case():
    q = W.lmsys_queue(3000, 11, seed=4, heavy_frac=0.5)
    return H.StepCase(client=q["client"], arrival=q["arrival"], in_tokens=q["in_tokens"], true_out=q["true_out"],
                      tag=q["tag"], client_names=q["client_names"], model=default_model(), profile=default_profile())


def test_gloo_world2_record_exchange():
    """world_size 2 over gloo: every rank ends with the same gathered buffer, and decoding it
    gives the unsharded queue's per-client lengths, first arrivals and first-W heads."""
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    assert got[0] == got[1]
    case = _exchange_case()
    want = H.run_step(case, "oracle")
    lay = SH.ShardLayout(SH.shard_owners(case.client_names, world), world)
    window = 5
    dec = SH.decode_records(np.frombuffer(got[0], np.uint8), world, _stride(lay.cmax, window), lay.cmax, window)
    client = np.asarray(case.client)
    for g in range(len(case.client_names)):
        r = int(np.searchsorted(lay.off, g, side="right") - 1)
        l = g - lay.off[r]
        rows = np.nonzero(client == lay.perm[g])[0]
        assert dec["count"][r, l] == len(rows)
        assert dec["first"][r, l] == (rows[0] if len(rows) else np.iinfo(np.int64).max)
        k = min(window, len(rows))
        np.testing.assert_array_equal(dec["id"][r, l, :k], case.id[rows[:k]])
        np.testing.assert_array_equal(dec["win"][r, l, :k]["pred"], want["pred"][rows[:k]])
        np.testing.assert_array_equal(dec["win"][r, l, :k]["ufc_inc"], want["ufc_inc"][rows[:k]])
        np.testing.assert_array_equal(SH.ordered_bits_to_double(dec["win"][r, l, :k]["abits"]),
                                      case.arrival[rows[:k]])


# ---------------------------------------------------------------------------------- GPU ----
def sharded_sim(case, world, window=None, owner=None, device_columns=False):
    """`world` ranks on one GPU: per-shard contexts export into their slice of the gathered
    buffer; one selection context runs the step.  Returns (events, ledger in caller order,
    per-request scores in row order, retries)."""
    import torch
    from paper_2508_16646_b200.scheduler import GpuScheduler
    clients = case_clients(case)
    kw = case_kwargs(case)
    lay = SH.ShardLayout(SH.shard_owners(case.client_names, world) if owner is None else owner, world)
    ts = torch.cuda.Stream()
    stream = ts.cuda_stream
    running = np.asarray(case.running, np.int32)
    sel = GpuScheduler([clients[i] for i in lay.perm], running=running[lay.perm], **kw)
    sel.set_stream(stream)
    members, reserved = case_batch(case)
    sel.set_batch(members, reserved)
    cols = case_columns(case)
    owner_of_row = lay.owner[cols["client"]] if len(cols["client"]) else np.zeros(0, np.int32)
    locs, rows_of = [], []
    for r in range(world):
        blk = lay.perm[lay.off[r]:lay.off[r + 1]]
        loc = GpuScheduler([clients[i] for i in blk], running=running[blk], **kw)
        loc.set_stream(stream)
        rows = np.nonzero(owner_of_row == r)[0]
        c = {k: v[rows] for k, v in cols.items()}
        c["client"] = lay.local_index(r, c["client"])
        if device_columns:
            c = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in c.items()}
            torch.cuda.synchronize()
        loc.drain(**c)
        locs.append(loc)
        rows_of.append(rows)
    Wd = window or max(1, min(case.max_batch - members, 64) + 1)
    sel.checkpoint()
    retries = 0
    while True:
        stride = _stride(lay.cmax, Wd)
        with torch.cuda.stream(ts):
            recv = torch.empty(world * stride, dtype=torch.uint8, device="cuda")
        for r, loc in enumerate(locs):
            loc.shard_export_async(case.now, lay.cmax, Wd, recv[r * stride:(r + 1) * stride])
        sel.shard_select_async(recv, world, stride, lay.off, lay.cmax, Wd, case.now)
        res = sel.collect()
        if not res.window_underflow:
            break
        retries += 1
        sel.restore_async()
        Wd *= 4
    res.clients = lay.perm[res.clients].astype(np.int32) if len(res.clients) else res.clients
    led = {k: v[lay.inv] for k, v in sel.ledger().items()}
    n = len(cols["client"])
    sc = {"pred": np.zeros(n, np.int32), "bucket": np.zeros(n, np.int32), "ufc_inc": np.zeros(n),
          "rfc_inc": np.zeros(n)}
    for loc, rows in zip(locs, rows_of):
        if len(rows):
            s = loc.scores()
            for k in sc:
                sc[k][rows] = s[k]
    return res, led, sc, retries


def compare_sharded(res, led, sc, want):
    np.testing.assert_array_equal(res.ids, want["ev_id"], err_msg="event ids / order")
    np.testing.assert_array_equal(res.kinds, want["ev_kind"], err_msg="event kinds")
    np.testing.assert_array_equal(res.clients, want["ev_client"])
    adm = want["ev_kind"] == H.EV_ADMIT
    for k in ("ufc_inc", "rfc_inc", "vtc_inc"):
        np.testing.assert_array_equal(getattr(res, k)[adm], want["ev_" + k][adm], err_msg=k)
    np.testing.assert_array_equal(res.wait_s[adm], want["ev_wait"][adm])
    assert res.n_admitted == want["n_admitted"] and res.n_rejected == want["n_rejected"]
    assert res.new_prefill_tokens == want["new_prefill"]
    for k in ("ufc", "rfc", "counter", "backlogged"):
        np.testing.assert_array_equal(led[k], want[k], err_msg="ledger " + k)
    for k in ("pred", "bucket", "ufc_inc", "rfc_inc"):
        np.testing.assert_array_equal(sc[k], want[k], err_msg=k)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", golden_names())
def test_sharded_golden(name, world):
    meta, ins, outs = load_golden(name)
    case = case_from_golden(meta, ins)
    res, led, sc, _ = sharded_sim(case, world)
    if res.noisy_near_ties and compare_flagged(res, sc, outs, res.noisy_near_ties, case.id):
        return
    compare_sharded(res, led, sc, outs)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(16))
def test_sharded_random_vs_oracle(seed):
    from test_gpu_parity import _random_case
    rng = np.random.default_rng(5000 + seed)
    C = int(rng.choice([2, 9, 64, 300, 1300]))
    n = int(rng.integers(0, 40000))
    world = int(rng.choice([2, 4, 8]))
    case = _random_case(seed, n, C)
    want = H.run_step(case, "oracle")
    owner = rng.integers(0, world, C).astype(np.int32) if seed % 4 == 1 else None  # arbitrary ownership
    res, led, sc, _ = sharded_sim(case, world, owner=owner, window=int(rng.choice([1, 2, 8])) if seed % 2 else None)
    compare_sharded(res, led, sc, want)


@pytest.mark.gpu
def test_sharded_underflow_retry_is_exact():
    """A window of 1 must underflow on any client picked twice; the retry stays exact."""
    meta, ins, outs = load_golden("reject_stream")
    case = case_from_golden(meta, ins)
    res, led, sc, retries = sharded_sim(case, 2, window=1)
    assert retries >= 1
    compare_sharded(res, led, sc, outs)


@pytest.mark.gpu
@pytest.mark.slow
def test_sharded_cfg4_shape_vs_oracle():
    """cfg4's per-GPU shape on a simulated 8-way split: 2M requests over 1,250 clients here
    (16M / 10k over 8 GPUs), device-resident columns, warm ledger."""
    q = W.lmsys_queue(2_000_000, 1250, seed=11)
    led0 = W.warm_ledger(1250, seed=12)
    case = H.StepCase(client=q["client"], arrival=q["arrival"], in_tokens=q["in_tokens"], true_out=q["true_out"],
                      tag=q["tag"], client_names=q["client_names"], model=default_model(),
                      profile=default_profile(), ufc0=led0["ufc"], rfc0=led0["rfc"], counter0=led0["counter"])
    res, led, sc, _ = sharded_sim(case, 8, device_columns=True)
    for which in (["ref", "oracle"] if H.available("ref") else ["oracle"]):
        compare_sharded(res, led, sc, H.run_step(case, which))
    assert res.n_admitted == 64


@pytest.mark.gpu
@pytest.mark.slow
def test_sharded_cfg4_global_shape_vs_reference():
    """BASELINE configs[3] at its global shape: 16M queued requests over 10,000 clients,
    client-sharded 8 ways (2M / 1,250 per rank) as 8 simulated ranks on this GPU, against the
    reference's own step (oracle/_ref) over the unsharded 16M queue.  Every rank's replicated
    selection runs over the gathered heads of all 10k clients, as on an 8-GPU box."""
    if not H.available("ref"):
        pytest.skip("reference build not present")
    q = W.lmsys_queue(16_000_000, 10_000, seed=13)
    led0 = W.warm_ledger(10_000, seed=14)
    case = H.StepCase(client=q["client"], arrival=q["arrival"], in_tokens=q["in_tokens"], true_out=q["true_out"],
                      tag=q["tag"], client_names=q["client_names"], model=default_model(),
                      profile=default_profile(), ufc0=led0["ufc"], rfc0=led0["rfc"], counter0=led0["counter"])
    res, led, sc, retries = sharded_sim(case, 8, device_columns=True)
    compare_sharded(res, led, sc, H.run_step(case, "ref"))
    assert res.n_admitted == 64


def _gpu_gloo_worker(rank, world, port, q, seed):
    """One rank of a real two-process sharded step on cuda:0 (gloo: the exchange is staged
    through the host): ShardedScheduler drains this rank's clients, exports its record with
    shard_export_kernel, all-gathers it with the other process and runs the replicated selection."""
    import sys
    sys.path[:0] = [os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), d) for d in ("", "oracle", "tests")]
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2508_16646_b200.sharded import ShardedScheduler
        from test_gpu_parity import _random_case
        case = _random_case(seed, 20000, 50 + seed)
        case.finalize()
        kw = case_kwargs(case)
        sch = ShardedScheduler(case_clients(case), rank, world, running=case.running, device=0, **kw)
        sch.set_batch(*case_batch(case))
        cols = case_columns(case)
        owner = sch.layout.owner[cols["client"]]
        rows = np.nonzero(owner == rank)[0]
        sch.drain(**{k: v[rows] for k, v in cols.items()})
        res = sch.step(case.now)
        led = sch.ledger()
        q.put((rank, res.ids.tolist(), res.kinds.tolist(), res.clients.tolist(), res.ufc_inc.tolist(),
               {k: led[k].tolist() for k in ("ufc", "rfc", "counter", "backlogged")}, sch.retries))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [1, 2])
def test_two_process_sharded_step_on_one_gpu(seed):
    """The multi-process path of bench.py --gpus N with real kernels: two processes on cuda:0,
    each exporting its shard with shard_export_kernel, exchanged through torch.distributed
    (gloo; NCCL needs distinct GPUs), identical schedules on both ranks, bit-exact against the
    oracle of the unsharded queue, with the adaptive head-window depth (8, grown on underflow)."""
    import torch.multiprocessing as mp
    from test_gpu_parity import _random_case
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gpu_gloo_worker, args=(r, world, port, q, seed)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict((r[0], r[1:]) for r in (q.get(timeout=300) for _ in range(world)))
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert got[0][:5] == got[1][:5]  # identical schedule and ledger on both ranks
    case = _random_case(seed, 20000, 50 + seed)
    want = H.run_step(case, "oracle")
    ids, kinds, clients, ufc_inc, led, _ = got[0]
    np.testing.assert_array_equal(ids, want["ev_id"])
    np.testing.assert_array_equal(kinds, want["ev_kind"])
    np.testing.assert_array_equal(clients, want["ev_client"])
    adm = want["ev_kind"] == H.EV_ADMIT
    np.testing.assert_array_equal(np.asarray(ufc_inc)[adm], want["ev_ufc_inc"][adm])
    for k in ("ufc", "rfc", "counter", "backlogged"):
        np.testing.assert_array_equal(led[k], want[k], err_msg=k)
