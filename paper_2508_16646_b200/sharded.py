"""Client-sharded scheduling step over the GPUs of one box.

The queue shards by client: every queued request of a client lives on the rank that owns the
client, so the drain (per-client FIFO order), the whole-queue scoring and each client's head
window are rank-local.  The one exchange per step is an all-gather of each rank's *exchange
record* -- per client the queue length, the trace position of its first arrival and its first W
queued requests already scored at ``now`` (include/eqx.h, ``eqx_shard_export_async``).  Every
rank then runs the identical exact selection (``eqx_shard_select_async``) over the gathered
heads with a replicated ledger, so all ranks hold the same schedule and ledger without a
second collective.  This is exact for every policy and norm mode -- including the default
``max_over_clients``, whose maxima move mid-step (scheduler.cpp:40-48) -- because the selection
is the reference's own sequential admit_requests loop (engine.cpp:207-271); a head beyond the
gathered depth is detected on the device and the step is re-run from its checkpoint deeper.

Host code here only partitions the roster, remaps client indices and moves the records
through torch.distributed (NCCL on the GPU box, gloo in the CPU tests); every per-request and
per-pick decision is made by the sm_100a kernels behind the C ABI.
"""
from __future__ import annotations

from typing import Sequence

import numpy as np

from . import _lib as L
from .scheduler import ClientState, ConfigError, EngineError, GpuScheduler, StepResult

# WinEntry (csrc/eqx_kernels.h): one scored head-of-queue request, 40 bytes.
WIN_DTYPE = np.dtype([("ufc_inc", "<f8"), ("rfc_inc", "<f8"), ("abits", "<u8"), ("in_tokens", "<i4"),
                      ("pred", "<i4"), ("row", "<i4"), ("alone", "<i4")])
assert WIN_DTYPE.itemsize == 40


def _a16(x: int) -> int:
    return (x + 15) & ~15


def rec_layout(cmax: int, window: int) -> dict:
    """Byte offsets of one rank's exchange record (mirror of rec_layout in eqx_kernels.h)."""
    count = 0
    first = _a16(4 * cmax)
    win = first + _a16(8 * cmax)
    ids = win + _a16(WIN_DTYPE.itemsize * cmax * window)
    return {"count": count, "first": first, "win": win, "id": ids, "bytes": ids + _a16(8 * cmax * window)}


def record_bytes(cmax: int, window: int) -> int:
    """eqx_shard_record_bytes (the C ABI is the authority; this mirror is checked against it)."""
    return int(L.load().eqx_shard_record_bytes(int(cmax), int(window)))


def ordered_bits_to_double(bits: np.ndarray) -> np.ndarray:
    """Inverse of the device's order-preserving double -> uint64 map (eqx_device.cuh)."""
    bits = np.asarray(bits, np.uint64)
    neg = (bits >> np.uint64(63)) == 0
    raw = np.where(neg, ~bits, bits & np.uint64(0x7FFFFFFFFFFFFFFF))
    return raw.view(np.float64)


def double_to_ordered_bits(x: np.ndarray) -> np.ndarray:
    x = np.where(np.asarray(x, np.float64) == 0.0, 0.0, x).astype(np.float64)
    b = x.view(np.uint64)
    return np.where((b >> np.uint64(63)) == 1, ~b, b | np.uint64(0x8000000000000000))


def decode_records(buf, world: int, stride: int, cmax: int, window: int) -> dict:
    """Gathered records (bytes) -> numpy views: count/first [world][cmax], win/id [world][cmax][W]."""
    raw = np.frombuffer(bytes(buf) if not isinstance(buf, np.ndarray) else buf.tobytes(), np.uint8)
    lay = rec_layout(cmax, window)
    out = {"count": [], "first": [], "win": [], "id": []}
    for r in range(world):
        base = raw[r * stride:(r + 1) * stride]
        out["count"].append(base[lay["count"]:lay["count"] + 4 * cmax].view(np.int32))
        out["first"].append(base[lay["first"]:lay["first"] + 8 * cmax].view(np.int64))
        out["win"].append(base[lay["win"]:lay["win"] + 40 * cmax * window].view(WIN_DTYPE).reshape(cmax, window))
        out["id"].append(base[lay["id"]:lay["id"] + 8 * cmax * window].view(np.int64).reshape(cmax, window))
    return {k: np.stack(v) if v else np.zeros(0) for k, v in out.items()}


def shard_owners(client_ids: Sequence[str], world: int) -> np.ndarray:
    """Owner rank of every client: contiguous blocks of the client_id byte order (the order
    select_next breaks ties in, scheduler.cpp:144-146), sizes differing by at most one."""
    n = len(client_ids)
    order = sorted(range(n), key=lambda i: (client_ids[i].encode(), i))
    sizes = [n // world + (1 if r < n % world else 0) for r in range(world)]
    owner = np.empty(n, np.int32)
    pos = 0
    for r, sz in enumerate(sizes):
        for i in order[pos:pos + sz]:
            owner[i] = r
        pos += sz
    return owner


class ShardLayout:
    """Global roster order used on the devices: clients grouped by owner rank (stable), so rank
    r's clients are the contiguous global block [off[r], off[r+1])."""

    def __init__(self, owner: np.ndarray, world: int):
        owner = np.asarray(owner, np.int32)
        if owner.size and (owner.min() < 0 or owner.max() >= world):
            raise ConfigError("client owner rank out of range")
        self.world = world
        self.owner = owner
        self.perm = np.argsort(owner, kind="stable").astype(np.int64)  # global position -> client
        self.inv = np.empty_like(self.perm)
        self.inv[self.perm] = np.arange(len(self.perm))
        sizes = np.bincount(owner, minlength=world)
        self.off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
        self.cmax = int(sizes.max()) if len(sizes) else 0

    def local_index(self, rank: int, client: np.ndarray) -> np.ndarray:
        client = np.asarray(client, np.int64)
        if client.size and np.any(self.owner[client] != rank):
            raise ConfigError(f"drain on rank {rank}: request of a client owned by another rank")
        return (self.inv[client] - self.off[rank]).astype(np.int32)


def all_gather_records(send, world: int, group=None):
    """The step's one collective: every rank's record -> [world * stride] on every rank
    (ncclAllGather over NVLink on the box; gloo with CPU tensors in the tests)."""
    import torch
    import torch.distributed as dist
    recv = torch.empty(world * send.numel(), dtype=send.dtype, device=send.device)
    if world == 1:
        recv.copy_(send)
    elif send.is_cuda and dist.get_backend(group) == "gloo":  # CPU-staged (single-GPU tests)
        host = torch.empty(world * send.numel(), dtype=send.dtype)
        dist.all_gather_into_tensor(host, send.cpu(), group=group)
        recv.copy_(host)
    else:
        dist.all_gather_into_tensor(recv, send, group=group)
    return recv


class ShardedScheduler:
    """One rank of a client-sharded scheduler (one process per GPU, torch.distributed).

    ``clients`` is the global roster (ClientState, scheduler.hpp:35-43) in the caller's order;
    events and ledgers are reported in that order.  ``owner[c]`` is the rank holding client c
    (default: contiguous client_id blocks).  The remaining keyword arguments are those of
    GpuScheduler (policy, perf, profile, predictor, model, tag_names, backfill, ...).
    """

    def __init__(self, clients: Sequence[ClientState], rank: int, world: int, owner=None, group=None,
                 running=None, window: int | None = None, device: int = 0, **kw):
        import torch
        if world > 64:
            raise ConfigError("at most 64 ranks per sharded scheduler")
        self.rank, self.world, self.group = rank, world, group
        self.client_ids = [c.client_id for c in clients]
        self.layout = ShardLayout(shard_owners(self.client_ids, world) if owner is None else owner, world)
        lay = self.layout
        run = np.zeros(len(clients), np.int32) if running is None else np.asarray(running, np.int32)
        glob = [clients[i] for i in lay.perm]
        self.sel = GpuScheduler(glob, running=run[lay.perm], device=device, **kw)
        mine = glob[lay.off[rank]:lay.off[rank + 1]]
        self.local = GpuScheduler(mine, running=run[lay.perm][lay.off[rank]:lay.off[rank + 1]],
                                  device=device, **kw)
        self.device = torch.device("cuda", device)
        self.stream = torch.cuda.Stream(self.device)  # contexts + the NCCL all-gather, in order
        self.sel.set_stream(self.stream.cuda_stream)
        self.local.set_stream(self.stream.cuda_stream)
        self.max_batch = int(self.sel.perf.max_batch)
        self.members = 0
        self.window = window
        self.retries = 0
        self._bufs: dict = {}
        self._lmap = None
        # one step per drain: shard_ingest treats every queued request as a fresh arrival (queue
        # length before = 0, counter lift in arrival order), which is the reference's state only
        # right after drain_arrivals of the whole queue (engine.cpp:171-197)
        self._drained = False

    def set_batch(self, members: int, reserved_kv_tokens: int) -> None:
        self.members = int(members)
        self.sel.set_batch(members, reserved_kv_tokens)

    def drain(self, client, arrival_s, input_tokens, tag=None, true_output_tokens=None, ids=None,
              local: bool = False) -> None:
        """Queue this rank's arrivals (every request of a client this rank owns; ``ids`` are the
        global trace positions).  ``client`` holds caller roster indices, or local indices of
        this rank's block when ``local`` is set (the resident-queue fast path)."""
        if ids is None:
            raise ConfigError("sharded drain needs the global trace ids (arrival order across ranks)")
        if not local:
            if type(client).__module__.startswith("torch"):
                import torch
                if self._lmap is None:
                    lm = np.full(len(self.client_ids), -1, np.int64)
                    lo, hi = self.layout.off[self.rank], self.layout.off[self.rank + 1]
                    lm[self.layout.perm[lo:hi]] = np.arange(hi - lo)
                    self._lmap = torch.from_numpy(lm).to(client.device)
                client = self._lmap[client.long()].int()
            else:
                client = self.layout.local_index(self.rank, client)
        self.local.drain(client, arrival_s, input_tokens, tag=tag, true_output_tokens=true_output_tokens,
                         ids=ids)
        self._drained = True

    def _buf(self, name: str, nbytes: int):
        import torch
        b = self._bufs.get(name)
        if b is None or b.numel() < nbytes:
            with torch.cuda.stream(self.stream):
                b = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            self._bufs[name] = b
        return b[:nbytes]

    def step_async(self, now: float, window: int) -> None:
        """Export -> all-gather -> selection, all enqueued on the shared stream.  Exactly one
        step per drain (the sharded step treats the drained queue as fresh arrivals)."""
        if not self._drained:
            raise EngineError("sharded step without a drain: ShardedScheduler runs one step per drain of the "
                              "rank's whole queue")
        self._drained = False
        stride = _a16(record_bytes(self.layout.cmax, window))
        send = self._buf("send", stride)
        self.local.shard_export_async(now, self.layout.cmax, window, send)
        import torch
        with torch.cuda.stream(self.stream):
            recv = all_gather_records(send, self.world, self.group)
        self._bufs["recv_keep"] = recv
        self.sel.shard_select_async(recv, self.world, stride, self.layout.off, self.layout.cmax, window, now)

    def default_window(self) -> int:
        """Head-window depth exchanged per client: small by default (a client rarely takes more
        than a few of the free slots when many clients are backlogged), grown 4x after an
        underflow and kept; the depth never exceeds free slots + 1, which is always exact without
        rejection streams."""
        free = max(0, self.max_batch - self.members)
        if self.window:
            return min(self.window, free + 1) if free else 1
        return max(1, min(free + 1, 8))

    def step(self, now: float, window: int | None = None, with_events: bool = True) -> StepResult:
        """One exact scheduling step over the whole sharded queue; identical on every rank."""
        if not self._drained:
            raise EngineError("sharded step without a drain: ShardedScheduler runs one step per drain of the "
                              "rank's whole queue")
        W = window or self.default_window()
        self.sel.checkpoint()
        while True:
            self._drained = True  # a retry re-runs the same drained step from its checkpoint
            self.step_async(now, W)
            res = self.sel.collect(with_events=with_events)
            if not res.window_underflow:
                break
            # a client needed a head beyond the gathered windows (a rejection stream or more
            # admissions than W - 1): re-run from the checkpoint with deeper windows
            self.retries += 1
            self.sel.restore_async()
            W *= 4
        if window is None and W > self.default_window():
            self.window = W  # keep the depth that sufficed for the next steps
        res.clients = self.layout.perm[res.clients].astype(np.int32) if len(res.clients) else res.clients
        return res

    def ledger(self) -> dict:
        led = self.sel.ledger()
        return {k: v[self.layout.inv] for k, v in led.items()}

    def scores(self) -> dict:
        """Per-request scores of this rank's queue (drain order of its requests)."""
        return self.local.scores()

    def close(self) -> None:
        self.sel.close()
        self.local.close()
