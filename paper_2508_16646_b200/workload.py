"""Synthetic queued-request workloads for the scheduling step (host-side fixture data).

The reference ships no LMSYS/ShareGPT files and this box has no network, so the configs of
BASELINE.json are builder-defined shapes built from the reference's own
prediction-corpus mixture (workload.cpp:430-476: three latent classes with output ranges
[4,52] / [53,209] / [210,1500] and input ranges [8,96] / [64,320] / [192,1024]) and its tag
assignment rule (workload.cpp:179-200: bucket by the 33rd/66th output percentiles, flipped
to a different bucket with probability ``tag_noise``).  Draws use numpy's PCG64 seeded by
``seed``; arrays are identical for identical arguments on every host.

Everything here is plain data preparation (numpy), not part of the device hot path.
"""
from __future__ import annotations

import numpy as np

TAG_NAMES = ["short", "medium", "long"]


def _nearest_rank(sorted_vals: np.ndarray, pct: float) -> int:
    """workload.cpp:154-160 percentile_nearest_rank."""
    n = len(sorted_vals)
    rank = int(np.ceil(pct / 100.0 * float(n)))
    rank = min(max(rank, 1), n)
    return int(sorted_vals[rank - 1])


def assign_category_tags(true_out: np.ndarray, rng: np.random.Generator, noise: float) -> np.ndarray:
    """workload.cpp:179-200 assign_category_tags -> tag index into TAG_NAMES."""
    if len(true_out) == 0:
        return np.zeros(0, np.int32)
    s = np.sort(true_out)
    b1, b2 = _nearest_rank(s, 33.0), _nearest_rank(s, 66.0)
    bucket = np.where(true_out <= b1, 0, np.where(true_out <= b2, 1, 2)).astype(np.int32)
    flip = rng.random(len(true_out)) < noise
    offset = 1 + rng.integers(0, 2, len(true_out))
    return np.where(flip, (bucket + offset) % 3, bucket).astype(np.int32)


def lmsys_queue(n: int, n_clients: int, seed: int = 1, heavy_frac: float | None = None,
                tag_noise: float = 0.2, untagged_frac: float = 0.0) -> dict:
    """One arrival-ordered queue of ``n`` requests over ``n_clients`` clients.

    cfg2: ``lmsys_queue(1_000_000, 64)``; cfg3: ``lmsys_queue(1_000_000, 1000, heavy_frac=0.5)``
    (client 0 sends ``heavy_frac`` of the load, the rest share the remainder uniformly).
    Arrival of request i is i/n seconds, so a step at now=1.0 drains the whole queue.
    """
    rng = np.random.default_rng(seed)
    if heavy_frac is not None and n_clients > 1:
        heavy = rng.random(n) < heavy_frac
        client = np.where(heavy, 0, rng.integers(1, n_clients, n)).astype(np.int32)
    else:
        client = rng.integers(0, n_clients, n).astype(np.int32)
    cls = rng.integers(0, 3, n)
    lo_out, hi_out = np.array([4, 53, 210]), np.array([52, 209, 1500])
    lo_in, hi_in = np.array([8, 64, 192]), np.array([96, 320, 1024])
    true_out = rng.integers(lo_out[cls], hi_out[cls] + 1).astype(np.int32)
    in_tokens = rng.integers(lo_in[cls], hi_in[cls] + 1).astype(np.int32)
    tag = assign_category_tags(true_out, rng, tag_noise)
    if untagged_frac > 0:
        tag = np.where(rng.random(n) < untagged_frac, -1, tag).astype(np.int32)
    return {
        "client": client,
        "arrival": np.arange(n, dtype=np.float64) / float(max(n, 1)),
        "in_tokens": in_tokens,
        "true_out": true_out,
        "tag": tag,
        "id": np.arange(n, dtype=np.int64),
        "client_names": [f"client{i}" for i in range(n_clients)],
        "tag_names": list(TAG_NAMES),
    }


def warm_ledger(n_clients: int, seed: int = 2) -> dict:
    """Seeded pre-step ledger: ufc U[0,1e6], rfc U[0,1e5], counter U[0,1e6]."""
    rng = np.random.default_rng(seed)
    return {
        "ufc": rng.uniform(0.0, 1e6, n_clients),
        "rfc": rng.uniform(0.0, 1e5, n_clients),
        "counter": rng.uniform(0.0, 1e6, n_clients),
    }
