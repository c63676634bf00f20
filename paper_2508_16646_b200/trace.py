"""Request traces: the reference's CSV trace format and a binary
struct-of-arrays format, parsed natively by libeqx_b200.so (csrc/eqx_trace.cpp).

Mirrors ``equinox::load_trace`` / ``write_trace_csv`` / ``trace_hash`` (workload.cpp:312-428):
same validation and ParseError messages, stable re-sort of out-of-order rows with one warning,
ids = arrival-order positions, roster in first-appearance order.  The columns live in the
library's pinned host arena when a GPU is present, so ``requests()`` feeds ``stage_async`` /
``drain`` without another copy::

    tr = Trace.load("trace.csv")              # or .eqxt (binary, carries trace_hash)
    sch = GpuScheduler([ClientState(c) for c in tr.client_names], tag_names=tr.tag_names, ...)
    sch.drain(**tr.requests())
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .scheduler import ParseError


def _names(ptr, n: int) -> list:
    """n NUL-terminated strings packed at ptr."""
    out = []
    for _ in range(n):
        b = C.string_at(ptr)
        out.append(b.decode())
        ptr += len(b) + 1
    return out


class Trace:
    """A request trace: columns client / arrival_s / input_tokens / output_tokens / tag (numpy
    views over the library's memory), client_names, tag_names, warnings, hash()."""

    def __init__(self, handle):
        self._lib = L.load()
        self._h = handle
        v = L.TraceView()
        self._lib.eqx_trace_view_get(self._h, C.byref(v))
        n = v.n
        def col(p, dt):  # a numpy view over the library's column; the view keeps the trace alive
            if not n:
                return np.zeros(0, dt)
            buf = (C.c_uint8 * (n * np.dtype(dt).itemsize)).from_address(p)
            buf._owner = self
            return np.frombuffer(buf, dt)
        self.client = col(v.client, np.int32)
        self.arrival_s = col(v.arrival_s, np.float64)
        self.input_tokens = col(v.input_tokens, np.int32)
        self.output_tokens = col(v.output_tokens, np.int32)
        self.tag = col(v.tag, np.int32)
        self.client_names = _names(v.client_names, v.n_clients)
        self.tag_names = _names(v.tag_names, v.n_tags)
        self.warnings = _names(v.warnings, v.n_warnings)
        self.duration_s = v.duration_s
        self.pinned = bool(v.pinned)
        self.stored_hash = v.stored_hash.decode()

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            self._lib.eqx_trace_free(h)

    def __len__(self) -> int:
        return len(self.client)

    # -- constructors --
    @classmethod
    def load_csv(cls, path: str) -> "Trace":
        return cls._load(L.load().eqx_trace_load_csv, path)

    @classmethod
    def load_bin(cls, path: str) -> "Trace":
        return cls._load(L.load().eqx_trace_load_bin, path)

    @classmethod
    def load(cls, path: str) -> "Trace":
        return cls.load_bin(path) if str(path).endswith(".eqxt") else cls.load_csv(path)

    @classmethod
    def _load(cls, fn, path: str) -> "Trace":
        h = C.c_void_p()
        err = C.create_string_buffer(1024)
        st = fn(str(path).encode(), C.byref(h), err, 1024)
        if st != L.EQX_OK:
            raise ParseError(err.value.decode() or f"trace load failed ({st})")
        return cls(h)

    @classmethod
    def from_columns(cls, client, arrival_s, input_tokens, output_tokens, client_names, tag=None,
                     tag_names=()) -> "Trace":
        """A trace from columns already in arrival order (e.g. workload generators)."""
        cols = [np.ascontiguousarray(client, np.int32), np.ascontiguousarray(arrival_s, np.float64),
                np.ascontiguousarray(input_tokens, np.int32), np.ascontiguousarray(output_tokens, np.int32)]
        tg = None if tag is None else np.ascontiguousarray(tag, np.int32)
        names = b"".join(s.encode() + b"\0" for s in client_names)
        tnames = b"".join(s.encode() + b"\0" for s in tag_names)
        h = C.c_void_p()
        st = L.load().eqx_trace_create(len(cols[0]), *(c.ctypes.data for c in cols),
                                       None if tg is None else tg.ctypes.data, len(client_names), names,
                                       len(tag_names), tnames, C.byref(h))
        if st != L.EQX_OK:
            raise ValueError(f"eqx_trace_create failed ({st}): client / tag index out of range")
        return cls(h)

    # -- output --
    def hash(self) -> str:
        """trace_hash (workload.cpp:422-428): FNV-1a of the canonical CSV, 16 hex digits."""
        out = C.create_string_buffer(17)
        self._lib.eqx_trace_hash(self._h, out)
        return out.value.decode()

    def save_csv(self, path: str) -> None:
        if self._lib.eqx_trace_save_csv(self._h, str(path).encode()) != L.EQX_OK:
            raise OSError(f"cannot write trace file '{path}'")

    def save_bin(self, path: str) -> None:
        if self._lib.eqx_trace_save_bin(self._h, str(path).encode()) != L.EQX_OK:
            raise OSError(f"cannot write trace file '{path}'")

    def tag_ids(self) -> np.ndarray:
        """Tag ids for a scheduler built with tag_names=self.tag_names (0 = untagged)."""
        if len(self.tag_names) > 255:
            raise ValueError("more than 255 distinct category tags")
        return np.where(self.tag < 0, 0, self.tag + 1).astype(np.uint8)

    def requests(self) -> dict:
        """Keyword columns for GpuScheduler.drain / stage_async / drain_step_async / append
        (ids = arrival-order positions, as load_trace assigns them)."""
        return dict(client=self.client, arrival_s=self.arrival_s, input_tokens=self.input_tokens,
                    tag=self.tag_ids(), true_output_tokens=self.output_tokens)
