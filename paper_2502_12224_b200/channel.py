"""The transfer channel C1 as a standalone object (SURVEY §8b
``prefetch_{enqueue, promote, drop_stale, wait}``): the reference's ``_Channel``
(pipeline.py:163-264) over real copies, bound from ``fate_channel_*``.

Pending transfers form a host FIFO that ``promote_ondemand`` / ``drop_stale``
reorder and discard until they start, exactly as in the reference; ``settle``
starts them in queue order on the channel's copy stream (at most
``max_inflight`` in flight) and ``completion(t, stream)`` makes a consumer
stream wait for a transfer without blocking the host.  The engine runs the same
discipline internally; this object serves callers that drive their own step
loop.  ``device=None`` keeps only the queue bookkeeping (no GPU needed)."""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import _lib
from ._lib import check

KINDS = {"prefetch": 0, "ondemand": 1}


@dataclass(frozen=True)
class Transfer:
    id: int
    kind: str
    token: int
    layer: int
    expert: int
    bits: int

    @property
    def step(self) -> tuple:
        return (self.token, self.layer)


class Channel:
    def __init__(self, device: int | None = 0, max_inflight: int = 2):
        self._L = _lib.lib() if device is not None else _lib.load()
        h = C.c_void_p()
        check(self._L.fate_channel_create(-1 if device is None else int(device), int(max_inflight), C.byref(h)),
              "fate_channel_create")
        self._h = h
        self._by_id: dict = {}

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._L.fate_channel_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def enqueue(self, kind: str, token: int, layer: int, expert: int, bits: int, src: int = 0, dst: int = 0,
                nbytes: int = 0) -> Transfer:
        """_Channel.enqueue (pipeline.py:196): a copy of ``nbytes`` from ``src`` to ``dst``."""
        i = C.c_int64()
        check(self._L.fate_channel_enqueue(self._h, KINDS[kind], token, layer, expert, bits, C.c_void_p(src or None),
                                           C.c_void_p(dst or None), int(nbytes), C.byref(i)), "fate_channel_enqueue")
        t = Transfer(int(i.value), kind, token, layer, expert, bits)
        self._by_id[t.id] = t
        return t

    def promote_ondemand(self) -> None:
        check(self._L.fate_channel_promote(self._h), "fate_channel_promote")

    def drop_stale(self, current_step: tuple) -> int:
        n = C.c_int()
        check(self._L.fate_channel_drop_stale(self._h, int(current_step[0]), int(current_step[1]), C.byref(n)),
              "fate_channel_drop_stale")
        return int(n.value)

    def settle(self) -> None:
        """Start pending transfers in queue order while fewer than max_inflight are in flight."""
        check(self._L.fate_channel_pump(self._h), "fate_channel_pump")

    def completion(self, t: Transfer, stream=None) -> None:
        """Start everything up to ``t`` and make ``stream`` (a torch stream or raw handle) wait for it."""
        s = getattr(stream, "cuda_stream", stream)
        check(self._L.fate_channel_wait(self._h, t.id, C.c_void_p(s or None)), "fate_channel_wait")

    def find(self, token: int, layer: int, expert: int):
        """(state, transfer): state None / "pending" / "in_flight" / "done" (pipeline.py:232)."""
        st, i = C.c_int(), C.c_int64(-1)
        check(self._L.fate_channel_find(self._h, token, layer, expert, C.byref(st), C.byref(i)), "fate_channel_find")
        names = {-1: None, 0: "pending", 1: "in_flight", 2: "done"}
        return names[st.value], self._by_id.get(int(i.value))

    @property
    def pending(self) -> list:
        n, fl = C.c_int(), C.c_int()
        check(self._L.fate_channel_pending(self._h, None, 0, C.byref(n), C.byref(fl)), "fate_channel_pending")
        ids = (C.c_int64 * max(1, n.value))()
        check(self._L.fate_channel_pending(self._h, ids, n.value, C.byref(n), C.byref(fl)), "fate_channel_pending")
        return [self._by_id[int(ids[k])] for k in range(n.value)]
