"""Host control plane (include/blockhost.h bh_pool_*, bh_kv_*): the block-instance queues that
form per-block batches and the paged KV bookkeeping that yields GPU page tables.

Method names and meaning follow blocksim's InstancePool (proj/core/include/blocksim/agent.hpp:
69-140) and KvStore (kv.hpp:72-128); errors raise ValueError (std::invalid_argument) or
RuntimeError("logic") (std::logic_error) as the reference throws.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from ._lib import lib

PREFILL, DECODE = 0, 1


class Entry(C.Structure):
    """QueueEntry (agent.hpp:20-30)."""
    _fields_ = [("request_id", C.c_int32), ("chain_step", C.c_int32), ("phase", C.c_int32),
                ("tokens", C.c_int32), ("context_tokens", C.c_int32), ("kv_resident", C.c_int32),
                ("est_cost_us", C.c_double), ("enqueue_seq", C.c_uint64)]

    def key(self):
        return (self.request_id, self.chain_step, self.phase, self.tokens, self.context_tokens,
                self.kv_resident, round(self.est_cost_us, 9), self.enqueue_seq)


class LogicError(RuntimeError):
    pass


def _raise(code: int, msg: str):
    if code == 1:
        raise ValueError(msg)
    if code == 2:
        raise LogicError(msg)
    raise RuntimeError(msg)


_bound = set()


def _bind(prefix: str, L):
    if prefix in _bound:
        return
    P, I, I64, U64, D = C.c_void_p, C.c_int, C.c_int64, C.c_uint64, C.c_double
    EP = C.POINTER(Entry)
    sigs = {
        "pool_new": (P, []) if prefix == "bh_" else (P, [I, I]),
        "pool_free": (None, [P]),
        "pool_last_error": (C.c_char_p, [P]),
        "pool_create_instance": (I, [P, C.c_char_p, I, I64, I64, C.c_char_p, I]),
        "pool_mark_ready": (I, [P, C.c_char_p, I64]),
        "pool_enqueue": (I, [P, C.c_char_p, EP]),
        "pool_pop_batch": (I, [P, C.c_char_p, I, I64, EP, I, C.POINTER(I), C.POINTER(I)]),
        "pool_finish_batch": (I, [P, C.c_char_p, I64]),
        "pool_next_runnable": (I, [P, I, I64, C.c_char_p, I]),
        "pool_remove_queued": (I, [P, C.c_char_p, I, EP, I, C.POINTER(I)]),
        "pool_take_tail": (I, [P, C.c_char_p, I, EP, I, C.POINTER(I)]),
        "pool_queue": (I, [P, C.c_char_p, EP, I, C.POINTER(I), C.POINTER(D), C.POINTER(I)]),
        "kv_new": (P, []) if prefix == "bh_" else (P, [I]),
        "kv_free": (None, [P]),
        "kv_last_error": (C.c_char_p, [P]),
        "kv_create_segment": (I, [P, U64, C.c_char_p, I, I64]),
        "kv_append_tokens": (I, [P, U64, C.c_char_p, I, C.POINTER(I)]),
        "kv_share_prefix": (I, [P, U64, U64, C.c_char_p, I, C.POINTER(I)]),
        "kv_release": (I, [P, U64, C.c_char_p]),
        "kv_release_request": (I, [P, U64]),
        "kv_move_segment": (I, [P, U64, C.c_char_p, I]),
        "kv_query": (I64, [P, U64, C.c_char_p, I]),
        "kv_bytes_saved": (I64, [P]),
        "kv_used": (I64, [P, I]),
        "kv_page_ids": (I, [P, U64, C.c_char_p, C.POINTER(U64), I, C.POINTER(I)]),
    }
    if prefix == "bh_":
        sigs["kv_attach_pool"] = (I, [P, C.c_char_p, I, I])
        sigs["kv_page_slots"] = (I, [P, U64, C.c_char_p, C.POINTER(C.c_int32), I, C.POINTER(I)])
        sigs["kv_move_segment_slots"] = (I, [P, U64, C.c_char_p, I, C.POINTER(C.c_int32),
                                             C.POINTER(C.c_int32), I, C.POINTER(I)])
    for name, (res, args) in sigs.items():
        fn = getattr(L, prefix + name)
        fn.restype, fn.argtypes = res, args
    _bound.add(prefix)


class Pool:
    """Block instances, their queues and the greedy prefix-merge batch rule."""

    prefix = "bh_"

    def __init__(self, _lib=None, _handle=None):
        self.L = _lib or lib()
        _bind(self.prefix, self.L)
        self.h = _handle if _handle is not None else self.L.bh_pool_new()
        self._f = lambda n: getattr(self.L, self.prefix + n)

    def _ck(self, rc):
        if rc != 0:
            _raise(rc, self._f("pool_last_error")(self.h).decode())

    def create(self, block_id: str, device: int, now: int = 0, ready_at: int = 0) -> str:
        buf = C.create_string_buffer(64)
        self._ck(self._f("pool_create_instance")(self.h, block_id.encode(), device, now,
                                                 ready_at, buf, 64))
        return buf.value.decode()

    def mark_ready(self, inst: str, now: int):
        self._ck(self._f("pool_mark_ready")(self.h, inst.encode(), now))

    def enqueue(self, inst: str, request_id: int, chain_step: int, phase: int, tokens: int,
                context_tokens: int, est_cost_us: float = 0.0, kv_resident: bool = False):
        e = Entry(request_id, chain_step, phase, tokens, context_tokens, int(kv_resident),
                  est_cost_us, 0)
        self._ck(self._f("pool_enqueue")(self.h, inst.encode(), C.byref(e)))

    def _entries(self, fn, *args, cap=4096):
        out = (Entry * cap)()
        n = C.c_int(0)
        extra = []
        rc = fn(self.h, *args, out, cap, C.byref(n), *extra)
        self._ck(rc)
        return [out[i] for i in range(n.value)]

    def pop_batch(self, inst: str, max_batch_tokens: int, now: int = 0):
        out = (Entry * 4096)()
        n, ph = C.c_int(0), C.c_int(0)
        self._ck(self._f("pool_pop_batch")(self.h, inst.encode(), max_batch_tokens, now, out,
                                          4096, C.byref(n), C.byref(ph)))
        return ph.value, [out[i] for i in range(n.value)]

    def finish_batch(self, inst: str, now: int = 0):
        self._ck(self._f("pool_finish_batch")(self.h, inst.encode(), now))

    def next_runnable(self, device: int, now: int = 0):
        buf = C.create_string_buffer(64)
        rc = self._f("pool_next_runnable")(self.h, device, now, buf, 64)
        if rc < 0:
            _raise(-rc, "next_runnable")
        return buf.value.decode() if rc == 1 else None

    def remove_queued(self, inst: str, request_id: int):
        return self._entries(self._f("pool_remove_queued"), inst.encode(), request_id)

    def take_tail(self, inst: str, count: int):
        return self._entries(self._f("pool_take_tail"), inst.encode(), count)

    def queue(self, inst: str):
        out = (Entry * 4096)()
        n, ex = C.c_int(0), C.c_int(0)
        cost = C.c_double(0)
        self._ck(self._f("pool_queue")(self.h, inst.encode(), out, 4096, C.byref(n),
                                      C.byref(cost), C.byref(ex)))
        return [out[i] for i in range(n.value)], cost.value, bool(ex.value)

    def __del__(self):
        try:
            self._f("pool_free")(self.h)
        except Exception:
            pass


@dataclass
class SegmentInfo:
    device: int
    tokens: int
    pages: int
    shared_pages: int
    bytes: int


class KvStore:
    """Block-local paged KV bookkeeping (16-token pages, global page ids, prefix sharing)."""

    prefix = "bh_"

    def __init__(self, _lib=None, _handle=None):
        self.L = _lib or lib()
        _bind(self.prefix, self.L)
        self.h = _handle if _handle is not None else self.L.bh_kv_new()
        self._f = lambda n: getattr(self.L, self.prefix + n)

    def _ck(self, rc):
        if rc != 0:
            _raise(rc, self._f("kv_last_error")(self.h).decode())

    def attach_pool(self, pool_key: str, device: int, n_pages: int):
        self._ck(self.L.bh_kv_attach_pool(self.h, pool_key.encode(), device, n_pages))

    def create_segment(self, request: int, block: str, device: int, bytes_per_token: int):
        self._ck(self._f("kv_create_segment")(self.h, request, block.encode(), device,
                                             bytes_per_token))

    def append_tokens(self, request: int, block: str, n: int) -> int:
        a = C.c_int(0)
        self._ck(self._f("kv_append_tokens")(self.h, request, block.encode(), n, C.byref(a)))
        return a.value

    def share_prefix(self, request: int, from_request: int, block: str, tokens: int) -> int:
        c = C.c_int(0)
        self._ck(self._f("kv_share_prefix")(self.h, request, from_request, block.encode(),
                                           tokens, C.byref(c)))
        return c.value

    def release(self, request: int, block: str):
        self._ck(self._f("kv_release")(self.h, request, block.encode()))

    def release_request(self, request: int):
        self._ck(self._f("kv_release_request")(self.h, request))

    def move_segment(self, request: int, block: str, dst_device: int):
        self._ck(self._f("kv_move_segment")(self.h, request, block.encode(), dst_device))

    def move_segment_slots(self, request: int, block: str, dst_device: int, cap: int = 4096):
        """move_segment plus the (source slot, destination slot) page copies it implies."""
        src = (C.c_int32 * cap)()
        dst = (C.c_int32 * cap)()
        n = C.c_int(0)
        self._ck(self._f("kv_move_segment_slots")(self.h, request, block.encode(), dst_device,
                                                  src, dst, cap, C.byref(n)))
        return list(src[:n.value]), list(dst[:n.value])

    def info(self, request: int, block: str) -> SegmentInfo:
        q = self._f("kv_query")
        b = block.encode()
        return SegmentInfo(*(int(q(self.h, request, b, w)) for w in range(5)))

    def has_segment(self, request: int, block: str) -> bool:
        return bool(self._f("kv_query")(self.h, request, block.encode(), 5))

    def bytes_saved_by_sharing(self) -> int:
        return int(self._f("kv_bytes_saved")(self.h))

    def used(self, device: int) -> int:
        return int(self._f("kv_used")(self.h, device))

    def page_ids(self, request: int, block: str):
        out = (C.c_uint64 * 65536)()
        n = C.c_int(0)
        self._ck(self._f("kv_page_ids")(self.h, request, block.encode(), out, 65536, C.byref(n)))
        return [int(out[i]) for i in range(n.value)]

    def page_slots(self, request: int, block: str):
        out = (C.c_int32 * 65536)()
        n = C.c_int(0)
        self._ck(self.L.bh_kv_page_slots(self.h, request, block.encode(), out, 65536, C.byref(n)))
        return [int(out[i]) for i in range(n.value)]

    def __del__(self):
        try:
            self._f("kv_free")(self.h)
        except Exception:
            pass
