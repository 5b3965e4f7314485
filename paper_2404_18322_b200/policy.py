"""Routing / speculation-marking / placement policy (include/blockpolicy.h; SURVEY §8 a10, a14,
a15) over ctypes.

Method names and meaning follow blocksim's Scheduler (proj/core/include/blocksim/scheduler.hpp:
62-118): `choose_binding` (scheduler.cpp:80-160), `estimate` (:23-78), `speculation_marks`
(:180-215), `scale_decisions` (:227-260), `choose_device` (:262-314), `placement_moves`
(:321-366), `migration_rates` (:368-381). Errors raise ValueError (std::invalid_argument).

The state is a snapshot the host keeps current (`put_instance`, `set_ledger`, `set_lane`,
`set_kv`, `note_adjacency`); `load_static` / `load_state` fill it from a plain description
(dicts / lists, the layout `oracle/ref_shim.cpp rs_policy_trace_run` emits).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import lib

PREF_LOCALITY, PREF_TIGHTEST_FIT, PREF_MOST_FREE = 0, 1, 2
KIND = {"attention": 0, "ffn": 1, "embedding": 2, "lm_head": 3, "adapter": 4}


class _Config(C.Structure):
    _fields_ = [("adaptive", C.c_int), ("least_busy", C.c_int), ("frag_min", C.c_int),
                ("speculation", C.c_int), ("spec_fraction", C.c_double),
                ("scale_queue_us", C.c_int64), ("expected_tokens", C.c_int),
                ("sur_attention_only", C.c_double), ("sur_ffn_only", C.c_double),
                ("sur_one_layer", C.c_double), ("sur_multi_layer", C.c_double),
                ("sur_allow_adapter_blocks", C.c_int)]


class _Grid(C.Structure):
    _fields_ = [("xs", C.c_void_p), ("nx", C.c_int), ("ys", C.c_void_p), ("ny", C.c_int),
                ("v", C.c_void_p)]


class _Instance(C.Structure):
    _fields_ = [("id", C.c_char_p), ("block_id", C.c_char_p), ("device", C.c_int),
                ("ready", C.c_int), ("ready_at", C.c_int64), ("last_used", C.c_int64),
                ("created_seq", C.c_uint64), ("executing", C.c_int), ("queue_len", C.c_int),
                ("queued_cost_us", C.c_double), ("queued_cost_hwm", C.c_double)]


class _QueuedDecode(C.Structure):
    _fields_ = [("instance", C.c_char_p), ("inst_block", C.c_char_p), ("device", C.c_int),
                ("request_id", C.c_uint64), ("chain_block", C.c_char_p), ("owner", C.c_int),
                ("pages", C.c_int), ("shared_pages", C.c_int), ("pending", C.c_int),
                ("pending_key", C.c_char_p), ("t_call", C.c_int64)]


class _Query(C.Structure):
    _fields_ = [("request_id", C.c_uint64), ("chain_block", C.c_char_p), ("phase", C.c_int),
                ("tokens", C.c_int), ("context_tokens", C.c_int), ("from_device", C.c_int),
                ("now", C.c_int64)]


class _Choice(C.Structure):
    _fields_ = [("block_id", C.c_char * 96), ("stitch_class", C.c_char * 96),
                ("instance_id", C.c_char * 32), ("device", C.c_int), ("adaptive", C.c_int),
                ("evict_bytes", C.c_int64), ("queue_us", C.c_double), ("compute_us", C.c_double),
                ("transfer_us", C.c_double), ("load_us", C.c_double)]


_bound = False


def _bind():
    global _bound
    if _bound:
        return lib()
    L = lib()
    P, I, I64, U64, D, S = C.c_void_p, C.c_int, C.c_int64, C.c_uint64, C.c_double, C.c_char_p
    SS = C.POINTER(C.c_char_p)
    sig = {
        "bh_policy_new": (P, [C.POINTER(_Config)]),
        "bh_policy_free": (None, [P]),
        "bh_policy_last_error": (S, [P]),
        "bh_policy_add_cost_class": (I, [P, S, C.POINTER(_Grid), C.POINTER(_Grid), I64]),
        "bh_policy_add_stitch_class": (I, [P, S, C.POINTER(_Grid)]),
        "bh_policy_set_device_class": (I, [P, S, D]),
        "bh_policy_add_component": (I, [P, S, I, I, I, I, SS, P]),
        "bh_policy_add_block": (I, [P, S, I, SS, I]),
        "bh_policy_add_chain": (I, [P, S, I, SS]),
        "bh_policy_add_candidate": (I, [P, S, S, S, D]),
        "bh_policy_add_server": (I, [P, I, D]),
        "bh_policy_set_inter_bandwidth": (I, [P, I, I, D]),
        "bh_policy_set_inter_default": (I, [P, D]),
        "bh_policy_add_device": (I, [P, I, I, S, I64, D, D]),
        "bh_policy_clear_state": (I, [P]),
        "bh_policy_put_instance": (I, [P, C.POINTER(_Instance)]),
        "bh_policy_remove_instance": (I, [P, S]),
        "bh_policy_set_ledger": (I, [P, I, I64, I64, I64]),
        "bh_policy_set_lane": (I, [P, I, I64]),
        "bh_policy_set_kv": (I, [P, U64, S, I, I]),
        "bh_policy_set_adjacency": (I, [P, S, S, I64]),
        "bh_policy_note_adjacency": (I, [P, S, S]),
        "bh_policy_choose_binding": (I, [P, C.POINTER(_Query), C.POINTER(_Choice), C.POINTER(I)]),
        "bh_policy_estimate": (I, [P, C.POINTER(_Query), S, S, S, I, P, C.POINTER(I64)]),
        "bh_policy_speculation_marks": (I, [P, P, I, C.POINTER(I)]),
        "bh_policy_scale_decisions": (I, [P, P, I, P, I, C.POINTER(I)]),
        "bh_policy_choose_device": (I, [P, S, I, P, I, C.POINTER(I)]),
        "bh_policy_placement_moves": (I, [P, P, I, P, I, C.POINTER(I)]),
        "bh_policy_migration_rates": (I, [P, S, I, I, C.POINTER(I64), C.POINTER(I64)]),
        "bh_policy_param_bytes_needed": (I, [P, S, I, C.POINTER(I64)]),
        "bh_plan_migration": (I, [I, I64, I64, P]),
        "bh_policy_interception_record": (I, [P, S, I64]),
        "bh_policy_interception_set": (I, [P, S, D, U64]),
        "bh_policy_interception_predict": (I, [P, S, I64, I64, C.POINTER(I64), C.POINTER(I)]),
        "bh_policy_kv_review": (I, [P, C.POINTER(_QueuedDecode), I, I64, I, P, I, C.POINTER(I)]),
    }
    for n, (r, a) in sig.items():
        fn = getattr(L, n)
        fn.restype, fn.argtypes = r, a
    _bound = True
    return L


def _b(s) -> bytes:
    return s.encode() if isinstance(s, str) else s


def _strs(v):
    arr = (C.c_char_p * max(1, len(v)))(*[_b(x) for x in v])
    return arr


def plan_migration(pages: int, rec_us: int, cp_us: int):
    """(pages, recompute_pages, copy_pages, completion_us) of a two-path page migration."""
    out = (C.c_int64 * 6)()
    if _bind().bh_plan_migration(pages, rec_us, cp_us, out) != 0:
        raise ValueError("plan_migration rejected its input")
    return tuple(out[:4])


class Policy:
    def __init__(self, adaptive=True, least_busy=False, frag_min=False, speculation=True,
                 spec_fraction=0.10, scale_queue_us=0, expected_tokens=256,
                 surrogate=(37.43, 1.71, 22.91, 18.55, False)):
        self._L = _bind()
        cfg = _Config(int(adaptive), int(least_busy), int(frag_min), int(speculation),
                      float(spec_fraction), int(scale_queue_us), int(expected_tokens),
                      *[float(x) for x in surrogate[:4]], int(surrogate[4]))
        self.h = self._L.bh_policy_new(C.byref(cfg))
        self._keep = []

    def close(self):
        if self.h:
            self._L.bh_policy_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _ck(self, rc):
        if rc != 0:
            msg = self._L.bh_policy_last_error(self.h).decode()
            raise ValueError(msg) if rc == 1 else RuntimeError(msg)

    # ---- static description
    @staticmethod
    def _grid(g):
        xs = np.ascontiguousarray(g["xs"], np.float64)
        ys = np.ascontiguousarray(g["ys"], np.float64)
        v = np.ascontiguousarray(g["v"], np.float64).reshape(-1)
        return _Grid(xs.ctypes.data, xs.size, ys.ctypes.data, ys.size, v.ctypes.data), (xs, ys, v)

    def add_cost_class(self, key, prefill, decode, kv_bytes_per_token=-1):
        gp, kp = self._grid(prefill)
        gd, kd = self._grid(decode)
        self._ck(self._L.bh_policy_add_cost_class(self.h, _b(key), C.byref(gp), C.byref(gd),
                                                  int(kv_bytes_per_token)))

    def add_stitch_class(self, key, grid):
        g, k = self._grid(grid)
        self._ck(self._L.bh_policy_add_stitch_class(self.h, _b(key), C.byref(g)))

    def set_device_class(self, name, speed):
        self._ck(self._L.bh_policy_set_device_class(self.h, _b(name), float(speed)))

    def add_component(self, cid, kind, embed_dim, layer, pieces):
        kind = KIND[kind] if isinstance(kind, str) else int(kind)
        ids = _strs([p[0] for p in pieces])
        nb = np.ascontiguousarray([p[1] for p in pieces] or [0], np.int64)
        self._ck(self._L.bh_policy_add_component(self.h, _b(cid), kind, embed_dim, layer,
                                                 len(pieces), ids, nb.ctypes.data))

    def add_block(self, bid, comps, embed_dim_out):
        self._ck(self._L.bh_policy_add_block(self.h, _b(bid), len(comps), _strs(comps),
                                             embed_dim_out))

    def add_chain(self, model, blocks):
        self._ck(self._L.bh_policy_add_chain(self.h, _b(model), len(blocks), _strs(blocks)))

    def add_candidate(self, block, cand, stitch_class="", score=1.0):
        self._ck(self._L.bh_policy_add_candidate(self.h, _b(block), _b(cand), _b(stitch_class),
                                                 float(score)))

    def add_server(self, sid, intra_bps):
        self._ck(self._L.bh_policy_add_server(self.h, sid, float(intra_bps)))

    def set_inter_bandwidth(self, a, b, bps):
        self._ck(self._L.bh_policy_set_inter_bandwidth(self.h, a, b, float(bps)))

    def set_inter_default(self, bps):
        self._ck(self._L.bh_policy_set_inter_default(self.h, float(bps)))

    def add_device(self, did, server, cls, capacity, mem_bps, load_bps):
        self._ck(self._L.bh_policy_add_device(self.h, did, server, _b(cls), int(capacity),
                                              float(mem_bps), float(load_bps)))

    # ---- dynamic state
    def clear_state(self):
        self._ck(self._L.bh_policy_clear_state(self.h))

    def put_instance(self, iid, block, device, ready=True, ready_at=0, last_used=0,
                     created_seq=0, executing=False, queue_len=0, queued_cost_us=0.0,
                     queued_cost_hwm=0.0):
        x = _Instance(_b(iid), _b(block), device, int(ready), ready_at, last_used, created_seq,
                      int(executing), queue_len, float(queued_cost_us), float(queued_cost_hwm))
        self._ck(self._L.bh_policy_put_instance(self.h, C.byref(x)))

    def remove_instance(self, iid):
        self._ck(self._L.bh_policy_remove_instance(self.h, _b(iid)))

    def set_ledger(self, device, params, kv=0, act=0):
        self._ck(self._L.bh_policy_set_ledger(self.h, device, int(params), int(kv), int(act)))

    def set_lane(self, device, busy_until):
        self._ck(self._L.bh_policy_set_lane(self.h, device, int(busy_until)))

    def set_kv(self, request, block, owner, pages):
        self._ck(self._L.bh_policy_set_kv(self.h, request, _b(block), owner, pages))

    def set_adjacency(self, a, b, count):
        self._ck(self._L.bh_policy_set_adjacency(self.h, _b(a), _b(b), int(count)))

    def note_adjacency(self, a, b):
        self._ck(self._L.bh_policy_note_adjacency(self.h, _b(a), _b(b)))

    # ---- decisions
    @staticmethod
    def _query(request_id, chain_block, decode, tokens, context, from_device, now):
        return _Query(request_id, _b(chain_block), 1 if decode else 0, tokens, context,
                      from_device, now)

    def choose_binding(self, request_id, chain_block, decode, tokens, context, from_device=-1,
                       now=0):
        """None when nothing is feasible, else dict(block, stitch, instance ('' = create on
        device), device, adaptive, evict, est=(queue, compute, transfer, load))."""
        q = self._query(request_id, chain_block, decode, tokens, context, from_device, now)
        out, found = _Choice(), C.c_int(0)
        self._ck(self._L.bh_policy_choose_binding(self.h, C.byref(q), C.byref(out),
                                                  C.byref(found)))
        if not found.value:
            return None
        return {"block": out.block_id.decode(), "stitch": out.stitch_class.decode(),
                "instance": out.instance_id.decode(), "device": out.device,
                "adaptive": bool(out.adaptive), "evict": out.evict_bytes,
                "est": (out.queue_us, out.compute_us, out.transfer_us, out.load_us)}

    def estimate(self, request_id, chain_block, decode, tokens, context, from_device, now,
                 block, stitch_class="", instance=None, device=0):
        q = self._query(request_id, chain_block, decode, tokens, context, from_device, now)
        out, ev = (C.c_double * 4)(), C.c_int64(0)
        self._ck(self._L.bh_policy_estimate(self.h, C.byref(q), _b(block), _b(stitch_class),
                                            _b(instance) if instance else None, device, out,
                                            C.byref(ev)))
        return tuple(out), ev.value

    def _ids(self, fn, with_devs):
        cap = 1 << 16
        buf = C.create_string_buffer(cap)
        n = C.c_int(0)
        if with_devs:
            devs = (C.c_int * 4096)()
            self._ck(fn(self.h, buf, cap, devs, 4096, C.byref(n)))
        else:
            self._ck(fn(self.h, buf, cap, C.byref(n)))
        ids = buf.value.decode().split("\n") if n.value else []
        return list(zip(ids, devs[:n.value])) if with_devs else ids

    def speculation_marks(self):
        return self._ids(self._L.bh_policy_speculation_marks, False)

    def scale_decisions(self):
        return self._ids(self._L.bh_policy_scale_decisions, True)

    def placement_moves(self):
        return self._ids(self._L.bh_policy_placement_moves, True)

    def choose_device(self, block, pref=PREF_LOCALITY, exclude=()):
        ex = (C.c_int * max(1, len(exclude)))(*exclude)
        d = C.c_int(-1)
        self._ck(self._L.bh_policy_choose_device(self.h, _b(block), pref, ex, len(exclude),
                                                 C.byref(d)))
        return d.value

    def migration_rates(self, block, src, dst):
        r, c = C.c_int64(0), C.c_int64(0)
        self._ck(self._L.bh_policy_migration_rates(self.h, _b(block), src, dst, C.byref(r),
                                                   C.byref(c)))
        return r.value, c.value

    def param_bytes_needed(self, block, device):
        n = C.c_int64(0)
        self._ck(self._L.bh_policy_param_bytes_needed(self.h, _b(block), device, C.byref(n)))
        return n.value

    # ---- proactive KV review
    def interception_record(self, key, sample):
        self._ck(self._L.bh_policy_interception_record(self.h, _b(key), int(sample)))

    def interception_set(self, key, total, n):
        """key None: the global accumulator."""
        self._ck(self._L.bh_policy_interception_set(self.h, _b(key) if key is not None else None,
                                                    float(total), int(n)))

    def predicted_remaining(self, key, t_call, now):
        out, found = C.c_int64(0), C.c_int(0)
        self._ck(self._L.bh_policy_interception_predict(self.h, _b(key), int(t_call), int(now),
                                                        C.byref(out), C.byref(found)))
        return out.value if found.value else None

    def kv_review(self, entries, now, recalc_only=False):
        """entries: dicts (instance, inst_block, device, request, chain_block, owner, pages,
        shared, pending, pending_key, t_call); returns indices to migrate, in order."""
        arr = (_QueuedDecode * max(1, len(entries)))()
        keep = []
        for i, e in enumerate(entries):
            vals = [_b(e["instance"]), _b(e["inst_block"]), e["device"], e["request"],
                    _b(e["chain_block"]), e["owner"], e["pages"], e["shared"],
                    int(e["pending"]), _b(e.get("pending_key") or ""), e["t_call"]]
            keep.append(vals)
            arr[i] = _QueuedDecode(*vals)
        out = (C.c_int * max(1, len(entries)))()
        n = C.c_int(0)
        self._ck(self._L.bh_policy_kv_review(self.h, arr, len(entries), int(now),
                                             int(recalc_only), out, len(entries), C.byref(n)))
        return list(out[:n.value])

    # ---- descriptions
    @classmethod
    def from_static(cls, st: dict) -> "Policy":
        c = st["config"]
        p = cls(adaptive=c["adaptive"], least_busy=c["least_busy"], frag_min=c["frag_min"],
                speculation=c["speculation"], spec_fraction=c["spec_fraction"],
                scale_queue_us=c["scale_queue_us"], expected_tokens=c["expected_tokens"],
                surrogate=tuple(st.get("surrogate", (37.43, 1.71, 22.91, 18.55, False))))
        for k, cc in st["classes"].items():
            p.add_cost_class(k, cc["prefill"], cc["decode"], cc.get("kv", -1))
        for k, g in st.get("stitches", {}).items():
            p.add_stitch_class(k, g)
        for k, s in st["device_classes"].items():
            p.set_device_class(k, s)
        for comp in st["components"]:
            p.add_component(comp["id"], comp["kind"], comp["dim"], comp["layer"],
                            [tuple(x) for x in comp["pieces"]])
        for b in st["blocks"]:
            p.add_block(b["id"], b["comps"], b["dim_out"])
        for b in st["blocks"]:
            for cand, stitch, score in b.get("candidates", []):
                p.add_candidate(b["id"], cand, stitch, score)
        for model, chain in st["chains"]:
            p.add_chain(model, chain)
        for sid, bps in st["servers"]:
            p.add_server(sid, bps)
        p.set_inter_default(st.get("inter_default", 0.0))
        for a, b, bps in st.get("inter", []):
            p.set_inter_bandwidth(a, b, bps)
        for did, server, cls_, cap, mem, load in st["devices"]:
            p.add_device(did, server, cls_, cap, mem, load)
        return p

    def load_state(self, sn: dict):
        self.clear_state()
        for i in sn["instances"]:
            self.put_instance(i["id"], i["block"], i["device"], i["ready"], i["ready_at"],
                              i["last_used"], i["created_seq"], i["executing"], i["queue_len"],
                              i["queued_cost"], i["queued_hwm"])
        for dev, params, kv, act in sn["ledger"]:
            self.set_ledger(dev, params, kv, act)
        for dev, busy in sn["lanes"]:
            self.set_lane(dev, busy)
        for a, b, n in sn["adjacency"]:
            self.set_adjacency(a, b, n)
        for q in sn.get("queries", []):
            if q["kv_owner"] >= 0:
                self.set_kv(q["request"], q["block"], q["kv_owner"], q["kv_pages"])
