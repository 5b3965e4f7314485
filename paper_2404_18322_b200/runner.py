"""Python handle over the C++ executor loop (include/blockhost.h bh_runner_*)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import check, lib, BlockDesc, BlockExecError
from .device import Context
from .workloads import Workload


class BatchRec(C.Structure):
    _fields_ = [("instance", C.c_int32), ("block", C.c_int32), ("phase", C.c_int32),
                ("n_members", C.c_int32), ("first_member", C.c_int32)]


class StepStats(C.Structure):
    _fields_ = [("weight_bytes", C.c_double), ("kv_bytes", C.c_double),
                ("act_bytes", C.c_double), ("flops", C.c_double), ("launches", C.c_int),
                ("graph_replayed", C.c_int)]


class WorkloadC(C.Structure):
    _fields_ = [("n_blocks", C.c_int), ("blocks", C.c_void_p), ("n_tenants", C.c_int),
                ("chain_ptr", C.c_void_p), ("chain_blocks", C.c_void_p),
                ("n_requests", C.c_int), ("req_tenant", C.c_void_p),
                ("req_prompt", C.c_void_p), ("req_output", C.c_void_p),
                ("max_batch_tokens", C.c_int), ("mode", C.c_int), ("use_graphs", C.c_int),
                ("seed", C.c_uint64), ("dry_run", C.c_int), ("plan_ahead", C.c_int),
                ("block_lora_base", C.c_void_p), ("block_lora_name", C.c_void_p),
                ("n_spec_blocks", C.c_int), ("spec_blocks", C.c_void_p),
                ("spec_threshold", C.c_float), ("spec_keep", C.c_float),
                ("req_prefix_group", C.c_void_p), ("req_prefix_tokens", C.c_void_p)]


class SpecStats(C.Structure):
    _fields_ = [("runs", C.c_int64), ("rows", C.c_int64), ("accepted", C.c_int64),
                ("cos_sum", C.c_double), ("cos_min", C.c_double)]


_bound = False


def _bind():
    global _bound
    if _bound:
        return
    L = lib()
    P, I = C.c_void_p, C.c_int
    for name, res, args in [
        ("bh_runner_create", I, [P, P, C.POINTER(C.c_void_p)]),
        ("bh_runner_free", I, [P]),
        ("bh_runner_last_error", C.c_char_p, [P]),
        ("bh_runner_run", I, [P, I]),
        ("bh_runner_decode_step", I, [P, P, P, P]),
        ("bh_runner_live_requests", I, [P]),
        ("bh_runner_tokens_generated", C.c_int64, [P]),
        ("bh_runner_trace", I, [P, P, I, P, P, P, P, I, P]),
        ("bh_runner_clear_trace", I, [P]),
        ("bh_runner_arena", P, [P]),
        ("bh_runner_prefill_arena", P, [P, C.POINTER(C.c_int64)]),
        ("bh_runner_decode_group", I, [P, I, P, I, P, P, P]),
        ("bh_runner_step_stats", I, [P, P]),
        ("bh_runner_serve", I, [P, P, P, P]),
        ("bh_runner_spec_stats", I, [P, P]),
        ("bh_runner_kv_bytes", I, [P, P, P]),
        ("bh_runner_adopt", I, [P, I, P, P, P]),
        ("bh_runner_request_state", I, [P, I, P, P, P]),
        ("bh_runner_kv_segment", I, [P, I, I, P, I, P, P]),
        ("bh_runner_kv_pool", P, [P, I]),
    ]:
        fn = getattr(L, name)
        fn.restype, fn.argtypes = res, args
    _bound = True


class Runner:
    """Multi-tenant block-chain execution on one GPU.

    mode 0: the reference's event order (arrivals at t=0, interleaved prefill/decode);
    mode 1: lockstep (all prompts prefilled, then decode one token for everyone per step).
    """

    def __init__(self, ctx: Context | None, wl: Workload, mode: int = 1, use_graphs: bool = True,
                 dry_run: bool = False, plan_ahead: bool = False, spec_blocks=None,
                 spec_threshold: float = 0.95, spec_keep: float = 0.5):
        """ctx None with dry_run=True runs the control plane alone (no GPU work).
        spec_blocks: block indices whose decode runs speculatively (bh_workload.spec_blocks)."""
        _bind()
        self.ctx, self.wl = ctx, wl
        s = wl.shape
        self._names = [n.encode() for n in wl.block_names]
        comps = wl.block_comps or [s.comps] * len(wl.block_names)
        self._comps = [c.encode() for c in comps]
        descs = (BlockDesc * len(wl.block_names))()
        for i, nm in enumerate(self._names):
            descs[i] = BlockDesc(s.n_layers, s.d_model, s.n_heads, s.head_dim, s.d_ff, s.max_pos,
                                 s.norm_eps, s.rope_theta, s.init_scale, wl.seed, nm,
                                 self._comps[i], s.ffn_src)
        ptr = np.zeros(len(wl.chains) + 1, np.int32)
        flat = []
        for t, ch in enumerate(wl.chains):
            flat += ch
            ptr[t + 1] = len(flat)
        self._keep = [descs, ptr, np.array(flat, np.int32),
                      np.array(wl.req_tenant, np.int32), np.array(wl.req_prompt, np.int32),
                      np.array(wl.req_output, np.int32)]
        k = self._keep
        lora_base, lora_names = None, None
        if getattr(wl, "block_lora", None):
            base = np.array([-1 if x is None else x[0] for x in wl.block_lora], np.int32)
            names = (C.c_char_p * len(wl.block_lora))(
                *[None if x is None else x[1].encode() for x in wl.block_lora])
            self._keep += [base, names]
            lora_base, lora_names = base.ctypes.data, C.cast(names, C.c_void_p)
        spec = np.ascontiguousarray(list(spec_blocks or []) or [0], np.int32)
        self._keep.append(spec)
        pg = pt = None
        if getattr(wl, "req_prefix_group", None) is not None:
            pga = np.ascontiguousarray(wl.req_prefix_group, np.int32)
            pta = np.ascontiguousarray(wl.req_prefix_tokens, np.int32)
            self._keep += [pga, pta]
            pg, pt = pga.ctypes.data, pta.ctypes.data
        w = WorkloadC(len(wl.block_names), C.cast(descs, C.c_void_p), len(wl.chains),
                      k[1].ctypes.data, k[2].ctypes.data, wl.n_requests, k[3].ctypes.data,
                      k[4].ctypes.data, k[5].ctypes.data, wl.max_batch_tokens, mode,
                      1 if use_graphs else 0, wl.seed, 1 if dry_run else 0,
                      1 if plan_ahead else 0, lora_base, lora_names,
                      len(spec_blocks or []), spec.ctypes.data, spec_threshold, spec_keep,
                      pg, pt)
        h = C.c_void_p()
        rc = lib().bh_runner_create(ctx.h if ctx is not None else None, C.byref(w), C.byref(h))
        if rc != 0:
            msg = lib().be_last_error(ctx.h).decode() if ctx is not None else ""
            raise BlockExecError(rc, "bh_runner_create failed (see stderr): " + msg)
        self.h = h

    def _check(self, rc):
        if rc != 0:
            raise BlockExecError(rc, lib().bh_runner_last_error(self.h).decode())

    def run(self, max_batches: int = 0) -> None:
        self._check(lib().bh_runner_run(self.h, max_batches))

    def decode_step(self, host_in=None, host_out=None) -> int:
        n = C.c_int(0)
        pin = C.c_void_p(host_in.data_ptr() if hasattr(host_in, "data_ptr") else
                         (host_in.ctypes.data if host_in is not None else 0))
        pout = C.c_void_p(host_out.data_ptr() if hasattr(host_out, "data_ptr") else
                          (host_out.ctypes.data if host_out is not None else 0))
        self._check(lib().bh_runner_decode_step(self.h, pin, pout, C.byref(n)))
        return n.value

    def decode_group(self, group: int, requests, host_in=None, host_out=None) -> int:
        """One lockstep token for a request group (pipeline micro-batch) only."""
        req = np.ascontiguousarray(requests, np.int32)
        n = C.c_int(0)
        pin = C.c_void_p(host_in.data_ptr() if host_in is not None else 0)
        pout = C.c_void_p(host_out.data_ptr() if host_out is not None else 0)
        self._check(lib().bh_runner_decode_group(self.h, group, req.ctypes.data, req.size, pin,
                                                 pout, C.byref(n)))
        return n.value

    def serve(self, arrival_us):
        """Live serving on a fresh lockstep runner (bh_runner_serve): request i arrives
        arrival_us[i] after the call; returns (first_token_us, completion_us) arrays."""
        arr = np.ascontiguousarray(arrival_us, np.int64)
        if arr.size != self.wl.n_requests:
            raise ValueError("one arrival time per request")
        first = np.full(arr.size, -1, np.int64)
        done = np.full(arr.size, -1, np.int64)
        self._check(lib().bh_runner_serve(self.h, arr.ctypes.data, first.ctypes.data,
                                          done.ctypes.data))
        return first, done

    def prefill_arena(self):
        """(device pointer, rows) of the prompt hidden-state rows (all requests, in order)."""
        rows = C.c_int64(0)
        ptr = lib().bh_runner_prefill_arena(self.h, C.byref(rows))
        return ptr, rows.value

    @property
    def live(self) -> int:
        return lib().bh_runner_live_requests(self.h)

    @property
    def tokens_generated(self) -> int:
        return lib().bh_runner_tokens_generated(self.h)

    @property
    def arena_ptr(self) -> int:
        return lib().bh_runner_arena(self.h)

    def step_stats(self) -> dict:
        s = StepStats()
        self._check(lib().bh_runner_step_stats(self.h, C.byref(s)))
        return {f: getattr(s, f) for f, _ in StepStats._fields_}

    def adopt(self, idx, ctx, generated) -> None:
        """Take over requests mid-decode (bh_runner_adopt): KV segments are created empty of
        content on fresh page slots; copy the migrated pages in before the next step."""
        a = [np.ascontiguousarray(v, np.int32) for v in (idx, ctx, generated)]
        self._check(lib().bh_runner_adopt(self.h, a[0].size, a[0].ctypes.data, a[1].ctypes.data,
                                          a[2].ctypes.data))

    def request_state(self, idx: int) -> tuple[int, int, bool]:
        c, g, d = C.c_int32(0), C.c_int32(0), C.c_int32(0)
        self._check(lib().bh_runner_request_state(self.h, idx, C.byref(c), C.byref(g),
                                                  C.byref(d)))
        return c.value, g.value, bool(d.value)

    def kv_segment(self, idx: int, block: int) -> tuple[list, int]:
        """(page slots in token order, tokens) of request idx's segment at block."""
        buf = (C.c_int32 * 4096)()
        n, t = C.c_int(0), C.c_int(0)
        self._check(lib().bh_runner_kv_segment(self.h, idx, block, buf, 4096, C.byref(n),
                                               C.byref(t)))
        return list(buf[:n.value]), t.value

    def kv_pool(self, block: int) -> int:
        return lib().bh_runner_kv_pool(self.h, block) or 0

    def kv_bytes(self) -> tuple[int, int]:
        """(bytes of KV pages in use, bytes saved by prefix sharing)."""
        u, sv = C.c_int64(0), C.c_int64(0)
        self._check(lib().bh_runner_kv_bytes(self.h, C.byref(u), C.byref(sv)))
        return u.value, sv.value

    def spec_stats(self) -> dict:
        s = SpecStats()
        self._check(lib().bh_runner_spec_stats(self.h, C.byref(s)))
        d = {f: getattr(s, f) for f, _ in SpecStats._fields_}
        d["accept_rate"] = d["accepted"] / d["rows"] if d["rows"] else None
        d["cos_mean"] = d["cos_sum"] / d["rows"] if d["rows"] else None
        return d

    def trace(self):
        """[(instance_idx, block_idx, phase, [(req, step, ctx), ...]), ...]"""
        n, m = C.c_int(0), C.c_int(0)
        self._check(lib().bh_runner_trace(self.h, None, 0, C.byref(n), None, None, None, 0,
                                          C.byref(m)))
        recs = (BatchRec * max(1, n.value))()
        req = np.zeros(max(1, m.value), np.int32)
        step = np.zeros_like(req)
        ctxs = np.zeros_like(req)
        self._check(lib().bh_runner_trace(self.h, C.cast(recs, C.c_void_p), n.value, C.byref(n),
                                          req.ctypes.data, step.ctypes.data, ctxs.ctypes.data,
                                          m.value, C.byref(m)))
        out = []
        for i in range(n.value):
            r = recs[i]
            mem = [(int(req[j]), int(step[j]), int(ctxs[j]))
                   for j in range(r.first_member, r.first_member + r.n_members)]
            out.append((r.instance, r.block, r.phase, mem))
        return out

    def clear_trace(self):
        self._check(lib().bh_runner_clear_trace(self.h))

    def close(self):
        if getattr(self, "h", None):
            lib().bh_runner_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
