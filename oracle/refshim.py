"""TEST INFRASTRUCTURE: Python handles over oracle/_ref/libblocksim_ref.so, i.e. the reference's
own blocksim classes (compiled in place from /root/reference by oracle/Makefile). Only tests/
use this, as the parity checker for paper_2404_18322_b200.host and the runner's batch traces.
"""
from __future__ import annotations

import ctypes as C
import os

from paper_2404_18322_b200 import host as H

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(_HERE, "_ref", "libblocksim_ref.so")

_lib = None


def available() -> bool:
    return os.path.exists(REF_LIB)


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(REF_LIB)
        P, I, I64, D = C.c_void_p, C.c_int, C.c_int64, C.c_double
        L.rs_cosine.restype = D
        L.rs_cosine.argtypes = [P, I, P, I, C.POINTER(I)]
        L.rs_plan_migration.restype = I
        L.rs_plan_migration.argtypes = [I, I64, I64, C.POINTER(I64)]
        L.rs_percentile.restype = I
        L.rs_percentile.argtypes = [P, I, D, C.POINTER(D)]
        L.rs_sim_run.restype = P
        L.rs_sim_run.argtypes = [I, I, I, I, I, P, P, I, I64]
        L.rs_sim_run_prefix.restype = P
        L.rs_sim_run_prefix.argtypes = [I, I, I, I, I, P, P, I, P, P]
        L.rs_sim_run_gpu.restype = P
        L.rs_sim_run_gpu.argtypes = [C.c_char_p, I, I, I, I, I, I, I, P, P, I, I64, C.c_uint64,
                                     C.c_float, P]
        for n, r, a in [("rs_sim_free", None, [P]), ("rs_sim_error", C.c_char_p, [P]),
                        ("rs_sim_report", C.c_char_p, [P]), ("rs_sim_n_blocks", I, [P]),
                        ("rs_sim_block_id", C.c_char_p, [P, I]),
                        ("rs_sim_block_kinds", C.c_char_p, [P, I]), ("rs_sim_n_chains", I, [P]),
                        ("rs_sim_chain", I, [P, I, P, I]), ("rs_sim_req_model", I, [P, I]),
                        ("rs_sim_n_batches", I, [P]), ("rs_sim_batch", I, [P, I, P, P, I])]:
            fn = getattr(L, n)
            fn.restype, fn.argtypes = r, a
        _lib = L
    return _lib


class RefPool(H.Pool):
    prefix = "rs_"

    def __init__(self, n_blocks: int = 8, n_devices: int = 2):
        L = lib()
        H._bind("rs_", L)
        super().__init__(_lib=L, _handle=L.rs_pool_new(n_blocks, n_devices))


class RefKvStore(H.KvStore):
    prefix = "rs_"

    def __init__(self, n_devices: int = 2):
        L = lib()
        H._bind("rs_", L)
        super().__init__(_lib=L, _handle=L.rs_kv_new(n_devices))


def cosine(a, b) -> float:
    import numpy as np
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    err = C.c_int(0)
    v = lib().rs_cosine(a.ctypes.data, a.size, b.ctypes.data, b.size, C.byref(err))
    if err.value:
        raise ValueError("signature_similarity rejected its input")
    return v


def plan_migration(pages: int, rec_us: int, cp_us: int):
    out = (C.c_int64 * 6)()
    rc = lib().rs_plan_migration(pages, rec_us, cp_us, out)
    if rc:
        raise ValueError("plan_migration rejected its input")
    return tuple(int(x) for x in out)


def percentile(values, q: float) -> float:
    import numpy as np
    v = np.ascontiguousarray(values, np.float64)
    out = C.c_double(0)
    rc = lib().rs_percentile(v.ctypes.data, v.size, q, C.byref(out))
    if rc:
        raise ValueError("percentile rejected q")
    return out.value


def simulate(n_layers: int, dim: int, n_lora: int, first_adapted: int, prompts, outputs,
             max_batch_tokens: int = 4096, arrival_gap_us: int = 0):
    """Runs the reference Simulation; returns (blocks, kinds, chains, req_model, trace)."""
    import numpy as np
    p = np.ascontiguousarray(prompts, np.int32)
    o = np.ascontiguousarray(outputs, np.int32)
    L = lib()
    h = L.rs_sim_run(n_layers, dim, n_lora, first_adapted, len(p), p.ctypes.data, o.ctypes.data,
                     max_batch_tokens, arrival_gap_us)
    try:
        err = L.rs_sim_error(h).decode()
        if err:
            raise RuntimeError(err)
        nb = L.rs_sim_n_blocks(h)
        blocks = [L.rs_sim_block_id(h, i).decode() for i in range(nb)]
        kinds = [L.rs_sim_block_kinds(h, i).decode() for i in range(nb)]
        chains = []
        buf = (C.c_int32 * 4096)()
        for m in range(L.rs_sim_n_chains(h)):
            n = L.rs_sim_chain(h, m, buf, 4096)
            chains.append([int(buf[i]) for i in range(n)])
        req_model = [L.rs_sim_req_model(h, r) for r in range(len(p))]
        trace = []
        rec = (C.c_int32 * 4)()
        mem = (C.c_int32 * (3 * 65536))()
        for i in range(L.rs_sim_n_batches(h)):
            L.rs_sim_batch(h, i, rec, mem, 65536)
            members = [(int(mem[3 * j]), int(mem[3 * j + 1]), int(mem[3 * j + 2]))
                       for j in range(rec[3])]
            trace.append((int(rec[0]), int(rec[1]), int(rec[2]), members))
        return blocks, kinds, chains, req_model, trace
    finally:
        L.rs_sim_free(h)


def simulate_prefix(n_layers: int, dim: int, n_lora: int, first_adapted: int, prompts, outputs,
                    prefix_group, prefix_tokens, max_batch_tokens: int = 4096):
    """The reference Simulation with prefix groups: (report dict, batch trace)."""
    import json
    import numpy as np
    p = np.ascontiguousarray(prompts, np.int32)
    o = np.ascontiguousarray(outputs, np.int32)
    g = np.ascontiguousarray(prefix_group, np.int32)
    t = np.ascontiguousarray(prefix_tokens, np.int32)
    L = lib()
    h = L.rs_sim_run_prefix(n_layers, dim, n_lora, first_adapted, len(p), p.ctypes.data,
                            o.ctypes.data, max_batch_tokens, g.ctypes.data, t.ctypes.data)
    try:
        err = L.rs_sim_error(h).decode()
        if err:
            raise RuntimeError(err)
        rep = json.loads(L.rs_sim_report(h).decode())
        trace = []
        rec = (C.c_int32 * 4)()
        mem = (C.c_int32 * (3 * 65536))()
        for i in range(L.rs_sim_n_batches(h)):
            L.rs_sim_batch(h, i, rec, mem, 65536)
            members = [(int(mem[3 * j]), int(mem[3 * j + 1]), int(mem[3 * j + 2]))
                       for j in range(rec[3])]
            trace.append((int(rec[0]), int(rec[1]), int(rec[2]), members))
        return rep, trace
    finally:
        L.rs_sim_free(h)


def simulate_gpu(n_layers: int, dim: int, n_heads: int, n_lora: int, first_adapted: int,
                 prompts, outputs, max_batch_tokens: int = 4096, seed: int = 1,
                 init_scale: float = 0.02 * 3 ** 0.5, device: int = 0, product_lib=None):
    """The reference Simulation (the same zoo and requests as simulate) driving the product's
    batch executor (bh_executor_run_batch) through its Engine trace hook: every batch it forms
    runs on the GPU. Returns (decode rows [n_requests][dim] as float32, batch trace)."""
    import numpy as np
    if product_lib is None:
        product_lib = os.path.join(os.path.dirname(_HERE), "paper_2404_18322_b200",
                                   "libblockexec.so")
    p = np.ascontiguousarray(prompts, np.int32)
    o = np.ascontiguousarray(outputs, np.int32)
    rows = np.zeros((len(p), dim), np.uint16)
    L = lib()
    h = L.rs_sim_run_gpu(product_lib.encode(), device, n_layers, dim, n_heads, n_lora,
                         first_adapted, len(p), p.ctypes.data, o.ctypes.data, max_batch_tokens,
                         0, seed, init_scale, rows.ctypes.data)
    try:
        err = L.rs_sim_error(h).decode()
        if err:
            raise RuntimeError(err)
        trace = []
        rec = (C.c_int32 * 4)()
        mem = (C.c_int32 * (3 * 65536))()
        for i in range(L.rs_sim_n_batches(h)):
            L.rs_sim_batch(h, i, rec, mem, 65536)
            members = [(int(mem[3 * j]), int(mem[3 * j + 1]), int(mem[3 * j + 2]))
                       for j in range(rec[3])]
            trace.append((int(rec[0]), int(rec[1]), int(rec[2]), members))
    finally:
        L.rs_sim_free(h)
    f32 = (rows.astype(np.uint32) << 16).view(np.float32)
    return f32, trace


def profile_component_us(path: str, cls: str, prefill: bool, batch: float, tokens: float) -> float:
    """The reference's load_profiles + CostModel::component_us on a profiles.json."""
    L = lib()
    fn = L.rs_profile_component_us
    fn.restype = C.c_int
    fn.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_double, C.c_double,
                   C.POINTER(C.c_double), C.c_char_p, C.c_int]
    out = C.c_double(0)
    err = C.create_string_buffer(512)
    if fn(path.encode(), cls.encode(), 1 if prefill else 0, batch, tokens, C.byref(out), err,
          512) != 0:
        raise ValueError(err.value.decode())
    return out.value


def policy_trace(spec: dict) -> dict:
    """Runs the reference Simulation described by `spec` (see rs_policy_trace_run in
    oracle/ref_shim.cpp) and returns its static description plus the Scheduler's decisions at
    snapshots taken while it runs."""
    import json
    L = lib()
    if not getattr(L, "_policy_bound", False):
        L.rs_policy_trace_run.restype = C.c_void_p
        L.rs_policy_trace_run.argtypes = [C.c_char_p]
        for n in ("rs_policy_trace_json", "rs_policy_trace_error"):
            getattr(L, n).restype = C.c_char_p
            getattr(L, n).argtypes = [C.c_void_p]
        L.rs_policy_trace_free.restype = None
        L.rs_policy_trace_free.argtypes = [C.c_void_p]
        L._policy_bound = True
    h = L.rs_policy_trace_run(json.dumps(spec).encode())
    try:
        err = L.rs_policy_trace_error(h).decode()
        if err:
            raise RuntimeError(err)
        return json.loads(L.rs_policy_trace_json(h).decode())
    finally:
        L.rs_policy_trace_free(h)
