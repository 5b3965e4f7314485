"""ctypes binding of libblockexec.so (include/blockexec.h, include/blockhost.h).

The product path has no CPU fallback: if the in-tree library is missing or cannot load, every
entry point raises. Build it with ``python -c "import __graft_entry__ as g; g.build()"`` or
``make -C paper_2404_18322_b200/csrc``.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BE_LIB_PATH") or os.path.join(_HERE, "libblockexec.so")

BE_OK = 0
BE_ERRORS = {1: "invalid argument", 2: "bad state", 3: "CUDA failure", 4: "out of device memory",
             5: "runtime error"}
PHASE_PREFILL = 0
PHASE_DECODE = 1


class BlockExecError(RuntimeError):
    """Raised on a non-zero status; `code` mirrors the reference's exception classes."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"{BE_ERRORS.get(code, code)}: {msg}")
        self.code = code


class BlockDesc(C.Structure):
    _fields_ = [("n_layers", C.c_int), ("d_model", C.c_int), ("n_heads", C.c_int),
                ("head_dim", C.c_int), ("d_ff", C.c_int), ("max_pos", C.c_int),
                ("norm_eps", C.c_float), ("rope_theta", C.c_float), ("init_scale", C.c_float),
                ("seed", C.c_uint64), ("name", C.c_char_p), ("components", C.c_char_p),
                ("ffn_src", C.c_int)]


class Token(C.Structure):
    _fields_ = [("src_row", C.c_int32), ("dst_row", C.c_int32), ("kv_slot", C.c_int32),
                ("pos", C.c_int32), ("pt_row", C.c_int32)]


_lib = None


def lib() -> C.CDLL:
    """Loads libblockexec.so once; raises if it is absent (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built; run __graft_entry__.build()")
    L = C.CDLL(LIB_PATH)
    P, I, I64, U64, F = C.c_void_p, C.c_int, C.c_int64, C.c_uint64, C.c_float
    PP = C.POINTER(C.c_void_p)
    sig = {
        "be_ctx_create": (I, [I, PP]),
        "be_ctx_destroy": (I, [P]),
        "be_last_error": (C.c_char_p, [P]),
        "be_ctx_num_sms": (I, [P]),
        "be_ctx_stream": (P, [P]),
        "be_synchronize": (I, [P]),
        "be_block_load": (I, [P, C.POINTER(BlockDesc), PP]),
        "be_block_free": (I, [P]),
        "be_block_param_bytes": (I64, [P]),
        "be_block_kv_bytes_per_token": (I64, [P]),
        "be_block_read_weight": (I, [P, I, C.c_char_p, P]),
        "be_kv_pool_create": (I, [P, P, I, PP]),
        "be_kv_pool_free": (I, [P]),
        "be_kv_pool_data": (P, [P]),
        "be_kv_pool_page_bytes": (I64, [P]),
        "be_kv_pool_read": (I, [P, I64, I64, P]),
        "be_workspace_create": (I, [P, I, I, I, I, I, I, PP]),
        "be_workspace_free": (I, [P]),
        "be_exec_batch": (I, [P, P, P, P, I, I, P, I, I, P, P, P, P]),
        "be_exec_speculative": (I, [P, P, P, P, I, P, P, P, P, F, P, P, P]),
        "be_kv_copy_pages": (I, [P, P, P, P, P, I, P]),
        "be_kv_migrate": (I, [P, P, P, P, P, P, P, I, I, I, P, P]),
        "be_lora_load": (I, [P, P, C.c_char_p, U64, F, F, PP]),
        "be_lora_free": (I, [P]),
        "be_stitch_load": (I, [P, I, I, C.c_char_p, U64, F, PP]),
        "be_stitch_free": (I, [P]),
        "be_stitch_rows": (I, [P, P, P, I, P, P]),
        "be_exec_lora_batch": (I, [P, P, P, P, I, I, P, I, I, P, I, P, P, P, P, P]),
        "be_exec_lora_batch_dev": (I, [P, P, P, P, I, I, P, I, P, I, P, P, P, P, P]),
        "be_exec_batch_dev": (I, [P, P, P, P, I, I, P, I, P, P, P, P]),
        "be_gather_rows": (I, [P, P, P, I, I, P, P]),
        "be_scatter_rows": (I, [P, P, P, I, I, P, P]),
        "be_cosine": (I, [P, P, P, I, I, F, P, P, P]),
        "be_synth_rows": (I, [P, P, I64, U64, C.c_char_p, F, P]),
        "be_gemm_bf16": (I, [P, P, P, P, I, I, I, I, P]),
        "be_pack_weight": (I, [P, P, P, I, I, P]),
        "be_bench_gemm": (I, [P, P, I, P, P, I, I, I, I, C.POINTER(C.c_float)]),
        "be_exec_batch_launches": (I, [P, P, I, I]),
        "be_prof_enable": (I, [P, I]),
        "be_prof_active": (I, [P]),
        "be_prof_read": (I, [P, P, I, P]),
        "be_timeline_enable": (I, [P, I]),
        "be_timeline_begin": (I, [P]),
        "be_timeline_read": (I, [P, P, I, P]),
        "be_attention": (I, [P, P, P, I, I, I, I, P, I, P, P, I, I, P, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def check(rc: int, ctx=None) -> None:
    if rc != BE_OK:
        msg = lib().be_last_error(ctx).decode() if ctx else ""
        raise BlockExecError(rc, msg)
