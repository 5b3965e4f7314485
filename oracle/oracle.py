"""TEST INFRASTRUCTURE: ctypes wrapper of the CPU oracle (oracle/liboracle.so).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg import
this module, always as the checker or the timed CPU baseline, never as the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(_HERE, "liboracle.so")


class OrBlockDesc(C.Structure):
    _fields_ = [("n_layers", C.c_int), ("d_model", C.c_int), ("n_heads", C.c_int),
                ("head_dim", C.c_int), ("d_ff", C.c_int), ("max_pos", C.c_int),
                ("norm_eps", C.c_float), ("rope_theta", C.c_float), ("init_scale", C.c_float),
                ("seed", C.c_uint64), ("name", C.c_char_p), ("components", C.c_char_p),
                ("ffn_src", C.c_int)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            subprocess.run(["make", "-C", _HERE, "liboracle.so"], check=True,
                           stdout=subprocess.DEVNULL)
        L = C.CDLL(LIB)
        P = C.c_void_p
        L.or_block_create.restype = P
        L.or_block_create.argtypes = [C.POINTER(OrBlockDesc)]
        L.or_block_free.argtypes = [P]
        L.or_block_weight.restype = C.POINTER(C.c_float)
        L.or_block_weight.argtypes = [P, C.c_int, C.c_char_p]
        L.or_block_add_delta.restype = C.c_int
        L.or_block_add_delta.argtypes = [P, C.c_int, C.c_char_p, P]
        L.or_seq_create.restype = P
        L.or_seq_create.argtypes = [P, C.c_int]
        L.or_seq_free.argtypes = [P]
        L.or_seq_len.restype = C.c_int
        L.or_seq_len.argtypes = [P]
        L.or_seq_fill.argtypes = [P, C.c_int, C.c_uint64]
        L.or_seq_kv.restype = C.POINTER(C.c_float)
        L.or_seq_kv.argtypes = [P, C.c_int, C.c_int]
        L.or_block_forward.restype = C.c_int
        L.or_block_forward.argtypes = [P, C.POINTER(P), C.c_int, P, P, P, P, C.c_int]
        L.or_cosine.restype = C.c_double
        L.or_cosine.argtypes = [P, P, C.c_int, C.POINTER(C.c_int)]
        L.or_cosine_rows.argtypes = [P, P, C.c_int, C.c_int, C.c_float, P, P]
        L.or_synth.restype = C.c_float
        L.or_synth.argtypes = [C.c_uint64, C.c_char_p, C.c_uint64, C.c_float]
        L.or_synth_fill.argtypes = [P, C.c_uint64, C.c_uint64, C.c_char_p, C.c_float, C.c_int]
        _lib = L
    return _lib


def _p(a: np.ndarray) -> C.c_void_p:
    return a.ctypes.data_as(C.c_void_p)


class OracleBlock:
    def __init__(self, shape, name: str, seed: int = 1):
        self.shape, self.name = shape, name
        self._nb = name.encode()
        comps = getattr(shape, "comps", None) or "af" * shape.n_layers
        self._cb = comps.encode()
        d = OrBlockDesc(shape.n_layers, shape.d_model, shape.n_heads, shape.head_dim, shape.d_ff,
                        shape.max_pos, shape.norm_eps, shape.rope_theta, shape.init_scale, seed,
                        self._nb, self._cb, getattr(shape, "ffn_src", 0))
        self.h = lib().or_block_create(C.byref(d))
        if not self.h:
            raise ValueError("oracle: bad block shape")

    def weight(self, layer: int, tensor: str) -> np.ndarray:
        s = self.shape
        rows, cols = {"wq": (s.d_model, s.d_model), "wk": (s.d_model, s.d_model),
                      "wv": (s.d_model, s.d_model), "wo": (s.d_model, s.d_model),
                      "wg": (s.d_ff, s.d_model), "wu": (s.d_ff, s.d_model),
                      "wd": (s.d_model, s.d_ff)}[tensor]
        ptr = lib().or_block_weight(self.h, layer, tensor.encode())
        return np.ctypeslib.as_array(ptr, shape=(rows, cols)).copy()

    def add_lora(self, name: str, seed: int, scale_a: float, scale_b: float, rank: int = 16):
        """Folds a LoRA adapter into the restated weights: W_x += B_x A_x for x in q, k, v, o of
        every attention layer, the factors being the synthetic streams be_lora_load generates
        ("lora:<name>:<l>:<t>", include/blockexec.h)."""
        s = self.shape
        d = s.d_model
        n_att = (getattr(s, "comps", None) or "af" * s.n_layers).count("a")
        for layer in range(n_att):
            for x in "qkvo":
                a = synth(rank * d, seed, f"lora:{name}:{layer}:a{x}", scale_a).reshape(rank, d)
                b = synth(d * rank, seed, f"lora:{name}:{layer}:b{x}", scale_b).reshape(d, rank)
                delta = np.ascontiguousarray(b.astype(np.float64) @ a.astype(np.float64),
                                             np.float32)
                if lib().or_block_add_delta(self.h, layer, f"w{x}".encode(), _p(delta)) != 0:
                    raise ValueError("oracle: add_delta failed")

    def new_seq(self, max_tokens: int) -> "OracleSeq":
        return OracleSeq(self, max_tokens)

    def forward(self, seqs, tok_seq, tok_pos, x_in: np.ndarray, threads: int = 0) -> np.ndarray:
        n = len(tok_seq)
        arr = (C.c_void_p * max(1, len(seqs)))(*[s.h for s in seqs])
        ts = np.ascontiguousarray(tok_seq, np.int32)
        tp = np.ascontiguousarray(tok_pos, np.int32)
        x = np.ascontiguousarray(x_in, np.float32)
        out = np.empty_like(x)
        rc = lib().or_block_forward(self.h, arr, n, _p(ts), _p(tp), _p(x), _p(out), threads)
        if rc != 0:
            raise ValueError("oracle: bad token metadata")
        return out

    def __del__(self):
        if getattr(self, "h", None):
            lib().or_block_free(self.h)
            self.h = None


class OracleSeq:
    def __init__(self, block: OracleBlock, max_tokens: int):
        self.block = block
        self.max_tokens = max_tokens
        self.h = lib().or_seq_create(block.h, max_tokens)

    def fill(self, length: int, seed: int = 1) -> None:
        lib().or_seq_fill(self.h, length, seed)

    def kv(self, layer: int, which: int) -> np.ndarray:
        """K (which=0) or V (1) cache of the layer-th attention component, [max_tokens][d]."""
        d = self.block.shape.d_model
        ptr = lib().or_seq_kv(self.h, layer, which)
        return np.ctypeslib.as_array(ptr, shape=(self.max_tokens, d)).copy()

    def __del__(self):
        if getattr(self, "h", None):
            lib().or_seq_free(self.h)
            self.h = None


def cosine(a, b) -> float:
    """signature_similarity restatement; raises ValueError like the reference's invalid_argument."""
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    if a.shape != b.shape:
        raise ValueError("signature length mismatch")
    err = C.c_int(0)
    v = lib().or_cosine(_p(a), _p(b), a.size, C.byref(err))
    if err.value:
        raise ValueError("zero-norm signature")
    return v


def cosine_rows(a: np.ndarray, b: np.ndarray, thr: float):
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    rows, d = a.shape
    cos = np.empty(rows, np.float32)
    acc = np.empty(rows, np.int32)
    lib().or_cosine_rows(_p(a), _p(b), rows, d, thr, _p(cos), _p(acc))
    return cos, acc


def synth(n: int, seed: int, stream_id: str, scale: float, round_bf16: bool = True) -> np.ndarray:
    out = np.empty(n, np.float32)
    lib().or_synth_fill(_p(out), n, seed, stream_id.encode(), scale, 1 if round_bf16 else 0)
    return out
