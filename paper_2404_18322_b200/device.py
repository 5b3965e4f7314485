"""Python handles over the C ABI (include/blockexec.h): context, blocks, KV pools, workspaces.

PyTorch is only plumbing here (device buffers and streams); every computation runs in the
sm_100a kernels of libblockexec.so.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from dataclasses import dataclass

import numpy as np

from ._lib import BlockDesc, Token, check, lib, PHASE_DECODE, PHASE_PREFILL  # noqa: F401

PAGE_TOKENS = 16  # blocksim kPageTokens (proj/core/include/blocksim/kv.hpp:16)


@dataclass(frozen=True)
class BlockShape:
    """Decoder-layer run served as one block (zoo.hpp:29-54 BlockDescriptor, as layers)."""
    n_layers: int
    d_model: int
    n_heads: int
    d_ff: int
    max_pos: int = 4096
    norm_eps: float = 1e-5
    rope_theta: float = 10000.0
    init_scale: float = 0.02 * 3 ** 0.5  # uniform with std 0.02
    components: str | None = None  # 'a'/'f' sequence (zoo components); None = n_layers x "af"
    ffn_src: int = 0  # > d_ff: FFN pruned to the first d_ff channels of a d_ff = ffn_src block

    def surrogate(self, keep: float = 0.5) -> "BlockShape":
        """The speculation draft of this block: same attention, FFN structured-pruned to the
        first keep*d_ff channels (PAPER.md:501-507 surrogate; C5 uses 50%)."""
        f = max(64, int(self.d_ff * keep) // 64 * 64)
        return dataclasses.replace(self, d_ff=f, ffn_src=self.ffn_src or self.d_ff)

    @property
    def head_dim(self) -> int:
        return self.d_model // self.n_heads

    @property
    def comps(self) -> str:
        return self.components if self.components is not None else "af" * self.n_layers

    @property
    def n_attention(self) -> int:
        return self.comps.count("a")

    @property
    def kv_bytes_per_token(self) -> int:
        # CostModel::kv_bytes_per_token: 4 * embed_dim per attention component (costmodel.cpp:114-127)
        return 4 * self.d_model * self.n_attention

    @property
    def param_bytes(self) -> int:
        d, f = self.d_model, self.d_ff
        return 2 * (self.comps.count("a") * 4 * d * d + self.comps.count("f") * 3 * d * f)


def _ptr(t) -> C.c_void_p:
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


PROF_CLASSES = ["gather", "rms", "gemm_qkv", "attention", "gemm_o", "gemm_gate_up", "gemm_down",
                "scatter"]


class ProfRec(C.Structure):
    _fields_ = [("cls", C.c_int32), ("ntok", C.c_int32), ("n", C.c_int32), ("k", C.c_int32),
                ("ms", C.c_float), ("bytes", C.c_double), ("flops", C.c_double)]


class TimelineRec(C.Structure):
    _fields_ = [("slot", C.c_int32), ("cls", C.c_int32), ("start_first", C.c_uint64),
                ("start_last", C.c_uint64), ("go_first", C.c_uint64), ("end_last", C.c_uint64)]


class Context:
    def __init__(self, device: int = 0):
        self.device = device
        h = C.c_void_p()
        rc = lib().be_ctx_create(device, C.byref(h))
        if rc != 0:
            check(rc)
        self.h = h

    @property
    def stream(self) -> C.c_void_p:
        return C.c_void_p(lib().be_ctx_stream(self.h))

    @property
    def num_sms(self) -> int:
        return lib().be_ctx_num_sms(self.h)

    def sync(self) -> None:
        check(lib().be_synchronize(self.h), self.h)

    def prof_enable(self, on: bool = True) -> None:
        """Per-launch event timing of exec_batch kernels (include/blockexec.h be_prof_*)."""
        check(lib().be_prof_enable(self.h, 1 if on else 0), self.h)

    def timeline_enable(self, cap: int = 4096) -> None:
        """Kernel timeline inside graph replays (include/blockexec.h be_timeline_*)."""
        check(lib().be_timeline_enable(self.h, cap), self.h)

    def timeline_begin(self) -> None:
        check(lib().be_timeline_begin(self.h), self.h)

    def timeline_read(self) -> list[dict]:
        n = C.c_int(0)
        check(lib().be_timeline_read(self.h, None, 0, C.byref(n)), self.h)
        recs = (TimelineRec * max(1, n.value))()
        check(lib().be_timeline_read(self.h, C.cast(recs, C.c_void_p), n.value, C.byref(n)),
              self.h)
        return [{"slot": r.slot, "cls": PROF_CLASSES[r.cls], "start_first": r.start_first,
                 "start_last": r.start_last, "go_first": r.go_first, "end_last": r.end_last}
                for r in recs[:n.value]]

    def prof_read(self) -> list[dict]:
        n = C.c_int(0)
        check(lib().be_prof_read(self.h, None, 0, C.byref(n)), self.h)
        recs = (ProfRec * max(1, n.value))()
        check(lib().be_prof_read(self.h, C.cast(recs, C.c_void_p), n.value, C.byref(n)), self.h)
        return [{"cls": PROF_CLASSES[r.cls], "ntok": r.ntok, "n": r.n, "k": r.k, "ms": r.ms,
                 "bytes": r.bytes, "flops": r.flops} for r in recs[:n.value]]

    def close(self) -> None:
        if self.h:
            lib().be_ctx_destroy(self.h)
            self.h = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass


class Block:
    """One block's weights on the device (synthetic, generated from (seed, name))."""

    def __init__(self, ctx: Context, shape: BlockShape, name: str, seed: int = 1):
        self.ctx, self.shape, self.name, self.seed = ctx, shape, name, seed
        self._name_b = name.encode()
        self._comps_b = shape.comps.encode()
        desc = BlockDesc(shape.n_layers, shape.d_model, shape.n_heads, shape.head_dim, shape.d_ff,
                         shape.max_pos, shape.norm_eps, shape.rope_theta, shape.init_scale, seed,
                         self._name_b, self._comps_b, shape.ffn_src)
        h = C.c_void_p()
        check(lib().be_block_load(ctx.h, C.byref(desc), C.byref(h)), ctx.h)
        self.h = h

    def read_weight(self, layer: int, tensor: str) -> np.ndarray:
        s = self.shape
        rows, cols = {"wq": (s.d_model, s.d_model), "wk": (s.d_model, s.d_model),
                      "wv": (s.d_model, s.d_model), "wo": (s.d_model, s.d_model),
                      "wg": (s.d_ff, s.d_model), "wu": (s.d_ff, s.d_model),
                      "wd": (s.d_model, s.d_ff)}[tensor]
        out = np.empty((rows, cols), np.float32)
        check(lib().be_block_read_weight(self.h, layer, tensor.encode(),
                                         out.ctypes.data_as(C.c_void_p)), self.ctx.h)
        return out

    def free(self):
        if self.h:
            lib().be_block_free(self.h)
            self.h = None


class KvPool:
    """Block-local paged KV pool: [page][layer][K|V][head][16][head_dim] bf16."""

    def __init__(self, ctx: Context, block: Block, n_pages: int):
        self.ctx, self.block, self.n_pages = ctx, block, n_pages
        h = C.c_void_p()
        check(lib().be_kv_pool_create(ctx.h, block.h, n_pages, C.byref(h)), ctx.h)
        self.h = h

    @property
    def data_ptr(self) -> int:
        return lib().be_kv_pool_data(self.h)

    @property
    def page_bytes(self) -> int:
        return lib().be_kv_pool_page_bytes(self.h)

    def read(self, n_elems: int, offset_elems: int = 0) -> np.ndarray:
        """Copies bf16 pool elements to host, returned as fp32."""
        raw = np.empty(n_elems, np.uint16)
        check(lib().be_kv_pool_read(self.h, offset_elems * 2, n_elems * 2,
                                    raw.ctypes.data_as(C.c_void_p)), self.ctx.h)
        return (raw.astype(np.uint32) << 16).view(np.float32)

    def free(self):
        if self.h:
            lib().be_kv_pool_free(self.h)
            self.h = None


class Workspace:
    def __init__(self, ctx: Context, shape: BlockShape, max_tokens: int, max_rows: int,
                 max_pages: int):
        self.ctx, self.shape = ctx, shape
        self.max_tokens, self.max_rows, self.max_pages = max_tokens, max_rows, max_pages
        h = C.c_void_p()
        check(lib().be_workspace_create(ctx.h, shape.d_model, shape.d_ff, shape.n_heads,
                                        max_tokens, max_rows, max_pages, C.byref(h)), ctx.h)
        self.h = h

    def free(self):
        if self.h:
            lib().be_workspace_free(self.h)
            self.h = None


def tokens_array(rows) -> "C.Array":
    """rows: iterable of (src_row, dst_row, kv_slot, pos, pt_row)."""
    rows = list(rows)
    arr = (Token * max(1, len(rows)))()
    for i, r in enumerate(rows):
        arr[i] = Token(*[int(v) for v in r])
    return arr


def exec_batch(ctx: Context, block: Block, pool: KvPool, ws: Workspace, phase: int, tokens,
               page_table: np.ndarray, arena_in, arena_out, stream=None) -> None:
    """One per-block batched execution (the call that replaces batch_duration_us)."""
    toks = tokens_array(tokens)
    n = len(tokens)
    pt = np.ascontiguousarray(page_table, dtype=np.int32)
    check(lib().be_exec_batch(ctx.h, block.h, pool.h, ws.h, phase, n, C.cast(toks, C.c_void_p),
                              pt.shape[0], pt.shape[1], pt.ctypes.data_as(C.c_void_p),
                              _ptr(arena_in), _ptr(arena_out),
                              stream if stream is not None else C.c_void_p(0)), ctx.h)


class Lora:
    """A rank-16 LoRA adapter of a block's attention components (be_lora_load): W'_x = W_x +
    B_x A_x, x in q, k, v, o; synthetic factors from the stream "lora:<name>:<layer>:<t>"."""

    def __init__(self, ctx: Context, base: "Block", name: str, seed: int = 1,
                 scale_a: float | None = None, scale_b: float | None = None):
        self.ctx, self.name, self.seed = ctx, name, seed
        s = base.shape.init_scale
        self.scale_a = s if scale_a is None else scale_a
        self.scale_b = s if scale_b is None else scale_b
        h = C.c_void_p()
        check(lib().be_lora_load(ctx.h, base.h, name.encode(), seed, self.scale_a, self.scale_b,
                                 C.byref(h)), ctx.h)
        self.h = h

    def free(self):
        if self.h:
            lib().be_lora_free(self.h)
            self.h = None


def exec_lora_batch(ctx: Context, block: "Block", pool: "KvPool", ws: "Workspace", phase: int,
                    tokens, page_table: np.ndarray, loras, lora_idx, arena_in, arena_out,
                    stream=None) -> None:
    """exec_batch with adapters: token i uses loras[lora_idx[i]] (-1: the base block)."""
    toks = tokens_array(tokens)
    n = len(tokens)
    pt = np.ascontiguousarray(page_table, dtype=np.int32)
    idx = np.ascontiguousarray(lora_idx, dtype=np.int32)
    arr = (C.c_void_p * max(1, len(loras)))(*[lo.h.value for lo in loras])
    check(lib().be_exec_lora_batch(ctx.h, block.h, pool.h, ws.h, phase, n,
                                   C.cast(toks, C.c_void_p), pt.shape[0], pt.shape[1],
                                   pt.ctypes.data_as(C.c_void_p), len(loras), arr,
                                   idx.ctypes.data_as(C.c_void_p), _ptr(arena_in),
                                   _ptr(arena_out),
                                   stream if stream is not None else C.c_void_p(0)), ctx.h)


class Stitch:
    """Width adapter between equivalent blocks of different embed dims (be_stitch_load):
    y = x W^T, W [dim_out][dim_in] synthetic from stream "stitch:<name>"."""

    def __init__(self, ctx: Context, dim_in: int, dim_out: int, name: str, seed: int = 1,
                 scale: float = 0.02 * 3 ** 0.5):
        self.ctx, self.dim_in, self.dim_out, self.name, self.seed, self.scale = (
            ctx, dim_in, dim_out, name, seed, scale)
        h = C.c_void_p()
        check(lib().be_stitch_load(ctx.h, dim_in, dim_out, name.encode(), seed, scale,
                                   C.byref(h)), ctx.h)
        self.h = h

    def __call__(self, x, out, stream=None) -> None:
        check(lib().be_stitch_rows(self.ctx.h, self.h, _ptr(x), x.shape[0], _ptr(out),
                                   stream if stream is not None else C.c_void_p(0)), self.ctx.h)

    def free(self):
        if self.h:
            lib().be_stitch_free(self.h)
            self.h = None


class SpecStage(C.Structure):
    _fields_ = [("blk", C.c_void_p), ("pool", C.c_void_p), ("ws", C.c_void_p),
                ("tokens", C.c_void_p), ("n_pt_rows", C.c_int), ("pt_stride", C.c_int),
                ("page_table", C.c_void_p)]


def exec_speculative(ctx: Context, verify, draft, nxt, x_in, y_draft, y_true, z_out,
                     threshold: float = 0.95):
    """One speculative decode step (include/blockexec.h be_exec_speculative). Each stage is
    (Block, KvPool, Workspace, tokens, page_table). Returns (cos[n], accept[n], n_accepted)."""
    keep, stages = [], []
    for blk, pool, ws, tokens, pt in (verify, draft, nxt):
        toks = tokens_array(tokens)
        pt = np.ascontiguousarray(pt, dtype=np.int32)
        keep += [toks, pt]
        stages.append(SpecStage(blk.h.value, pool.h.value, ws.h.value,
                                C.cast(toks, C.c_void_p).value, pt.shape[0], pt.shape[1],
                                pt.ctypes.data))
    n = len(verify[3])
    cos = np.zeros(n, np.float32)
    acc = np.zeros(n, np.int32)
    n_acc = C.c_int(0)
    check(lib().be_exec_speculative(ctx.h, C.byref(stages[0]), C.byref(stages[1]),
                                    C.byref(stages[2]), n, _ptr(x_in), _ptr(y_draft),
                                    _ptr(y_true), _ptr(z_out), threshold,
                                    cos.ctypes.data_as(C.c_void_p),
                                    acc.ctypes.data_as(C.c_void_p), C.byref(n_acc)), ctx.h)
    return cos, acc, n_acc.value


def kv_copy_pages(ctx: Context, src_pool: "KvPool", dst_pool: "KvPool", src_slots, dst_slots,
                  stream=None) -> None:
    """Copy whole KV pages between pools (same GPU or peer GPUs): the data path of a KV
    migration whose page pairs come from KvStore.move_segment_slots."""
    s = np.ascontiguousarray(src_slots, np.int32)
    d = np.ascontiguousarray(dst_slots, np.int32)
    check(lib().be_kv_copy_pages(ctx.h, src_pool.h, dst_pool.h, s.ctypes.data_as(C.c_void_p),
                                 d.ctypes.data_as(C.c_void_p), len(s),
                                 stream if stream is not None else C.c_void_p(0)), ctx.h)


def kv_migrate(ctx: Context, blk: "Block", src_pool: "KvPool", dst_pool: "KvPool",
               ws: "Workspace", src_slots, dst_slots, n_recompute: int = 0, head_rows=None,
               head_tokens: int | None = None, stream=None) -> None:
    """KV migration with overlapped recompute / copy (be_kv_migrate): the first n_recompute
    pages are rebuilt on the destination by a chunked prefill of `blk` over `head_rows` (the
    head tokens' block-input rows, bf16 [head_tokens][d] on ctx's GPU); the rest are copied
    from src_pool on a side stream. n_recompute comes from plan_migration (policy.py)."""
    s = np.ascontiguousarray(src_slots, np.int32)
    d = np.ascontiguousarray(dst_slots, np.int32)
    if head_tokens is None:
        head_tokens = head_rows.shape[0] if head_rows is not None else 0
    check(lib().be_kv_migrate(ctx.h, blk.h, src_pool.h, dst_pool.h, ws.h,
                              s.ctypes.data_as(C.c_void_p), d.ctypes.data_as(C.c_void_p),
                              len(s), n_recompute, head_tokens, _ptr(head_rows),
                              stream if stream is not None else C.c_void_p(0)), ctx.h)


def pack_weight(ctx: Context, w):
    """Row-major [N][K] bf16 -> packed GEMM tile layout (csrc/ptx.cuh packed_index)."""
    out = w.new_empty(w.shape)
    N, K = w.shape
    check(lib().be_pack_weight(ctx.h, _ptr(w), _ptr(out), N, K, C.c_void_p(0)), ctx.h)
    return out


def gemm_bf16(ctx: Context, w, x, out, grid_cap: int = 0, packed: bool = False) -> None:
    """out[t] = x[t] @ w^T (bf16 in/out, fp32 accumulate) on the tcgen05 stream-K kernel."""
    N, K = w.shape
    wp = w if packed else pack_weight(ctx, w)
    check(lib().be_gemm_bf16(ctx.h, _ptr(wp), _ptr(x), _ptr(out), N, K, x.shape[0], grid_cap,
                             C.c_void_p(0)), ctx.h)


def cosine(ctx: Context, pred, actual, threshold: float, cos_out, accept_out) -> None:
    rows, d = pred.shape
    check(lib().be_cosine(ctx.h, _ptr(pred), _ptr(actual), rows, d, threshold, _ptr(cos_out),
                          _ptr(accept_out), C.c_void_p(0)), ctx.h)


def gather_rows(ctx: Context, arena, src_idx, out) -> None:
    check(lib().be_gather_rows(ctx.h, _ptr(arena), _ptr(src_idx), src_idx.shape[0],
                               arena.shape[1], _ptr(out), C.c_void_p(0)), ctx.h)


def scatter_rows(ctx: Context, rows, dst_idx, arena) -> None:
    check(lib().be_scatter_rows(ctx.h, _ptr(rows), _ptr(dst_idx), dst_idx.shape[0],
                                rows.shape[1], _ptr(arena), C.c_void_p(0)), ctx.h)


def synth_rows(ctx: Context, dst, seed: int, stream_id: str, scale: float) -> None:
    check(lib().be_synth_rows(ctx.h, _ptr(dst), dst.numel(), seed, stream_id.encode(), scale,
                              C.c_void_p(0)), ctx.h)
