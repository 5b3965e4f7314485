"""GPU parity of one per-block batched execution against the CPU oracle.

Tolerance (bf16 storage, fp32 accumulation vs the fp32 oracle, stated in BASELINE.md §4):
  per-call output rel-L2 <= 1e-2 and min per-row cosine >= 0.999; KV pages within rel-L2 1e-2.
Routing (which arena rows are read/written, which page slots hold which token) is exact.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2404_18322_b200 import device as dev  # noqa: E402

pytestmark = pytest.mark.gpu

REL_L2 = 1e-2
MIN_COS = 0.999


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def row_cos(a, b):
    num = (a * b).sum(1)
    den = np.linalg.norm(a, axis=1) * np.linalg.norm(b, axis=1)
    return num / den


def bf16_np(t):
    return t.float().cpu().numpy()


class PagedSeqs:
    """Test-local page bookkeeping: request r owns pages perm[...] of the pool (16 tok/page)."""

    def __init__(self, n_req, max_tokens, n_pages, seed=0):
        rng = np.random.default_rng(seed)
        self.max_pages = (max_tokens + 15) // 16
        slots = rng.permutation(n_pages)[: n_req * self.max_pages]
        self.pt = slots.reshape(n_req, self.max_pages).astype(np.int32)

    def slot(self, r, pos):
        return int(self.pt[r, pos // 16]) * 16 + pos % 16


def run_case(ctx, shape, prompts, decode_steps, seed=1):
    from oracle import oracle as O
    n_req = len(prompts)
    max_tok = max(prompts) + decode_steps + 1
    blk = dev.Block(ctx, shape, "b0", seed=seed)
    ob = O.OracleBlock(shape, "b0", seed=seed)
    n_pages = n_req * ((max_tok + 15) // 16) + 5
    pool = dev.KvPool(ctx, blk, n_pages)
    total_prompt = sum(prompts)
    ws = dev.Workspace(ctx, shape, max_tokens=max(total_prompt, n_req), max_rows=n_req,
                       max_pages=(max_tok + 15) // 16)
    ps = PagedSeqs(n_req, max_tok, n_pages, seed)
    seqs = [ob.new_seq(max_tok) for _ in range(n_req)]
    d = shape.d_model

    # prefill: one batch with every prompt token (ragged prompts)
    g = torch.Generator().manual_seed(seed)
    arena_in = (torch.randn(total_prompt, d, generator=g)).to(torch.bfloat16).cuda()
    arena_out = torch.zeros(total_prompt, d, dtype=torch.bfloat16, device="cuda")
    toks, tok_seq, tok_pos = [], [], []
    row = 0
    for r, p in enumerate(prompts):
        for pos in range(p):
            toks.append((row, row, ps.slot(r, pos), pos, r))
            tok_seq.append(r)
            tok_pos.append(pos)
            row += 1
    dev.exec_batch(ctx, blk, pool, ws, dev.PHASE_PREFILL, toks, ps.pt, arena_in, arena_out)
    ctx.sync()
    y_gpu = bf16_np(arena_out)
    y_ref = ob.forward(seqs, tok_seq, tok_pos, bf16_np(arena_in))
    assert rel_l2(y_gpu, y_ref) <= REL_L2
    assert row_cos(y_gpu, y_ref).min() >= MIN_COS

    # decode: each step feeds every request's last output row back (greedy, no LM head)
    last_rows = np.cumsum(prompts) - 1
    x = arena_out[torch.as_tensor(last_rows, device="cuda")].contiguous()
    lens = list(prompts)
    for step in range(decode_steps):
        order = list(range(n_req))[::-1] if step % 2 else list(range(n_req))  # batch order varies
        toks = [(r, r, ps.slot(r, lens[r]), lens[r], r) for r in order]
        xin = x
        xout = torch.zeros_like(x)
        dev.exec_batch(ctx, blk, pool, ws, dev.PHASE_DECODE, toks, ps.pt, xin, xout)
        ctx.sync()
        y_gpu = bf16_np(xout)
        y_ref = ob.forward(seqs, order, [lens[r] for r in order], bf16_np(xin)[order])
        y_gpu_o = y_gpu[order]
        assert rel_l2(y_gpu_o, y_ref) <= REL_L2, step
        assert row_cos(y_gpu_o, y_ref).min() >= MIN_COS, step
        for r in range(n_req):
            lens[r] += 1
        x = xout

    # KV pages: unpermute the pair-interleaved K head dims and compare with the oracle cache
    hd, H, L = shape.head_dim, shape.n_heads, shape.n_layers
    kv = _read_pool(pool, n_pages * L * 2 * H * 16 * hd).reshape(n_pages, L, 2, H, 16, hd)
    inv = np.empty(hd, np.int64)
    for e in range(hd):
        inv[e] = (e >> 1) + (hd // 2 if e & 1 else 0)  # physical e holds logical inv[e]
    for r in range(n_req):
        for layer in range(L):
            kref = seqs[r].kv(layer, 0)[: lens[r]].reshape(lens[r], H, hd)
            vref = seqs[r].kv(layer, 1)[: lens[r]].reshape(lens[r], H, hd)
            kg = np.empty_like(kref)
            vg = np.empty_like(vref)
            for pos in range(lens[r]):
                page, t = ps.pt[r, pos // 16], pos % 16
                kphys = kv[page, layer, 0, :, t, :]
                kg[pos][:, inv] = kphys
                vg[pos] = kv[page, layer, 1, :, t, :]
            assert rel_l2(kg, kref) <= REL_L2
            assert rel_l2(vg, vref) <= REL_L2
    ws.free()
    pool.free()
    blk.free()


def _read_pool(pool, n_elems):
    pool.ctx.sync()
    return pool.read(n_elems)


def test_block_tiny_hd64(ctx):
    # C1 shape (BASELINE.json configs[0]): d=256, 4 heads x 64, d_ff=768, 2-layer block
    shape = dev.BlockShape(n_layers=2, d_model=256, n_heads=4, d_ff=768, max_pos=256)
    run_case(ctx, shape, prompts=[20, 13, 1, 33], decode_steps=5)


def test_block_hd128(ctx):
    # Llama head geometry (hd=128) at a small width
    shape = dev.BlockShape(n_layers=2, d_model=512, n_heads=4, d_ff=1536, max_pos=512)
    run_case(ctx, shape, prompts=[40, 17, 64], decode_steps=4, seed=2)


def test_block_llama13b_shape(ctx):
    # C4 (BASELINE.json configs[3]) geometry: d=5120, 40 heads x 128, d_ff=13824 - 40 m-tiles of
    # O/down, 216 of gate/up, a 215-k-block down projection; one decoder layer, ragged prompts
    shape = dev.BlockShape(n_layers=1, d_model=5120, n_heads=40, d_ff=13824, max_pos=128)
    run_case(ctx, shape, prompts=[9, 17, 3], decode_steps=3, seed=4)


def test_block_llama7b_shape_batch64(ctx):
    # C2 geometry at the decode batch the bench runs (64 rows; BN=64 tiles, stream-K partials)
    shape = dev.BlockShape(n_layers=1, d_model=4096, n_heads=32, d_ff=11008, max_pos=64)
    run_case(ctx, shape, prompts=[1 + (r * 7) % 5 for r in range(64)], decode_steps=2, seed=6)
