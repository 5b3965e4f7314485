"""§8(f) rank 4: prefix-shared KV pages on the GPU.

Two requests of a prefix group share their prompt's first pages (KvStore::share_prefix,
kv.cpp:135-152, mirrored bit-exact by bh_kv_share_prefix): the host maps request B's leading
page-table entries to request A's physical page slots (bh_kv_page_slots), and B's prefill runs
only its own suffix tokens - a chunked prefill whose causal attention reads the shared prefix
pages. Checks against B computed alone with a private copy of the prefix:
  * B's suffix outputs and the next decode token of A and B match (bf16 tolerance);
  * A's pages are byte-identical before and after B's prefill (nothing writes shared pages);
  * the shared pages are counted once (bytes_saved_by_sharing = 3 pages).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2404_18322_b200 import device as dev  # noqa: E402
from paper_2404_18322_b200 import host as H  # noqa: E402

pytestmark = pytest.mark.gpu

SHAPE = dev.BlockShape(n_layers=2, d_model=512, n_heads=8, d_ff=1536, max_pos=256)
PREFIX, SUF_A, SUF_B = 48, 20, 30  # 3 shared pages


def rel_l2(a, b):
    a, b = a.float().cpu().numpy(), b.float().cpu().numpy()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def toks_for(slots, row0, positions, pt_row):
    return [(row0 + i, row0 + i, slots[p // 16] * 16 + p % 16, p, pt_row)
            for i, p in enumerate(positions)]


def table(rows):
    w = max(len(r) for r in rows)
    return np.asarray([list(r) + [-1] * (w - len(r)) for r in rows], np.int32)


def test_prefix_shared_pages(ctx):
    d = SHAPE.d_model
    bpt = SHAPE.kv_bytes_per_token
    kv = H.KvStore()
    kv.attach_pool("blk", 0, 64)
    kv.create_segment(1, "blk", 0, bpt)
    kv.append_tokens(1, "blk", PREFIX + SUF_A + 1)
    kv.create_segment(2, "blk", 0, bpt)
    assert kv.share_prefix(2, 1, "blk", PREFIX) == PREFIX
    kv.append_tokens(2, "blk", SUF_B + 1)
    sa, sb = kv.page_slots(1, "blk"), kv.page_slots(2, "blk")
    assert sb[:3] == sa[:3] and not set(sb[3:]) & set(sa)
    page_bytes = 16 * bpt
    assert kv.bytes_saved_by_sharing() == 3 * page_bytes

    blk = dev.Block(ctx, SHAPE, "pfx", seed=6)
    pool = dev.KvPool(ctx, blk, 64)
    ws = dev.Workspace(ctx, SHAPE, max_tokens=128, max_rows=2, max_pages=8)
    g = torch.Generator().manual_seed(8)
    prefix = torch.randn(PREFIX, d, generator=g).to(torch.bfloat16)
    xa = torch.cat([prefix, torch.randn(SUF_A, d, generator=g).to(torch.bfloat16)]).cuda()
    xb = torch.cat([prefix, torch.randn(SUF_B, d, generator=g).to(torch.bfloat16)]).cuda()
    pt = table([sa, sb])
    # A: whole prompt
    ya = torch.empty_like(xa)
    dev.exec_batch(ctx, blk, pool, ws, dev.PHASE_PREFILL,
                   toks_for(sa, 0, range(PREFIX + SUF_A), 0), pt, xa, ya)
    ctx.sync()
    pe = pool.page_bytes // 2
    a_pages = np.stack([pool.read(pe, s * pe) for s in sa])
    # B: its suffix only, attending to the shared prefix pages
    xb_suf = xb[PREFIX:].contiguous()
    yb_suf = torch.empty_like(xb_suf)
    dev.exec_batch(ctx, blk, pool, ws, dev.PHASE_PREFILL,
                   toks_for(sb, 0, range(PREFIX, PREFIX + SUF_B), 1), pt, xb_suf, yb_suf)
    ctx.sync()
    a_after = np.stack([pool.read(pe, s * pe) for s in sa])
    assert np.array_equal(a_pages.view(np.uint32), a_after.view(np.uint32))

    # reference: B alone with a private prefix
    pool2 = dev.KvPool(ctx, blk, 16)
    own = list(range(1, 1 + len(sb)))
    pt2 = table([own])
    yb_ref = torch.empty_like(xb)
    dev.exec_batch(ctx, blk, pool2, ws, dev.PHASE_PREFILL,
                   toks_for(own, 0, range(PREFIX + SUF_B), 0), pt2, xb, yb_ref)
    ctx.sync()
    assert rel_l2(yb_suf, yb_ref[PREFIX:]) <= 1e-2

    # next token for A and B in one decode batch over the shared pages, and B alone
    x1 = torch.randn(2, d, generator=g).to(torch.bfloat16).cuda()
    y1 = torch.empty_like(x1)
    dec = [(0, 0, sa[(PREFIX + SUF_A) // 16] * 16 + (PREFIX + SUF_A) % 16, PREFIX + SUF_A, 0),
           (1, 1, sb[(PREFIX + SUF_B) // 16] * 16 + (PREFIX + SUF_B) % 16, PREFIX + SUF_B, 1)]
    dev.exec_batch(ctx, blk, pool, ws, dev.PHASE_DECODE, dec, pt, x1, y1)
    y1_ref = torch.empty_like(x1[1:])
    dev.exec_batch(ctx, blk, pool2, ws, dev.PHASE_DECODE,
                   [(0, 0, own[(PREFIX + SUF_B) // 16] * 16 + (PREFIX + SUF_B) % 16,
                     PREFIX + SUF_B, 0)], pt2, x1[1:].contiguous(), y1_ref)
    ctx.sync()
    assert rel_l2(y1[1:], y1_ref) <= 1e-2
    for o in (ws, pool, pool2, blk):
        o.free()
