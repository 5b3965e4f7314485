"""GPU parity of the individual sm_100a kernels (run with -m gpu on a B200).

Integer/byte work (gather, scatter, synthetic weights) must be bit-exact; the floating-point
kernels are checked against an fp32 reference with the tolerance written in each test.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2404_18322_b200 import device as dev  # noqa: E402

pytestmark = pytest.mark.gpu


def _bf16(a: np.ndarray):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16).cuda()


@pytest.mark.parametrize("N,K,ntok,ksplit", [
    (128, 64, 1, 1), (256, 256, 8, 1), (768, 512, 300, 1), (1024, 1024, 16, 4),
    (4096, 4096, 64, 0), (12288, 4096, 64, 0), (4096, 11008, 16, 0), (512, 256, 200, 2),
    # prefill sizes: M > 4096 with >= 4 x 148 tiles takes the round-robin whole-tile schedule
    # (gemm_plan rr), a partial last token tile included
    (2560, 512, 8192 + 77, 0), (12288, 1024, 4097, 0),
])
def test_gemm_matches_fp32(ctx, N, K, ntok, ksplit):
    g = torch.Generator().manual_seed(N * 7 + K + ntok)
    w = (torch.randn(N, K, generator=g) * 0.05).to(torch.bfloat16).cuda()
    x = torch.randn(ntok, K, generator=g).to(torch.bfloat16).cuda()
    out = torch.empty(ntok, N, dtype=torch.bfloat16, device="cuda")
    dev.gemm_bf16(ctx, w, x, out, ksplit)
    ctx.sync()
    ref = x.float() @ w.float().t()
    err = (out.float() - ref).abs().max().item()
    scale = ref.abs().max().item()
    # bf16 output rounding (2^-8 relative) dominates; fp32 accumulation order differs
    assert err <= 8e-3 * scale + 1e-3, (err, scale)


def test_gather_scatter_bit_exact(ctx):
    d = 4096
    arena = torch.randn(300, d).to(torch.bfloat16).cuda()
    src = torch.tensor([5, 0, 299, 17, 17, 42, 8], dtype=torch.int32, device="cuda")
    out = torch.empty(len(src), d, dtype=torch.bfloat16, device="cuda")
    dev.gather_rows(ctx, arena, src, out)
    ctx.sync()
    assert torch.equal(out, arena[src.long()])
    dst_arena = torch.zeros_like(arena)
    dst = torch.tensor([3, 1, 4, 100, 5, 9, 2], dtype=torch.int32, device="cuda")
    dev.scatter_rows(ctx, out, dst, dst_arena)
    ctx.sync()
    expect = torch.zeros_like(arena)
    expect[dst.long()] = out
    assert torch.equal(dst_arena, expect)


def test_cosine_rows(ctx):
    from oracle import oracle as O
    rows, d = 256, 5120
    g = torch.Generator().manual_seed(3)
    a = torch.randn(rows, d, generator=g)
    b = a + 0.35 * torch.randn(rows, d, generator=g) * torch.linspace(0, 1, rows)[:, None]
    ab, bb = a.to(torch.bfloat16), b.to(torch.bfloat16)
    cos = torch.empty(rows, dtype=torch.float32, device="cuda")
    acc = torch.empty(rows, dtype=torch.int32, device="cuda")
    dev.cosine(ctx, ab.cuda(), bb.cuda(), 0.95, cos, acc)
    ctx.sync()
    rc, racc = O.cosine_rows(ab.float().numpy(), bb.float().numpy(), 0.95)
    np.testing.assert_allclose(cos.cpu().numpy(), rc, atol=2e-6)
    # verdicts may only differ inside the fp32-vs-fp64 rounding band around the threshold
    band = np.abs(rc - 0.95) < 1e-5
    assert np.array_equal(acc.cpu().numpy()[~band], racc[~band])


def test_synth_rows_bit_exact(ctx):
    from oracle import oracle as O
    n = 100003
    t = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    dev.synth_rows(ctx, t, 7, "inputs:test", 1.7320508)
    ctx.sync()
    ref = O.synth(n, 7, "inputs:test", 1.7320508, round_bf16=True)
    assert np.array_equal(t.float().cpu().numpy(), ref)


def test_block_weights_bit_exact(ctx):
    from oracle import oracle as O
    shape = dev.BlockShape(n_layers=2, d_model=256, n_heads=4, d_ff=768, max_pos=64)
    blk = dev.Block(ctx, shape, "b0", seed=1)
    ob = O.OracleBlock(shape, "b0", seed=1)
    for layer in range(2):
        for t in ["wq", "wk", "wv", "wo", "wg", "wu", "wd"]:
            assert np.array_equal(blk.read_weight(layer, t), ob.weight(layer, t)), (layer, t)
    blk.free()


def test_kv_copy_pages_moves_whole_pages(ctx):
    """be_kv_copy_pages (KV migration data path): pages land byte-identical at their new slots,
    contiguous runs coalesced, other pages untouched."""
    shape = dev.BlockShape(n_layers=1, d_model=256, n_heads=4, d_ff=768, max_pos=64)
    blk = dev.Block(ctx, shape, "m0", seed=2)
    a = dev.KvPool(ctx, blk, 8)
    b = dev.KvPool(ctx, blk, 8)
    page_elems = shape.n_attention * 2 * shape.n_heads * 16 * shape.head_dim
    n = 8 * page_elems

    class _View:  # the pools' device memory as int16 tensors
        def __init__(self, ptr):
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i2",
                                             "data": (ptr, False), "version": 3}

    ta = torch.as_tensor(_View(a.data_ptr), device="cuda")
    tb = torch.as_tensor(_View(b.data_ptr), device="cuda")
    ta.copy_(torch.randint(-30000, 30000, (n,), dtype=torch.int16, device="cuda"))
    tb.zero_()
    torch.cuda.synchronize()
    src, dst = [2, 3, 4, 7], [5, 6, 7, 0]
    dev.kv_copy_pages(ctx, a, b, src, dst)
    ctx.sync()
    pa = ta.view(8, page_elems).cpu()
    pb = tb.view(8, page_elems).cpu()
    for s_, d_ in zip(src, dst):
        assert torch.equal(pa[s_], pb[d_])
    for d_ in (1, 2, 3, 4):
        assert not pb[d_].any()
    a.free()
    b.free()
    blk.free()


@pytest.mark.parametrize("dims,rows", [((4096, 5120), 16), ((5120, 4096), 64), ((256, 512), 3)])
def test_stitch_rows_match_fp32(ctx, dims, rows):
    """§8(f) rank 3 stitch: y = x W^T on the tcgen05 GEMM equals the fp32 product of the same
    synthetic W (stream "stitch:<name>") within bf16 output rounding."""
    from oracle import oracle as O
    din, dout = dims
    st = dev.Stitch(ctx, din, dout, "s01", seed=5)
    w = O.synth(din * dout, 5, "stitch:s01", st.scale).reshape(dout, din)
    g = torch.Generator().manual_seed(2)
    x = torch.randn(rows, din, generator=g).to(torch.bfloat16).cuda()
    y = torch.empty(rows, dout, dtype=torch.bfloat16, device="cuda")
    st(x, y)
    ctx.sync()
    ref = x.float().cpu().numpy() @ w.T
    got = y.float().cpu().numpy()
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-2
    st.free()


def test_prefill_large_batch_matches_small_batches(ctx):
    """A prefill batch of 4352 tokens (17 prompts x 256) at d=2048 runs its QKV (RoPE + paged KV
    append) and gate/up GEMMs with the round-robin whole-tile schedule (M > 4096); the same
    prompts prefilled one per batch (stream-K) give the same rows and the same K/V pages within
    bf16 rounding."""
    shape = dev.BlockShape(n_layers=1, d_model=2048, n_heads=16, d_ff=5504, max_pos=512)
    n, p = 17, 256
    pages = p // 16
    blk = dev.Block(ctx, shape, "rr", seed=4)
    pool_a = dev.KvPool(ctx, blk, n * pages)
    pool_b = dev.KvPool(ctx, blk, n * pages)
    ws = dev.Workspace(ctx, shape, max_tokens=n * p, max_rows=n, max_pages=pages)
    pt = np.arange(n * pages, dtype=np.int32).reshape(n, pages)
    g = torch.Generator().manual_seed(9)
    x = torch.randn(n * p, shape.d_model, generator=g).to(torch.bfloat16).cuda()
    toks = [(r * p + j, r * p + j, int(pt[r, j // 16]) * 16 + j % 16, j, r)
            for r in range(n) for j in range(p)]
    ya = torch.empty_like(x)
    dev.exec_batch(ctx, blk, pool_a, ws, dev.PHASE_PREFILL, toks, pt, x, ya)
    yb = torch.empty_like(x)
    for r in range(n):
        tr = [(j, j, int(pt[r, j // 16]) * 16 + j % 16, j, 0) for j in range(p)]
        dev.exec_batch(ctx, blk, pool_b, ws, dev.PHASE_PREFILL, tr, pt[r:r + 1],
                       x[r * p:(r + 1) * p].contiguous(), yb[r * p:(r + 1) * p])
    ctx.sync()
    ra = (ya.float() - yb.float()).norm() / yb.float().norm()
    assert ra.item() <= 1e-2
    pe = pool_a.page_bytes // 2
    ka, kb = pool_a.read(n * pages * pe), pool_b.read(n * pages * pe)
    assert np.linalg.norm(ka - kb) / np.linalg.norm(kb) <= 1e-2
    for o in (ws, pool_a, pool_b, blk):
        o.free()
