"""§8 a14 speculation on the GPU (be_exec_speculative): the draft lane (a 50%-FFN-pruned
surrogate) feeds the next block early on a second stream, the true block
verifies, K7 decides per row (cos >= threshold) and rejected rows re-run the next
block from the true rows (finish_verified, scenario.cpp:740-807).

Checked against the fp32 oracle: the surrogate's weights are the base block's first channels;
the verdict equals the oracle cosine of draft vs true rows; the next block's output is the
oracle's next(draft) for accepted rows and next(true) for rejected ones; tolerances as in
test_gpu_block.py (rel-L2 <= 1e-2 per call, bf16 hops <= 3e-2).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2404_18322_b200 import device as dev  # noqa: E402

pytestmark = pytest.mark.gpu


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def f32(t):
    return t.float().cpu().numpy()


def test_surrogate_weights_are_the_base_prefix(ctx):
    base = dev.BlockShape(n_layers=1, d_model=256, n_heads=4, d_ff=768, max_pos=64)
    sur = base.surrogate(0.5)
    assert (sur.d_ff, sur.ffn_src) == (384, 768)
    b = dev.Block(ctx, base, "b7", seed=3)
    s = dev.Block(ctx, sur, "b7", seed=3)
    for t in ("wq", "wo"):
        assert np.array_equal(b.read_weight(0, t), s.read_weight(0, t))
    assert np.array_equal(b.read_weight(0, "wg")[:384], s.read_weight(0, "wg"))
    assert np.array_equal(b.read_weight(0, "wu")[:384], s.read_weight(0, "wu"))
    assert np.array_equal(b.read_weight(0, "wd")[:, :384], s.read_weight(0, "wd"))
    b.free()
    s.free()


@pytest.mark.parametrize("threshold,d,n", [(-2.0, 256, 8), (0.95, 256, 8), (2.0, 256, 8),
                                         (0.95, 512, 256), (None, 512, 256)])
def test_speculative_step_matches_oracle(ctx, threshold, d, n):
    """8 rows at C1 width, and C5's batch of 256 rows (configs[4]) at d=512 (hd 128) so the
    oracle stays fast; threshold None = the median cosine (the batch splits into accepted and
    rejected rows)."""
    from oracle import oracle as O
    heads = d // 64 if d == 256 else d // 128
    shape = dev.BlockShape(n_layers=2, d_model=d, n_heads=heads, d_ff=3 * d, max_pos=64)
    sur = shape.surrogate(0.5)
    prompt = 5
    d = shape.d_model
    names = {"verify": ("b1", shape), "draft": ("b1", sur), "next": ("b2", shape)}
    gpu, orc, pools, seqs = {}, {}, {}, {}
    pt = np.arange(n, dtype=np.int32).reshape(n, 1)  # request r owns page r (16 tokens)
    for k, (nm, sh) in names.items():
        gpu[k] = dev.Block(ctx, sh, nm, seed=5)
        orc[k] = O.OracleBlock(sh, nm, seed=5)
        pools[k] = dev.KvPool(ctx, gpu[k], n + 1)
        seqs[k] = [orc[k].new_seq(16) for _ in range(n)]
    ws_main = dev.Workspace(ctx, shape, max_tokens=n * prompt, max_rows=n, max_pages=1)
    ws_side = dev.Workspace(ctx, shape, max_tokens=n * prompt, max_rows=n, max_pages=1)
    g = torch.Generator().manual_seed(11)
    # prefill every block's pool with its own prompt states (the draft lane keeps its own KV)
    xp = torch.randn(n * prompt, d, generator=g).to(torch.bfloat16).cuda()
    toks = [(r * prompt + p, r * prompt + p, r * 16 + p, p, r) for r in range(n)
            for p in range(prompt)]
    tok_seq = [r for r in range(n) for _ in range(prompt)]
    tok_pos = [p for _ in range(n) for p in range(prompt)]
    for k in names:
        out = torch.empty_like(xp)
        dev.exec_batch(ctx, gpu[k], pools[k], ws_main, dev.PHASE_PREFILL, toks, pt, xp, out)
        orc[k].forward(seqs[k], tok_seq, tok_pos, f32(xp))
    ctx.sync()
    # the speculative decode step at position `prompt`
    x = torch.randn(n, d, generator=g).to(torch.bfloat16).cuda()
    y_draft, y_true, z = (torch.zeros(n, d, dtype=torch.bfloat16, device="cuda") for _ in range(3))
    dtoks = [(r, r, r * 16 + prompt, prompt, r) for r in range(n)]
    st = {k: (gpu[k], pools[k], ws_main if k == "verify" else ws_side, dtoks, pt) for k in names}
    if threshold is None:
        # a dry pass to find the median cosine; then the real step (the KV slots of position
        # `prompt` are rewritten with the same values)
        cos0, _, _ = dev.exec_speculative(ctx, st["verify"], st["draft"], st["next"], x,
                                          y_draft, y_true, z, 0.95)
        threshold = float(np.median(cos0))
    cos, acc, n_acc = dev.exec_speculative(ctx, st["verify"], st["draft"], st["next"], x,
                                           y_draft, y_true, z, threshold)
    if n == 256 and threshold == float(np.median(cos)):
        assert 0 < n_acc < n
    pos = [prompt] * n
    seq_ids = list(range(n))
    yt_ref = orc["verify"].forward(seqs["verify"], seq_ids, pos, f32(x))
    yd_ref = orc["draft"].forward(seqs["draft"], seq_ids, pos, f32(x))
    assert rel_l2(f32(y_true), yt_ref) <= 1e-2
    assert rel_l2(f32(y_draft), yd_ref) <= 1e-2
    cos_ref, _ = O.cosine_rows(f32(y_draft), f32(y_true), threshold)
    np.testing.assert_allclose(cos, cos_ref, atol=1e-5)
    assert np.array_equal(acc, (cos >= threshold).astype(np.int32))
    assert n_acc == int(acc.sum())
    if threshold < -1:
        assert n_acc == n
    if threshold > 1:
        assert n_acc == 0
    # next block: accepted rows ran on the draft, rejected ones were redone on the true rows
    z_in = np.where(acc[:, None] == 1, f32(y_draft), f32(y_true))
    z_ref = orc["next"].forward(seqs["next"], seq_ids, pos, z_in)
    assert rel_l2(f32(z), z_ref) <= 3e-2
    for k in names:
        pools[k].free()
        gpu[k].free()
    ws_main.free()
    ws_side.free()


def test_speculative_stage_at_c5_scale(ctx):
    """configs[4] (C5): the cosine equivalence check at batch 256 over 8 tenants on 7B-shaped
    4-layer blocks (verify = a shared block, draft = its 50%-FFN surrogate, next = the following
    shared block). Size-independent properties instead of the CPU oracle:
      * the verify lane's rows equal a plain be_exec_batch of the block within bf16 rounding
        (the two lanes split the SMs, so the verify GEMMs run stream-K over half the CTAs and
        sum their k-slices in another grouping);
      * K7's cosine equals an fp32 torch cosine of the draft/true rows; accept = cos >= thr;
      * the next block's rows equal next(draft) for accepted rows and next(true) for rejected
        ones (a plain run on the selected inputs; other batch composition, so within bf16
        rounding)."""
    from paper_2404_18322_b200.workloads import c5_llama7b_8tenant
    wl = c5_llama7b_8tenant()
    shape = dev.BlockShape(n_layers=4, d_model=4096, n_heads=32, d_ff=11008, max_pos=128)
    n, prompt, d = len(wl.req_tenant), 64, shape.d_model
    assert n == 256 and len(wl.chains) == 8
    pages = (prompt + 1 + 15) // 16
    pt = np.arange(n * pages, dtype=np.int32).reshape(n, pages)
    names = {"verify": ("b3", shape), "draft": ("b3", shape.surrogate(0.5)),
             "next": ("b4", shape)}
    gpu, pools = {}, {}
    for k, (nm, sh) in names.items():
        gpu[k] = dev.Block(ctx, sh, nm, seed=9)
        pools[k] = dev.KvPool(ctx, gpu[k], n * pages)
    ws_main = dev.Workspace(ctx, shape, max_tokens=8192, max_rows=n, max_pages=pages)
    ws_side = dev.Workspace(ctx, shape, max_tokens=n, max_rows=n, max_pages=pages)
    g = torch.Generator().manual_seed(5)
    for k in names:  # prompt KV for every lane, in 32-request prefill batches
        for r0 in range(0, n, 32):
            xp = torch.randn(32 * prompt, d, generator=g).to(torch.bfloat16).cuda()
            toks = [(i * prompt + p, i * prompt + p, int(pt[r0 + i, p // 16]) * 16 + p % 16, p,
                     r0 + i) for i in range(32) for p in range(prompt)]
            dev.exec_batch(ctx, gpu[k], pools[k], ws_main, dev.PHASE_PREFILL, toks, pt, xp,
                           torch.empty_like(xp))
    ctx.sync()
    x = torch.randn(n, d, generator=g).to(torch.bfloat16).cuda()
    dtoks = [(r, r, int(pt[r, prompt // 16]) * 16 + prompt % 16, prompt, r) for r in range(n)]
    st = {k: (gpu[k], pools[k], ws_main if k == "verify" else ws_side, dtoks, pt) for k in names}
    y_draft, y_true, z = (torch.zeros(n, d, dtype=torch.bfloat16, device="cuda")
                          for _ in range(3))
    cos0, _, _ = dev.exec_speculative(ctx, st["verify"], st["draft"], st["next"], x, y_draft,
                                      y_true, z, 0.95)
    thr = float(np.median(cos0))  # a threshold that splits the batch
    cos, acc, n_acc = dev.exec_speculative(ctx, st["verify"], st["draft"], st["next"], x,
                                           y_draft, y_true, z, thr)
    assert 0 < n_acc < n
    yd, yt = y_draft.float(), y_true.float()
    cos_t = (yd * yt).sum(1) / (yd.norm(dim=1) * yt.norm(dim=1))
    np.testing.assert_allclose(cos, cos_t.cpu().numpy(), atol=1e-5)
    assert np.array_equal(acc, (cos >= thr).astype(np.int32)) and n_acc == int(acc.sum())
    y_plain = torch.empty_like(x)
    dev.exec_batch(ctx, gpu["verify"], pools["verify"], ws_main, dev.PHASE_DECODE, dtoks, pt, x,
                   y_plain)
    ctx.sync()
    assert rel_l2(f32(y_true), f32(y_plain)) <= 1e-2
    yc = torch.nn.functional.cosine_similarity(y_true.float(), y_plain.float(), dim=1)
    assert float(yc.min()) >= 0.999
    a = torch.from_numpy(acc).cuda().bool()[:, None]
    z_in = torch.where(a, y_draft, y_true)
    z_plain = torch.empty_like(x)
    dev.exec_batch(ctx, gpu["next"], pools["next"], ws_main, dev.PHASE_DECODE, dtoks, pt, z_in,
                   z_plain)
    ctx.sync()
    assert rel_l2(f32(z), f32(z_plain)) <= 1e-2
    zc = torch.nn.functional.cosine_similarity(z.float(), z_plain.float(), dim=1)
    assert float(zc.min()) >= 0.999
    for k in names:
        pools[k].free()
        gpu[k].free()
    ws_main.free()
    ws_side.free()
