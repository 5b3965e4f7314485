"""§8(f) rank 3: multi-tenant LoRA adapter deltas in one launch (be_exec_lora_batch).

Requests of three LoRA variants of one block and of the base block itself share a launch: the
base weights stream once, each token adds its own adapter's B (A x) in the QKV and O epilogues.
Checked against the fp32 oracle with each adapter folded into the weights (W + B A; the reference
zoo's fused attention, attach "fuse"): prefill of ragged prompts, then a decode step, every
request against its own restated block (rel-L2 <= 1e-2 as test_gpu_block.py). Base-only rows
must equal a plain be_exec_batch of the same batch bit for bit.
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


@pytest.mark.parametrize("comps", ["afaf", "fafa"])
def test_lora_batch_matches_oracle(ctx, comps):
    from oracle import oracle as O
    shape = dev.BlockShape(n_layers=2, d_model=256, n_heads=4, d_ff=768, max_pos=64,
                           components=comps)
    names = ["t0", "t1", "t2"]
    adapter = [0, 1, 2, -1, 0, 1, 2, -1]  # per request; -1 = the base block
    prompts = [5, 3, 7, 4, 2, 6, 1, 5]
    n, d = len(adapter), shape.d_model
    blk = dev.Block(ctx, shape, "lb", seed=3)
    loras = [dev.Lora(ctx, blk, nm, seed=11) for nm in names]
    pool = dev.KvPool(ctx, blk, n)
    pool_plain = dev.KvPool(ctx, blk, n)
    ws = dev.Workspace(ctx, shape, max_tokens=64, max_rows=n, max_pages=1)
    pt = np.arange(n, dtype=np.int32).reshape(n, 1)  # request r owns page r
    orc = [O.OracleBlock(shape, "lb", seed=3) for _ in range(4)]
    for k, nm in enumerate(names):
        orc[k].add_lora(nm, 11, loras[k].scale_a, loras[k].scale_b)
    seqs = [orc[adapter[r]].new_seq(16) for r in range(n)]

    def run(phase, toks, x, tok_req, tok_pos):
        idx = [adapter[r] for r in tok_req]
        y = torch.zeros_like(x)
        dev.exec_lora_batch(ctx, blk, pool, ws, phase, toks, pt, loras, idx, x, y)
        y_plain = torch.zeros_like(x)
        dev.exec_batch(ctx, blk, pool_plain, ws, phase, toks, pt, x, y_plain)
        ctx.sync()
        ref = np.zeros((len(tok_req), d), np.float32)
        xs = f32(x)
        for k in range(4):  # each restated block runs its own requests' tokens
            rows = [i for i, r in enumerate(tok_req) if adapter[r] == (k if k < 3 else -1)]
            if not rows:
                continue
            ref[rows] = orc[k].forward(seqs, [tok_req[i] for i in rows],
                                       [tok_pos[i] for i in rows], xs[rows])
        out = f32(y)
        assert rel_l2(out, ref) <= 1e-2
        for r in range(n):
            rows = [i for i, q in enumerate(tok_req) if q == r]
            assert rel_l2(out[rows], ref[rows]) <= 1.5e-2, r
        base_rows = [i for i, r in enumerate(tok_req) if adapter[r] < 0]
        assert torch.equal(y[base_rows], y_plain[base_rows])
        lora_rows = [i for i, r in enumerate(tok_req) if adapter[r] >= 0]
        assert not torch.equal(y[lora_rows], y_plain[lora_rows])  # the deltas are live

    g = torch.Generator().manual_seed(4)
    toks, tok_req, tok_pos = [], [], []
    for r, p in enumerate(prompts):
        for j in range(p):
            toks.append((len(toks), len(toks), r * 16 + j, j, r))
            tok_req.append(r)
            tok_pos.append(j)
    xp = torch.randn(len(toks), d, generator=g).to(torch.bfloat16).cuda()
    run(dev.PHASE_PREFILL, toks, xp, tok_req, tok_pos)
    x1 = torch.randn(n, d, generator=g).to(torch.bfloat16).cuda()
    dtoks = [(r, r, r * 16 + prompts[r], prompts[r], r) for r in range(n)]
    run(dev.PHASE_DECODE, dtoks, x1, list(range(n)), prompts)
    for lo in loras:
        lo.free()
    ws.free()
    pool.free()
    pool_plain.free()
    blk.free()
