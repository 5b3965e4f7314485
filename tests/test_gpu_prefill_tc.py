"""The tcgen05 prefill attention (csrc/attention_prefill_tc.cu: S and O in TMEM, Q / K / V tiles
by TMA, V as an MN-major operand) against the mma.sync kernel (BE_PREFILL_TC=2) and the per-row
decode kernel (BE_PREFILL_TC=0) on identical inputs, and against the fp32 oracle: ragged prompts,
query tiles that start inside a 128-token window (a prefill resuming at position 40), and
contexts spanning several K/V tiles. Tolerance as test_gpu_block.py (rel-L2 <= 1e-2)."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2404_18322_b200 import device as dev  # noqa: E402

pytestmark = pytest.mark.gpu

SHAPE = dev.BlockShape(n_layers=2, d_model=512, n_heads=4, d_ff=1536, max_pos=1024)


def run(mode, prompts, start=0, seed=3):
    """Prefill `prompts` (positions start .. start+p-1 of each request; positions below `start`
    come from a first prefill of the same rows) and return the block output rows."""
    os.environ["BE_PREFILL_TC"] = str(mode)
    try:
        ctx = dev.Context(0)
    finally:
        del os.environ["BE_PREFILL_TC"]
    blk = dev.Block(ctx, SHAPE, "ptc", seed=seed)
    ppr = (max(prompts) + start + 15) // 16
    pool = dev.KvPool(ctx, blk, len(prompts) * ppr + 1)
    total = sum(prompts) + start * len(prompts)
    ws = dev.Workspace(ctx, SHAPE, max_tokens=total, max_rows=len(prompts), max_pages=ppr)
    pt = np.arange(len(prompts) * ppr, dtype=np.int32).reshape(len(prompts), ppr)
    g = torch.Generator().manual_seed(seed)
    outs = []
    for first, lens in ((0, [start] * len(prompts)), (start, prompts)):
        if max(lens) == 0:
            continue
        toks, row = [], 0
        for r, n in enumerate(lens):
            for i in range(n):
                p = first + i
                toks.append((row, row, int(pt[r, p // 16]) * 16 + p % 16, p, r))
                row += 1
        x = torch.randn(row, SHAPE.d_model, generator=g).to(torch.bfloat16).cuda()
        y = torch.empty_like(x)
        dev.exec_batch(ctx, blk, pool, ws, dev.PHASE_PREFILL, toks, pt, x, y)
        ctx.sync()
        outs.append((x.float().cpu().numpy(), y.float().cpu().numpy(), toks))
    ws.free()
    pool.free()
    blk.free()
    ctx.close()
    return outs


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("prompts,start", [([300, 17, 129, 1, 256], 0), ([90, 200], 40),
                                           ([700], 0)])
@pytest.mark.parametrize("mode", [1, 4])
def test_tcgen05_prefill_matches_other_kernels_and_oracle(prompts, start, mode):
    """mode 1: two CTAs per SM (the default); 4: the warp-specialised kernel (one CTA per SM, S
    double-buffered in TMEM, loader and MMA warps)."""
    from oracle import oracle as O
    tc = run(mode, prompts, start)
    ref = run(2, prompts, start)
    rowk = run(0, prompts, start)
    for (x1, y1, _), (x2, y2, _), (x3, y3, _) in zip(tc, ref, rowk):
        assert np.array_equal(x1, x2)
        assert rel(y1, y2) <= 1e-2 and rel(y1, y3) <= 1e-2
    # the oracle over both prefill passes (the second attends to the first's K/V)
    ob = O.OracleBlock(SHAPE, "ptc", seed=3)
    seqs = [ob.new_seq(max(prompts) + start + 1) for _ in prompts]
    for x, y, toks in tc:
        want = ob.forward(seqs, [t[4] for t in toks], [t[3] for t in toks], x)
        assert rel(y, want) <= 1e-2
