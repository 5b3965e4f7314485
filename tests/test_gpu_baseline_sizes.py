"""Oracle parity at the sizes of BASELINE.json's configs that the small-shape tests do not reach.

* C3 (configs[2]): 2k-token prompts and decode to context >= 2,304 (145 pages per segment), 4
  requests per private block, the tenants' private blocks at one chain position decoded in one
  grouped launch (8 blocks x 4 rows, each padded to a 16-row n-tile). A d=512 block keeps the
  fp32 oracle in seconds; the attention geometry (hd 128, 16-token pages) is the 7B one. At these
  row counts decode attention takes the flash-decoding split path (rows x heads < 4 x SMs).
* The split-K path forced (BE_ATTN_SPLITS) at several split counts, including more splits than a
  short row has pages (empty splits must drop out of the combine).

Tolerances as in test_gpu_block.py / test_gpu_runner.py: rel-L2 <= 1e-2 and min row cosine
>= 0.999 per block call; chains of two blocks with a bf16 hop: rel-L2 <= 2e-2, cosine >= 0.995.
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2404_18322_b200 import device as dev  # noqa: E402
from paper_2404_18322_b200.runner import Runner  # noqa: E402
from paper_2404_18322_b200.workloads import shared_prefix_zoo  # noqa: E402

pytestmark = pytest.mark.gpu


def _chain_check(outs, ref, tol=2e-2, min_cos=0.995):
    for k in range(1, len(outs)):
        g, r = outs[k], ref[k]
        rel = np.linalg.norm(g - r) / np.linalg.norm(r)
        cos = ((g * r).sum(1) / np.linalg.norm(g, axis=1) / np.linalg.norm(r, axis=1)).min()
        assert rel <= tol and cos >= min_cos, (k, rel, cos)


def test_c3_length_grouped_private_decode_matches_oracle(ctx):
    """C3's structure at d=512: 8 tenants x 4 requests share block 0, each tenant owns block 1;
    prompts of 2,296 tokens, 9 output tokens (the last decode step reads 2,304 tokens of context
    per segment). Decode runs lockstep: block 0 at 32 rows, then the 8 private blocks in one
    grouped launch; the executor loop's outputs are compared with the oracle run along the same
    chains, teacher-forced per step."""
    from test_gpu_runner import oracle_chain
    shape = dev.BlockShape(n_layers=1, d_model=512, n_heads=4, d_ff=1536, max_pos=2320)
    prompt, output, n_steps = 2296, 9, 8
    wl = shared_prefix_zoo("c3-narrow", shape, 2, 1, 8, 4, prompt, output,
                           max_batch_tokens=8192)
    assert wl.rows_at_block() == [32] + [4] * 8
    run = Runner(ctx, wl, mode=1, use_graphs=True)
    run.run()
    n, d = wl.n_requests, shape.d_model
    buf = torch.empty(n, d, dtype=torch.bfloat16)
    outs = []
    for _ in range(n_steps):
        nb = run.decode_step(None, buf)
        assert nb == 9  # block 0 plus the 8 private blocks
        outs.append(buf.float().numpy().copy())
    st = run.step_stats()
    # the 8 private blocks ran as ONE grouped launch (8 x 16-row n-tiles): the step's kernels are
    # those of a 32-token batch plus those of one 128-token batch
    assert st["launches"] == ctx_launches(ctx, shape, 32) + ctx_launches(ctx, shape, 128)
    run.close()
    first_ref, _ = oracle_chain(wl, 0, [])
    ins = [first_ref] + outs[:-1]
    _, ref = oracle_chain(wl, n_steps, ins)
    _chain_check(outs, ref)
    assert prompt + n_steps >= 2304


def ctx_launches(ctx, shape, n_tokens):
    from paper_2404_18322_b200._lib import lib
    blk = dev.Block(ctx, shape, "count", seed=1)
    try:
        return lib().be_exec_batch_launches(ctx.h, blk.h, n_tokens, 146)
    finally:
        blk.free()


@pytest.mark.parametrize("splits", [2, 3, 16])
def test_forced_attention_splits_match_oracle(splits):
    """Decode attention through the split-K partials + combine kernel at a forced split count,
    on ragged contexts from 1 to 100 tokens (a 1-page row over 16 splits leaves 15 empty)."""
    from test_gpu_block import run_case
    os.environ["BE_ATTN_SPLITS"] = str(splits)
    try:
        c = dev.Context(0)
    finally:
        del os.environ["BE_ATTN_SPLITS"]
    try:
        shape = dev.BlockShape(n_layers=2, d_model=512, n_heads=4, d_ff=1536, max_pos=512)
        run_case(c, shape, prompts=[40, 1, 96, 17], decode_steps=4, seed=splits)
    finally:
        c.close()


def test_c3_length_single_block_decode_with_splits_matches_oracle(ctx):
    """One 2-layer d=512 block, 4 requests at 2,300-2,310 tokens of context (the C3 private
    block's per-block batch), through be_exec_batch: prefill, then decode steps whose attention
    splits each row's 145 pages over 16 CTAs."""
    from test_gpu_block import run_case
    shape = dev.BlockShape(n_layers=2, d_model=512, n_heads=4, d_ff=1536, max_pos=2400)
    run_case(ctx, shape, prompts=[2300, 2290, 2305, 2297], decode_steps=3, seed=7)
