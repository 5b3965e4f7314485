"""Host-side validation of the routing metadata at the C ABI (be_exec_batch / be_kv_migrate):
the kernels trust what passes, so what cannot be executed safely must be refused with
BE_ERR_INVALID before anything is launched."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2404_18322_b200 import device as dev  # noqa: E402
from paper_2404_18322_b200._lib import BlockExecError  # noqa: E402

pytestmark = pytest.mark.gpu

SHAPE = dev.BlockShape(n_layers=2, d_model=256, n_heads=4, d_ff=768, max_pos=128)


@pytest.fixture
def parts(ctx):
    blk = dev.Block(ctx, SHAPE, "val", seed=2)
    pool = dev.KvPool(ctx, blk, 8)
    ws = dev.Workspace(ctx, SHAPE, max_tokens=64, max_rows=2, max_pages=4)
    yield blk, pool, ws
    ws.free()
    pool.free()
    blk.free()


def _decode(ctx, parts, pt, kv_slot, pos):
    blk, pool, ws = parts
    x = torch.zeros(1, SHAPE.d_model, dtype=torch.bfloat16, device="cuda")
    dev.exec_batch(ctx, blk, pool, ws, dev.PHASE_DECODE, [(0, 0, kv_slot, pos, 0)],
                   np.asarray([pt], np.int32), x, torch.empty_like(x))
    ctx.sync()


def test_unmapped_page_before_the_token_is_refused(ctx, parts):
    # position 20 reads pages 0 and 1; page 0 is unmapped (-1)
    with pytest.raises(BlockExecError):
        _decode(ctx, parts, [-1, 3, -1, -1], 3 * 16 + 4, 20)


def test_kv_slot_off_its_page_is_refused(ctx, parts):
    # the token's page-table page is 3, but its KV slot lies on page 5
    with pytest.raises(BlockExecError):
        _decode(ctx, parts, [1, 3, -1, -1], 5 * 16 + 4, 20)


def test_consistent_metadata_runs(ctx, parts):
    _decode(ctx, parts, [1, 3, -1, -1], 3 * 16 + 4, 20)


def test_migration_with_copied_tail_needs_full_head_pages(ctx, parts):
    """2 recomputed pages + copied tail pages: the head must cover all 32 tokens, or tokens
    20..31 would be neither recomputed nor copied."""
    blk, pool, ws = parts
    other = dev.KvPool(ctx, blk, 8)
    x = torch.zeros(32, SHAPE.d_model, dtype=torch.bfloat16, device="cuda")
    try:
        with pytest.raises(BlockExecError):
            dev.kv_migrate(ctx, blk, pool, other, ws, [0, 1, 2], [4, 5, 6], 2, x[:20], 20)
        dev.kv_migrate(ctx, blk, pool, other, ws, [0, 1, 2], [4, 5, 6], 2, x, 32)
        # all pages recomputed: a partial last page is fine
        dev.kv_migrate(ctx, blk, pool, other, ws, [0, 1], [4, 5], 2, x[:20], 20)
        ctx.sync()
    finally:
        other.free()
