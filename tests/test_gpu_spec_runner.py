"""Speculation inside the lockstep executor loop (bh_workload.spec_blocks; §8 a14): the marked
block runs be_exec_speculative with its 50%-FFN surrogate feeding the next block early.
  * threshold 2 (every row rejected): the next block re-runs from the true rows, so the step
    equals the plain runner's within bf16 rounding (the verify lane's GEMMs split the SMs with
    the draft lane: other stream-K partitions);
  * threshold -2 (every row accepted): the outputs are next(draft) - finite, close to the plain
    ones (the surrogate is the block with half its FFN);
  * the reference's marking rule picks the blocks (pipeline.speculation_blocks)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2404_18322_b200 import device as dev  # noqa: E402
from paper_2404_18322_b200.pipeline import _DevRows, speculation_blocks  # noqa: E402
from paper_2404_18322_b200.runner import Runner  # noqa: E402
from paper_2404_18322_b200.workloads import shared_prefix_zoo  # noqa: E402

pytestmark = pytest.mark.gpu


def narrow_c5(output=6):
    """C5's structure (8 tenants, 4 shared positions then 2 private) at d=512."""
    shape = dev.BlockShape(n_layers=1, d_model=512, n_heads=4, d_ff=1536, max_pos=128)
    return shared_prefix_zoo("c5-narrow", shape, 6, 4, 8, 4, 40, output)


def rows(run, n, d):
    return torch.as_tensor(_DevRows(run.arena_ptr, n, d), device="cuda").view(
        torch.bfloat16).float().cpu().numpy()


def test_marks_come_from_the_reference_rule():
    blocks, marked = speculation_blocks(narrow_c5())
    assert marked[:2] == ["b0", "b2"] and blocks[:2] == [0, 2]


@pytest.mark.parametrize("thr", [2.0, -2.0, 0.95])
def test_speculative_steps_in_the_runner(ctx, thr):
    wl = narrow_c5()
    n, d = wl.n_requests, wl.shape.d_model
    blocks, _ = speculation_blocks(wl)
    plain = Runner(ctx, wl, mode=1, use_graphs=False)
    spec = Runner(ctx, wl, mode=1, use_graphs=True, spec_blocks=blocks, spec_threshold=thr)
    plain.run()
    spec.run()
    for k in range(4):
        plain.decode_step()
        spec.decode_step()
        ctx.sync()
        a, b = rows(plain, n, d), rows(spec, n, d)
        assert np.isfinite(b).all()
        rel = np.linalg.norm(a - b) / np.linalg.norm(a)
        if thr > 1:
            assert rel <= 2e-2, (k, rel)
        else:
            assert rel <= 0.5, (k, rel)
    st = spec.spec_stats()
    assert st["runs"] == 4 * len(blocks) and st["rows"] == 4 * len(blocks) * n
    if thr > 1:
        assert st["accepted"] == 0
    elif thr < -1:
        assert st["accepted"] == st["rows"]
    assert -1.0 <= st["cos_min"] <= st["cos_mean"] <= 1.0
    plain.close()
    spec.close()
