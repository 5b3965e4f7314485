"""The drop-in, end to end: the reference's own Simulation (oracle/_ref, the unmodified
/root/reference sources) forms the batches and hands each one to the product's batch executor
(bh_executor_run_batch, the call replacing batch_duration_us at scenario.cpp:493), through the
reference Engine's trace hook. The GPU rows it leaves behind must be
  * bit-identical to the product's own executor loop (bh_runner, event order) on the same zoo -
    the same batches on the same blocks, so the same bits - and
  * within the oracle tolerance of the fp32 restatement along the chains (rel-L2 <= 3e-2,
    cosine >= 0.995 per request's final hidden state, as test_gpu_reference_zoo.py)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
R = pytest.importorskip("oracle.refshim")

from paper_2404_18322_b200.device import BlockShape  # noqa: E402
from paper_2404_18322_b200.pipeline import _DevRows  # noqa: E402
from paper_2404_18322_b200.runner import Runner  # noqa: E402
from paper_2404_18322_b200.workloads import Workload  # noqa: E402

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")]


@pytest.mark.parametrize("case", [
    # C1's width (d=256, 4 heads x 64): a foundation + 2 LoRA tenants fusing from layer 2
    (4, 256, 4, 2, 2, [16] * 8, [6] * 8, 4096),
    (3, 512, 4, 3, 1, [17, 40, 9, 25, 3, 12], [5, 3, 6, 2, 4, 5], 64),
])
def test_reference_simulation_drives_the_gpu_executor(ctx, case):
    from test_gpu_reference_zoo import oracle_outputs
    n_layers, dim, heads, n_lora, first, prompts, outputs, budget = case
    rows_sim, trace_sim = R.simulate_gpu(n_layers, dim, heads, n_lora, first, prompts, outputs,
                                         max_batch_tokens=budget)
    blocks, kinds, chains, req_model, trace = R.simulate(n_layers, dim, n_lora, first, prompts,
                                                         outputs, max_batch_tokens=budget)
    assert trace_sim == trace  # the hook ran every batch without changing the simulation
    shape = BlockShape(1, dim, heads, 3 * dim, max_pos=max(p + o for p, o in
                                                           zip(prompts, outputs)) + 16)
    wl = Workload("refzoo", shape, blocks, chains, req_model, prompts, outputs,
                  max_batch_tokens=budget, block_comps=kinds)
    run = Runner(ctx, wl, mode=0, use_graphs=False)
    run.run()
    ctx.sync()
    ours = torch.as_tensor(_DevRows(run.arena_ptr, wl.n_requests, dim), device="cuda").view(
        torch.bfloat16).float().cpu().numpy()
    run.close()
    assert np.array_equal(rows_sim, ours)
    ref = oracle_outputs(wl, blocks, kinds)
    for r in range(wl.n_requests):
        rel = np.linalg.norm(rows_sim[r] - ref[r]) / np.linalg.norm(ref[r])
        cos = float(rows_sim[r] @ ref[r] / np.linalg.norm(rows_sim[r]) / np.linalg.norm(ref[r]))
        assert rel <= 3e-2 and cos >= 0.995, (r, rel, cos)
