"""Prefix groups in the executor loop (create_kv_for_step's donor rule, scenario.cpp:671-695):
requests of a tenant share a 40-token prompt prefix; at every block the first member to finish
prefill donates its whole prefix pages and the others' page tables point at them (their prefill
rewrites the same K/V there). Sharing must not change a single bit of any output: the same
workload run with sharing disabled (BH_PREFIX_SHARE=0: every request keeps private pages) gives
identical rows after prefill and after every decode step, while holding fewer KV bytes."""
import dataclasses
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2404_18322_b200.pipeline import _DevRows  # noqa: E402
from paper_2404_18322_b200.runner import Runner  # noqa: E402
from paper_2404_18322_b200.workloads import c1_tiny  # noqa: E402

pytestmark = pytest.mark.gpu


def rows(run, n, d):
    return torch.as_tensor(_DevRows(run.arena_ptr, n, d), device="cuda").view(
        torch.bfloat16).float().cpu().numpy()


@pytest.mark.parametrize("mode", [0, 1])
def test_prefix_sharing_is_bit_transparent(ctx, mode):
    wl = c1_tiny(output=5)
    n, d = wl.n_requests, wl.shape.d_model
    wl = dataclasses.replace(wl, req_prompt=[48, 44, 60, 41, 48, 52, 47, 50],
                             req_prefix_group=list(wl.req_tenant), req_prefix_tokens=[40] * n)
    shared = Runner(ctx, wl, mode=mode, use_graphs=False)
    os.environ["BH_PREFIX_SHARE"] = "0"
    try:
        private = Runner(ctx, wl, mode=mode, use_graphs=False)
    finally:
        del os.environ["BH_PREFIX_SHARE"]
    if mode == 1:
        shared.run()
        private.run()
        ctx.sync()
        assert np.array_equal(rows(shared, n, d), rows(private, n, d))
        used_s, saved = shared.kv_bytes()
        used_p, saved_p = private.kv_bytes()
        assert saved > 0 and saved_p == 0 and used_s < used_p
        outs = [rows(shared, n, d)]
        for _ in range(4):
            shared.decode_step()
            private.decode_step()
            ctx.sync()
            outs.append(rows(shared, n, d))
            assert np.array_equal(outs[-1], rows(private, n, d))
        # and the shared run against the fp32 oracle along the chains (prefix rows from the
        # group's stream), teacher-forced per step as test_gpu_runner.py
        from test_gpu_runner import oracle_chain
        first_ref, ref = oracle_chain(wl, 4, outs[:-1])
        for k, (g, r) in enumerate(zip([outs[0]] + outs[1:], [first_ref] + ref)):
            rel = np.linalg.norm(g - r) / np.linalg.norm(r)
            cos = ((g * r).sum(1) / np.linalg.norm(g, axis=1) / np.linalg.norm(r, axis=1)).min()
            assert rel <= 2e-2 and cos >= 0.995, (k, rel, cos)
    else:  # the reference's event order, to completion
        shared.run()
        private.run()
        ctx.sync()
        assert shared.trace() == private.trace()
        assert np.array_equal(rows(shared, n, d), rows(private, n, d))
        assert shared.kv_bytes()[1] > 0
    shared.close()
    private.close()
