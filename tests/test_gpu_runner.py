"""End-to-end GPU parity of the executor loop on the C1 workload (BASELINE.json configs[0]):
2 tenants sharing block 0, batch 8, prompts 16, decode steps, against the fp32 oracle run along
the same chains. Activations cross block boundaries as bf16 on both sides (act_bytes_per_token =
2*d, costmodel.cpp:129-131). Decode steps are teacher-forced: the oracle consumes the GPU's
step input so errors do not compound. Tolerance: rel-L2 <= 2e-2, min row cosine >= 0.995 per
step (two blocks of bf16 storage per step)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2404_18322_b200 import device as dev  # noqa: E402
from paper_2404_18322_b200.runner import Runner  # noqa: E402
from paper_2404_18322_b200.workloads import c1_tiny  # noqa: E402

pytestmark = pytest.mark.gpu


def bf16_round(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16).float().numpy()


def oracle_chain(wl, n_steps, gpu_inputs):
    """Runs the oracle over the workload; gpu_inputs[k] = GPU input rows of decode step k."""
    from oracle import oracle as O
    s = wl.shape
    blocks = {}
    lora = getattr(wl, "block_lora", None) or [None] * len(wl.block_names)
    for b, name in enumerate(wl.block_names):
        if lora[b] is None:
            blocks[b] = O.OracleBlock(s, name, seed=wl.seed)
        else:  # LoRA variant: the base's weights with the adapter folded in
            blocks[b] = O.OracleBlock(s, wl.block_names[lora[b][0]], seed=wl.seed)
            blocks[b].add_lora(lora[b][1], wl.seed, s.init_scale, s.init_scale)
    max_tok = max(p + o for p, o in zip(wl.req_prompt, wl.req_output)) + 1
    seqs = {}
    first = []
    for r in range(wl.n_requests):
        p = wl.req_prompt[r]
        x = O.synth(p * s.d_model, wl.seed, f"inputs:req{r + 1}", 1.7320508).reshape(p, s.d_model)
        pg = getattr(wl, "req_prefix_group", None)
        if pg is not None and pg[r] >= 0:  # the group's common prefix (bh_workload.req_prefix_*)
            t = min(wl.req_prefix_tokens[r], p)
            x[:t] = O.synth(t * s.d_model, wl.seed, f"inputs:prefix{pg[r]}",
                            1.7320508).reshape(t, s.d_model)
        for b in wl.chains[wl.req_tenant[r]]:
            seqs[(r, b)] = blocks[b].new_seq(max_tok)
            x = bf16_round(blocks[b].forward([seqs[(r, b)]], [0] * p, list(range(p)), x))
        first.append(x[-1])
    outs = []
    for k in range(n_steps):
        xin = gpu_inputs[k]
        out = np.empty_like(xin)
        for r in range(wl.n_requests):
            pos = wl.req_prompt[r] + k
            x = xin[r:r + 1]
            for b in wl.chains[wl.req_tenant[r]]:
                x = bf16_round(blocks[b].forward([seqs[(r, b)]], [0], [pos], x))
            out[r] = x[0]
        outs.append(out)
    return np.stack(first), outs


def test_c1_runner_matches_oracle(ctx):
    wl = c1_tiny(output=6)
    run = Runner(ctx, wl, mode=1, use_graphs=True)
    run.run()
    n, d = wl.n_requests, wl.shape.d_model
    ins, outs = [], []
    buf = torch.empty(n, d, dtype=torch.bfloat16)
    for k in range(5):
        nb = run.decode_step(None, buf)
        assert nb == 3  # b0 (8 rows), t0.b1 (4), t1.b1 (4)
        outs.append(buf.float().numpy().copy())
    # inputs of step k are the outputs of step k-1; step 0 input is the prefill's first token
    first_ref, _ = oracle_chain(wl, 0, [])
    ins = [first_ref] + outs[:-1]
    _, ref = oracle_chain(wl, 5, ins)
    for k in range(1, 5):
        g, r = outs[k], ref[k]
        rel = np.linalg.norm(g - r) / np.linalg.norm(r)
        cos = ((g * r).sum(1) / np.linalg.norm(g, axis=1) / np.linalg.norm(r, axis=1)).min()
        assert rel <= 2e-2 and cos >= 0.995, (k, rel, cos)
    st = run.step_stats()
    assert st["graph_replayed"] == 1
    run.close()


def test_c1_lockstep_trace_is_convoy(ctx):
    wl = c1_tiny(output=4)
    run = Runner(ctx, wl, mode=1, use_graphs=False)
    run.run()
    run.clear_trace()
    run.decode_step()
    tr = run.trace()
    assert [t[1] for t in tr] == [0, 1, 2]
    assert [m[0] for m in tr[0][3]] == list(range(1, 9))
    assert [m[0] for m in tr[1][3]] == [1, 3, 5, 7]  # tenant 0 requests (round-robin arrivals)
    assert [m[0] for m in tr[2][3]] == [2, 4, 6, 8]
    assert all(m[2] == 17 for m in tr[0][3])  # context = prompt + first token
    run.close()


def test_c1_lora_runner_matches_oracle(ctx):
    """The executor loop with LoRA variants (workloads.lora_variant): the tenants' private
    blocks share one base block's weights plus their own rank-16 adapters; prefill runs each
    variant alone, decode runs both variants in one launch (be_exec_lora_group_dev). Same
    oracle comparison as the full-weight C1 test, the oracle folding each adapter into W."""
    from paper_2404_18322_b200.workloads import lora_variant
    wl = lora_variant(c1_tiny(output=6), "c1-lora")
    run = Runner(ctx, wl, mode=1, use_graphs=True)
    run.run()
    n, d = wl.n_requests, wl.shape.d_model
    outs = []
    buf = torch.empty(n, d, dtype=torch.bfloat16)
    for k in range(5):
        run.decode_step(None, buf)
        outs.append(buf.float().numpy().copy())
    first_ref, _ = oracle_chain(wl, 0, [])
    ins = [first_ref] + outs[:-1]
    _, ref = oracle_chain(wl, 5, ins)
    for k in range(1, 5):
        g, r = outs[k], ref[k]
        rel = np.linalg.norm(g - r) / np.linalg.norm(r)
        cos = ((g * r).sum(1) / np.linalg.norm(g, axis=1) / np.linalg.norm(r, axis=1)).min()
        assert rel <= 2e-2 and cos >= 0.995, (k, rel, cos)
    st = run.step_stats()
    assert st["graph_replayed"] == 1
    run.close()
