"""LoRA zoos on the host side (no GPU): workloads.lora_variant builds the reference zoo's
fused-attention variants (each tenant-private block = a shared base block's weights + its
adapter), and the executor loop's control plane (dry run) accepts them, batches them exactly as
the full-weight zoo (same batch trace), and rejects malformed LoRA descriptions."""
import pytest

from paper_2404_18322_b200.runner import Runner
from paper_2404_18322_b200.workloads import c1_tiny, c2_llama7b, lora_variant


def test_lora_variant_structure():
    wl = lora_variant(c2_llama7b(), "c2-lora")
    base = c2_llama7b()
    assert wl.chains == base.chains
    assert wl.block_names[:len(base.block_names)] == base.block_names
    extra = wl.block_names[len(base.block_names):]
    assert extra == ["base.b6", "base.b7"]
    for b, name in enumerate(base.block_names):
        lo = wl.block_lora[b]
        if name.startswith("t"):  # private: a variant of the position's base block
            pos = int(name.split(".b")[1])
            assert lo is not None and wl.block_names[lo[0]] == f"base.b{pos}"
        else:
            assert lo is None
    assert all(wl.block_lora[len(base.block_names) + i] is None for i in range(2))


def test_lora_zoo_batches_like_the_full_zoo():
    plain, lora = c1_tiny(output=4), lora_variant(c1_tiny(output=4), "c1-lora")
    traces = []
    for wl in (plain, lora):
        run = Runner(None, wl, mode=1, dry_run=True)
        run.run()
        run.clear_trace()
        run.decode_step()
        traces.append([(t[1], [m[0] for m in t[3]]) for t in run.trace()])
        run.close()
    assert traces[0] == traces[1]


def test_runner_rejects_bad_lora_base():
    wl = lora_variant(c1_tiny(output=4), "c1-lora")
    bad = list(wl.block_lora)
    bad[1] = (1, "self")  # a block cannot be its own base
    import dataclasses
    with pytest.raises(Exception):
        Runner(None, dataclasses.replace(wl, block_lora=bad), mode=1, dry_run=True)
