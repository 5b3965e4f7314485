"""Synthetic multi-tenant block-chain workloads of BASELINE.json `configs`.

A workload is a zoo of blocks (runs of Llama decoder layers), one chain of blocks per tenant
(ModelDescriptor::chain, proj/core/include/blocksim/zoo.hpp:56-63) and a burst of requests.
Shared blocks are the foundation layers every tenant routes through; private blocks are a
tenant's fine-tuned layers.
"""
from __future__ import annotations

from dataclasses import dataclass, field

from .device import BlockShape


@dataclass
class Workload:
    name: str
    shape: BlockShape                 # every block of the zoo has this shape
    block_names: list[str]
    chains: list[list[int]]           # per tenant: block indices in chain order
    req_tenant: list[int]
    req_prompt: list[int]
    req_output: list[int]
    max_batch_tokens: int = 4096      # configs/base.json:27
    seed: int = 1
    notes: dict = field(default_factory=dict)
    block_comps: list[str] | None = None  # per block 'a'/'f' component sequence (zoo blocks)
    # per block: None, or (base block index, adapter name) for a LoRA variant that shares the
    # base's weights (the reference zoo's fused attention, attach "fuse"; gen_configs.py:88-106)
    block_lora: list | None = None
    # per request: prefix group (-1 none) and shared prefix tokens (workload.hpp:19-20)
    req_prefix_group: list | None = None
    req_prefix_tokens: list | None = None

    @property
    def n_requests(self) -> int:
        return len(self.req_tenant)

    def rows_at_block(self) -> list[int]:
        """Decode rows each block serves per token step (per-block batch size)."""
        rows = [0] * len(self.block_names)
        for t in self.req_tenant:
            for b in self.chains[t]:
                rows[b] += 1
        return rows


def llama_blocks(n_layers_total: int, layers_per_block: int, d: int, heads: int, d_ff: int,
                 max_pos: int) -> tuple[BlockShape, int]:
    assert n_layers_total % layers_per_block == 0
    return (BlockShape(n_layers=layers_per_block, d_model=d, n_heads=heads, d_ff=d_ff,
                       max_pos=max_pos), n_layers_total // layers_per_block)


def shared_prefix_zoo(name: str, shape: BlockShape, n_positions: int, n_shared: int,
                      n_tenants: int, per_tenant: int, prompt: int, output: int,
                      max_batch_tokens: int = 4096) -> Workload:
    """n_shared foundation blocks used by every tenant, then private blocks per tenant."""
    names = [f"b{i}" for i in range(n_shared)]
    chains = []
    for t in range(n_tenants):
        chain = list(range(n_shared))
        for p in range(n_shared, n_positions):
            chain.append(len(names))
            names.append(f"t{t}.b{p}")
        chains.append(chain)
    # requests interleave tenants (arrival order round-robins apps, scenario.cpp:198-199)
    n = n_tenants * per_tenant
    req_tenant = [i % n_tenants for i in range(n)]
    return Workload(name, shape, names, chains, req_tenant, [prompt] * n, [output] * n,
                    max_batch_tokens)


def c1_tiny(output: int = 64) -> Workload:
    """configs[0]: tiny 4-layer decoder (d=256, 4 heads) in 2 blocks, 2 tenants share block 0,
    batch 8, 64-token decode (prompt 16, d_ff 768)."""
    shape = BlockShape(n_layers=2, d_model=256, n_heads=4, d_ff=768, max_pos=256)
    return shared_prefix_zoo("c1-tiny", shape, 2, 1, 2, 4, 16, output)


def c2_llama7b(prompt: int = 512, output: int = 128) -> Workload:
    """configs[1]: Llama-2-7B-shaped, 32 layers in 4-layer blocks, 4 fine-tuned variants share
    the first 24 layers (6 blocks), each owns 2 private blocks; mixed batch 64 (16 per tenant)."""
    shape, npos = llama_blocks(32, 4, 4096, 32, 11008, prompt + output + 16)
    return shared_prefix_zoo("c2-llama7b-4tenant", shape, npos, 6, 4, 16, prompt, output)


def c3_llama7b_16tenant(prompt: int = 2048, output: int = 256) -> Workload:
    """configs[2]: 7B shape, 16 tenants x 4 requests share blocks 0-5, private blocks 6-7."""
    shape, npos = llama_blocks(32, 4, 4096, 32, 11008, prompt + output + 16)
    return shared_prefix_zoo("c3-llama7b-16tenant", shape, npos, 6, 16, 4, prompt, output,
                             max_batch_tokens=8192)


def c4_llama13b(prompt: int = 512, output: int = 128) -> Workload:
    """configs[3]: Llama-2-13B shape (d=5120, 40 heads, d_ff=13824), 10 blocks x 4 layers,
    4 tenants share blocks 0-7."""
    shape, npos = llama_blocks(40, 4, 5120, 40, 13824, prompt + output + 16)
    return shared_prefix_zoo("c4-llama13b-4tenant", shape, npos, 8, 4, 16, prompt, output)


def c5_llama7b_8tenant(prompt: int = 512, output: int = 128) -> Workload:
    """configs[4]: the speculative-execution case - batch 256 over 8 tenants (32 requests each),
    7B shape, blocks 0-5 shared, 6-7 private. Its cosine equivalence check at batch 256 is
    tests/test_gpu_speculation.py::test_speculative_stage_at_c5_scale; the decode step of the
    workload runs like the others (bench.py --config c5); 8 B200 = one replica per GPU."""
    shape, npos = llama_blocks(32, 4, 4096, 32, 11008, prompt + output + 16)
    return shared_prefix_zoo("c5-llama7b-8tenant", shape, npos, 6, 8, 32, prompt, output,
                             max_batch_tokens=8192)


def lora_variant(wl: Workload, name: str) -> Workload:
    """The same zoo with every tenant-private block made a rank-16 LoRA variant of one shared
    base block per chain position (the base's weights + the tenant's adapter): the reference's
    LoRA models whose fused attention layers are their own blocks. Private positions then decode
    in one launch per position that streams the base weights once (be_exec_lora_group_dev)."""
    import dataclasses
    names = list(wl.block_names)
    comps = list(wl.block_comps) if wl.block_comps else None
    lora = [None] * len(names)
    base_of = {}
    shared = set.intersection(*[set(c) for c in wl.chains]) if len(wl.chains) > 1 else set()
    for t, ch in enumerate(wl.chains):
        for p, b in enumerate(ch):
            if b in shared:
                continue
            if p not in base_of:
                base_of[p] = len(names)
                names.append(f"base.b{p}")
                lora.append(None)
                if comps is not None:
                    comps.append(comps[b])
            lora[b] = (base_of[p], f"t{t}.p{p}")
    return dataclasses.replace(wl, name=name, block_names=names, block_comps=comps,
                               block_lora=lora)


def c2_lora(prompt: int = 512, output: int = 128) -> Workload:
    """C2 with the tenants' private blocks as LoRA variants of shared base blocks (not a BASELINE
    config: the multi-tenant adapter path of SURVEY §8(f) rank 3, measured beside C2)."""
    return lora_variant(c2_llama7b(prompt, output), "c2-lora-llama7b-4tenant")


CONFIGS = {"c1": c1_tiny, "c2": c2_llama7b, "c3": c3_llama7b_16tenant, "c4": c4_llama13b,
           "c5": c5_llama7b_8tenant, "c2lora": c2_lora}
