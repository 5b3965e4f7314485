"""B200-native per-block batched execution path of BlockLLM (arXiv 2404.18322).

Multi-tenant requests are gathered into one batch at each shared block, run through the block's
decoder layers on hand-written sm_100a kernels (tcgen05/TMEM GEMMs fed by TMA, paged attention
over a block-local KV cache) and scattered back along their block chains.
"""
__all__ = ["device", "host"]
