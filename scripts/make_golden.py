#!/usr/bin/env python3
"""Generates tests/golden/llama_layer_*.npz: HuggingFace transformers' LlamaDecoderLayer (fp32)
run with the oracle's synthetic weights on synthetic inputs. These fixtures pin the CPU oracle's
decoder-layer arithmetic (RMSNorm, rotate_half RoPE, causal softmax attention, SwiGLU,
residuals) to an independent, widely used implementation; the reference itself (blocksim) holds
no arithmetic for the block forward.

  python scripts/make_golden.py     # writes tests/golden/*.npz (run in the build container)
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2404_18322_b200.device import BlockShape  # noqa: E402


def golden(d, heads, dff, tokens, seed, name, out_path):
    from transformers import LlamaConfig
    from transformers.models.llama.modeling_llama import LlamaDecoderLayer, LlamaRotaryEmbedding
    shape = BlockShape(n_layers=1, d_model=d, n_heads=heads, d_ff=dff, max_pos=256)
    ob = O.OracleBlock(shape, name, seed=seed)
    cfg = LlamaConfig(hidden_size=d, intermediate_size=dff, num_attention_heads=heads,
                      num_key_value_heads=heads, rms_norm_eps=shape.norm_eps,
                      rope_theta=shape.rope_theta, max_position_embeddings=256,
                      attention_bias=False, mlp_bias=False)
    cfg._attn_implementation = "eager"
    layer = LlamaDecoderLayer(cfg, layer_idx=0).float().eval()
    with torch.no_grad():
        sd = layer.self_attn
        sd.q_proj.weight.copy_(torch.from_numpy(ob.weight(0, "wq")))
        sd.k_proj.weight.copy_(torch.from_numpy(ob.weight(0, "wk")))
        sd.v_proj.weight.copy_(torch.from_numpy(ob.weight(0, "wv")))
        sd.o_proj.weight.copy_(torch.from_numpy(ob.weight(0, "wo")))
        layer.mlp.gate_proj.weight.copy_(torch.from_numpy(ob.weight(0, "wg")))
        layer.mlp.up_proj.weight.copy_(torch.from_numpy(ob.weight(0, "wu")))
        layer.mlp.down_proj.weight.copy_(torch.from_numpy(ob.weight(0, "wd")))
        layer.input_layernorm.weight.fill_(1.0)
        layer.post_attention_layernorm.weight.fill_(1.0)
    x = O.synth(tokens * d, seed, f"golden:{name}:inputs", 1.7320508).reshape(tokens, d)
    rope = LlamaRotaryEmbedding(cfg)
    pos = torch.arange(tokens)[None]
    hs = torch.from_numpy(x)[None]
    cos, sin = rope(hs, pos)
    mask = torch.full((tokens, tokens), float("-inf")).triu(1)[None, None]
    with torch.no_grad():
        out = layer(hs, attention_mask=mask, position_ids=pos, position_embeddings=(cos, sin))
    y = (out[0] if isinstance(out, tuple) else out)[0].numpy()
    np.savez_compressed(out_path, x=x, y=y, d=d, heads=heads, dff=dff, seed=seed,
                        name=np.array(name))
    return x, y


def main():
    gdir = os.path.join(ROOT, "tests", "golden")
    os.makedirs(gdir, exist_ok=True)
    for d, h, f, t, seed in [(256, 4, 768, 12, 7), (512, 4, 1536, 9, 11)]:
        path = os.path.join(gdir, f"llama_layer_d{d}.npz")
        golden(d, h, f, t, seed, f"golden{d}", path)
        print("wrote", path)


if __name__ == "__main__":
    main()
