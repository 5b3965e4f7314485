"""One prefill batch through an FFN-only 7B block (gather, gate/up GEMM with the SwiGLU
epilogue, down GEMM with the residual epilogue) - a target for ncu on the round-robin GEMMs.
  python scripts/prefill_ffn_probe.py [--batch 4 --prompt 2048]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2404_18322_b200 import device as dev  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=4)
ap.add_argument("--prompt", type=int, default=2048)
a = ap.parse_args()
d = 4096
ctx = dev.Context(0)
shape = dev.BlockShape(n_layers=1, d_model=d, n_heads=32, d_ff=11008, max_pos=4096, components="f")
blk = dev.Block(ctx, shape, "probe", seed=1)
ppr = (a.prompt + 15) // 16
pool = dev.KvPool(ctx, blk, a.batch * ppr + 1)
n = a.batch * a.prompt
ws = dev.Workspace(ctx, shape, max_tokens=n, max_rows=a.batch, max_pages=ppr)
pt = np.arange(a.batch * ppr, dtype=np.int32).reshape(a.batch, ppr)
toks = [(r * a.prompt + p, r * a.prompt + p, int(pt[r, p // 16]) * 16 + p % 16, p, r)
        for r in range(a.batch) for p in range(a.prompt)]
x = torch.randn(n, d, device="cuda").to(torch.bfloat16)
y = torch.empty_like(x)
for _ in range(2):
    ctx.prof_enable(True)
    dev.exec_batch(ctx, blk, pool, ws, dev.PHASE_PREFILL, toks, pt, x, y)
    recs = ctx.prof_read()
    ctx.prof_enable(False)
    print(" ".join(f"{r['cls']}={r['ms']:.3f}ms" for r in recs))
