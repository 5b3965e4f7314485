"""Per-kernel times of one prefill batch of one attention component (be_prof event timing):
QKV GEMM, prefill attention (tile index + tensor-core kernel), O GEMM.
  python scripts/prefill_attn_probe.py [--batch 32 --prompt 1024 --d 4096]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2404_18322_b200 import device as dev  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=32)
ap.add_argument("--prompt", type=int, default=1024)
ap.add_argument("--d", type=int, default=4096)
a = ap.parse_args()
H = a.d // 128
ctx = dev.Context(0)
shape = dev.BlockShape(n_layers=1, d_model=a.d, n_heads=H, d_ff=11008, max_pos=4096, components="a")
blk = dev.Block(ctx, shape, "probe", seed=1)
ppr = (a.prompt + 15) // 16
pool = dev.KvPool(ctx, blk, a.batch * ppr + 1)
n = a.batch * a.prompt
ws = dev.Workspace(ctx, shape, max_tokens=n, max_rows=a.batch, max_pages=ppr)
pt = np.arange(a.batch * ppr, dtype=np.int32).reshape(a.batch, ppr)
toks = [(r * a.prompt + p, r * a.prompt + p, int(pt[r, p // 16]) * 16 + p % 16, p, r)
        for r in range(a.batch) for p in range(a.prompt)]
x = torch.randn(n, a.d, device="cuda").to(torch.bfloat16)
y = torch.empty_like(x)
dev.exec_batch(ctx, blk, pool, ws, dev.PHASE_PREFILL, toks, pt, x, y)
ctx.sync()
for _ in range(2):
    ctx.prof_enable(True)
    dev.exec_batch(ctx, blk, pool, ws, dev.PHASE_PREFILL, toks, pt, x, y)
    recs = ctx.prof_read()
    ctx.prof_enable(False)
    print(" ".join(f"{r['cls']}={r['ms']:.3f}ms" for r in recs))
flops = a.batch * (a.prompt * (a.prompt + 1) / 2) * H * 128 * 4
print(f"attention flops {flops / 1e9:.1f} GFLOP")
