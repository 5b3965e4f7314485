"""Per-tile timeline of CTA 0 in a round-robin (prefill) GEMM launch of one epilogue mode
(library built with -DBE_EXP_RR_TRACE=<mode>: 1 kResid, 2 kSwiGLU, 3 kQKV): how long the MMA
warp waits for a free accumulator, the tile's MMA time, how long the epilogue waits for the
accumulator and how long it runs.
  BE_LIB_PATH=scripts/variants/libblockexec_rrtrace3.so python scripts/rr_trace.py"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2404_18322_b200 import device as dev  # noqa: E402
from paper_2404_18322_b200._lib import lib  # noqa: E402

batch, prompt, d = 4, 2048, 4096
ctx = dev.Context(0)
shape = dev.BlockShape(n_layers=1, d_model=d, n_heads=32, d_ff=11008, max_pos=4096)
blk = dev.Block(ctx, shape, "probe", seed=1)
ppr = prompt // 16
pool = dev.KvPool(ctx, blk, batch * ppr + 1)
n = batch * prompt
ws = dev.Workspace(ctx, shape, max_tokens=n, max_rows=batch, max_pages=ppr)
pt = np.arange(batch * ppr, dtype=np.int32).reshape(batch, ppr)
toks = [(r * prompt + p, r * prompt + p, int(pt[r, p // 16]) * 16 + p % 16, p, r)
        for r in range(batch) for p in range(prompt)]
x = torch.randn(n, d, device="cuda").to(torch.bfloat16)
y = torch.empty_like(x)
for _ in range(3):
    dev.exec_batch(ctx, blk, pool, ws, dev.PHASE_PREFILL, toks, pt, x, y)
ctx.sync()
buf = np.zeros((64, 6), np.uint64)
f = lib().be_exp_rr_trace
f.argtypes = [C.c_void_p]
assert f(buf.ctypes.data) == 0
ld = np.zeros(64, np.uint64)
g = lib().be_exp_rr_ld
g.argtypes = [C.c_void_p]
g(ld.ctypes.data)
tr = buf.astype(np.int64)
tr = tr[tr[:, 5] > 0]
t0 = tr[0, 0]
print(f"{len(tr)} tiles of CTA 0 (us from its first tile)")
print(" tile  mma_wait_acc  mma(start->commit)  epi_wait_acc  epilogue  (warp 2)")
for i, r in enumerate(tr):
    print(f"{i:5d} {(r[1]-r[0])/1e3:12.2f} {(r[5]-r[1])/1e3:18.2f} {(r[3]-r[2])/1e3:13.2f} {(r[4]-r[3])/1e3:9.2f}")
