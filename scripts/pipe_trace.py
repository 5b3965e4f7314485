"""Per-tile timeline of CTA 0 of the warp-specialised prefill attention (BE_PREFILL_TC=1,
library built with -DBE_EXP_PTC_TRACE): when the softmax starts waiting for S(t), gets it,
finishes P(t); when the MMA warp issued S(t), saw P(t), saw V(t).
  BE_LIB_PATH=scripts/variants/libblockexec_pipetrace.so python scripts/pipe_trace.py"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("BE_PREFILL_TC", "1")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2404_18322_b200 import device as dev  # noqa: E402
from paper_2404_18322_b200._lib import lib  # noqa: E402

batch, prompt, d = 16, 2048, 4096
ctx = dev.Context(0)
shape = dev.BlockShape(n_layers=1, d_model=d, n_heads=32, d_ff=11008, max_pos=4096, components="a")
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
for _ in range(2):
    dev.exec_batch(ctx, blk, pool, ws, dev.PHASE_PREFILL, toks, pt, x, y)
ctx.sync()
buf = np.zeros((4, 64, 9), np.uint64)
f = lib().be_exp_ptc_trace
f.argtypes = [C.c_void_p]
assert f(buf.ctypes.data) == 0
tr = buf[0].astype(np.int64)
t0 = tr[0, 0]
print(" tile  sm_wait_S  softmax  | mma: S issued  P seen  V seen   (us from the first S wait)")
for i in range(40):
    r = tr[i]
    if r[5] == 0:
        break
    print(f"{i:5d} {(r[1]-r[0])/1e3:9.2f} {(r[5]-r[1])/1e3:8.2f}  | {(r[2]-t0)/1e3:9.2f} {(r[3]-t0)/1e3:8.2f} {(r[4]-t0)/1e3:8.2f}")
