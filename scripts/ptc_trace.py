"""Phase timeline of the tcgen05 prefill attention (library built with -DBE_EXP_PTC_TRACE):
per kv iteration of CTAs 0..3 (thread 0), the ns spent waiting for S = Q K^T (and the P V
before it), in the softmax, at the CTA barrier + waiting for V, issuing P V and the next S.
  BE_LIB_PATH=scripts/variants/libblockexec_ptctrace.so python scripts/ptc_trace.py"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2404_18322_b200 import device as dev  # noqa: E402
from paper_2404_18322_b200._lib import lib  # noqa: E402

batch, prompt, d = 16, 2048, 4096
H = d // 128
ctx = dev.Context(0)
shape = dev.BlockShape(n_layers=1, d_model=d, n_heads=H, d_ff=11008, max_pos=4096, components="a")
blk = dev.Block(ctx, shape, "probe", seed=1)
ppr = (prompt + 15) // 16
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
names = ["wait_S", "softmax", "bar+wait_V", "issue PV+S", "tmem_ld", "max", "exp+pack", "st+rest"]
cols = [(0, 2), (2, 3), (3, 4), (4, 5), (2, 6), (6, 7), (7, 8), (8, 3)]
for c in range(4):
    tr = buf[c].astype(np.int64)
    tr = tr[tr[:, 5] > 0]
    nxt = tr[1:, 0] - tr[:-1, 5]
    print(f"cta {c}: {len(tr)} iterations; median ns:",
          {n: int(np.median(tr[:, b] - tr[:, a])) for n, (a, b) in zip(names, cols)},
          "next-iter gap", int(np.median(nxt)) if len(nxt) else None,
          "total us", round((tr[-1, 5] - tr[0, 0]) / 1e3, 1))
