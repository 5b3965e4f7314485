"""Multi-tenant LoRA at a private chain position, C2 shape (7B 4-layer blocks, 4 tenants x 16
decode rows, context 512): (a) four fully fine-tuned private blocks in one grouped launch
(be_exec_group_dev, each streams its own weights), (b) one base block + four rank-16 adapters
in one launch (be_exec_lora_batch_dev: the base weights stream once), (c) the base block alone
at 64 rows. Device time per block run, median of 20. Prints one JSON line.

  python scripts/lora_probe.py
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2404_18322_b200 import device as dev  # noqa: E402
from paper_2404_18322_b200._lib import check, lib  # noqa: E402


def main():
    ctx = dev.Context(0)
    L = lib()
    P, I = C.c_void_p, C.c_int
    L.be_exec_group_dev.restype = I
    L.be_exec_group_dev.argtypes = [P, I, P, P, P, I, I, P, I, P, P, P, P]
    shape = dev.BlockShape(n_layers=4, d_model=4096, n_heads=32, d_ff=11008, max_pos=640)
    T, rows, ctxlen = 4, 16, 512
    n = T * rows
    pages = ctxlen // 16 + 1
    pt = torch.arange(n * pages, dtype=torch.int32, device="cuda").reshape(n, pages)
    toks = torch.tensor([(r, r, int(pt[r, ctxlen // 16]) * 16 + ctxlen % 16, ctxlen, r)
                         for r in range(n)], dtype=torch.int32, device="cuda")
    x = torch.randn(n, shape.d_model, device="cuda").to(torch.bfloat16)
    y = torch.empty_like(x)
    ws = dev.Workspace(ctx, shape, max_tokens=n, max_rows=n, max_pages=pages)
    stream = torch.cuda.ExternalStream(ctx.stream.value)

    def timed(fn, reps=20):
        fn()
        ctx.sync()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            ctx.sync()
            ts.append(a.elapsed_time(b) * 1e3)
        return round(float(np.median(ts)), 1)

    res = {"case": "private position of C2: 4 tenants x 16 decode rows, 7B 4-layer blocks, "
                   "ctx 512"}
    blks = [dev.Block(ctx, shape, f"t{t}.b6", seed=1) for t in range(T)]
    pools = [dev.KvPool(ctx, b, n * pages) for b in blks]
    bh = (C.c_void_p * T)(*[b.h.value for b in blks])
    ph = (C.c_void_p * T)(*[p.h.value for p in pools])

    def grouped():
        check(L.be_exec_group_dev(ctx.h, T, bh, ph, ws.h, dev.PHASE_DECODE, n,
                                  C.c_void_p(toks.data_ptr()), pages, C.c_void_p(pt.data_ptr()),
                                  C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()),
                                  C.c_void_p(0)), ctx.h)
    res["grouped_full_blocks_us"] = timed(grouped) if "--only-lora" not in sys.argv else None
    for p in pools[1:]:
        p.free()
    for b in blks[1:]:
        b.free()
    base, pool = blks[0], pools[0]
    loras = [dev.Lora(ctx, base, f"t{t}", seed=1) for t in range(T)]
    lh = (C.c_void_p * T)(*[lo.h.value for lo in loras])
    idx = torch.tensor([r // rows for r in range(n)], dtype=torch.int32, device="cuda")

    def lora():
        check(L.be_exec_lora_batch_dev(ctx.h, base.h, pool.h, ws.h, dev.PHASE_DECODE, n,
                                       C.c_void_p(toks.data_ptr()), pages,
                                       C.c_void_p(pt.data_ptr()), T, lh,
                                       C.c_void_p(idx.data_ptr()), C.c_void_p(x.data_ptr()),
                                       C.c_void_p(y.data_ptr()), C.c_void_p(0)), ctx.h)

    def plain():
        check(L.be_exec_batch_dev(ctx.h, base.h, pool.h, ws.h, dev.PHASE_DECODE, n,
                                  C.c_void_p(toks.data_ptr()), pages, C.c_void_p(pt.data_ptr()),
                                  C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()),
                                  C.c_void_p(0)), ctx.h)
    res["base_plus_4_lora_us"] = timed(lora, 3 if "--only-lora" in sys.argv else 20)
    res["base_alone_us"] = timed(plain) if "--only-lora" not in sys.argv else None
    res["weight_bytes_grouped"] = T * shape.param_bytes
    res["weight_bytes_lora"] = shape.param_bytes + T * 4 * 4 * 2 * 4096 * 16 * 2
    print(json.dumps(res), flush=True)
    for lo in loras:
        lo.free()
    ws.free()
    pool.free()
    base.free()
    ctx.close()


if __name__ == "__main__":
    main()
