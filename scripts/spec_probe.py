"""Cost of the speculative stage at C5 scale (batch 256, 7B-shaped 4-layer blocks) on one GPU:
plain (verify block, then the next block on its output) vs be_exec_speculative (draft surrogate
+ next block on a side stream, verify concurrently, K7 verdict, rejected rows re-run) with every
row accepted, half, and none. Prints one JSON line.

  python scripts/spec_probe.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2404_18322_b200 import device as dev  # noqa: E402


def main():
    ctx = dev.Context(0)
    shape = dev.BlockShape(n_layers=4, d_model=4096, n_heads=32, d_ff=11008, max_pos=640)
    n, prompt, d = 256, 512, shape.d_model
    pages = (prompt + 16) // 16
    pt = np.arange(n * pages, dtype=np.int32).reshape(n, pages)
    names = {"verify": ("b3", shape), "draft": ("b3", shape.surrogate(0.5)), "next": ("b4", shape)}
    gpu, pools = {}, {}
    for k, (nm, sh) in names.items():
        gpu[k] = dev.Block(ctx, sh, nm, seed=9)
        pools[k] = dev.KvPool(ctx, gpu[k], n * pages)
    ws_main = dev.Workspace(ctx, shape, max_tokens=8192, max_rows=n, max_pages=pages)
    ws_side = dev.Workspace(ctx, shape, max_tokens=n, max_rows=n, max_pages=pages)
    for k in names:  # prompt KV in 16-request prefill batches
        for r0 in range(0, n, 16):
            xp = torch.randn(16 * prompt, d, device="cuda").to(torch.bfloat16)
            toks = [(i * prompt + p, i * prompt + p, int(pt[r0 + i, p // 16]) * 16 + p % 16, p,
                     r0 + i) for i in range(16) for p in range(prompt)]
            dev.exec_batch(ctx, gpu[k], pools[k], ws_main, dev.PHASE_PREFILL, toks, pt, xp,
                           torch.empty_like(xp))
    ctx.sync()
    x = torch.randn(n, d, device="cuda").to(torch.bfloat16)
    dtoks = [(r, r, int(pt[r, prompt // 16]) * 16 + prompt % 16, prompt, r) for r in range(n)]
    y_draft, y_true, z = (torch.zeros(n, d, dtype=torch.bfloat16, device="cuda")
                          for _ in range(3))
    st = {k: (gpu[k], pools[k], ws_main if k == "verify" else ws_side, dtoks, pt) for k in names}
    stream = torch.cuda.ExternalStream(ctx.stream.value)

    def timed(fn, reps=10):
        fn()
        ctx.sync()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            out = fn()
            b.record(stream)
            ctx.sync()
            ts.append(a.elapsed_time(b))
        return float(np.median(ts)), out

    def plain():
        dev.exec_batch(ctx, gpu["verify"], pools["verify"], ws_main, dev.PHASE_DECODE, dtoks, pt,
                       x, y_true)
        dev.exec_batch(ctx, gpu["next"], pools["next"], ws_main, dev.PHASE_DECODE, dtoks, pt,
                       y_true, z)

    res = {"case": "C5 speculative stage, batch 256, 7B 4-layer blocks, ctx 512"}
    res["plain_ms"], _ = timed(plain)
    cos, _, _ = dev.exec_speculative(ctx, st["verify"], st["draft"], st["next"], x, y_draft,
                                     y_true, z, 0.95)
    for label, thr in (("all_accepted", -2.0), ("half", float(np.median(cos))),
                       ("none_accepted", 2.0)):
        ms, out = timed(lambda: dev.exec_speculative(ctx, st["verify"], st["draft"], st["next"],
                                                     x, y_draft, y_true, z, thr))
        res[f"spec_{label}_ms"] = ms
        res[f"spec_{label}_accepted"] = int(out[2])
    res["cos_median"] = float(np.median(cos))
    res["cos_min"] = float(cos.min())
    print(json.dumps(res), flush=True)
    for k in names:
        pools[k].free()
        gpu[k].free()
    ws_main.free()
    ws_side.free()
    ctx.close()


if __name__ == "__main__":
    main()
