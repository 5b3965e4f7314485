"""Times be_kv_migrate on a Llama-7B-shaped 4-layer block for one request's 2048-token segment
(128 pages): all-copy, all-recompute, and the split plan_migration picks from the measured
per-page rates (the reference's rule, kv.cpp:16-58), on one GPU and across two (NVLink peer copy).

  python scripts/migration_probe.py            # prints one JSON line per case
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2404_18322_b200 import device as dev  # noqa: E402
from paper_2404_18322_b200 import policy as P  # noqa: E402

SHAPE = dev.BlockShape(n_layers=4, d_model=4096, n_heads=32, d_ff=11008, max_pos=4096)
TOK = 2048
NP = TOK // 16


def timed(ctx, fn, reps=5):
    st = torch.cuda.ExternalStream(ctx.stream.value, device=f"cuda:{ctx.device}")
    fn()
    ctx.sync()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        ctx.sync()
        ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))


def case(c_src, c_dst, label):
    blk_a = dev.Block(c_src, SHAPE, "mig", seed=1)
    blk_b = blk_a if c_dst is c_src else dev.Block(c_dst, SHAPE, "mig", seed=1)
    a = dev.KvPool(c_src, blk_a, NP + 1)
    b = dev.KvPool(c_dst, blk_b, NP + 1)
    ws = dev.Workspace(c_dst, SHAPE, max_tokens=TOK, max_rows=1, max_pages=NP)
    src = list(range(NP))
    dst = list(range(1, NP + 1))
    x = torch.randn(TOK, SHAPE.d_model, device=f"cuda:{c_dst.device}").to(torch.bfloat16)
    t_copy = timed(c_dst, lambda: dev.kv_migrate(c_dst, blk_b, a, b, ws, src, dst, 0))
    t_rec = timed(c_dst, lambda: dev.kv_migrate(c_dst, blk_b, a, b, ws, src, dst, NP, x, TOK))
    rec_pp = max(1, round(t_rec / NP))
    cp_pp = max(1, round(t_copy / NP))
    _, n_rec, n_cp, plan_us = P.plan_migration(NP, rec_pp, cp_pp)
    head = n_rec * 16
    t_plan = timed(c_dst, lambda: dev.kv_migrate(c_dst, blk_b, a, b, ws, src, dst, n_rec,
                                                 x[:head] if n_rec else None, head))
    seg_bytes = NP * a.page_bytes
    print(json.dumps({"case": label, "pages": NP, "segment_MB": round(seg_bytes / 1e6, 1),
                      "all_copy_us": round(t_copy, 1),
                      "copy_GBps": round(seg_bytes / t_copy / 1e3, 1),
                      "all_recompute_us": round(t_rec, 1),
                      "plan": {"recompute_pages": n_rec, "copy_pages": n_cp,
                               "modelled_us": plan_us},
                      "planned_us": round(t_plan, 1)}), flush=True)
    ws.free()
    a.free()
    b.free()
    blk_a.free()
    if blk_b is not blk_a:
        blk_b.free()


def main():
    c0 = dev.Context(0)
    case(c0, c0, "same GPU")
    if torch.cuda.device_count() > 1:
        c1 = dev.Context(1)
        case(c0, c1, "GPU0 -> GPU1 (NVLink)")
        c1.close()
    c0.close()


if __name__ == "__main__":
    main()
