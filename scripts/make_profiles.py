"""Measured B200 cost profiles in the reference's own format (§8 f rank 2).

blocksim prices a block run by bilinear lookup in per-component grids
(`profiles.json`: classes "attention:<dim>" / "ffn:<dim>", each with prefill and decode grids
us[batch][tokens]; `load_profiles`, proj/core/src/config.cpp:356-384; `Interp2D`,
costmodel.cpp:49-59). This script measures those grids on the GPU with the real kernels - one
component (a one-component block, 'a' or 'f') run through be_exec_batch, CUDA-event timed,
median of reps - so the reference's router and placement price B200 kernels instead of
synthetic curves:

  python scripts/make_profiles.py --out profiles/b200_profiles.json [--dims 4096 5120]

Decode point (batch n, tokens t): n requests each decoding one token at context t.
Prefill point (batch n, tokens t): n requests each prefilling a t-token prompt.
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import ctypes as C  # noqa: E402

from paper_2404_18322_b200 import device as dev  # noqa: E402
from paper_2404_18322_b200._lib import check, lib  # noqa: E402

BATCH = [1, 2, 4, 8, 16, 32, 64]
TOKENS = [1, 64, 256, 512, 1024, 2048]
PREFILL_BATCH = [1, 2, 4, 8, 16, 32]
PREFILL_TOKENS = [1, 64, 256, 512, 1024]
SHAPES = {4096: (32, 11008), 5120: (40, 13824), 8192: (64, 28672)}


def time_call(ctx, fn, reps):
    """Median device time of fn() with CUDA events on the context's stream (where it runs)."""
    st = torch.cuda.ExternalStream(ctx.stream.value)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(reps)]
    fn()  # warm
    ctx.sync()
    for a, b in ev:
        a.record(st)
        fn()
        b.record(st)
    ctx.sync()
    return statistics.median(a.elapsed_time(b) * 1e3 for a, b in ev)


def grid(ctx, kind, d, phase, batches, tokens, reps):
    heads, dff = SHAPES[d]
    shape = dev.BlockShape(n_layers=1, d_model=d, n_heads=heads, d_ff=dff, max_pos=4096,
                           components=kind)
    blk = dev.Block(ctx, shape, f"prof.{kind}", seed=1)
    max_rows = max(batches)
    pages_per_row = (max(tokens) + 1 + 15) // 16
    n_pages = max_rows * pages_per_row + 1
    pool = dev.KvPool(ctx, blk, n_pages)
    max_tok = max(batches) * (max(tokens) if phase == dev.PHASE_PREFILL else 1)
    ws = dev.Workspace(ctx, shape, max_tokens=max_tok, max_rows=max_rows,
                       max_pages=pages_per_row)
    pt = np.arange(max_rows * pages_per_row, dtype=np.int32).reshape(max_rows, pages_per_row)
    x = torch.randn(max_tok, d, device="cuda").to(torch.bfloat16)
    y = torch.empty_like(x)
    us = []
    for n in batches:
        row = []
        for t in tokens:
            if phase == dev.PHASE_DECODE:
                toks = [(r, r, int(pt[r, (t - 1) // 16]) * 16 + (t - 1) % 16, t - 1, r)
                        for r in range(n)]
            else:
                toks = [(r * t + p, r * t + p, int(pt[r, p // 16]) * 16 + p % 16, p, r)
                        for r in range(n) for p in range(t)]
            # metadata on the device once (be_exec_batch_dev): the timing is the block run only
            tk = torch.tensor(toks, dtype=torch.int32).cuda()
            ptd = torch.from_numpy(np.ascontiguousarray(pt[:n])).cuda()

            def run():
                check(lib().be_exec_batch_dev(ctx.h, blk.h, pool.h, ws.h, phase, len(toks),
                                              C.c_void_p(tk.data_ptr()), pt.shape[1],
                                              C.c_void_p(ptd.data_ptr()),
                                              C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()),
                                              C.c_void_p(0)),  # the context's stream
                      ctx.h)
            torch.cuda.synchronize()  # metadata copies (torch's stream) before the run
            row.append(round(time_call(ctx, run, reps), 3))
        us.append(row)
    ws.free()
    pool.free()
    blk.free()
    return {"batch": list(batches), "tokens": list(tokens), "us": us}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="profiles/b200_profiles.json")
    ap.add_argument("--dims", type=int, nargs="+", default=[4096, 5120])
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    ctx = dev.Context(0)
    classes = {}
    for d in a.dims:
        for kind, name in (("a", "attention"), ("f", "ffn")):
            classes[f"{name}:{d}"] = {
                "prefill": grid(ctx, kind, d, dev.PHASE_PREFILL, PREFILL_BATCH, PREFILL_TOKENS,
                                a.reps),
                "decode": grid(ctx, kind, d, dev.PHASE_DECODE, BATCH, TOKENS, a.reps),
                # CostModel::kv_bytes_per_token convention: 4 * embed_dim for an attention
                # component (K and V, bf16), nothing for an ffn
                "kv_bytes_per_token": 4 * d if kind == "a" else 0,
            }
            print(name, d, "done", flush=True)
    out = {
        "schema_version": 1,
        "source": "measured on B200 (sm_100a kernels of this repo, be_exec_batch, CUDA events, "
                  "median of reps); scripts/make_profiles.py",
        "device_classes": {"b200": 1.0},
        "classes": classes,
        "surrogate": {"attention_only": 37.43, "ffn_only": 1.71, "one_layer": 22.91,
                      "multi_layer": 18.55, "allow_adapter_blocks": False,
                      "accept_threshold": 0.95},
    }
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    ctx.close()


if __name__ == "__main__":
    main()
