#!/usr/bin/env python3
"""Device-time sweep of the tcgen05 stream-K GEMM (graph replay, weights > L2).

  python scripts/gemm_bench.py [--reps 40]
Prints us/launch, achieved GB/s (algorithmic bytes 2*(NK+MK+MN)) and TFLOP/s per shape.
"""
import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2404_18322_b200 import device as dev  # noqa: E402
from paper_2404_18322_b200._lib import lib, check  # noqa: E402

SHAPES = [  # (name, N, K, ntok)
    ("qkv7b", 12288, 4096, 64), ("o7b", 4096, 4096, 64), ("gu7b", 22016, 4096, 64),
    ("down7b", 4096, 11008, 64),
    ("qkv7b_m16", 12288, 4096, 16), ("o7b_m16", 4096, 4096, 16), ("gu7b_m16", 22016, 4096, 16),
    ("down7b_m16", 4096, 11008, 16),
    ("gu7b_m256", 22016, 4096, 256), ("gu7b_m2048", 22016, 4096, 2048),
    ("qkv7b_m4096", 12288, 4096, 4096), ("qkv7b_m8192", 12288, 4096, 8192),
    ("qkv7b_m16384", 12288, 4096, 16384), ("qkv7b_m32768", 12288, 4096, 32768),
    ("o7b_m32768", 4096, 4096, 32768),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=40)
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    ctx = dev.Context(0)
    out_rows = []
    for name, N, K, ntok in SHAPES:
        if args.only and args.only not in name:
            continue
        copies = max(2, int(3 * 126e6 // (N * K * 2)) + 1)
        ws = [dev.pack_weight(ctx, (torch.rand(N, K, device="cuda", dtype=torch.bfloat16) - 0.5) * 0.05)
              for _ in range(copies)]
        x = torch.randn(ntok, K, device="cuda").to(torch.bfloat16)
        out = torch.empty(ntok, N, device="cuda", dtype=torch.bfloat16)
        ptrs = (C.c_void_p * copies)(*[w.data_ptr() for w in ws])
        us = C.c_float(0)
        torch.cuda.synchronize()
        check(lib().be_bench_gemm(ctx.h, ptrs, copies, C.c_void_p(x.data_ptr()),
                                  C.c_void_p(out.data_ptr()), N, K, ntok, args.reps, C.byref(us)),
              ctx.h)
        t = us.value * 1e-6
        byts = 2 * (N * K + ntok * K + ntok * N)
        row = {"shape": name, "N": N, "K": K, "M": ntok, "us": round(us.value, 2),
               "GBps": round(byts / t / 1e9), "TFLOPs": round(2 * N * K * ntok / t / 1e12, 1)}
        out_rows.append(row)
        print(json.dumps(row), flush=True)
        del ws
        torch.cuda.empty_cache()
    ctx.close()


if __name__ == "__main__":
    main()
