#!/usr/bin/env python3
"""Phase timeline of one GEMM launch (BE_GEMM_TRACE=1 prints globaltimer stamps per phase)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2404_18322_b200 import device as dev  # noqa: E402

ctx = dev.Context(0)
shapes = [(4096, 4096, 64), (4096, 4096, 16), (12288, 4096, 64), (22016, 4096, 64), (4096, 11008, 64)]
if os.environ.get("BE_TRACE_SHAPES"):  # e.g. "12288x4096x256,22016x4096x256"
    shapes = [tuple(int(v) for v in sh.split("x")) for sh in os.environ["BE_TRACE_SHAPES"].split(",")]
for N, K, M in shapes:
    w = dev.pack_weight(ctx, (torch.rand(N, K, device="cuda", dtype=torch.bfloat16) - 0.5) * 0.05)
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    os.environ.pop("BE_GEMM_TRACE", None)
    for _ in range(3):
        dev.gemm_bf16(ctx, w, x, out, packed=True)
    ctx.sync()
    junk = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    junk.fill_(1)
    torch.cuda.synchronize()
    os.environ["BE_GEMM_TRACE"] = "1"
    dev.gemm_bf16(ctx, w, x, out, packed=True)
    ctx.sync()
    os.environ.pop("BE_GEMM_TRACE", None)
    del junk
