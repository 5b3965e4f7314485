#!/usr/bin/env python3
"""Per-launch time of the decode GEMM shapes (64 rows) from one CUDA-graph replay of `reps`
PDL-chained launches cycling over weight copies > L2 (be_bench_gemm), for the library in
BE_LIB_PATH - e.g. the experiment builds without epilogue (-DBE_EXP_NO_EPI) or without MMAs
(-DBE_EXP_NO_MMA), to split a launch into streaming, MMA and epilogue / fixup time.

  BE_LIB_PATH=scripts/variants/libblockexec_noepi.so python scripts/gemm_floor.py
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2404_18322_b200 import device as dev  # noqa: E402
from paper_2404_18322_b200._lib import check, lib  # noqa: E402

ctx = dev.Context(0)
out = {"lib": os.environ.get("BE_LIB_PATH", "default")}
for name, N, K in [("o", 4096, 4096), ("qkv", 12288, 4096), ("gate_up", 22016, 4096),
                   ("down", 4096, 11008)]:
    for M in [int(m) for m in os.environ.get("BE_FLOOR_M", "64,16").split(",")]:
        # BE_FLOOR_L2=1: one weight copy, re-read every launch (L2-resident when it fits)
        copies = 1 if os.environ.get("BE_FLOOR_L2") else max(2, int(3 * 126e6 / (N * K * 2)) + 1)
        ws = [dev.pack_weight(ctx, (torch.rand(N, K, device="cuda", dtype=torch.bfloat16) - 0.5)
                              * 0.05) for _ in range(copies)]
        x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        ptrs = (C.c_void_p * copies)(*[w.data_ptr() for w in ws])
        us = C.c_float(0)
        check(lib().be_bench_gemm(ctx.h, ptrs, copies, C.c_void_p(x.data_ptr()),
                                  C.c_void_p(y.data_ptr()), N, K, M, 4 * copies, C.byref(us)),
              ctx.h)
        mb = 2 * (N * K + M * K + M * N) / 1e6
        out[f"{name}_m{M}"] = {"us": round(us.value, 2), "MB": round(mb, 1),
                               "GBps": round(mb * 1e3 / us.value, 0),
                               "TFLOPs": round(2 * M * N * K / us.value / 1e6, 1)}
        del ws
        torch.cuda.empty_cache()
print(json.dumps(out))
