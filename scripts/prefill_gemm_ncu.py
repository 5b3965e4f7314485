import sys, os, torch
sys.path.insert(0, '.')
from paper_2404_18322_b200 import device as dev
ctx = dev.Context(0)
for (N, K, M) in [(12288, 4096, 16384), (22016, 4096, 8192)]:
    w = (torch.randn(N, K) * 0.05).to(torch.bfloat16).cuda()
    x = torch.randn(M, K).to(torch.bfloat16).cuda()
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    wp = dev.pack_weight(ctx, w)
    for _ in range(2):
        dev.gemm_bf16(ctx, wp, x, out, 0, packed=True)
    ctx.sync()
print("ok")
