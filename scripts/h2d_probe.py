import torch
x = torch.empty(64*4096, dtype=torch.bfloat16).pin_memory()
y = torch.empty(64*4096, dtype=torch.bfloat16, device="cuda")
for n in [1, 8, 64]:
    ts=[]
    for _ in range(20):
        e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(n):
            y[i*(64*4096//n):(i+1)*(64*4096//n)].copy_(x[i*(64*4096//n):(i+1)*(64*4096//n)], non_blocking=True)
        e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    ts.sort(); print("h2d 512KB in", n, "copies: %.1f us" % (1e3*ts[len(ts)//2]))
    ts=[]
    for _ in range(20):
        e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
        e0.record(); x.copy_(y, non_blocking=True); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    ts.sort(); print("d2h 512KB: %.1f us" % (1e3*ts[len(ts)//2]))
