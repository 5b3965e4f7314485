import time, torch, numpy as np, sys
sys.path.insert(0, '.')
from paper_2404_18322_b200.device import Context
from paper_2404_18322_b200.runner import Runner
from paper_2404_18322_b200.workloads import CONFIGS
wl = CONFIGS["c2"](prompt=512, output=128)
ctx = Context(0)
run = Runner(ctx, wl, mode=1, use_graphs=True, plan_ahead=True)
run.run()
for _ in range(4): run.decode_step()
ctx.sync()
d = wl.shape.d_model
hin = torch.empty(run.live, d, dtype=torch.bfloat16).pin_memory()
hout = torch.empty(run.live, d, dtype=torch.bfloat16).pin_memory()
s = torch.cuda.ExternalStream(ctx.stream.value)
def t(fn, n=12):
    ctx.sync(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(n): fn()
    e1.record(s); ctx.sync(); return e0.elapsed_time(e1)/n
print("none", t(lambda: run.decode_step()))
print("none+sync", t(lambda: (run.decode_step(), ctx.sync())))
print("in", t(lambda: run.decode_step(hin, None)))
print("out", t(lambda: run.decode_step(None, hout)))
print("both", t(lambda: run.decode_step(hin, hout)))
scratch = torch.empty(run.live, d, dtype=torch.bfloat16, device="cuda")
def manual_in():
    with torch.cuda.stream(s):
        scratch.copy_(hin, non_blocking=True)
    run.decode_step()
print("manual 512KB h2d + step", t(manual_in))
import os
os.environ["BE_RUNNER_DEBUG"] = "1"
run.decode_step(hin, None)
