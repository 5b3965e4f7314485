import time, torch, numpy as np, sys
sys.path.insert(0, '.')
from paper_2404_18322_b200.device import Context
from paper_2404_18322_b200.runner import Runner
from paper_2404_18322_b200.workloads import CONFIGS
wl = CONFIGS["c2"](prompt=512, output=128)
ctx = Context(0)
run = Runner(ctx, wl, mode=1, use_graphs=True)
run.run()
for _ in range(4): run.decode_step()
ctx.sync()
d = wl.shape.d_model
hin = torch.empty(run.live, d, dtype=torch.bfloat16).pin_memory()
hout = torch.empty(run.live, d, dtype=torch.bfloat16).pin_memory()
# host time of a decode_step call that only launches (GPU busy with previous steps)
ts = []
for _ in range(10):
    t0 = time.perf_counter(); run.decode_step(); ts.append(time.perf_counter() - t0)
ctx.sync()
print("launch-only decode_step host ms: med %.3f max %.3f" % (1e3*np.median(ts), 1e3*max(ts)))
ts = []
for _ in range(10):
    t0 = time.perf_counter(); run.decode_step(hin, hout); ts.append(time.perf_counter() - t0)
print("decode_step with host in/out ms: med %.3f" % (1e3*np.median(ts)))
ctx.sync()
# pure GPU time of a step
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
s = torch.cuda.ExternalStream(ctx.stream.value)
e0.record(s)
for _ in range(10): run.decode_step()
e1.record(s); ctx.sync()
print("device ms/step: %.3f" % (e0.elapsed_time(e1)/10))
t0 = time.perf_counter()
for _ in range(10):
    hin.copy_(hout)
print("hin.copy_ ms: %.3f" % ((time.perf_counter()-t0)*100))
