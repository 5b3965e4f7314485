"""Host time of one lockstep decode step call (planning + staging + graph launch), measured on
calls that do not block on the device (the first calls after a sync), for a config.
  python scripts/host_step_time.py [--config c2]"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_18322_b200.device import Context  # noqa: E402
from paper_2404_18322_b200.runner import Runner  # noqa: E402
from paper_2404_18322_b200.workloads import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
a = ap.parse_args()
wl = CONFIGS[a.config](prompt=64, output=40)
ctx = Context(0)
for plan_ahead in (False, True):
    run = Runner(ctx, wl, mode=1, use_graphs=True, plan_ahead=plan_ahead)
    run.run()
    for _ in range(3):
        run.decode_step()
    ctx.sync()
    samples = []
    for _ in range(5):
        ctx.sync()
        t = time.perf_counter()
        run.decode_step()
        samples.append((time.perf_counter() - t) * 1e3)
    ctx.sync()
    print(f"{a.config} plan_ahead={plan_ahead}: host ms per decode_step call (device idle at "
          f"entry): {[round(x, 3) for x in samples]}")
    run.close()
ctx.close()
