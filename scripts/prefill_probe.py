"""Where a config's prefill goes: wall time of Runner.run() (every prompt prefilled, untimed in
bench.py's decode legs), then a second runner with be_prof event timing summed per kernel class.

  python scripts/prefill_probe.py [--config c3 --prompt 2048]
"""
import argparse
import collections
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_18322_b200.device import Context  # noqa: E402
from paper_2404_18322_b200.runner import Runner  # noqa: E402
from paper_2404_18322_b200.workloads import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--prompt", type=int, default=2048)
    ap.add_argument("--output", type=int, default=8)
    a = ap.parse_args()
    wl = CONFIGS[a.config](prompt=a.prompt, output=a.output)
    ctx = Context(0)
    res = {"config": wl.name, "prompt": a.prompt, "requests": wl.n_requests}
    for rep in range(2):
        run = Runner(ctx, wl, mode=1, use_graphs=True)
        ctx.sync()
        t0 = time.time()
        run.run()
        ctx.sync()
        res[f"wall_s_{rep}"] = round(time.time() - t0, 4)
        run.close()
    run = Runner(ctx, wl, mode=1, use_graphs=True)
    ctx.prof_enable(True)
    run.run()
    recs = ctx.prof_read()
    ctx.prof_enable(False)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for r in recs:
        g = agg[r["cls"]]
        g[0] += 1
        g[1] += r["ms"]
        g[2] += r["flops"]
    res["kernels"] = {k: {"launches": v[0], "ms": round(v[1], 2),
                          "tflops": round(v[2] / v[1] / 1e9, 1) if v[1] > 0 else None}
                      for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])}
    res["kernel_ms_total"] = round(sum(v[1] for v in agg.values()), 2)
    run.close()
    ctx.close()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
