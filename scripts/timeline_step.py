"""Kernel timeline of one graph-replayed C2 decode step (be_timeline_*): per kernel its span
(first CTA start -> last CTA end), the PDL wait and the gap to the previous kernel.

  python scripts/timeline_step.py [--config c2] [--out gpurun_out/timeline.json]
"""
import argparse
import json
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2404_18322_b200.device import Context  # noqa: E402
from paper_2404_18322_b200.runner import Runner  # noqa: E402
from paper_2404_18322_b200.workloads import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--prompt", type=int, default=512)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    wl = CONFIGS[a.config](prompt=a.prompt, output=128)
    ctx = Context(0)
    ctx.timeline_enable(8192)
    run = Runner(ctx, wl, mode=1, use_graphs=True)
    run.run()
    for i in range(5):  # plain, capture, replays
        ctx.timeline_begin()
        run.decode_step()
        ctx.sync()
    assert run.step_stats()["graph_replayed"]
    recs = ctx.timeline_read()
    t0 = min(r["start_first"] for r in recs)
    rows, prev_end = [], None
    fam = defaultdict(lambda: {"n": 0, "span_us": 0.0, "gap_us": 0.0, "wait_us": 0.0})
    for r in recs:
        span = (r["end_last"] - r["start_first"]) / 1e3
        wait = (r["go_first"] - r["start_first"]) / 1e3
        gap = (r["start_first"] - prev_end) / 1e3 if prev_end is not None else 0.0
        prev_end = r["end_last"] if prev_end is None else max(prev_end, r["end_last"])
        rows.append({"slot": r["slot"], "cls": r["cls"], "t_us": (r["start_first"] - t0) / 1e3,
                     "span_us": span, "wait_us": wait, "gap_us": gap,
                     "start_spread_us": (r["start_last"] - r["start_first"]) / 1e3})
        f = fam[r["cls"]]
        f["n"] += 1
        f["span_us"] += span
        f["gap_us"] += gap
        f["wait_us"] += wait
    total = (max(r["end_last"] for r in recs) - t0) / 1e3
    summary = {"step_us": total, "kernels": len(recs),
               "families": {k: {kk: (round(vv, 1) if isinstance(vv, float) else vv)
                                for kk, vv in v.items()} for k, v in fam.items()}}
    print(json.dumps(summary, indent=1))
    for r in rows[:60]:
        print(f"{r['slot']:4d} {r['cls']:14s} t={r['t_us']:8.1f} span={r['span_us']:7.1f} "
              f"wait={r['wait_us']:6.1f} gap={r['gap_us']:6.1f} spread={r['start_spread_us']:5.1f}")
    if a.out:
        with open(a.out, "w") as f:
            json.dump({"summary": summary, "rows": rows}, f, indent=1)
    run.close()
    ctx.close()


if __name__ == "__main__":
    main()
