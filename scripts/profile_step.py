"""One C2 decode step for profilers: prefill, warm-up steps (graphs captured), an event-timed
step (bench.profile_step: per-launch classes, algorithmic bytes), then `--steps` plain decode
steps inside an NVTX range "step" for `ncu --nvtx --nvtx-include step/`.

  python scripts/profile_step.py --out gpurun_out/step_prof.json
  ncu --nvtx --nvtx-include step/ --metrics gpu__time_duration.sum,dram__bytes_read.sum,\
dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/step_launches.csv \
python scripts/profile_step.py --steps 1
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2404_18322_b200.device import Context  # noqa: E402
from paper_2404_18322_b200.runner import Runner  # noqa: E402
from paper_2404_18322_b200.workloads import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--prompt", type=int, default=512)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    wl = CONFIGS[a.config](prompt=a.prompt, output=128)
    ctx = Context(0)
    stream = torch.cuda.ExternalStream(ctx.stream.value)
    run = Runner(ctx, wl, mode=1, use_graphs=True)
    run.run()
    for _ in range(a.warmup):
        run.decode_step()
    ctx.sync()
    peaks, kind = bench.load_peaks()
    prof = bench.profile_step(ctx, run, wl, stream, peaks, kind)
    torch.cuda.nvtx.range_push("step")
    for _ in range(a.steps):
        run.decode_step()
    ctx.sync()
    torch.cuda.nvtx.range_pop()
    if a.out:
        with open(a.out, "w") as f:
            json.dump(prof, f, indent=1)
    print(json.dumps(prof["roofline"]))
    run.close()
    ctx.close()


if __name__ == "__main__":
    main()
