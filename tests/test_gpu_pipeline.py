"""Block-placed pipeline over >= 2 GPUs (NCCL P2P hops) vs the one-GPU lockstep run, bit-exact
(scripts/pipeline_check.py --exact). Skipped on boxes with fewer than two GPUs."""
import json
import os
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs two GPUs")
def test_pipeline_two_gpus_bit_exact():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29561",
           os.path.join(ROOT, "scripts", "pipeline_check.py"), "--config", "c2", "--prompt", "64",
           "--ticks", "8", "--exact"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert out.returncode == 0 and lines, out.stderr[-3000:]
    res = json.loads(lines[-1])
    assert res["ok"] and all(p["bit_exact"] for p in res["passes"]), res
