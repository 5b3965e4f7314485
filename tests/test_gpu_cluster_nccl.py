"""The block-placed cluster over NCCL on >= 2 GPUs (scripts/cluster_check.py): home rows of every
rank bit-identical to the same plan run in one process with device-copy hops, and the NCCL byte
counters equal to the plan's hops. Skipped on boxes with fewer than two GPUs."""
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
def test_cluster_nccl_two_gpus_bit_exact_vs_loopback():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29563",
           os.path.join(ROOT, "scripts", "cluster_check.py"), "--config", "c2n", "--steps", "4"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert out.returncode == 0 and lines, out.stderr[-3000:]
    res = json.loads(lines[-1])
    assert res["ok"], res
