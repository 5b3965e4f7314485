"""The block-placed cluster over NCCL (one process per GPU, torchrun) vs the same plan executed
in one process on one GPU with device-copy hops: every decode step's home rows must be
bit-identical on every rank (the transport must not change a bit), and the NCCL byte counters
must equal the plan's hop bytes.

  torchrun --nproc-per-node N scripts/cluster_check.py [--config c2n|c2|c4] [--steps 4]

Prints one JSON line on rank 0: {"ok": bool, "world": N, "steps": [...], ...}.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def narrow_c2(output):
    from paper_2404_18322_b200 import device as dev
    from paper_2404_18322_b200.workloads import shared_prefix_zoo
    shape = dev.BlockShape(n_layers=1, d_model=512, n_heads=4, d_ff=1536, max_pos=128)
    return shared_prefix_zoo("c2-narrow", shape, 4, 2, 4, 4, 40, output)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2n")
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--migrate", action="store_true",
                    help="after half the steps move tenant 0's private blocks to the next rank "
                         "(Cluster.migrate: KV pages over NCCL) and keep decoding")
    args = ap.parse_args()
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2404_18322_b200 import device as dev
    from paper_2404_18322_b200.cluster import Cluster, Comm, block_plan
    from paper_2404_18322_b200.pipeline import _DevRows
    from paper_2404_18322_b200.workloads import CONFIGS

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    wl = narrow_c2(args.steps + 2) if args.config == "c2n" else \
        CONFIGS[args.config](prompt=64, output=args.steps + 2)
    mig_at = args.steps // 2 if args.migrate else -1
    idx = sorted(range(wl.n_requests), key=lambda i: (wl.req_tenant[i], i))
    wl = dataclasses.replace(wl, req_tenant=[wl.req_tenant[i] for i in idx])
    n, d = wl.n_requests, wl.shape.d_model
    plan = block_plan(wl, world)
    moved = list(plan.placement)
    for b, name in enumerate(wl.block_names):
        if name.startswith("t0.") and moved[b] >= 0:
            moved[b] = (moved[b] + 1) % world

    def rows(run):
        t = torch.as_tensor(_DevRows(run.arena_ptr, n, d), device="cuda").view(torch.bfloat16)
        return t.clone()

    # --- over NCCL, one rank per process
    ctx = dev.Context(local)
    uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
    if rank == 0:
        uid.copy_(torch.frombuffer(bytearray(Comm.unique_id()), dtype=torch.uint8))
    dist.broadcast(uid, 0)
    comm = Comm(ctx, world, rank, bytes(uid.cpu().numpy().tobytes()))
    cl = Cluster({rank: ctx}, plan, comm)
    cl.prefill()
    got = [rows(cl.home(rank))]
    mig = None
    for k in range(args.steps):
        if k == mig_at:
            mig = cl.migrate(moved)
        cl.decode_step()
        ctx.sync()
        got.append(rows(cl.home(rank)))
    st = cl.stats()
    sent, recv = plan.hop_bytes_per_step(rank, d)
    counters_ok = args.migrate or (st["sent_bytes"] >= args.steps * sent and
                                   st["recv_bytes"] >= args.steps * recv)
    cl.close()
    comm.close()
    # every rank's rows, gathered on rank 0
    allg = [[torch.empty_like(g) for _ in range(world)] for g in got]
    for k, g in enumerate(got):
        dist.all_gather(allg[k], g)
    ok_counters = torch.tensor([1 if counters_ok else 0], device="cuda")
    dist.all_reduce(ok_counters, op=dist.ReduceOp.MIN)
    res = None
    if rank == 0:
        # --- the same plan in this process: every rank a context on GPU 0, device-copy hops
        ctxs = {r: dev.Context(local) for r in range(world)}
        lb = Cluster(ctxs, plan)
        lb.prefill()
        ref = [[rows(lb.home(r)) for r in range(world)]]
        for k in range(args.steps):
            if k == mig_at:
                lb.migrate(moved)
            lb.decode_step()
            for c in ctxs.values():
                c.sync()
            ref.append([rows(lb.home(r)) for r in range(world)])
        lb.close()
        for c in ctxs.values():
            c.close()
        steps = []
        for k in range(args.steps + 1):
            same = all(torch.equal(allg[k][r], ref[k][r]) for r in range(world))
            steps.append({"step": k, "bit_exact": bool(same)})
        res = {"ok": all(s["bit_exact"] for s in steps) and bool(ok_counters.item()),
               "world": world, "config": wl.name, "placement": plan.note,
               "hop_bytes_per_step_rank0": plan.hop_bytes_per_step(0, d),
               "nccl_counters_ok": bool(ok_counters.item()), "steps": steps,
               "migration_rank0": mig}
        print(json.dumps(res), flush=True)
    ctx.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
