"""Multi-GPU block placement: chains placed across GPUs as pipeline stages, activations moving
between consecutive stages by NCCL point-to-point send/recv over NVLink (the inter-block hop of
Simulation::deliver / LinkManager::transfer, proj/core/src/scenario.cpp:282-308,
cluster.cpp:170-192; hop payload 2*d bytes per token, costmodel.cpp:129-131).

Placement (placement_stages): contiguous chain-position ranges per GPU, cut to minimise the
most loaded stage (weights + KV bytes streamed per decode step) - consecutive blocks of a chain
stay together, so a decode token crosses one GPU boundary per stage (under NVSwitch,
locality = fewest hops). N micro-batches are in flight: at tick t, stage s runs micro-batch
(t - s) mod N through its blocks, then in one grouped NCCL call sends the rows on and receives
the next micro-batch's rows (the grouped send+recv cannot deadlock around the ring). The last
stage feeds the first (greedy next-token input).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .workloads import Workload


def position_costs(wl: Workload, ctx_tokens: int) -> list[float]:
    """Bytes streamed per decode step at each chain position (all tenants' blocks there)."""
    s = wl.shape
    npos = max(len(c) for c in wl.chains)
    w_bytes = s.param_bytes
    kv_row = ctx_tokens * s.kv_bytes_per_token  # K+V read per request per block
    rows = wl.rows_at_block()
    cost = [0.0] * npos
    for p in range(npos):
        blocks = {c[p] for c in wl.chains if p < len(c)}
        for b in blocks:
            cost[p] += w_bytes + rows[b] * kv_row
    return cost


def placement_stages(costs: list[float], n: int) -> list[tuple[int, int]]:
    """Contiguous partition of positions into n stages minimising the max stage cost (DP)."""
    P = len(costs)
    n = min(n, P)
    pre = [0.0]
    for c in costs:
        pre.append(pre[-1] + c)
    INF = float("inf")
    best = [[INF] * (P + 1) for _ in range(n + 1)]
    cut = [[0] * (P + 1) for _ in range(n + 1)]
    best[0][0] = 0.0
    for k in range(1, n + 1):
        for j in range(k, P + 1):
            for i in range(k - 1, j):
                v = max(best[k - 1][i], pre[j] - pre[i])
                if v < best[k][j]:
                    best[k][j], cut[k][j] = v, i
    ranges, j = [], P
    for k in range(n, 0, -1):
        i = cut[k][j]
        ranges.append((i, j))
        j = i
    return ranges[::-1]


def stage_memory(wl: Workload, rng: tuple[int, int], n_micro: int) -> float:
    """HBM bytes a stage holds: its blocks' weights plus full-length KV of n_micro request mixes."""
    s = wl.shape
    a, b = rng
    blocks = {blk for ch in wl.chains for blk in ch[a:b]}
    kv = 0.0
    for t, n_out, n_in in zip(wl.req_tenant, wl.req_output, wl.req_prompt):
        nb = len(set(wl.chains[t][a:b]))
        kv += nb * (n_in + n_out) * s.kv_bytes_per_token
    return len(blocks) * s.param_bytes + n_micro * kv


def choose_layout(wl: Workload, world: int, hbm_bytes: float = 0.85 * 180e9) -> dict:
    """Block placement over `world` GPUs: pipeline depth P (chain positions cut into P stages,
    NCCL hops between them) times R = world / P replica groups, each group serving its own
    request mixes. Among depths whose stages fit in HBM, pick the highest modelled throughput
    R / max_stage_cost (every GPU streams its stage's weights + KV once per token step); with
    180 GB per GPU a 7B/13B zoo fits whole, so replication (P = 1, no hop) wins unless memory
    forces a cut - the same trade the reference's placement makes between replicas and spread."""
    npos = max(len(c) for c in wl.chains)
    costs = position_costs(wl, wl.req_prompt[0] + wl.req_output[0] // 2)
    best = None
    for P in range(1, min(world, npos) + 1):
        if world % P:
            continue
        st = placement_stages(costs, P)
        mem = max(stage_memory(wl, r, P) for r in st)
        if mem > hbm_bytes:
            continue
        score = (world // P) / max(sum(costs[a:b]) for a, b in st)
        if best is None or score > best["score"] * (1 + 1e-9):
            best = {"depth": P, "replicas": world // P, "stages": st, "score": score,
                    "stage_mem": mem}
    if best is None:
        raise ValueError(f"{wl.name}: no placement fits {world} GPUs")
    return best


def _profile_classes(path: str | None):
    import json
    import os
    if path is None:
        path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                            "profiles", "b200_profiles.json")
    if not os.path.exists(path):
        return {}
    return json.load(open(path))["classes"]


def routing_policy(wl: Workload, n_devices: int, profiles: str | None = None,
                   hbm_bytes: int = 180 * 10**9, instances: bool = True,
                   speculation: bool = False, spec_fraction: float = 0.10,
                   scale_queue_us: int = 0):
    """A bh_policy (include/blockpolicy.h) describing replica placement of `wl`: every block on
    each of n_devices GPUs of one NVLink server, priced by the measured B200 cost profiles
    (profiles/b200_profiles.json, scripts/make_profiles.py; §8(f) rank 2). Classes the profile
    file lacks are priced by streamed bytes at the measured copy peak."""
    from .policy import Policy
    s = wl.shape
    d = s.d_model
    prof = _profile_classes(profiles)
    pol = Policy(adaptive=False, speculation=speculation, spec_fraction=spec_fraction,
                 scale_queue_us=scale_queue_us)
    att_bytes, ffn_bytes = 2 * 4 * d * d, 2 * 3 * d * s.d_ff
    for kind, wbytes, kv in (("attention", att_bytes, 4 * d), ("ffn", ffn_bytes, 0)):
        key = f"{kind}:{d}"
        if key in prof:
            c = prof[key]
            grids = [{"xs": c[p]["batch"], "ys": c[p]["tokens"], "v": c[p]["us"]}
                     for p in ("prefill", "decode")]
            kv = c.get("kv_bytes_per_token", kv)
        else:  # bytes model: weights once + K/V of batch x tokens, at 6.37 TB/s
            xs, ys = [1, 8, 64], [1, 256, 4096]
            us = [[(wbytes + b * t * kv) / 6.37e12 * 1e6 for t in ys] for b in xs]
            grids = [{"xs": xs, "ys": ys, "v": us}] * 2
        pol.add_cost_class(key, grids[0], grids[1], kv)
    pol.set_device_class("b200", 1.0)
    for bi, name in enumerate(wl.block_names):
        comps = []
        for ci, k in enumerate(wl.block_comps[bi] if wl.block_comps else s.comps):
            cid = f"{name}.c{ci}"
            pol.add_component(cid, "attention" if k == "a" else "ffn", d, ci // 2,
                              [(cid + ".w", att_bytes if k == "a" else ffn_bytes)])
            comps.append(cid)
        pol.add_block(name, comps, d)
    for t, ch in enumerate(wl.chains):
        pol.add_chain(f"tenant{t}", [wl.block_names[b] for b in ch])
    pol.add_server(0, 900e9)  # NVLink 5 per direction
    for dev in range(n_devices):
        pol.add_device(dev, 0, "b200", hbm_bytes, 7.7e12, 55e9)
    if not instances:  # the caller places the blocks (cluster.place_blocks)
        return pol
    seq = 0
    for dev in range(n_devices):
        for name in wl.block_names:
            seq += 1
            pol.put_instance(f"r{dev}.{name}", name, dev, ready=True, created_seq=seq)
        pol.set_ledger(dev, s.param_bytes * len(wl.block_names))
    return pol


def route_requests(wl: Workload, n_devices: int, copies: int = 1,
                   profiles: str | None = None) -> list[int]:
    """Routes `copies` x the workload's requests (request i of copy c is global request
    i * copies + c) over n_devices replicas with the reference's binding rule
    (bh_policy_choose_binding = Scheduler::choose_binding, scheduler.cpp:80-160): each prefill
    binds to the lowest (queue + compute + transfer + load) estimate, ties to the lower device;
    the chosen instance's queue grows by the step's standalone cost (InstancePool::enqueue,
    agent.cpp:132-137). Decode steps then stick to the device holding the request's KV, so the
    prefill choice is the request's replica. Returns the device per global request."""
    pol = routing_policy(wl, n_devices, profiles)
    queued = {}
    out = []
    for i in range(wl.n_requests):
        blk = wl.block_names[wl.chains[wl.req_tenant[i]][0]]
        for c in range(copies):
            ch = pol.choose_binding(i * copies + c, blk, False, wl.req_prompt[i],
                                    wl.req_prompt[i], -1, 0)
            if ch is None:
                raise ValueError(f"no feasible replica for block {blk}")
            iid = ch["instance"]
            queued[iid] = queued.get(iid, 0.0) + ch["est"][1]
            pol.put_instance(iid, blk, ch["device"], ready=True,
                             created_seq=1 + ch["device"] * len(wl.block_names)
                             + wl.block_names.index(blk),
                             queue_len=1, queued_cost_us=queued[iid],
                             queued_cost_hwm=queued[iid])
            out.append(ch["device"])
    return out


def stage_workload(wl: Workload, rng: tuple[int, int], n_micro: int) -> Workload:
    """The blocks of chain positions [a, b) and n_micro copies of the request mix."""
    a, b = rng
    names, comps, remap, chains = [], [], {}, []
    for ch in wl.chains:
        sub = []
        for blk in ch[a:b]:
            if blk not in remap:
                remap[blk] = len(names)
                names.append(wl.block_names[blk])
                if wl.block_comps:
                    comps.append(wl.block_comps[blk])
            sub.append(remap[blk])
        chains.append(sub)
    n = wl.n_requests
    return Workload(f"{wl.name}@{a}-{b}", wl.shape, names, chains,
                    wl.req_tenant * n_micro, wl.req_prompt * n_micro, wl.req_output * n_micro,
                    wl.max_batch_tokens, wl.seed, dict(wl.notes, stage=(a, b)),
                    comps or None)


class _DevRows:
    """__cuda_array_interface__ over raw bf16 rows (int16 typestr: the interface has no bf16; the
    tensor is viewed back as bfloat16 for NCCL)."""

    def __init__(self, ptr: int, rows: int, cols: int):
        self.__cuda_array_interface__ = {"shape": (rows, cols), "typestr": "<i2",
                                         "data": (ptr, False), "version": 3, "strides": None}


@dataclass
class TickStats:
    computed: int = 0   # micro-batch steps this rank ran
    finished: int = 0   # tokens completed by this rank as the last stage


class PipelineStage:
    """One rank of the block-placed pipeline (torch.distributed with the NCCL backend)."""

    def __init__(self, ctx, wl: Workload, world: int, rank: int, n_micro: int | None = None,
                 ctx_for_cost: int | None = None, base_rank: int = 0):
        """`world` = pipeline depth, `rank` = stage index; the group occupies global ranks
        base_rank .. base_rank + world - 1 (replica groups side by side)."""
        import torch
        import torch.distributed as dist
        from .runner import Runner
        self.torch, self.dist = torch, dist
        self.world, self.rank, self.base = world, rank, base_rank
        self.n_micro = n_micro or world
        costs = position_costs(wl, ctx_for_cost or (wl.req_prompt[0] + wl.req_output[0] // 2))
        self.stages = placement_stages(costs, world)
        self.stage_costs = [sum(costs[a:b]) for a, b in self.stages]
        self.wl = stage_workload(wl, self.stages[rank], self.n_micro)
        self.per_mb = wl.n_requests
        self.ctx = ctx
        self.run = Runner(ctx, self.wl, mode=1, use_graphs=True)
        self.stream = torch.cuda.ExternalStream(ctx.stream.value)
        d = wl.shape.d_model
        self.d = d
        dptr = self.run.arena_ptr
        self.arena = torch.as_tensor(_DevRows(dptr, self.wl.n_requests, d),
                                     device="cuda").view(torch.bfloat16)
        pptr, prow = self.run.prefill_arena()
        self.parena = torch.as_tensor(_DevRows(pptr, prow, d), device="cuda").view(torch.bfloat16)
        self.stats = TickStats()

    # ------------------------------------------------------------------ prefill
    def prefill(self):
        """Stage by stage: receive the prompts' hidden states, prefill, pass them on; the last
        stage returns the first-token rows to stage 0."""
        dist, torch = self.dist, self.torch
        r, W = self.rank, self.world

        def p2p(op, t, peer):
            for w in dist.batch_isend_irecv([dist.P2POp(op, t, self.base + peer)]):
                w.wait()

        with torch.cuda.stream(self.stream):
            if W > 1 and r > 0:
                p2p(dist.irecv, self.parena, r - 1)
            self.run.run()
            if W > 1 and r < W - 1:
                p2p(dist.isend, self.parena, r + 1)
            if W > 1 and r == W - 1:
                p2p(dist.isend, self.arena, 0)
            if W > 1 and r == 0:
                p2p(dist.irecv, self.arena, W - 1)
        self.ctx.sync()
        torch.cuda.synchronize()

    # ------------------------------------------------------------------ decode ticks
    def mb_rows(self, m: int):
        return self.arena[m * self.per_mb:(m + 1) * self.per_mb]

    def tick(self, t: int, total_ticks: int) -> None:
        with self.torch.cuda.stream(self.stream):
            run_tick(self.dist, t, total_ticks, self.rank, self.world, self.n_micro,
                     self._compute, self.mb_rows, self.base)

    def set_host_io(self, on: bool) -> None:
        """End-to-end leg: stage 0 uploads each micro-batch's input rows from pinned host memory
        and the last stage reads its output rows back (synchronously) every tick."""
        self.host_in = self.host_out = None
        if not on:
            return
        d = self.wl.shape.d_model
        t = self.torch
        if self.rank == 0:
            self.host_in = t.zeros(self.per_mb, d, dtype=t.bfloat16).pin_memory()
        if self.rank == self.world - 1:
            self.host_out = t.empty(self.per_mb, d, dtype=t.bfloat16).pin_memory()

    def _compute(self, m: int) -> None:
        reqs = np.arange(m * self.per_mb, (m + 1) * self.per_mb, dtype=np.int32)
        self.run.decode_group(m, reqs, getattr(self, "host_in", None),
                              getattr(self, "host_out", None))
        self.stats.computed += 1
        if self.rank == self.world - 1:
            self.stats.finished += self.per_mb

    def close(self):
        self.run.close()


def tick_plan(t: int, total_ticks: int, r: int, W: int, N: int):
    """(compute, send, recv) micro-batch indices (or None) of stage r at tick t.

    Stage r first computes at tick r (micro-batch 0), so at tick t it runs micro-batch
    (t - r) mod N; its output goes to stage r+1 (the last stage wraps to stage 0: the next token's
    input), and it receives the micro-batch it runs at tick t+1. Stage 0 owns every micro-batch's
    first input (from prefill), so it only receives once the last stage has produced something.
    """
    comp = (t - r) % N if t >= r else None
    if W == 1:
        return comp, None, None
    send = comp if comp is not None and t + 1 < total_ticks else None
    recv = None
    if t + 1 >= r and t + 1 < total_ticks and (r > 0 or t >= W - 1):
        recv = (t + 1 - r) % N
    return comp, send, recv


def run_tick(dist, t, total_ticks, r, W, N, compute, rows, base=0) -> None:
    """One tick: compute, then one grouped send-on / receive-next (cannot deadlock the ring).
    Stage s of the group is global rank base + s."""
    comp, send, recv = tick_plan(t, total_ticks, r, W, N)
    if comp is not None:
        compute(comp)
    ops = []
    if send is not None:
        ops.append(dist.P2POp(dist.isend, rows(send), base + (r + 1) % W))
    if recv is not None:
        ops.append(dist.P2POp(dist.irecv, rows(recv), base + (r - 1) % W))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()


def ticks_needed(world: int, steps: int, warmup: int) -> int:
    return warmup + steps + world


def tokens_per_request_needed(world: int, total_ticks: int, n_micro: int) -> int:
    return math.ceil(total_ticks / n_micro) + 2


def speculation_blocks(wl: Workload, spec_fraction: float = 0.10, us_per_row: float = 1.0):
    """Blocks a lockstep decode step runs speculatively: the reference's marking rule
    (bh_policy_speculation_marks = Scheduler::speculation_marks, scheduler.cpp:180-215: the top
    ceil(fraction x instances) instances by queued cost, skipping blocks without a surrogate,
    chain-final blocks and chain neighbours of marked ones) over the instances of one GPU, each
    queue holding its per-block decode batch (queued cost = rows x us_per_row). Returns
    (marked block indices the executor can speculate - every member continues to one block -,
    all marked block names)."""
    pol = routing_policy(wl, 1, instances=False, speculation=True, spec_fraction=spec_fraction)
    rows = wl.rows_at_block()
    for b, name in enumerate(wl.block_names):
        pol.put_instance(f"r0.{name}", name, 0, ready=True, created_seq=b + 1,
                         queue_len=rows[b], queued_cost_us=rows[b] * us_per_row,
                         queued_cost_hwm=rows[b] * us_per_row)
    marked = [iid.split(".", 1)[1] for iid in pol.speculation_marks()]
    pol.close()
    ok = []
    for name in marked:
        b = wl.block_names.index(name)
        succ = {ch[ch.index(b) + 1] for ch in wl.chains if b in ch and ch.index(b) + 1 < len(ch)}
        if len(succ) == 1:
            ok.append(b)
    return ok, marked
