"""Block placement plans (paper_2404_18322_b200/cluster.py) on CPU: where choose_device puts the
private blocks, the legs and runners of a plan, and the hop schedule executed by a world-2/4
gloo group with the same row ranges the NCCL path moves (rows carry their (home, request)
identity; every runner must see exactly its items, and every row must come home)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2404_18322_b200.cluster import (ARENA_DECODE, PHASE_DECODE, PHASE_PREFILL,
                                          block_plan, place_blocks, shared_blocks, stage_plan)
from paper_2404_18322_b200.workloads import CONFIGS


@pytest.mark.parametrize("cfg", ["c2", "c4", "c5"])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_private_blocks_follow_locality(cfg, world):
    wl = CONFIGS[cfg]()
    place = place_blocks(wl, world)
    shared = shared_blocks(wl)
    assert all(place[b] == -1 for b in shared)
    n_t = len(wl.chains)
    for t, ch in enumerate(wl.chains):
        priv = [b for b in ch if b not in shared]
        # a tenant's private blocks stay together (one hop out, one back) ...
        assert len({place[b] for b in priv}) == 1
        # ... and tenants spread over the emptiest GPUs in turn (ties to the lower device)
        assert place[priv[0]] == (t % world if world > 1 else -1)
    used = {place[wl.chains[t][-1]] for t in range(n_t)}
    assert len(used) == min(world, n_t)
    if world == 1:
        assert set(place) == {-1}


def test_c4_world8_layout():
    """configs[3] on 8 GPUs: 8 shared 13B blocks on every GPU, the 4 tenants' private blocks
    (positions 8-9) on GPUs 0-3; every rank's 64 requests hop 48 rows out and back."""
    wl = CONFIGS["c4"]()
    plan = block_plan(wl, 8)
    assert [wl.block_names[b] for b in sorted(shared_blocks(wl))] == [f"b{i}" for i in range(8)]
    assert {(wl.block_names[b], p) for b, p in enumerate(plan.placement) if p >= 0} == {
        (f"t{t}.b{p}", t) for t in range(4) for p in (8, 9)}
    for r in range(8):
        leg1 = plan.runner(r, 1)
        if r < 4:
            assert leg1.wl.n_requests == 8 * 16 and len(leg1.wl.block_names) == 2
        else:
            assert leg1 is None
        sent, recv = plan.hop_bytes_per_step(r, wl.shape.d_model)
        own = 16 if r < 4 else 0  # rows of this rank's own tenant stay
        assert sent == (64 - own) * 5120 * 2 + (7 * 16 if r < 4 else 0) * 5120 * 2
        assert recv == sent


def _plan_invariants(wl, plan):
    n_phase = max(r.slot for r in plan.runners) + 1
    for p in range(n_phase):
        items = [it for r in plan.runners if r.slot == p for it in r.items]
        assert len(items) == len(set(items))
    for spec in plan.runners:
        assert spec.wl.n_requests == len(spec.items)
        for (s, i), t in zip(spec.items, spec.wl.req_tenant):
            assert [spec.wl.block_names[b] for b in spec.wl.chains[t]] == \
                [wl.block_names[b] for b in wl.chains[wl.req_tenant[i]]
                 if plan.placement[b] == plan.placement[wl.chains[wl.req_tenant[i]]
                                                       [_first_of_leg(wl, plan, i, spec.slot)]]][
                    :len(spec.wl.chains[t])]


def _first_of_leg(wl, plan, i, slot):
    ch = wl.chains[wl.req_tenant[i]]
    leg, k = 0, 0
    for j in range(1, len(ch)):
        if plan.placement[ch[j]] != plan.placement[ch[j - 1]]:
            leg += 1
            if leg == slot:
                return j
    return k


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_block_plan_runners_hold_each_leg_once(world):
    wl = CONFIGS["c2"]()
    plan = block_plan(wl, world)
    _plan_invariants(wl, plan)
    homes = [r for r in plan.runners if r.slot == 0]
    assert [r.rank for r in homes] == list(range(world))
    assert all(r.wl.n_requests == wl.n_requests for r in homes)
    if world == 1:
        assert all(not hops for _, _, hops in plan.phases)


def test_stage_plan_keeps_request_order():
    wl = CONFIGS["c2"]()
    plan = stage_plan(wl, [(0, 4), (4, 8)])
    r0, r1 = plan.runner(0, 0), plan.runner(1, 1)
    assert [i for _, i in r0.items] == list(range(wl.n_requests)) == [i for _, i in r1.items]
    assert r0.wl.block_names == [f"b{i}" for i in range(4)]
    assert sorted(r1.wl.block_names) == sorted(
        [f"b{i}" for i in (4, 5)] + [f"t{t}.b{p}" for t in range(4) for p in (6, 7)])


# ------------------------------------------------------------------------ the hops over gloo
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _exec_plan(rank, world, port, cfg, out_q):
    """Executes one decode step of the block plan with identity 'blocks': arenas hold each row's
    (home, request) identity; hops use the plan's row ranges, remote ones as gloo send/recv in
    one batch per phase (the NCCL group of bh_cluster)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        wl = CONFIGS[cfg]()
        plan = block_plan(wl, world)
        arenas = {}
        for spec in plan.runners:
            if spec.rank == rank:
                arenas[spec.slot] = torch.full((spec.wl.n_requests, 2), -1, dtype=torch.int64)
        home = arenas[0]
        for j, i in enumerate(plan.order):
            home[j] = torch.tensor([rank, i])
        seen_ok = True
        for kind, runs, hops in plan.phases:
            if kind != PHASE_DECODE:
                continue
            for (r, slot) in runs:
                if r == rank:  # the runner sees exactly its items
                    spec = plan.runner(r, slot)
                    want = torch.tensor(spec.items, dtype=torch.int64)
                    seen_ok &= bool(torch.equal(arenas[slot], want))
            ops, copies = [], []
            for h in hops:
                sr, ss, dr, ds, arena, _, s0, d0, n = h
                assert arena == ARENA_DECODE
                if sr == rank and dr == rank:
                    copies.append((ss, ds, s0, d0, n))
                elif sr == rank:
                    ops.append(dist.P2POp(dist.isend, arenas[ss][s0:s0 + n].contiguous(), dr))
                elif dr == rank:
                    buf = torch.empty(n, 2, dtype=torch.int64)
                    ops.append(dist.P2POp(dist.irecv, buf, sr))
                    copies.append((None, ds, buf, d0, n))
            if ops:
                for w in dist.batch_isend_irecv(ops):
                    w.wait()
            for ss, ds, s0, d0, n in copies:
                src = s0 if ss is None else arenas[ss][s0:s0 + n].clone()
                arenas[ds][d0:d0 + n] = src
        back = all(home[j].tolist() == [rank, i] for j, i in enumerate(plan.order))
        out_q.put((rank, seen_ok, back))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg,world", [("c2", 2), ("c4", 4), ("c5", 2)])
def test_block_plan_hops_over_gloo(cfg, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exec_plan, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r for r, _, _ in res) == list(range(world))
    assert all(ok and back for _, ok, back in res), res


def test_prefill_phases_move_prompt_rows():
    wl = CONFIGS["c2"](prompt=32, output=4)
    plan = block_plan(wl, 2)
    pre = [hops for k, _, hops in plan.phases if k == PHASE_PREFILL]
    # phase 0: prompt rows (32 per request) to the private leg; phase 1: first tokens home
    assert all(h[4] == 1 and h[8] % 32 == 0 for h in pre[0] if h[0] != h[2] or h[1] != h[3])
    assert all(h[4] == ARENA_DECODE for h in pre[1])
    rows = sum(h[8] for h in pre[0]) // 32
    assert rows == 2 * wl.n_requests  # every request of both ranks reaches its private leg


def test_shared_blocks_replicated_by_the_reference_scale_out():
    """place_blocks replicates the shared blocks through bh_policy_scale_decisions (the
    reference's Scheduler::scale_decisions): one instance per shared block on rank 0 holding
    every rank's decode queue is hot; each round adds replicas on the most-free devices until
    every rank holds one (weak scaling: each replica then serves one rank's rows)."""
    from paper_2404_18322_b200.cluster import place_blocks, shared_blocks
    from paper_2404_18322_b200.workloads import CONFIGS
    wl = CONFIGS["c2"](prompt=64, output=8)
    shared = shared_blocks(wl)
    for world in (2, 4, 8):
        trace = []
        place = place_blocks(wl, world, trace=trace)
        assert all(place[b] == -1 for b in shared)
        assert len(trace) == len(shared) * (world - 1)
        for b in shared:
            devs = sorted(d for _, inst, d in trace if inst.endswith("." + wl.block_names[b]))
            assert devs == list(range(1, world))
