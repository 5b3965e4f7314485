"""Block placement across GPUs (paper_2404_18322_b200/pipeline.py) on CPU: the stage cut, the
per-stage workloads and the tick schedule, the last over a real world-size 2/3 gloo group with the
same grouped send/recv calls the NCCL path makes."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2404_18322_b200.pipeline import (choose_layout, placement_stages, position_costs,
                                           run_tick, stage_memory, stage_workload, tick_plan,
                                           ticks_needed, tokens_per_request_needed)
from paper_2404_18322_b200.workloads import CONFIGS


def brute_minmax(costs, n):
    import itertools
    P = len(costs)
    n = min(n, P)
    best = None
    for cuts in itertools.combinations(range(1, P), n - 1):
        b = [0, *cuts, P]
        v = max(sum(costs[b[i]:b[i + 1]]) for i in range(n))
        best = v if best is None else min(best, v)
    return best


@pytest.mark.parametrize("n", [1, 2, 3, 4, 8])
def test_placement_is_minmax_contiguous(n):
    rng = np.random.default_rng(n)
    for _ in range(20):
        costs = list(rng.uniform(1, 10, size=int(rng.integers(1, 10))))
        st = placement_stages(costs, n)
        assert st[0][0] == 0 and st[-1][1] == len(costs)
        assert all(a < b for a, b in st)
        assert all(st[i][1] == st[i + 1][0] for i in range(len(st) - 1))
        got = max(sum(costs[a:b]) for a, b in st)
        assert got == pytest.approx(brute_minmax(costs, n))


def test_c2_stage_workloads_cover_the_chains():
    wl = CONFIGS["c2"]()
    costs = position_costs(wl, 576)
    assert len(costs) == 8
    # private positions serve 4 blocks (one per tenant), shared ones a single block
    assert costs[7] > 2 * costs[0]
    for n in (2, 4, 8):
        stages = placement_stages(costs, n)
        assert len(stages) == n
        blocks_seen = []
        for a, b in stages:
            sw = stage_workload(wl, (a, b), n)
            assert sw.n_requests == n * wl.n_requests
            assert sw.req_tenant[:wl.n_requests] == wl.req_tenant
            for t, ch in enumerate(sw.chains):
                assert [sw.block_names[i] for i in ch] == \
                    [wl.block_names[i] for i in wl.chains[t][a:b]]
            blocks_seen += sw.block_names
        # every block is placed on exactly one GPU
        assert sorted(blocks_seen) == sorted(wl.block_names)


def test_layout_replicates_when_the_zoo_fits():
    # 180 GB per GPU holds a whole 7B/13B zoo: replicas (no hop) beat any cut under weak scaling
    for c in ("c2", "c4"):
        wl = CONFIGS[c]()
        for W in (1, 2, 4, 8):
            lay = choose_layout(wl, W)
            assert (lay["depth"], lay["replicas"]) == (1, W)


def test_layout_cuts_the_chain_when_memory_forces_it():
    wl = CONFIGS["c2"]()
    whole = stage_memory(wl, (0, 8), 1)
    lay = choose_layout(wl, 8, hbm_bytes=0.8 * whole)
    assert lay["depth"] > 1 and lay["depth"] * lay["replicas"] == 8
    assert lay["stage_mem"] <= 0.8 * whole
    # every stage of the chosen cut fits, with its micro-batches' KV
    for r in lay["stages"]:
        assert stage_memory(wl, r, lay["depth"]) <= 0.8 * whole
    with pytest.raises(ValueError):
        choose_layout(wl, 8, hbm_bytes=1e9)


@pytest.mark.parametrize("W", [1, 2, 3, 4, 8])
def test_tick_plan_sends_match_receives(W):
    N = W
    total = 3 * W + 5
    for t in range(total):
        plans = [tick_plan(t, total, r, W, N) for r in range(W)]
        for r in range(W):
            _, send, _ = plans[r]
            _, _, recv_next = plans[(r + 1) % W]
            assert send == recv_next, (t, r)
    # each stage computes a micro-batch only after its rows arrived, in pass order
    have = {(0, m): 0 for m in range(N)}  # stage 0 holds every first input from prefill
    passes = {}
    for t in range(total):
        plans = [tick_plan(t, total, r, W, N) for r in range(W)]
        for r, (comp, _, _) in enumerate(plans):
            if comp is not None:
                assert (r, comp) in have, (t, r, comp)
                if W > 1:  # one stage keeps its rows in place
                    del have[(r, comp)]
                passes[(r, comp)] = passes.get((r, comp), 0) + 1
        for r, (_, _, recv) in enumerate(plans):
            if recv is not None:
                have[(r, recv)] = t
    # steady state: every stage ran every micro-batch about total/N times
    for r in range(W):
        for m in range(N):
            assert passes.get((r, m), 0) >= (total - r) // N - 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, W, port, total, q):
    """W = pipeline depth; world / W groups side by side (stage s of group g = rank g*W + s)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g, s = divmod(rank, W)
    N, rows_per = W, 3
    arena = torch.full((N * rows_per, 4), 1000.0 * g)
    log = []

    def compute(m):
        arena[m * rows_per:(m + 1) * rows_per] += s + 1
        if s == W - 1:
            log.append((m, float(arena[m * rows_per, 0]) - 1000.0 * g))

    for t in range(total):
        run_tick(dist, t, total, s, W, N, compute,
                 lambda m: arena[m * rows_per:(m + 1) * rows_per], base=g * W)
    dist.barrier()
    q.put((rank, log))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,W", [(2, 2), (3, 3), (4, 2)])
def test_gloo_pipeline_ring(world, W):
    total = ticks_needed(W, 4, 3)
    assert tokens_per_request_needed(W, total, W) > total // W
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, W, port, total, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    # a micro-batch's k-th pass through all W stages adds k * (1 + 2 + ... + W); groups never mix
    per_pass = W * (W + 1) / 2
    for g in range(world // W):
        seen = {}
        last = out[g * W + W - 1]
        for m, v in last:
            seen[m] = seen.get(m, 0) + 1
            assert v == seen[m] * per_pass, (g, m, v, seen[m])
        assert len(last) >= total - W
