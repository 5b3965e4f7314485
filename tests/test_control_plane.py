"""CPU parity of the host control plane against the reference's own blocksim classes.

The checker is oracle/_ref/libblocksim_ref.so: the unmodified reference sources compiled in place
(oracle/Makefile) behind a C shim. Everything here is integer/queue/page bookkeeping, so the bar
is bit-exact: batch membership and order, enqueue sequence numbers, arbitration, page counts,
page ids, ledger bytes, and whole-simulation batch traces.
"""
import random

import pytest

from paper_2404_18322_b200 import host as H

R = pytest.importorskip("oracle.refshim")
if not R.available():  # pragma: no cover
    pytest.skip("oracle/_ref not built (make -C oracle ref)", allow_module_level=True)

PRE, DEC = H.PREFILL, H.DECODE


def both_pools():
    ours = H.Pool()
    ref = R.RefPool(n_blocks=8, n_devices=2)
    return ours, ref


def keys(entries):
    return [e.key() for e in entries]


# ---------------------------------------------------------------- golden cases (test_agent.cpp)
@pytest.mark.parametrize("impl", ["ours", "ref"])
def test_pop_batch_budget_golden(impl):
    """test_agent.cpp:105-136: 4,6,8 under budget 16 -> {1,2}; oversized head alone; phase cut."""
    P = H.Pool() if impl == "ours" else R.RefPool()
    a = P.create("b0", 0)
    for rid, tok in [(1, 4), (2, 6), (3, 8)]:
        P.enqueue(a, rid, 0, PRE, tok, tok)
    ph, b = P.pop_batch(a, 16)
    assert [e.request_id for e in b] == [1, 2] and ph == PRE
    q, _, executing = P.queue(a)
    assert len(q) == 1 and executing
    P2 = H.Pool() if impl == "ours" else R.RefPool()
    c = P2.create("b0", 0)
    P2.enqueue(c, 1, 0, PRE, 20, 20)
    P2.enqueue(c, 2, 0, PRE, 20, 20)
    assert [e.request_id for e in P2.pop_batch(c, 32)[1]] == [1]
    P3 = H.Pool() if impl == "ours" else R.RefPool()
    d = P3.create("b0", 0)
    P3.enqueue(d, 1, 0, DEC, 1, 5)
    P3.enqueue(d, 2, 0, PRE, 4, 4)
    P3.enqueue(d, 3, 0, DEC, 1, 5)
    ph, b = P3.pop_batch(d, 16)
    assert ph == DEC and [e.request_id for e in b] == [1]


@pytest.mark.parametrize("impl", ["ours", "ref"])
def test_priority_segment_golden(impl):
    """test_agent.cpp:138-154: resident entries ahead, stable -> {2,3,1,4}; cost 20 -> 15."""
    P = H.Pool() if impl == "ours" else R.RefPool()
    a = P.create("b0", 0)
    for rid, res in [(1, False), (2, True), (3, True), (4, False)]:
        P.enqueue(a, rid, 0, DEC, 1, 1, est_cost_us=5.0, kv_resident=res)
    q, cost, _ = P.queue(a)
    assert [e.request_id for e in q] == [2, 3, 1, 4] and cost == pytest.approx(20.0)
    removed = P.remove_queued(a, 3)
    q, cost, _ = P.queue(a)
    assert len(removed) == 1 and len(q) == 3 and cost == pytest.approx(15.0)


@pytest.mark.parametrize("impl", ["ours", "ref"])
def test_arbitration_golden(impl):
    """test_agent.cpp:156-170: earliest head wins; an executing instance is skipped."""
    P = H.Pool() if impl == "ours" else R.RefPool()
    a = P.create("b0", 0)
    b = P.create("b1", 0)
    P.enqueue(b, 1, 0, DEC, 1, 1)
    P.enqueue(a, 2, 0, DEC, 1, 1)
    assert P.next_runnable(0) == b
    P.pop_batch(b, 16)
    assert P.next_runnable(0) == a
    P.finish_batch(b, 10)
    P.enqueue(b, 3, 0, DEC, 1, 1)
    assert P.next_runnable(0, 10) == a


def test_pool_errors_match_reference():
    for P in both_pools():
        a = P.create("b0", 0)
        with pytest.raises(H.LogicError):
            P.create("b0", 0)  # device already serves the block
        with pytest.raises(H.LogicError):
            P.pop_batch(a, 16)  # empty queue
        P.enqueue(a, 1, 0, PRE, 4, 4)
        P.pop_batch(a, 16)
        P.enqueue(a, 2, 0, PRE, 4, 4)
        with pytest.raises(H.LogicError):
            P.pop_batch(a, 16)  # already executing
        with pytest.raises(H.LogicError):
            P.finish_batch("i99")


@pytest.mark.parametrize("seed", range(12))
def test_pool_random_ops_bit_exact(seed):
    """Random interleavings of every queue operation give identical results step by step."""
    rng = random.Random(seed)
    ours, ref = both_pools()
    insts_o, insts_r = [], []
    for b in range(rng.randint(2, 6)):
        dev = rng.randint(0, 1)
        ready = rng.choice([0, 0, 50])
        insts_o.append(ours.create(f"b{b}", dev, 0, ready))
        insts_r.append(ref.create(f"b{b}", dev, 0, ready))
    assert insts_o == insts_r
    executing = set()
    now = 0
    for _ in range(400):
        now += rng.randint(0, 5)
        i = rng.randrange(len(insts_o))
        io, ir = insts_o[i], insts_r[i]
        op = rng.random()
        if op < 0.45:
            phase = rng.choice([PRE, DEC, DEC])
            tok = rng.randint(1, 40) if phase == PRE else 1
            args = (rng.randint(1, 60), rng.randint(0, 7), phase, tok, rng.randint(1, 900),
                    rng.choice([0.0, 1.5, 7.25]), phase == DEC and rng.random() < 0.5)
            ours.enqueue(io, *args)
            ref.enqueue(ir, *args)
        elif op < 0.65:
            budget = rng.choice([1, 8, 16, 64, 4096])
            if io in executing:
                with pytest.raises(H.LogicError):
                    ours.pop_batch(io, budget, now)
                with pytest.raises(H.LogicError):
                    ref.pop_batch(ir, budget, now)
                continue
            qo = ours.queue(io)[0]
            if not qo:
                continue
            po, pr = ours.pop_batch(io, budget, now), ref.pop_batch(ir, budget, now)
            assert po[0] == pr[0] and keys(po[1]) == keys(pr[1])
            executing.add(io)
        elif op < 0.8:
            if io in executing:
                ours.finish_batch(io, now)
                ref.finish_batch(ir, now)
                executing.discard(io)
        elif op < 0.87:
            rid = rng.randint(1, 60)
            assert keys(ours.remove_queued(io, rid)) == keys(ref.remove_queued(ir, rid))
        elif op < 0.92:
            n = rng.randint(0, 5)
            assert keys(ours.take_tail(io, n)) == keys(ref.take_tail(ir, n))
        elif op < 0.95:
            ours.mark_ready(io, now)
            ref.mark_ready(ir, now)
        for dev in (0, 1):
            assert ours.next_runnable(dev, now) == ref.next_runnable(dev, now)
        qo, co, eo = ours.queue(io)
        qr, cr, er = ref.queue(ir)
        assert keys(qo) == keys(qr) and eo == er and co == pytest.approx(cr, abs=1e-9)


# ---------------------------------------------------------------- KvStore (test_kv.cpp)
def both_kv():
    return H.KvStore(), R.RefKvStore(n_devices=3)


@pytest.mark.parametrize("impl", ["ours", "ref"])
def test_kv_pages_golden(impl):
    """test_kv.cpp:129-147: 17 tokens -> 2 pages; +10 -> no page; +10 -> 3 pages."""
    kv = H.KvStore() if impl == "ours" else R.RefKvStore()
    kv.create_segment(1, "blk", 0, 64)
    assert kv.append_tokens(1, "blk", 17) == 2
    i = kv.info(1, "blk")
    assert (i.tokens, i.pages, i.bytes) == (17, 2, 2 * 64 * 16) and kv.used(0) == 2 * 64 * 16
    assert kv.append_tokens(1, "blk", 10) == 0
    assert kv.append_tokens(1, "blk", 10) == 1
    kv.release(1, "blk")
    assert kv.used(0) == 0 and not kv.has_segment(1, "blk")


@pytest.mark.parametrize("impl", ["ours", "ref"])
def test_kv_prefix_sharing_golden(impl):
    """test_kv.cpp:149-177: 40 tokens shared -> 32 (whole pages); saved bytes; extend privately."""
    kv = H.KvStore() if impl == "ours" else R.RefKvStore()
    kv.create_segment(1, "blk", 0, 64)
    kv.append_tokens(1, "blk", 40)
    used = kv.used(0)
    kv.create_segment(2, "blk", 0, 64)
    assert kv.share_prefix(2, 1, "blk", 40) == 32
    assert kv.info(2, "blk").pages == 2 and kv.info(2, "blk").shared_pages == 2
    assert kv.info(1, "blk").shared_pages == 2 and kv.used(0) == used
    assert kv.bytes_saved_by_sharing() == 2 * 64 * 16
    assert kv.append_tokens(2, "blk", 16) == 1
    kv.release(1, "blk")
    assert kv.used(0) == 3 * 64 * 16
    kv.release(2, "blk")
    assert kv.used(0) == 0


@pytest.mark.parametrize("impl", ["ours", "ref"])
def test_kv_move_golden(impl):
    """test_kv.cpp:192-220: private pages move, shared pages are copied."""
    kv = H.KvStore() if impl == "ours" else R.RefKvStore()
    kv.create_segment(1, "blk", 0, 64)
    kv.append_tokens(1, "blk", 32)
    kv.create_segment(2, "blk", 0, 64)
    kv.share_prefix(2, 1, "blk", 32)
    kv.append_tokens(2, "blk", 16)
    page = 64 * 16
    assert kv.used(0) == 3 * page
    kv.move_segment(2, "blk", 1)
    assert kv.info(2, "blk").device == 1 and kv.info(1, "blk").device == 0
    assert kv.used(1) == 3 * page and kv.used(0) == 2 * page
    assert kv.info(1, "blk").shared_pages == 0 and kv.info(2, "blk").shared_pages == 0
    kv.release_request(1)
    kv.release_request(2)
    assert kv.used(0) == 0 and kv.used(1) == 0


def test_kv_errors_match_reference():
    for kv in both_kv():
        kv.create_segment(1, "blk", 0, 64)
        kv.append_tokens(1, "blk", 32)
        kv.create_segment(2, "blk", 0, 64)
        kv.append_tokens(2, "blk", 1)
        with pytest.raises(ValueError):
            kv.share_prefix(2, 1, "blk", 32)  # non-empty target
        kv.create_segment(3, "blk", 1, 64)
        with pytest.raises(ValueError):
            kv.share_prefix(3, 1, "blk", 32)  # across devices
        with pytest.raises(ValueError):
            kv.create_segment(1, "blk", 0, 64)  # exists
        with pytest.raises(ValueError):
            kv.append_tokens(9, "blk", 1)  # unknown
        with pytest.raises(ValueError):
            kv.create_segment(4, "blk", 0, 0)  # bytes_per_token must be positive


@pytest.mark.parametrize("seed", range(10))
def test_kv_random_ops_bit_exact_page_ids(seed):
    """Random create/append/share/move/release sequences: identical page counts, sharing,
    ledger bytes and the global page ids themselves (kv.hpp:126)."""
    rng = random.Random(1000 + seed)
    ours, ref = both_kv()
    blocks = ["b0", "b1", "b2"]
    live = set()
    for _ in range(300):
        op = rng.random()
        req = rng.randint(1, 12)
        blk = rng.choice(blocks)
        try_both = []
        if op < 0.2:
            args = (req, blk, rng.randint(0, 2), rng.choice([64, 128, 4096]))
            try_both = [("create_segment", args)]
        elif op < 0.55:
            try_both = [("append_tokens", (req, blk, rng.randint(0, 40)))]
        elif op < 0.65:
            try_both = [("share_prefix", (req, rng.randint(1, 12), blk, rng.randint(0, 70)))]
        elif op < 0.75:
            try_both = [("move_segment", (req, blk, rng.randint(0, 2)))]
        elif op < 0.85:
            try_both = [("release", (req, blk))]
        else:
            try_both = [("release_request", (req,))]
        for name, args in try_both:
            res = []
            for kv in (ours, ref):
                try:
                    res.append(("ok", getattr(kv, name)(*args)))
                except ValueError:
                    res.append(("invalid", None))
                except H.LogicError:
                    res.append(("logic", None))
            assert res[0] == res[1], (name, args, res)
        for r in range(1, 13):
            for b in blocks:
                assert ours.info(r, b) == ref.info(r, b)
                assert ours.page_ids(r, b) == ref.page_ids(r, b)
        for dev in range(3):
            assert ours.used(dev) == ref.used(dev)
        assert ours.bytes_saved_by_sharing() == ref.bytes_saved_by_sharing()
        live.add(req)


def test_kv_page_slots_are_physical_and_unique():
    kv = H.KvStore()
    kv.attach_pool("b0", 0, 10)
    kv.create_segment(1, "b0", 0, 64)
    kv.append_tokens(1, "b0", 40)
    kv.create_segment(2, "b0", 0, 64)
    kv.append_tokens(2, "b0", 17)
    s1, s2 = kv.page_slots(1, "b0"), kv.page_slots(2, "b0")
    assert s1 == [0, 1, 2] and s2 == [3, 4]
    kv.release(1, "b0")
    kv.create_segment(3, "b0", 0, 64)
    kv.append_tokens(3, "b0", 33)
    assert kv.page_slots(3, "b0") == [0, 1, 2]  # lowest free slots first
    with pytest.raises(H.LogicError):
        kv.append_tokens(3, "b0", 100)  # pool full (ledger over capacity)


def test_kv_move_segment_slots_gives_page_copies():
    """Moving a segment to another device yields one (old slot, new slot) copy per page: private
    pages free their old slot, a shared prefix page stays for its other reader (kv.cpp move)."""
    kv = H.KvStore()
    kv.attach_pool("b0", 0, 8)
    kv.attach_pool("b0", 1, 8)
    kv.create_segment(1, "b0", 0, 64)
    kv.append_tokens(1, "b0", 32)           # slots 0, 1
    kv.create_segment(2, "b0", 0, 64)
    kv.share_prefix(2, 1, "b0", 32)         # shares slots 0, 1
    kv.append_tokens(2, "b0", 16)           # slot 2
    assert kv.page_slots(2, "b0") == [0, 1, 2]
    src, dst = kv.move_segment_slots(2, "b0", 1)
    assert src == [0, 1, 2] and dst == [0, 1, 2]
    assert kv.page_slots(2, "b0") == [0, 1, 2] and kv.info(2, "b0").device == 1
    assert kv.page_slots(1, "b0") == [0, 1]  # the shared pages stay for request 1
    kv.create_segment(3, "b0", 0, 64)
    kv.append_tokens(3, "b0", 1)
    assert kv.page_slots(3, "b0") == [2]    # request 2's private page freed slot 2 on device 0


def test_kv_move_segment_full_pool_leaves_ledger_unchanged():
    """A move whose destination pool is full throws before the page's bytes are charged to the
    destination: the ledger still matches where the pages are (kv.cpp move)."""
    kv = H.KvStore()
    kv.attach_pool("b0", 0, 4)
    kv.attach_pool("b0", 1, 1)
    kv.create_segment(1, "b0", 0, 64)
    kv.append_tokens(1, "b0", 32)           # 2 private pages on device 0
    used0, used1 = kv.used(0), kv.used(1)
    with pytest.raises(H.LogicError):
        kv.move_segment_slots(1, "b0", 1)   # the second page finds no slot on device 1
    # the first page moved (slot and bytes together), the second stayed (slot and bytes)
    page = used0 // 2
    assert kv.used(0) == used0 - page and kv.used(1) == used1 + page


# ---------------------------------------------------------------- whole-simulation traces
SIM_CASES = [
    # n_layers, dim, n_lora, first_adapted, prompts, outputs, budget
    (4, 256, 2, 2, [20, 13, 7, 33, 16, 5], [4, 6, 3, 5, 2, 4], 48),
    (2, 256, 3, 1, [16] * 9, [5] * 9, 4096),
    (6, 512, 4, 3, [40, 3, 77, 12, 9, 64, 1, 30], [7, 2, 4, 9, 1, 3, 5, 6], 96),
    (3, 256, 1, 0, [100, 100, 100, 5], [3, 3, 3, 10], 128),
    (4, 256, 2, 4, [9, 17, 25], [12, 2, 6], 16),
]


@pytest.mark.parametrize("case", SIM_CASES)
def test_batch_trace_matches_reference_simulation(case):
    """The executor loop's batch sequence (instance, block, phase, members (request, chain step,
    context)) equals the reference Simulation's (scenario.cpp pump/on_batch_finish) on one lane,
    with prefill/decode interleaving, the kv-resident priority segment and the token budget."""
    from paper_2404_18322_b200.device import BlockShape
    from paper_2404_18322_b200.runner import Runner
    from paper_2404_18322_b200.workloads import Workload
    n_layers, dim, n_lora, first, prompts, outputs, budget = case
    blocks, kinds, chains, req_model, trace = R.simulate(n_layers, dim, n_lora, first, prompts,
                                                         outputs, max_batch_tokens=budget)
    shape = BlockShape(1, dim, dim // 64, 3 * dim, max_pos=1024)
    wl = Workload("parity", shape, blocks, chains, req_model, prompts, outputs,
                  max_batch_tokens=budget, block_comps=kinds)
    run = Runner(None, wl, mode=0, dry_run=True)
    run.run()
    mine = run.trace()
    assert len(mine) == len(trace)
    for i, (a, b) in enumerate(zip(mine, trace)):
        assert a == b, (i, a, b)
    assert run.live == 0 and run.tokens_generated == sum(outputs)


# ---------------------------------------------------------------- scalar functions
def test_cosine_golden_reference_and_restatement():
    """test_zoo.cpp:12-18 on both the reference and the oracle restatement."""
    from oracle import oracle as O
    for f in (R.cosine, O.cosine):
        assert f([1, 2, 3], [1, 2, 3]) == pytest.approx(1.0)
        assert f([0.5, 0.5, 0], [0.5, 0, 0.5]) == pytest.approx(0.5)
        assert f([1, 0], [0, 1]) == pytest.approx(0.0)
        with pytest.raises(ValueError):
            f([0, 0], [1, 1])
    with pytest.raises(ValueError):
        R.cosine([1, 2], [1, 2, 3])
    rng = random.Random(5)
    for _ in range(200):
        n = rng.randint(1, 40)
        a = [rng.uniform(-1, 1) for _ in range(n)]
        b = [rng.uniform(-1, 1) for _ in range(n)]
        assert O.cosine(a, b) == pytest.approx(R.cosine(a, b), rel=1e-12, abs=1e-14)


def test_percentile_nearest_rank_matches_reference():
    from paper_2404_18322_b200.metrics import percentile
    rng = random.Random(9)
    for _ in range(200):
        v = [rng.uniform(0, 100) for _ in range(rng.randint(1, 50))]
        q = rng.choice([0.5, 0.9, 0.95, 0.99, 1.0, rng.uniform(0.01, 1.0)])
        assert percentile(v, q) == R.percentile(v, q)
    assert percentile([], 0.95) == R.percentile([], 0.95) == 0.0


def test_measured_b200_profiles_load_in_the_reference():
    """profiles/b200_profiles.json (scripts/make_profiles.py: per-component B200 timings of this
    repo's kernels in blocksim's schema) is accepted by the reference's own load_profiles and its
    CostModel reads back the measured grid points."""
    import json
    import os
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "profiles", "b200_profiles.json")
    prof = json.load(open(path))
    for cls, c in prof["classes"].items():
        for phase in ("decode", "prefill"):
            g = c[phase]
            for i, b in enumerate(g["batch"]):
                for j, t in enumerate(g["tokens"]):
                    got = R.profile_component_us(path, cls, phase == "prefill", b, t)
                    assert got == pytest.approx(g["us"][i][j], rel=1e-12)
    # attention cost grows with context at a fixed batch (the KV read), as the kernels do
    dec = prof["classes"]["attention:4096"]["decode"]["us"]
    assert dec[-1][-1] > 2 * dec[-1][0]


PREFIX_CASES = [
    # n_layers, dim, n_lora, first_adapted, prompts, outputs, budget, prefix tokens
    (4, 256, 2, 2, [48] * 8, [4] * 8, 4096, 40),         # one prefill batch: donor in-batch
    (4, 256, 2, 2, [48, 20, 48, 33, 48, 16], [5, 3, 4, 2, 6, 3], 64, 33),  # across batches
    (3, 512, 3, 1, [64, 70, 40, 64, 80, 17], [3, 3, 3, 3, 3, 3], 4096, 64),
]


@pytest.mark.parametrize("case", PREFIX_CASES)
def test_prefix_sharing_matches_reference_simulation(case):
    """Prefix groups (Request::prefix_group = the app's model, prefix_tokens): the executor loop
    shares a donor's whole prefix pages exactly as create_kv_for_step (scenario.cpp:671-695) -
    the batch trace is unchanged and the bytes saved equal the reference report's
    kv.shared_bytes."""
    from paper_2404_18322_b200.device import BlockShape
    from paper_2404_18322_b200.runner import Runner
    from paper_2404_18322_b200.workloads import Workload
    n_layers, dim, n_lora, first, prompts, outputs, budget, ptok = case
    blocks, kinds, chains, req_model, trace = R.simulate(n_layers, dim, n_lora, first, prompts,
                                                         outputs, max_batch_tokens=budget)
    groups = list(req_model)
    toks = [ptok] * len(prompts)
    rep, ptrace = R.simulate_prefix(n_layers, dim, n_lora, first, prompts, outputs, groups, toks,
                                    max_batch_tokens=budget)
    assert ptrace == trace
    shape = BlockShape(1, dim, dim // 64, 3 * dim, max_pos=1024)
    wl = Workload("prefix", shape, blocks, chains, req_model, prompts, outputs,
                  max_batch_tokens=budget, block_comps=kinds, req_prefix_group=groups,
                  req_prefix_tokens=toks)
    run = Runner(None, wl, mode=0, dry_run=True)
    run.run()
    assert run.trace() == trace
    assert run.kv_bytes()[1] == rep["kv"]["shared_bytes"] > 0
