"""Multi-GPU block placement and the cluster executor (SURVEY §8 a11 / a15 / e).

Placement (place_blocks): the unit is a block instance on a device (agent.hpp:44-56).
  * A block every tenant routes through (a shared foundation block) serves every request, so
    each GPU holds an instance of it and runs its own requests through it - the reference's
    scale-out of its hottest instances to further devices (Scheduler::scale_decisions,
    scheduler.cpp:227-260), taken to every device since 180 GB holds them all.
  * A tenant's private blocks are placed one by one in chain order by the reference's device
    rule (Scheduler::choose_device with the locality preference, scheduler.cpp:262-314, mirrored
    bit-exactly by bh_policy_choose_device): the device whose resident blocks have the most
    adjacency weight (static chain neighbours) to the block, ties to the most free memory. The
    first private block of a tenant neighbours shared blocks present everywhere, so it lands on
    the emptiest GPU; the tenant's next private block follows it there (one hop out, one back).
  * Requests are served where they arrive (weak scaling: every GPU receives the config's request
    mix). A private block then runs ALL tenants' rows for it from every GPU in one batch - its
    weights stream once per token step instead of once per GPU.

Plan (block_plan / stage_plan): a request's chain is cut into legs (consecutive blocks on one
device); phase k runs every request's k-th leg, and after it the rows hop to their next leg's
runner (NCCL P2P across GPUs, a device copy inside a process) or back home after the last leg.
Each (rank, phase) pair with work is one single-device executor (bh_runner) whose workload is the
leg's blocks and rows. The plan is the same on every rank; bh_cluster (C++) executes it.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from dataclasses import dataclass, field

import numpy as np

from ._lib import BlockExecError, check, lib
from .workloads import Workload

PHASE_PREFILL, PHASE_DECODE = 0, 1
ARENA_DECODE, ARENA_PREFILL = 0, 1


class Hop(C.Structure):
    _fields_ = [("src_rank", C.c_int32), ("src_runner", C.c_int32), ("dst_rank", C.c_int32),
                ("dst_runner", C.c_int32), ("arena", C.c_int32), ("pad_", C.c_int32),
                ("src_row", C.c_int64), ("dst_row", C.c_int64), ("rows", C.c_int64)]


class ClusterStats(C.Structure):
    _fields_ = [("steps", C.c_int64), ("batches", C.c_int64), ("sent_bytes", C.c_int64),
                ("recv_bytes", C.c_int64), ("local_bytes", C.c_int64)]


_bound = False


def _bind():
    global _bound
    if _bound:
        return lib()
    L = lib()
    P, I, I64 = C.c_void_p, C.c_int, C.c_int64
    for name, res, args in [
        ("be_comm_unique_id", I, [P]),
        ("be_comm_init", I, [P, I, I, P, C.POINTER(C.c_void_p)]),
        ("be_comm_destroy", I, [P]),
        ("be_comm_last_error", C.c_char_p, [P]),
        ("be_comm_rank", I, [P]),
        ("be_comm_size", I, [P]),
        ("be_comm_bytes", I64, [P, I]),
        ("be_hop_begin", I, [P]),
        ("be_hop_end", I, [P]),
        ("be_hop_send", I, [P, I, P, I64, P]),
        ("be_hop_recv", I, [P, I, P, I64, P]),
        ("bh_cluster_create", I, [P, I, I, P, I, C.POINTER(C.c_void_p)]),
        ("bh_cluster_free", I, [P]),
        ("bh_cluster_last_error", C.c_char_p, [P]),
        ("bh_cluster_add_runner", I, [P, I, I, P]),
        ("bh_cluster_add_phase", I, [P, I, I, P, I, P]),
        ("bh_cluster_prefill", I, [P]),
        ("bh_cluster_decode_step", I, [P, I, P, P]),
        ("bh_cluster_get_stats", I, [P, P]),
        ("bh_runner_requests", I, [P]),
    ]:
        fn = getattr(L, name)
        fn.restype, fn.argtypes = res, args
    _bound = True
    return L


# ------------------------------------------------------------------------------ placement
def shared_blocks(wl: Workload) -> set[int]:
    """Blocks on more than one tenant's chain."""
    seen: dict[int, set[int]] = {}
    for t, ch in enumerate(wl.chains):
        for b in ch:
            seen.setdefault(b, set()).add(t)
    return {b for b, ts in seen.items() if len(ts) > 1}


def place_blocks(wl: Workload, world: int, hbm_bytes: int = 180 * 10**9,
                 trace: list | None = None) -> list[int]:
    """Block -> rank (-1: an instance on every rank).
    Shared blocks follow the reference's scale-out (bh_policy_scale_decisions =
    Scheduler::scale_decisions, scheduler.cpp:227-260): each starts as one instance on rank 0
    holding the decode queue of every rank's requests (weak scaling: world x the config's rows);
    an instance whose queued work exceeds one GPU's rows is hot and gets a replica on the device
    choose_device(most free) picks, the queue splitting over the replicas, until none is hot - on
    a server with room that is every rank. Private blocks by the locality rule
    (bh_policy_choose_device, scheduler.cpp:262-314), in chain order, each placement charged to
    its device's ledger before the next choice. `trace` (optional) receives the scale-out
    decisions as (round, instance, device)."""
    from .pipeline import routing_policy
    if world == 1:
        return [-1] * len(wl.block_names)  # one GPU holds every block: no leg ever leaves it
    shared = shared_blocks(wl)
    rows = wl.n_requests  # each rank's decode rows per step
    pol = routing_policy(wl, world, instances=False, hbm_bytes=hbm_bytes, scale_queue_us=rows)
    used = [0] * world
    seq = 0
    replicas = {b: [0] for b in sorted(shared)}
    for b in replicas:
        used[0] += wl.shape.param_bytes
    for rnd in range(world):
        for dev in range(world):
            pol.set_ledger(dev, used[dev])
        for b, devs in replicas.items():
            for dev in devs:
                seq += 1
                pol.put_instance(f"r{dev}.{wl.block_names[b]}", wl.block_names[b], dev,
                                 ready=True, created_seq=seq, queue_len=world * rows // len(devs),
                                 queued_cost_us=world * rows / len(devs))
        decisions = pol.scale_decisions()
        if not decisions:
            break
        for inst, dev in decisions:
            b = wl.block_names.index(inst.split(".", 1)[1])
            if dev not in replicas[b]:
                replicas[b].append(dev)
                used[dev] += wl.shape.param_bytes
                if trace is not None:
                    trace.append((rnd, inst, dev))
    for b, devs in replicas.items():
        if len(devs) != world:
            raise ValueError(f"{wl.name}: scale-out left block {wl.block_names[b]} on ranks "
                             f"{sorted(devs)} only (the plan needs shared blocks on every rank)")
    for dev in range(world):
        pol.set_ledger(dev, used[dev])
    place = [-1] * len(wl.block_names)
    for ch in wl.chains:
        for b in ch:
            if b in shared or place[b] >= 0:
                continue
            dev = pol.choose_device(wl.block_names[b])
            if dev < 0:
                raise ValueError(f"{wl.name}: no device fits block {wl.block_names[b]}")
            seq += 1
            pol.put_instance(f"r{dev}.{wl.block_names[b]}", wl.block_names[b], dev, ready=True,
                             created_seq=seq)
            used[dev] += wl.shape.param_bytes
            pol.set_ledger(dev, used[dev])
            place[b] = dev
    pol.close()
    return place


# ------------------------------------------------------------------------------ plans
@dataclass
class RunnerSpec:
    rank: int
    slot: int                      # = phase index
    wl: Workload                   # the leg's blocks and rows
    items: list = field(default_factory=list)  # (home rank, request index) per row


@dataclass
class Plan:
    world: int
    homes: list[int]                 # ranks that receive requests
    order: list[int]                 # request order of a home runner (row -> request index)
    runners: list[RunnerSpec]
    phases: list[tuple[int, list, list]]  # (kind, [(rank, slot)], [Hop fields tuple])
    placement: list[int]             # block -> rank (-1 = every rank / home)
    note: str = ""
    wl: Workload | None = None       # the whole workload the plan cuts

    def runner(self, rank: int, slot: int) -> RunnerSpec | None:
        for r in self.runners:
            if r.rank == rank and r.slot == slot:
                return r
        return None

    def hop_bytes_per_step(self, rank: int, d_model: int) -> tuple[int, int]:
        """(sent, received) NCCL bytes of one decode step on `rank`."""
        s = r = 0
        for kind, _, hops in self.phases:
            if kind != PHASE_DECODE:
                continue
            for h in hops:
                if h[0] == h[2]:
                    continue
                if h[0] == rank:
                    s += h[8] * d_model * 2
                if h[2] == rank:
                    r += h[8] * d_model * 2
        return s, r


def _legs(chain: list[int], placement: list[int]) -> list[tuple[int, list[int]]]:
    """Consecutive chain blocks on one location; location -1 = the request's home rank."""
    legs: list[tuple[int, list[int]]] = []
    for b in chain:
        loc = placement[b]
        if legs and legs[-1][0] == loc:
            legs[-1][1].append(b)
        else:
            legs.append((loc, [b]))
    return legs


def _sub_workload(wl: Workload, name: str, items, legs_of, phase) -> Workload:
    names, comps, remap, chains, tmap = [], [], {}, [], {}
    req_tenant, req_prompt, req_output = [], [], []
    for _, i in items:
        t = wl.req_tenant[i]
        if t not in tmap:
            sub = []
            for b in legs_of[t][phase][1]:
                if b not in remap:
                    remap[b] = len(names)
                    names.append(wl.block_names[b])
                    if wl.block_comps:
                        comps.append(wl.block_comps[b])
                sub.append(remap[b])
            tmap[t] = len(chains)
            chains.append(sub)
        req_tenant.append(tmap[t])
        req_prompt.append(wl.req_prompt[i])
        req_output.append(wl.req_output[i])
    return Workload(name, wl.shape, names, chains, req_tenant, req_prompt, req_output,
                    wl.max_batch_tokens, wl.seed, dict(wl.notes), comps or None)


def make_plan(wl: Workload, world: int, placement: list[int], homes: list[int],
              order: list[int], note: str = "") -> Plan:
    legs_of = [_legs(ch, placement) for ch in wl.chains]
    for t, lg in enumerate(legs_of):
        if lg[0][0] != -1 and len(homes) > 1:
            raise ValueError(f"tenant {t}: a chain must start on blocks present at every home")
    n_phase = max(len(lg) for lg in legs_of)

    def where(loc, home):
        return home if loc == -1 else loc

    # items per (rank, phase), in (home, request order) order
    runners: dict[tuple[int, int], RunnerSpec] = {}
    row_of: dict[tuple[int, int, int], int] = {}  # (phase, home, i) -> row in its runner
    poff_of: dict[tuple[int, int, int], int] = {}
    for p in range(n_phase):
        for s in homes:
            for i in order:
                lg = legs_of[wl.req_tenant[i]]
                if p >= len(lg):
                    continue
                q = where(lg[p][0], s)
                spec = runners.setdefault((q, p), RunnerSpec(q, p, None))
                row_of[(p, s, i)] = len(spec.items)
                poff_of[(p, s, i)] = sum(wl.req_prompt[j] for _, j in spec.items)
                spec.items.append((s, i))
    for (q, p), spec in runners.items():
        spec.wl = _sub_workload(wl, f"{wl.name}@r{q}.leg{p}", spec.items, legs_of, p)

    def merge(hops):
        out = []
        for h in hops:
            if out:
                o = out[-1]
                if (o[:6] == h[:6] and o[6] + o[8] == h[6] and o[7] + o[8] == h[7]):
                    out[-1] = o[:8] + (o[8] + h[8],)
                    continue
            out.append(h)
        return out

    phases = []
    for kind in (PHASE_PREFILL, PHASE_DECODE):
        for p in range(n_phase):
            runs = sorted((q, pp) for (q, pp) in runners if pp == p)
            hops = []
            for s in homes:
                for i in order:
                    lg = legs_of[wl.req_tenant[i]]
                    if p >= len(lg):
                        continue
                    src = where(lg[p][0], s)
                    if p + 1 < len(lg):
                        dst, dslot = where(lg[p + 1][0], s), p + 1
                        if kind == PHASE_PREFILL:
                            hops.append((src, p, dst, dslot, ARENA_PREFILL, 0,
                                         poff_of[(p, s, i)], poff_of[(p + 1, s, i)],
                                         wl.req_prompt[i]))
                        else:
                            hops.append((src, p, dst, dslot, ARENA_DECODE, 0, row_of[(p, s, i)],
                                         row_of[(p + 1, s, i)], 1))
                    elif p > 0 or src != s:
                        # the last leg's rows (prefill: the first token) go back home
                        hops.append((src, p, s, 0, ARENA_DECODE, 0, row_of[(p, s, i)],
                                     row_of[(0, s, i)], 1))
            phases.append((kind, runs, merge(hops)))
    return Plan(world, list(homes), list(order), sorted(runners.values(),
                key=lambda r: (r.rank, r.slot)), phases, placement, note, wl)


def block_plan(wl: Workload, world: int) -> Plan:
    """Weak scaling with block placement: every rank receives the config's requests (home rows
    ordered by tenant so each tenant's rows hop as one range)."""
    placement = place_blocks(wl, world)
    order = sorted(range(wl.n_requests), key=lambda i: (wl.req_tenant[i], i))
    owners = sorted({p for p in placement if p >= 0})
    note = (f"block placement over {world} GPU(s): {len(shared_blocks(wl))} shared blocks on "
            f"every GPU; private blocks by choose_device(locality) -> ranks "
            + ",".join(f"{wl.block_names[b]}:{p}" for b, p in enumerate(placement) if p >= 0)
            + f" ({len(owners)} GPU(s) hold private blocks)")
    return make_plan(wl, world, placement, list(range(world)), order, note)


def stage_plan(wl: Workload, cuts: list[tuple[int, int]]) -> Plan:
    """Chain positions [a, b) of cut k on rank k; all requests live on rank 0 (request order):
    the position pipeline of pipeline.py without micro-batches. Batches are composed exactly as
    in a one-GPU lockstep run."""
    placement = [-1] * len(wl.block_names)
    for k, (a, b) in enumerate(cuts):
        for ch in wl.chains:
            for blk in ch[a:b]:
                placement[blk] = k
    return make_plan(wl, len(cuts), placement, [0], list(range(wl.n_requests)),
                     f"positions {cuts} on ranks 0..{len(cuts) - 1}")


# ------------------------------------------------------------------------------ runtime
class Comm:
    """An NCCL communicator of the hop data path (be_comm_*)."""

    @staticmethod
    def unique_id() -> bytes:
        L = _bind()
        buf = C.create_string_buffer(128)
        if L.be_comm_unique_id(buf) != 0:
            raise BlockExecError(5, "be_comm_unique_id failed")
        return buf.raw

    def __init__(self, ctx, world: int, rank: int, uid: bytes):
        L = _bind()
        h = C.c_void_p()
        rc = L.be_comm_init(ctx.h, world, rank, C.create_string_buffer(uid, 128), C.byref(h))
        if rc != 0:
            raise BlockExecError(rc, "be_comm_init failed")
        self.h = h

    def bytes(self, sent: bool) -> int:
        return _bind().be_comm_bytes(self.h, 1 if sent else 0)

    def close(self):
        if getattr(self, "h", None):
            _bind().be_comm_destroy(self.h)
            self.h = None


class Cluster:
    """The local ranks' runners of a plan and the bh_cluster executing it. ctxs: {rank: ctx}
    for the ranks of this process (one with a communicator; any number without)."""

    def __init__(self, ctxs: dict, plan: Plan, comm: Comm | None = None, use_graphs=True,
                 plan_ahead=False, spec_blocks=None, spec_threshold: float = 0.95):
        """spec_blocks: blocks of plan.wl (global indices) whose decode runs speculatively
        (bh_workload.spec_blocks); every leg runner holding one speculates on it, the draft and
        its verification on that runner's GPU (a marked block's successor is in the same leg:
        the shared blocks the reference's marking rule picks are on every home rank)."""
        from .runner import Runner
        self.plan, self.ctxs, self.comm = plan, dict(ctxs), comm
        self.use_graphs, self.plan_ahead = use_graphs, plan_ahead
        self.spec_names = {plan.wl.block_names[b] for b in (spec_blocks or [])}
        self.spec_threshold = spec_threshold
        ranks = sorted(ctxs)
        if ranks != list(range(ranks[0], ranks[0] + len(ranks))):
            raise ValueError("local ranks must be consecutive")
        self.runners = {}
        for spec in plan.runners:
            if spec.rank in ctxs:
                self.runners[(spec.rank, spec.slot)] = self._runner(spec)
        self.h = None
        self._build()

    def _runner(self, spec: RunnerSpec):
        from .runner import Runner
        local = [b for b, n in enumerate(spec.wl.block_names) if n in self.spec_names]
        return Runner(self.ctxs[spec.rank], spec.wl, mode=1, use_graphs=self.use_graphs,
                      plan_ahead=self.plan_ahead, spec_blocks=local or None,
                      spec_threshold=self.spec_threshold)

    def spec_stats(self) -> dict:
        """Speculation counters summed over this process's runners (bh_runner_spec_stats)."""
        out = {}
        for run in self.runners.values():
            for k, v in run.spec_stats().items():
                if k == "cos_min":
                    out[k] = min(out.get(k, 1.0), v) if run.spec_stats()["rows"] else out.get(k)
                elif k not in ("accept_rate", "cos_mean"):
                    out[k] = out.get(k, 0) + v
        rows = out.get("rows", 0)
        out["accept_rate"] = out["accepted"] / rows if rows else None
        out["cos_mean"] = out["cos_sum"] / rows if rows else None
        return out

    def _build(self):
        """The bh_cluster of the current plan over the current runners."""
        L = _bind()
        if self.h:
            L.bh_cluster_free(self.h)
            self.h = None
        ranks = sorted(self.ctxs)
        arr = (C.c_void_p * len(ranks))(*[self.ctxs[r].h.value for r in ranks])
        h = C.c_void_p()
        d = self.plan.runners[0].wl.shape.d_model
        rc = L.bh_cluster_create(self.comm.h if self.comm else None, ranks[0], len(ranks), arr,
                                 d, C.byref(h))
        if rc != 0:
            raise BlockExecError(rc, "bh_cluster_create failed")
        self.h = h
        for (r, s), run in self.runners.items():
            self._ck(L.bh_cluster_add_runner(h, r, s, run.h))
        self._keep = []
        for kind, runs, hops in self.plan.phases:
            ra = np.asarray([x for rs in runs for x in rs] or [0], np.int32)
            ha = (Hop * max(1, len(hops)))(*[Hop(*x) for x in hops])
            self._keep += [ra, ha]
            self._ck(L.bh_cluster_add_phase(h, kind, len(runs), ra.ctypes.data, len(hops),
                                            C.cast(ha, C.c_void_p)))

    def _ck(self, rc):
        if rc != 0:
            raise BlockExecError(rc, _bind().bh_cluster_last_error(self.h).decode())

    def prefill(self):
        self._ck(_bind().bh_cluster_prefill(self.h))

    def decode_step(self, host_in=None, host_out=None):
        pin = C.c_void_p(host_in.data_ptr() if host_in is not None else 0)
        pout = C.c_void_p(host_out.data_ptr() if host_out is not None else 0)
        self._ck(_bind().bh_cluster_decode_step(self.h, 0, pin, pout))

    def stats(self) -> dict:
        s = ClusterStats()
        self._ck(_bind().bh_cluster_get_stats(self.h, C.byref(s)))
        return {f: getattr(s, f) for f, _ in ClusterStats._fields_}

    def home(self, rank: int):
        return self.runners[(rank, 0)]

    def step_stats(self) -> dict:
        """Summed per-step accounting of this process's runners (last decode step)."""
        out = {}
        for run in self.runners.values():
            for k, v in run.step_stats().items():
                out[k] = out.get(k, 0) + v
        return out

    # -------------------------------------------------------------- KV migration (§8 f rank 1)
    def migrate(self, placement: list[int]) -> dict:
        """Re-places private blocks mid-decode (placement: block -> rank, as place_blocks) and
        moves the KV the new layout needs: every leg runner whose rows change is rebuilt on its
        rank (the block weights loaded there - the reference's parameter load), adopts its rows
        at their current context (bh_runner_adopt) and receives each (request, block) segment's
        pages from the runner that held them - be_kv_copy_pages inside a process (peer copy when
        the contexts differ), NCCL send/recv of the pages across processes (be_hop_*): the copy
        path of start_kv_migration (scenario.cpp:361-431; plan_migration picks all-copy on
        NVLink). Home runners and their rows stay. Returns what moved."""
        import time
        from .runner import Runner
        if self.plan_ahead:
            raise ValueError("migrate needs runners without plan-ahead (their request counters "
                             "run one step ahead)")
        old = self.plan
        wl = old.wl
        new = make_plan(wl, old.world, placement, old.homes, old.order,
                        old.note + " -> migrated")
        t0 = time.perf_counter()
        for c in self.ctxs.values():
            c.sync()
        # every rank is in lockstep: a home runner's request state is every copy's state
        state = {}
        for (r, s), run in self.runners.items():
            if s == 0:
                for j, i in enumerate(old.order):
                    state[i] = run.request_state(j)[:2]
                break
        keep, fresh = {}, {}
        for spec in new.runners:
            if spec.rank not in self.ctxs:
                continue
            prev = old.runner(spec.rank, spec.slot)
            if spec.slot == 0 or (prev is not None and prev.items == spec.items):
                keep[(spec.rank, spec.slot)] = self.runners[(spec.rank, spec.slot)]
                continue
            run = self._runner(spec)
            idx = list(range(len(spec.items)))
            run.adopt(idx, [state[i][0] for _, i in spec.items],
                      [state[i][1] for _, i in spec.items])
            fresh[(spec.rank, spec.slot)] = (spec, run)
        # the page moves, in one canonical order on every rank: (new rank, slot, row, block)
        moves = []  # (src rank, src slot, src row, src block, dst rank, dst slot, dst row, dst block)
        for spec in new.runners:
            key = (spec.rank, spec.slot)
            if spec.slot == 0 or (old.runner(*key) is not None and
                                  old.runner(*key).items == spec.items):
                continue
            for j, (s, i) in enumerate(spec.items):
                src = next(r for r in old.runners if r.slot == spec.slot and (s, i) in r.items)
                jo = src.items.index((s, i))
                t = spec.wl.req_tenant[j]
                for b in spec.wl.chains[t]:
                    bo = src.wl.block_names.index(spec.wl.block_names[b])
                    moves.append((src.rank, src.slot, jo, bo, spec.rank, spec.slot, j, b))
        moved_pages = moved_bytes = remote_bytes = 0
        L = lib()
        local = [m for m in moves if m[0] in self.ctxs and m[4] in self.ctxs]
        for (sr, ss, sj, sb, dr, ds, dj, db) in local:
            src_run = self.runners[(sr, ss)]
            dst_run = fresh[(dr, ds)][1]
            src_slots, tok = src_run.kv_segment(sj, sb)
            if tok == 0 and not src_slots:
                continue  # a block without attention keeps no KV
            dst_slots, _ = dst_run.kv_segment(dj, db)
            n = min(len(src_slots), len(dst_slots))
            a = np.asarray(src_slots[:n], np.int32)
            b = np.asarray(dst_slots[:n], np.int32)
            dp = dst_run.kv_pool(db)
            check(L.be_kv_copy_pages(self.ctxs[dr].h, C.c_void_p(src_run.kv_pool(sb)),
                                     C.c_void_p(dp), a.ctypes.data_as(C.c_void_p),
                                     b.ctypes.data_as(C.c_void_p), n, C.c_void_p(0)),
                  self.ctxs[dr].h)
            moved_pages += n
            moved_bytes += n * L.be_kv_pool_page_bytes(C.c_void_p(dp))
        remote = [m for m in moves if (m[0] in self.ctxs) != (m[4] in self.ctxs)]
        if remote:
            remote_bytes = self._migrate_remote(remote, fresh)
        for c in self.ctxs.values():
            c.sync()
        # swap in the new runners and plan
        for key, run in self.runners.items():
            if key not in keep:
                run.close()
        self.runners = dict(keep)
        self.runners.update({k: v[1] for k, v in fresh.items()})
        self.plan = new
        self._build()
        return {"runners_rebuilt": len(fresh), "pages_copied_in_process": moved_pages,
                "bytes_copied_in_process": moved_bytes, "bytes_over_nccl": remote_bytes,
                "seconds": time.perf_counter() - t0}

    def _migrate_remote(self, moves, fresh) -> int:
        """Pages of segments changing process: per peer, the pages this rank sends are packed
        (canonical move order, the same list on both ranks) into one staging buffer, one NCCL
        group moves every buffer, and received buffers are unpacked into the fresh slots."""
        import torch
        from .pipeline import _DevRows
        L = lib()
        me = next(iter(self.ctxs))

        def pool_view(run, block, slots):
            pool = C.c_void_p(run.kv_pool(block))
            pb = L.be_kv_pool_page_bytes(pool)
            n = max(slots) + 1
            t = torch.as_tensor(_DevRows(L.be_kv_pool_data(pool), n, pb // 2),
                                device="cuda").view(torch.uint8).view(n, pb)
            return t, torch.as_tensor(slots, dtype=torch.long, device="cuda")

        for c in self.ctxs.values():
            c.sync()
        sends, recvs = {}, {}  # peer -> [(pool view, slot index)]
        for (sr, ss, sj, sb, dr, ds, dj, db) in moves:
            if sr == me:
                run = self.runners[(sr, ss)]
                slots, _ = run.kv_segment(sj, sb)
                if slots:
                    sends.setdefault(dr, []).append(pool_view(run, sb, slots))
            else:
                run = fresh[(dr, ds)][1]
                slots, _ = run.kv_segment(dj, db)
                if slots:
                    recvs.setdefault(sr, []).append(pool_view(run, db, slots))

        def staging(parts):
            n = sum(idx.numel() for _, idx in parts)
            return torch.empty(n, parts[0][0].shape[1], dtype=torch.uint8, device="cuda")

        sbuf = {p: staging(v) for p, v in sends.items()}
        rbuf = {p: staging(v) for p, v in recvs.items()}
        for p, parts in sends.items():
            off = 0
            for view, idx in parts:
                sbuf[p][off:off + idx.numel()] = view[idx]
                off += idx.numel()
        torch.cuda.synchronize()
        B = _bind()
        self._ck_comm(B.be_hop_begin(self.comm.h))
        for p, buf in sbuf.items():
            self._ck_comm(B.be_hop_send(self.comm.h, p, C.c_void_p(buf.data_ptr()), buf.numel(),
                                        C.c_void_p(0)))
        for p, buf in rbuf.items():
            self._ck_comm(B.be_hop_recv(self.comm.h, p, C.c_void_p(buf.data_ptr()), buf.numel(),
                                        C.c_void_p(0)))
        self._ck_comm(B.be_hop_end(self.comm.h))
        for c in self.ctxs.values():
            c.sync()
        for p, parts in recvs.items():
            off = 0
            for view, idx in parts:
                view[idx] = rbuf[p][off:off + idx.numel()]
                off += idx.numel()
        torch.cuda.synchronize()
        return sum(b.numel() for b in sbuf.values()) + sum(b.numel() for b in rbuf.values())

    def _ck_comm(self, rc):
        if rc != 0:
            raise BlockExecError(rc, _bind().be_comm_last_error(self.comm.h).decode())

    def close(self):
        if getattr(self, "h", None):
            _bind().bh_cluster_free(self.h)
            self.h = None
        for run in self.runners.values():
            run.close()
        self.runners = {}
