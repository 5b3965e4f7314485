"""Routing / speculation marking / placement: bh_policy against the
reference's own Scheduler.

oracle/ref_shim.cpp runs the reference Simulation (multi-server cluster, LoRA and fully
fine-tuned models with equivalence edges, loads, evictions, KV migrations, speculation, scale-out
and placement reviews) and at snapshots inside the run records the state the Scheduler reads and
every decision it makes from it. Each snapshot is loaded into bh_policy (include/blockpolicy.h)
and every decision must match exactly - ids, devices, and the estimate doubles bit for bit.
"""
import random

import pytest

from oracle import refshim
from paper_2404_18322_b200 import policy as P

pytestmark = pytest.mark.skipif(not refshim.available(), reason="oracle/_ref not built")

SPECS = {
    "locality": {"capacity": 80 << 20},
    "frag_min": {"frag_min": True, "capacity": 64 << 20, "seed": 3},
    "least_busy": {"least_busy": True, "spec_fraction": 0.5, "capacity": 64 << 20, "seed": 5},
    "tight_memory": {"capacity": 64 << 20, "n_servers": 1, "per_server": 3, "seed": 7,
                     "load_bps": 4e9},
    "no_adaptive": {"adaptive": False, "speculation": False, "n_servers": 3, "per_server": 1,
                    "capacity": 96 << 20, "seed": 9},
}


def _spec(name):
    rnd = random.Random(name)
    n = 48
    s = {"prompts": [rnd.choice([16, 40, 100, 200, 333]) for _ in range(n)],
         "outputs": [rnd.randint(1, 14) for _ in range(n)],
         "gaps": [rnd.randint(0, 500) for _ in range(n)], "every": 5, "max_snapshots": 50}
    s.update(SPECS[name])
    return s


_TRACES = {}


def trace(name):
    if name not in _TRACES:
        _TRACES[name] = refshim.policy_trace(_spec(name))
    return _TRACES[name]


@pytest.mark.parametrize("name", sorted(SPECS))
def test_choose_binding_matches_reference(name):
    t = trace(name)
    pol = P.Policy.from_static(t["static"])
    n = 0
    for sn in t["snapshots"]:
        pol.load_state(sn)
        for q in sn["queries"]:
            if "error" in q:
                with pytest.raises((ValueError, RuntimeError)):
                    pol.choose_binding(q["request"], q["block"], q["decode"], q["tokens"],
                                       q["context"], q["from"], sn["now"])
                continue
            got = pol.choose_binding(q["request"], q["block"], q["decode"], q["tokens"],
                                     q["context"], q["from"], sn["now"])
            want = q["choice"]
            if want is None:
                assert got is None
                continue
            assert got is not None, q
            assert (got["block"], got["stitch"], got["instance"], got["device"],
                    got["adaptive"], got["evict"]) == (
                want["block"], want["stitch"], want["instance"], want["device"],
                want["adaptive"], want["evict"]), (sn["now"], q)
            assert list(got["est"]) == want["est"], (sn["now"], q)  # bit-exact doubles
            n += 1
    assert n > 100


@pytest.mark.parametrize("name", sorted(SPECS))
def test_marks_scale_moves_devices_match_reference(name):
    t = trace(name)
    pol = P.Policy.from_static(t["static"])
    for sn in t["snapshots"]:
        pol.load_state(sn)
        assert pol.speculation_marks() == sn["marks"], sn["now"]
        assert [list(x) for x in pol.scale_decisions()] == sn["scale"], sn["now"]
        assert [list(x) for x in pol.placement_moves()] == sn["moves"], sn["now"]
        for block, pref, excl, dev in sn["devices"]:
            assert pol.choose_device(block, pref, excl) == dev, (sn["now"], block, pref, excl)
        for block, dev, need in sn["need"]:
            assert pol.param_bytes_needed(block, dev) == need
        for block, a, b, rec, cp in sn["rates"]:
            assert pol.migration_rates(block, a, b) == (rec, cp)


def test_traces_cover_the_decision_paths():
    """The snapshots exercise what the policy decides: adaptive (equivalent) bindings, decode
    stick-to-cache, new instances with evictions, loading instances, transfers, marks, scale-outs
    and placement moves."""
    seen = dict.fromkeys(["adaptive", "new", "evict", "loading", "transfer", "marks", "scale",
                          "moves", "decode_home"], 0)
    for name in SPECS:
        for sn in trace(name)["snapshots"]:
            seen["loading"] += sum(not i["ready"] for i in sn["instances"])
            seen["marks"] += len(sn["marks"])
            seen["scale"] += len(sn["scale"])
            seen["moves"] += len(sn["moves"])
            for q in sn["queries"]:
                c = q.get("choice")
                if not c:
                    continue
                seen["adaptive"] += c["adaptive"]
                seen["new"] += c["instance"] == ""
                seen["evict"] += c["evict"] > 0
                seen["transfer"] += c["est"][2] > 0
                seen["decode_home"] += q["decode"] and q["kv_owner"] == c["device"]
    assert all(v > 0 for v in seen.values()), seen


def test_plan_migration_matches_reference():
    rnd = random.Random(11)
    for _ in range(400):
        pages, rec, cp = rnd.randint(0, 40), rnd.randint(0, 9), rnd.randint(0, 9)
        try:
            want = refshim.plan_migration(pages, rec, cp)
        except ValueError:
            with pytest.raises(ValueError):
                P.plan_migration(pages, rec, cp)
            continue
        got = P.plan_migration(pages, rec, cp)
        assert got == (want[0], want[3], want[4], want[5]), (pages, rec, cp, got, want)


def test_policy_errors_mirror_reference():
    pol = P.Policy()
    with pytest.raises(ValueError):
        pol.choose_binding(1, "missing", False, 16, 16)
    with pytest.raises(ValueError):
        pol.set_device_class("x", 0.0)
    with pytest.raises(ValueError):
        pol.add_cost_class("attention:8", {"xs": [2, 1], "ys": [1], "v": [[1], [2]]},
                           {"xs": [1], "ys": [1], "v": [[1]]})


def test_replica_routing_balances_copies():
    """bench.py's replica placement: world copies of a config's requests routed by
    choose_binding land one copy per replica (equal queued cost after every group of identical
    requests; ties to the lower device), so each GPU serves the config's own mix."""
    from paper_2404_18322_b200.pipeline import route_requests
    from paper_2404_18322_b200.workloads import CONFIGS
    for cfg, n in (("c2", 4), ("c3", 2), ("c1", 8)):
        wl = CONFIGS[cfg]()
        dev = route_requests(wl, n, copies=n)
        assert len(dev) == n * wl.n_requests
        for i in range(wl.n_requests):
            assert sorted(dev[i * n:(i + 1) * n]) == list(range(n))


def test_routing_prices_with_measured_profiles():
    """The router's compute estimate for a 7B block is the measured B200 profile (profiles/
    b200_profiles.json) summed over the block's components, read through the reference's own
    bilinear rule (bit-exact vs the reference's CostModel in test_control_plane)."""
    import json
    import os
    from paper_2404_18322_b200.pipeline import routing_policy
    from paper_2404_18322_b200.workloads import CONFIGS
    wl = CONFIGS["c2"]()
    pol = routing_policy(wl, 2)
    blk = wl.block_names[0]
    ch = pol.choose_binding(1, blk, False, 512, 512)
    prof = json.load(open(os.path.join(os.path.dirname(os.path.dirname(__file__)), "profiles",
                                       "b200_profiles.json")))["classes"]

    def lookup(c, b, t):
        g = prof[c]["prefill"]
        return g["us"][g["batch"].index(b)][g["tokens"].index(t)]
    n_layers = wl.shape.n_layers
    want = n_layers * (lookup("attention:4096", 1, 512) + lookup("ffn:4096", 1, 512))
    assert abs(ch["est"][1] - want) <= 1e-9 * want
    assert ch["device"] == 0 and ch["est"][0] == 0.0


@pytest.mark.parametrize("name", sorted(SPECS))
def test_kv_review_matches_reference(name):
    """Proactive KV review (§8(f) rank 1): the interception tracker's predictions and the
    migration order over the queued decode entries with remote caches, at every snapshot, equal
    the reference's (InterceptionTracker, order_migrations, kv_review's selection rule)."""
    t = trace(name)
    pol = P.Policy.from_static(t["static"])
    for sn in t["snapshots"]:
        pol.load_state(sn)
        tint = sn["tint"]
        for key, total, n in tint["keys"]:
            pol.interception_set(key, total, n)
        pol.interception_set(None, *tint["global"])
        for key, t_call, want in sn.get("tint_predict", []):
            got = pol.predicted_remaining(key, t_call, sn["now"])
            assert (got if got is not None else -1) == want
        got = pol.kv_review(sn["kvq"], sn["now"])
        assert got == sn["kv_review"], sn["now"]


def test_kv_review_sees_migrations():
    seen = sum(len(sn["kv_review"]) for name in SPECS for sn in trace(name)["snapshots"])
    remote = sum(1 for name in SPECS for sn in trace(name)["snapshots"] for e in sn["kvq"]
                 if e["owner"] >= 0 and e["owner"] != e["device"])
    assert remote > 0 and seen > 0, (remote, seen)
