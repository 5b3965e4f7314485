"""Live serving (bh_runner_serve) on the control plane alone (dry run, no GPU): requests arrive
over wall-clock time, are prefilled on arrival and board the next lockstep decode iteration.
Checks the reference's report definitions (nearest-rank percentiles, tokens / drain,
metrics.cpp:30-38, 159-190) and the scheduling invariants of the batch trace."""
import numpy as np
import pytest

from paper_2404_18322_b200.metrics import (latency_stats, load_arrivals, percentile,
                                           poisson_arrivals, serving_report)
from paper_2404_18322_b200.runner import Runner
from paper_2404_18322_b200.workloads import c1_tiny, c2_llama7b


def test_poisson_arrivals_are_seeded_and_sorted():
    a = poisson_arrivals(100, 50.0, seed=3)
    assert a[0] == 0 and np.all(np.diff(a) >= 0)
    assert np.array_equal(a, poisson_arrivals(100, 50.0, seed=3))
    assert 1.2e6 < a[-1] < 3.2e6  # ~99 gaps of 20 ms


def test_latency_stats_nearest_rank():
    v = [5.0, 1.0, 4.0, 2.0, 3.0]
    st = latency_stats(v)
    assert st["count"] == 5 and st["mean"] == 3.0
    assert st["p50"] == 3.0 and st["p95"] == 5.0 and st["p90"] == 5.0
    assert st["p50"] == percentile(v, 0.5)


def test_load_arrivals_reads_the_reference_format(tmp_path):
    p = tmp_path / "arr.csv"
    p.write_text("t_us,app_id,prompt_tokens,output_tokens\n0,1,64,32\n1500,0,128,16,2,32\n")
    assert load_arrivals(str(p)) == [(0, 1, 64, 32), (1500, 0, 128, 16)]


@pytest.mark.parametrize("qps", [400.0, 5000.0])
def test_dry_serve_invariants(qps):
    wl = c1_tiny(output=5)
    arr = poisson_arrivals(wl.n_requests, qps, seed=7)
    run = Runner(None, wl, mode=1, dry_run=True)
    first, done = run.serve(arr)
    assert np.all(first >= arr) and np.all(done >= first)
    assert run.tokens_generated == sum(wl.req_output)
    rep = serving_report(arr, first, done, run.tokens_generated)
    assert rep["completed"] == wl.n_requests
    assert rep["latency_ms"]["p95"] >= rep["latency_ms"]["p50"]
    tr = run.trace()
    # every request: one prefill batch per chain step, then output-1 decode tokens per step
    pre = [m for (_, _, ph, mem) in tr if ph == 0 for m in mem]
    dec = [m for (_, _, ph, mem) in tr if ph == 1 for m in mem]
    assert len(pre) == wl.n_requests * 2
    assert len(dec) == wl.n_requests * 2 * (5 - 1)
    # a request's decode contexts run prompt+1 .. prompt+output-1, one token per iteration
    for r in range(1, wl.n_requests + 1):
        ctxs = sorted({c for (q, s, c) in dec if q == r})
        assert ctxs == list(range(17, 17 + 4))
    run.close()


def test_dry_serve_arrivals_join_running_decodes():
    """Arrivals spaced wider than a dry decode step: late requests board iterations in which
    earlier ones are already decoding (decode batches with mixed contexts)."""
    wl = c2_llama7b(prompt=32, output=400)
    arr = np.arange(wl.n_requests, dtype=np.int64) * 50
    run = Runner(None, wl, mode=1, dry_run=True)
    first, done = run.serve(arr)
    tr = run.trace()
    mixed = [mem for (_, _, ph, mem) in tr if ph == 1 and len({c for _, _, c in mem}) > 1]
    assert mixed, "no decode iteration mixed requests that arrived at different times"
    run.close()
