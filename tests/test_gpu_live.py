"""Live serving on the GPU (bh_runner_serve): Poisson arrivals prefilled on arrival, decoders
joining the running lockstep iterations; every request completes, time stamps are ordered, and
the final rows agree with a lockstep run of the same requests (other batch compositions, so
within bf16 rounding compounded over the chain: rel-L2 <= 5e-2, min row cosine >= 0.99)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2404_18322_b200.metrics import poisson_arrivals, serving_report  # noqa: E402
from paper_2404_18322_b200.pipeline import _DevRows  # noqa: E402
from paper_2404_18322_b200.runner import Runner  # noqa: E402
from paper_2404_18322_b200.workloads import c1_tiny  # noqa: E402

pytestmark = pytest.mark.gpu


def rows(run, n, d):
    return torch.as_tensor(_DevRows(run.arena_ptr, n, d), device="cuda").view(
        torch.bfloat16).float().cpu().numpy()


def test_c1_live_serve(ctx):
    wl = c1_tiny(output=6)
    n, d = wl.n_requests, wl.shape.d_model
    arr = poisson_arrivals(n, 2000.0, seed=5)
    live = Runner(ctx, wl, mode=1, use_graphs=True)
    first, done = live.serve(arr)
    ctx.sync()
    assert np.all(first >= arr) and np.all(done > first)
    rep = serving_report(arr, first, done, live.tokens_generated)
    assert rep["completed"] == n and live.tokens_generated == n * 6
    got = rows(live, n, d)
    ref = Runner(ctx, wl, mode=1, use_graphs=False)
    ref.run()
    for _ in range(5):
        ref.decode_step()
    ctx.sync()
    want = rows(ref, n, d)
    rel = np.linalg.norm(got - want) / np.linalg.norm(want)
    cos = ((got * want).sum(1) / np.linalg.norm(got, axis=1) / np.linalg.norm(want, axis=1)).min()
    assert rel <= 5e-2 and cos >= 0.99, (rel, cos)
    live.close()
    ref.close()
