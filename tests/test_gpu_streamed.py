"""solve_streamed: host inputs, uploads overlapped with asynchronous lane-group
solves (bench.py's e2e leg).  At tolerance 0 lanes are independent
(pkg/tests/test_batch.py:46-63), so the streamed result must equal one
device-resident solve of the whole batch, for equal groups, explicit group
sizes and every cost kind; with a tolerance it is one synchronous group.
"""

from __future__ import annotations

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _skb():
    import paper_1907_01729_b200 as skb

    return skb


def _inputs(kind, B, d, seed):
    skb = _skb()
    gen = torch.Generator()
    gen.manual_seed(seed)

    def hist():
        m = torch.rand(B, d, generator=gen, dtype=torch.float64) + 0.5
        return (m / m.sum(1, keepdim=True)).float().pin_memory()
    mu, nu = hist(), hist()
    if kind == "per_sample":
        cost = torch.rand(B, d, d, generator=gen).pin_memory()
    elif kind == "shared":
        i = torch.arange(d, dtype=torch.float64)
        cost = (((i[:, None] - i[None, :]).abs() / (d - 1)) ** 2).float().pin_memory()
    else:
        n = int(round(d ** 0.5))
        cost = skb.GridCost(n, n)
    return mu, nu, cost


def _dev(x, cuda):
    return x if isinstance(x, _skb().GridCost) else x.to(cuda)


def _close(a, ref):
    assert a.iterations_run == ref.iterations_run
    rel = ((a.cost_e0.double() - ref.cost_e0.double()).abs() / ref.cost_e0.double().abs())
    assert float(rel.max()) <= 1e-6
    assert float((a.log_u - ref.log_u).abs().max()) <= 1e-5
    assert float((a.log_v - ref.log_v).abs().max()) <= 1e-5


@pytest.mark.parametrize("kind,d", [("per_sample", 256), ("shared", 300), ("grid", 256)])
@pytest.mark.parametrize("chunks", [1, 3, 8, [5, 17, 9, 1]])
def test_streamed_equals_resident_solve(kind, d, chunks, cuda):
    skb = _skb()
    B = 32
    mu, nu, cost = _inputs(kind, B, d, 21)
    ref = skb.solve(mu.to(cuda), nu.to(cuda), _dev(cost, cuda), 0.05, 60, 0.0)
    for _ in range(2):   # the second pass replays the cached graphs
        res = skb.solve_streamed(mu, nu, cost, 0.05, 60, 0.0, chunks=chunks, device=cuda)
        _close(res, ref)


def test_streamed_with_tolerance_is_one_lockstep_group(cuda):
    skb = _skb()
    mu, nu, cost = _inputs("per_sample", 24, 128, 22)
    ref = skb.solve(mu.to(cuda), nu.to(cuda), cost.to(cuda), 0.05, 500, 1e-4)
    res = skb.solve_streamed(mu, nu, cost, 0.05, 500, 1e-4, chunks=4, device=cuda)
    assert res.iterations_run < 500
    _close(res, ref)


def test_streamed_group_sizes_must_cover_the_batch(cuda):
    skb = _skb()
    mu, nu, cost = _inputs("per_sample", 8, 64, 23)
    with pytest.raises(skb.InvalidConfig):
        skb.solve_streamed(mu, nu, cost, 0.05, 10, 0.0, chunks=[3, 3], device=cuda)


def test_streamed_reports_invalid_inputs(cuda):
    """Statuses from any group surface after the pipeline drains (the
    reference raises before returning any result)."""
    skb = _skb()
    mu, nu, cost = _inputs("per_sample", 16, 64, 24)
    cost[11, 3, 5] = -1.0
    with pytest.raises(skb.InvalidCost):
        skb.solve_streamed(mu, nu, cost, 0.05, 10, 0.0, chunks=4, device=cuda)
