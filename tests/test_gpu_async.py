"""Asynchronous forward (sinkhorn_forward_async_device_v1, tolerance 0).

SPEC.md:515-516 makes the FFI calls reentrant for disjoint buffers, and
SURVEY 8(b) asks for no host synchronisation at tolerance 0.  These tests
check that the call returns while the GPU is still working, that two solves
on two streams proceed independently, that results equal the synchronous
solve on every path, that the estimate-guard rerun is decided on the device
(forced through the diagnostics flag), and that device-detected statuses
surface through ``SolveResult.check()``.
"""

from __future__ import annotations

import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _skb():
    import paper_1907_01729_b200 as skb

    return skb


def _hist(B, d, gen, dev):
    m = torch.rand(B, d, generator=gen, device=dev, dtype=torch.float64) + 0.5
    return (m / m.sum(1, keepdim=True)).float()


def _index_cost(d, dev):
    i = torch.arange(d, device=dev, dtype=torch.float64)
    return (((i[:, None] - i[None, :]).abs() / (d - 1)) ** 2).float()


CASES = [
    pytest.param("shared", 100, {}, id="small"),
    pytest.param("shared", 400, {"tiled_only": True}, id="fused"),
    pytest.param("shared", 400, {"tiled_only": True, "fused": False, "gemm": False}, id="tiled"),
    pytest.param("shared", 400, {"tiled_only": True, "gemm": True}, id="gemm"),
    pytest.param("grid", 256, {}, id="separable"),
    pytest.param("per_sample", 256, {}, id="per_sample_fused"),
    pytest.param("per_sample", 256, {"fused": False}, id="per_sample_lane"),
]


def _problem(kind, d, B, seed, dev):
    skb = _skb()
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    mu, nu = _hist(B, d, gen, dev), _hist(B, d, gen, dev)
    if kind == "shared":
        c = _index_cost(d, dev)
    elif kind == "grid":
        n = int(round(d ** 0.5))
        c = skb.GridCost(n, n)
    else:
        c = torch.rand(B, d, d, generator=gen, device=dev)
    return mu, nu, c


def _same(a, b, tol):
    fa, fb = torch.isfinite(a), torch.isfinite(b)
    assert torch.equal(fa, fb)
    assert float((a[fa] - b[fb]).abs().max()) <= tol


@pytest.mark.parametrize("kind,d,kw", CASES)
def test_async_equals_sync(kind, d, kw, cuda):
    skb = _skb()
    mu, nu, c = _problem(kind, d, 24, 11, cuda)
    ref = skb.solve(mu, nu, c, 0.05, 50, 0.0, **kw)
    for _ in range(2):   # the second call replays the cached rerun graph
        res = skb.solve(mu, nu, c, 0.05, 50, 0.0, asynchronous=True, **kw).check()
        assert res.iterations_run == 50 and res.path == ref.path
        _same(res.cost_e0, ref.cost_e0, 1e-6 * float(ref.cost_e0.abs().max()))
        _same(res.log_u, ref.log_u, 1e-5)
        _same(res.log_v, ref.log_v, 1e-5)


@pytest.mark.parametrize("kind,d,kw", [c for c in CASES if c.id in
                                       ("fused", "tiled", "gemm", "per_sample_fused")])
def test_forced_rerun_is_decided_on_the_device(kind, d, kw, cuda):
    """With the guard forced, the asynchronous solve's conditional node runs the
    exact solve: its result equals the synchronous forced rerun (the same
    exact solve, decided on the host) and stays within the parity bar of the
    fast one."""
    skb = _skb()
    mu, nu, c = _problem(kind, d, 16, 12, cuda)
    fast = skb.solve(mu, nu, c, 0.05, 40, 0.0, **kw)
    sync_exact = skb.solve(mu, nu, c, 0.05, 40, 0.0, force_rerun=True, **kw)
    for _ in range(2):
        res = skb.solve(mu, nu, c, 0.05, 40, 0.0, asynchronous=True, force_rerun=True,
                        **kw).check()
        _same(res.cost_e0, sync_exact.cost_e0, 1e-7 * float(sync_exact.cost_e0.abs().max()))
        _same(res.log_u, sync_exact.log_u, 1e-6)
    rel = ((sync_exact.cost_e0.double() - fast.cost_e0.double()).abs() / fast.cost_e0.double())
    assert float(rel.max()) <= 1e-5


def test_call_returns_before_the_gpu_finishes(cuda):
    """A config-4-shaped solve (per-sample costs, ~20 ms of GPU work): the call
    returns while the stream is still busy."""
    skb = _skb()
    mu, nu, c = _problem("per_sample", 1024, 192, 13, cuda)
    ref = skb.solve(mu, nu, c, 0.05, 100, 0.0)
    skb.solve(mu, nu, c, 0.05, 100, 0.0, asynchronous=True).check()   # warm (graph capture)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = skb.solve(mu, nu, c, 0.05, 100, 0.0, asynchronous=True)
    t_call = time.perf_counter() - t0
    busy = not torch.cuda.current_stream(cuda).query()
    torch.cuda.synchronize()
    t_all = time.perf_counter() - t0
    res.check()
    assert busy, (t_call, t_all)
    assert t_call < 0.5 * t_all, (t_call, t_all)
    _same(res.cost_e0, ref.cost_e0, 1e-6 * float(ref.cost_e0.abs().max()))


def test_two_streams_proceed_independently(cuda):
    """Two asynchronous solves enqueued on two streams (disjoint buffers,
    SPEC.md:515-516) both return before either finishes and both equal their
    synchronous results."""
    skb = _skb()
    p1 = _problem("per_sample", 1024, 96, 14, cuda)
    p2 = _problem("per_sample", 1024, 96, 15, cuda)
    r1 = skb.solve(*p1, 0.05, 100, 0.0)
    r2 = skb.solve(*p2, 0.05, 100, 0.0)
    s1, s2 = torch.cuda.Stream(cuda), torch.cuda.Stream(cuda)
    for _ in range(2):   # warm both streams' workspaces and graphs
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(s1):
            a = skb.solve(*p1, 0.05, 100, 0.0, asynchronous=True)
        with torch.cuda.stream(s2):
            b = skb.solve(*p2, 0.05, 100, 0.0, asynchronous=True)
        t_enq = time.perf_counter() - t0
        pending = (not s1.query()) or (not s2.query())
        torch.cuda.synchronize()
        t_all = time.perf_counter() - t0
    assert pending and t_enq < t_all, (t_enq, t_all)
    a.check()
    b.check()
    _same(a.cost_e0, r1.cost_e0, 1e-6 * float(r1.cost_e0.abs().max()))
    _same(b.cost_e0, r2.cost_e0, 1e-6 * float(r2.cost_e0.abs().max()))


def test_device_status_surfaces_through_check(cuda):
    """The reference's NaNProduced instance (tests/test_gpu_batch_props.py):
    the asynchronous call returns 0, check() raises NaNProduced."""
    skb = _skb()
    gen = torch.Generator(device=cuda)
    gen.manual_seed(6)
    mu, nu = _hist(3, 64, gen, cuda), _hist(3, 64, gen, cuda)
    c = torch.full((64, 64), 1.0e30, device=cuda)
    res = skb.solve(mu, nu, c, 1e-300, 20, 0.0, asynchronous=True, tiled_only=True)
    with pytest.raises(skb.NaNProduced):
        res.check()


def test_async_needs_tolerance_zero(cuda):
    skb = _skb()
    mu, nu, c = _problem("shared", 100, 4, 16, cuda)
    with pytest.raises(skb.InvalidConfig):
        skb.solve(mu, nu, c, 0.05, 50, 1e-6, asynchronous=True)


def test_host_threads_solve_concurrently(cuda):
    """the calls are reentrant and thread-safe for disjoint
    buffers.  Four host threads (ctypes drops the GIL inside the library), each
    on its own stream and solver path, repeatedly; every result equals the same
    solve run alone."""
    import threading

    skb = _skb()
    jobs = [_problem("per_sample", 256, 24, 41, cuda) + ({},),
            _problem("shared", 400, 24, 42, cuda) + ({"tiled_only": True},),
            _problem("grid", 256, 24, 43, cuda) + ({},),
            _problem("shared", 100, 24, 44, cuda) + ({},)]
    want = [skb.solve(m, n, c, 0.05, 40, 0.0, **kw) for m, n, c, kw in jobs]
    torch.cuda.synchronize()
    errors, got = [], [None] * len(jobs)

    def work(k):
        try:
            m, n, c, kw = jobs[k]
            s = torch.cuda.Stream(cuda)
            with torch.cuda.stream(s):
                for _ in range(3):
                    got[k] = skb.solve(m, n, c, 0.05, 40, 0.0, **kw)
            s.synchronize()
        except Exception as e:   # noqa: BLE001 -- reported below
            errors.append((k, repr(e)))
    ts = [threading.Thread(target=work, args=(k,)) for k in range(len(jobs))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    for r, w in zip(got, want):
        assert r.path == w.path
        _same(r.cost_e0, w.cost_e0, 1e-6 * float(w.cost_e0.abs().max()))
        _same(r.log_u, w.log_u, 1e-5)


def test_graph_cache_eviction_keeps_results_right(cuda):
    """More distinct asynchronous problems than the instantiated-graph cache
    holds (8, LRU): every solve -- fresh capture, replay, in-place update or
    after eviction -- equals its synchronous result."""
    skb = _skb()
    probs = [_problem("per_sample", 64 + 4 * k, 8, 50 + k, cuda) for k in range(11)]
    want = [skb.solve(m, n, c, 0.05, 30, 0.0, fused=True) for m, n, c in probs]
    order = list(range(11)) + list(range(10, -1, -1)) + [0, 5, 10, 0]
    for k in order:
        m, n, c = probs[k]
        res = skb.solve(m, n, c, 0.05, 30, 0.0, fused=True, asynchronous=True,
                        force_rerun=(k % 3 == 0)).check()
        ref = want[k] if k % 3 else skb.solve(m, n, c, 0.05, 30, 0.0, fused=True, force_rerun=True)
        _same(res.cost_e0, ref.cost_e0, 1e-6 * float(ref.cost_e0.abs().max()))
        _same(res.log_v, ref.log_v, 1e-5)
