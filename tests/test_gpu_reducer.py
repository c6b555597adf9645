"""The cross-rank protocol of the residual reducer (sinkhorn_set_residual_reducer_v1),
checked in one process by standing in for the other ranks inside the callback.

With a reducer installed (batch-sharded solves with a tolerance) every rank
calls it at every convergence check (batch.py:318-322 lockstep), and once
more after its first attempt to agree on the exact rerun: if ANY rank's
estimate guard fired, every rank reruns exactly -- otherwise the ranks'
collectives would fall out of step (round-1 ADVICE, high).  Here a callback
that reports "a peer failed" at the decision call must make this rank rerun
(the result then equals the forced exact solve), and an honest callback must
not.
"""

from __future__ import annotations

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _skb():
    import paper_1907_01729_b200 as skb

    return skb


def _problem(cuda, d=300, B=12, seed=31):
    gen = torch.Generator(device=cuda)
    gen.manual_seed(seed)

    def hist():
        m = torch.rand(B, d, generator=gen, device=cuda, dtype=torch.float64) + 0.5
        return (m / m.sum(1, keepdim=True)).float()
    i = torch.arange(d, device=cuda, dtype=torch.float64)
    c = (((i[:, None] - i[None, :]).abs() / (d - 1)) ** 2).float()
    return hist(), hist(), c


class _Reducer:
    """Records every call; at call index `peer_fails_at` answers 1.0 (a peer's
    estimate guard fired), otherwise returns the local value (world size 1)."""

    def __init__(self, peer_fails_at=None):
        from paper_1907_01729_b200 import _lib

        self.calls = []
        self.peer_fails_at = peer_fails_at
        self.lib = _lib.load()
        self.cb = _lib.REDUCER(self._reduce)
        self.null = _lib.REDUCER(0)

    def _reduce(self, local, _user):
        self.calls.append(local)
        if self.peer_fails_at is not None and len(self.calls) - 1 == self.peer_fails_at:
            return 1.0
        return local

    def __enter__(self):
        self.lib.sinkhorn_set_residual_reducer_v1(self.cb, None)
        return self

    def __exit__(self, *exc):
        self.lib.sinkhorn_set_residual_reducer_v1(self.null, None)


KW = [pytest.param({"tiled_only": True}, id="fused"),
      pytest.param({"tiled_only": True, "fused": False, "gemm": False}, id="tiled"),
      pytest.param({"tiled_only": True, "gemm": True}, id="gemm")]


@pytest.mark.parametrize("kw", KW)
def test_peer_failure_makes_every_rank_rerun(kw, cuda):
    skb = _skb()
    from paper_1907_01729_b200 import _lib

    lib = _lib.load()
    mu, nu, c = _problem(cuda)
    args = (mu, nu, c, 0.05, 40, 1e-12, 10)   # never converges: checks at 10, 20, 30
    r0 = lib.sinkhorn_exact_reruns_v1()
    with _Reducer() as honest:
        fast = skb.solve(*args, **kw)
    assert lib.sinkhorn_exact_reruns_v1() == r0
    n = len(honest.calls)
    assert n == 4 and honest.calls[-1] == 0.0   # three checks, then the rerun decision
    exact = skb.solve(*args, force_rerun=True, **kw)   # the exact solve, decided locally
    r1 = lib.sinkhorn_exact_reruns_v1()
    with _Reducer(peer_fails_at=n - 1) as peer:
        res = skb.solve(*args, **kw)
    assert lib.sinkhorn_exact_reruns_v1() == r1 + 1
    # the rerun's own checks call the reducer in step; it makes no second decision
    assert len(peer.calls) == n + (n - 1)
    assert res.iterations_run == fast.iterations_run == 40
    assert torch.equal(res.cost_e0, exact.cost_e0)
    assert torch.equal(res.log_u, exact.log_u)


@pytest.mark.parametrize("kind", ["grid", "per_sample_lane"])
def test_decision_call_on_paths_without_a_global_rerun(kind, cuda):
    """The separable sweeps (estimate redone locally per thread tile) and the
    per-sample lane sweeps never rerun the solve, but a rank on them still
    makes the decision call -- and follows a peer's failure -- so ranks on
    different paths stay in step."""
    skb = _skb()
    from paper_1907_01729_b200 import _lib

    lib = _lib.load()
    mu, nu, c = _problem(cuda, d=256)
    kw = {}
    if kind == "grid":
        c = skb.GridCost(16, 16)
    else:
        c = c.expand(mu.shape[0], 256, 256).contiguous()
        kw = {"fused": False}
    with _Reducer() as honest:
        res = skb.solve(mu, nu, c, 0.05, 40, 1e-12, 10, **kw)
    assert res.path == {"grid": "separable", "per_sample_lane": "lane"}[kind]
    assert len(honest.calls) == 4 and honest.calls[-1] == 0.0
    r0 = lib.sinkhorn_exact_reruns_v1()
    with _Reducer(peer_fails_at=3) as peer:
        again = skb.solve(mu, nu, c, 0.05, 40, 1e-12, 10, **kw)
    assert lib.sinkhorn_exact_reruns_v1() == r0 + 1 and len(peer.calls) == 7
    rel = ((again.cost_e0.double() - res.cost_e0.double()).abs() / res.cost_e0.double()).max()
    assert float(rel) <= 1e-6
