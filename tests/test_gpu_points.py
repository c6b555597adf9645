"""Point-cloud costs c_ij = |x_i - y_j|^2 (SINKHORN_COST_POINTS; SURVEY 8(f) rank 3,
PAPER.md:147).  The library evaluates |x|^2 + |y|^2 - 2 x.y with
the x.y contraction on the tensor cores and solves with the materialised
cost.  The reference has no point-cloud API: the oracle is the reference
algorithm (oracle/, pinned to the reference's fixtures) on the float64 cost
materialised from the same points."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import GRAD_ATOL, LOSS_RTOL

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _case(d1, d2, D, B, seed):
    from oracle import sinkhorn_oracle as orc

    rng = np.random.default_rng(seed)
    x = orc.fp32_exact(rng.random((d1, D)))
    y = orc.fp32_exact(rng.random((d2, D)))
    mu = orc.fp32_exact(orc.random_histogram_batch(B, d1, rng))
    nu = orc.fp32_exact(orc.random_histogram_batch(B, d2, rng))
    c = ((x[:, None, :] - y[None, :, :]) ** 2).sum(-1)   # float64, exact from the points
    return x, y, mu, nu, c


@pytest.mark.parametrize("d1,d2,D,kw", [
    pytest.param(100, 80, 3, {}, id="small-D3"),
    pytest.param(300, 200, 2, {"tiled_only": True}, id="fused-D2"),
    pytest.param(257, 190, 7, {"tiled_only": True, "fused": False, "gemm": False}, id="tiled-D7"),
    pytest.param(300, 300, 64, {"tiled_only": True, "gemm": True}, id="gemm-D64"),
    pytest.param(130, 70, 100, {}, id="D100-two-chunks"),
])
def test_point_cloud_cost_matches_reference_algorithm(d1, d2, D, kw, cuda):
    import paper_1907_01729_b200 as skb
    from oracle import sinkhorn_oracle as orc

    x, y, mu, nu, c = _case(d1, d2, D, 6, d1 + D)
    lam, iters = 0.05 * D, 60   # |x - y|^2 grows with D: keep c / lambda comparable
    ref = orc.batch_forward(mu, nu, c, lam, iters, 0.0, workers=2)
    cost = skb.PointCloudCost(torch.tensor(x, device=cuda), torch.tensor(y, device=cuda))
    res = skb.solve(torch.tensor(mu, device=cuda), torch.tensor(nu, device=cuda), cost, lam,
                    iters, 0.0, **kw)
    rel = np.abs(res.cost_e0.double().cpu().numpy() - ref.cost_e0) / ref.cost_e0
    assert rel.max() <= LOSS_RTOL, rel.max()
    up = np.linspace(-1.0, 1.0, 6)
    gm, gn = skb.potentials_backward(res.log_u, res.log_v, lam, torch.tensor(up, device=cuda))
    gm_ref, gn_ref = orc.batch_backward(ref.log_u, ref.log_v, lam, up)
    assert np.abs(gm.double().cpu().numpy() - gm_ref).max() <= GRAD_ATOL
    assert np.abs(gn.double().cpu().numpy() - gn_ref).max() <= GRAD_ATOL


def test_point_cloud_loss_node_and_async(cuda):
    """The autograd node and the asynchronous entry point take point costs too
    (gradients reach mu and nu; the cost is not a tensor input)."""
    import paper_1907_01729_b200 as skb

    x, y, mu, nu, c = _case(120, 90, 3, 4, 9)
    cost = skb.PointCloudCost(torch.tensor(x, device=cuda), torch.tensor(y, device=cuda))
    mu_t = torch.tensor(mu, device=cuda, requires_grad=True)
    nu_t = torch.tensor(nu, device=cuda, requires_grad=True)
    loss = skb.sinkhorn_loss(mu_t, nu_t, cost, 0.1, max_iters=40)
    loss.sum().backward()
    dense = skb.solve(mu_t.detach(), nu_t.detach(), torch.tensor(c, dtype=torch.float32,
                                                                  device=cuda), 0.1, 40)
    # the expanded |x|^2 + |y|^2 - 2 x.y rounds differently from the direct fp32 cost
    assert float(((loss.detach() - dense.cost_e0).abs() / dense.cost_e0).max()) <= LOSS_RTOL
    assert mu_t.grad is not None and nu_t.grad is not None
    asy = skb.solve(mu_t.detach(), nu_t.detach(), cost, 0.1, 40, asynchronous=True).check()
    assert float(((asy.cost_e0 - loss.detach()).abs() / loss.detach()).max()) <= 1e-6


def test_point_cloud_large_support_on_the_gemm_path(cuda):
    """d = 4096 points in 16 dimensions: the materialised cost takes the tcgen05
    GEMM iteration; two lanes against the dense reference restatement."""
    import paper_1907_01729_b200 as skb
    from oracle import sinkhorn_oracle as orc

    x, y, mu, nu, c = _case(4096, 4096, 16, 2, 17)
    lam, iters = 0.5, 20
    cost = skb.PointCloudCost(torch.tensor(x, device=cuda), torch.tensor(y, device=cuda))
    res = skb.solve(torch.tensor(mu, device=cuda), torch.tensor(nu, device=cuda), cost, lam, iters)
    assert res.path == "gemm"
    for b in range(2):
        ref = orc.dense_forward(mu[b], nu[b], c, lam, iters)
        assert abs(float(res.cost_e0[b]) - float(ref.cost_e0[0])) <= LOSS_RTOL * float(ref.cost_e0[0])


def test_non_finite_point_is_an_invalid_cost(cuda):
    import paper_1907_01729_b200 as skb

    x, y, mu, nu, _ = _case(64, 64, 3, 2, 5)
    x[3, 1] = np.inf
    cost = skb.PointCloudCost(torch.tensor(x, device=cuda), torch.tensor(y, device=cuda))
    with pytest.raises(skb.InvalidCost):
        skb.solve(torch.tensor(mu, device=cuda), torch.tensor(nu, device=cuda), cost, 0.1, 10,
                  tiled_only=True)
