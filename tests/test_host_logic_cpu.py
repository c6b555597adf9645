"""Host-side logic of the Python mirror: config validation, shape contracts,
status -> exception mapping, cost descriptors.  CPU only."""

from __future__ import annotations

import math

import numpy as np
import pytest
import torch

import paper_1907_01729_b200 as skb
from oracle import sinkhorn_oracle as orc


def test_config_defaults_match_reference():
    """core.py:83-86."""
    cfg = skb.SinkhornConfig(lam=0.1)
    assert (cfg.max_iters, cfg.tolerance, cfg.check_interval) == (1000, 1e-9, 10)


@pytest.mark.parametrize("kw", [dict(lam=0.0), dict(lam=-1.0), dict(lam=math.inf),
                                dict(lam=math.nan), dict(lam=1.0, max_iters=0),
                                dict(lam=1.0, tolerance=-1e-3),
                                dict(lam=1.0, tolerance=math.inf),
                                dict(lam=1.0, check_interval=0)])
def test_config_validation(kw):
    """core.py:88-96 raises ValueError; ours is a ValueError subclass too."""
    with pytest.raises(ValueError):
        skb.SinkhornConfig(**kw)


def test_shape_mismatch_raised_before_device_work():
    """test_batch.py:127-134: batch sizes / cost dims disagree -> ShapeMismatch."""
    rng = np.random.default_rng(54)
    c = rng.uniform(size=(4, 4))
    cfg = skb.SinkhornConfig(lam=1.0)
    with pytest.raises(skb.ShapeMismatch):
        skb.batch_forward(orc.random_histogram_batch(2, 4, rng),
                          orc.random_histogram_batch(3, 4, rng), c, cfg)
    with pytest.raises(skb.ShapeMismatch):
        skb.batch_forward(orc.random_histogram_batch(2, 5, rng),
                          orc.random_histogram_batch(2, 4, rng), c, cfg)
    with pytest.raises(skb.ShapeMismatch):
        skb.solve(np.ones((2, 4)) / 4, np.ones((2, 4)) / 4, np.ones((3, 4, 4)), 1.0)
    with pytest.raises(skb.ShapeMismatch):
        skb.solve(np.ones((2, 9)) / 9, np.ones((2, 9)) / 9, skb.GridCost(4, 2), 1.0)


def test_grid_cost_descriptor_matches_oracle_grid():
    g = skb.GridCost(28, 28)
    assert g.d == 784
    np.testing.assert_allclose(g.materialize().numpy(), orc.grid2d_cost(28), rtol=0, atol=1e-15)
    hx, hy = skb.GridCost(64, 32).spacing()
    assert hx == pytest.approx(1 / 63) and hy == pytest.approx(1 / 31)


def test_status_to_exception_mapping():
    from paper_1907_01729_b200 import errors

    with pytest.raises(skb.ShapeMismatch):
        errors.raise_for_status(10, "x")
    with pytest.raises(skb.InvalidHistogram):
        errors.raise_for_status(11, "x")
    with pytest.raises(skb.NaNProduced):
        errors.raise_for_status(12, "x")
    with pytest.raises(skb.ZeroMassGradient) as exc:
        errors.raise_for_status(13, "x", lane=3)
    assert exc.value.lane == 3
    with pytest.raises(ValueError):
        errors.raise_for_status(14, "x")
    with pytest.raises(ValueError):
        errors.raise_for_status(15, "x")
    with pytest.raises(skb.DeviceError):
        errors.raise_for_status(20, "x")
    errors.raise_for_status(0, "x")


def test_backward_upstream_shape_check():
    """test_batch.py:215-224."""
    res = skb.SolveResult(torch.zeros(3), torch.zeros(3, 5), torch.zeros(3, 5), 0.5, 20,
                          torch.zeros(3))
    with pytest.raises(skb.ShapeMismatch):
        skb.batch_backward(res, np.ones(4))


def test_library_is_required_no_cpu_fallback(monkeypatch, tmp_path):
    """Without the built .so the product refuses to run (no CPU fallback)."""
    from paper_1907_01729_b200 import _build, _lib

    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "lib_path", lambda: str(tmp_path / "missing.so"))
    with pytest.raises(ImportError, match="no CPU fallback"):
        _lib.load()
    assert _build.LIB_NAME == "libsinkhorn_b200.so"


def test_point_cloud_cost_descriptor():
    """PointCloudCost: the (d1, d2) matrix it stands for, and the host-side shape
    checks solve() applies before touching the device."""
    import torch

    from paper_1907_01729_b200 import PointCloudCost, ShapeMismatch
    from paper_1907_01729_b200.loss import _check_shapes

    x = torch.tensor([[0.0, 0.0], [1.0, 0.0], [0.0, 2.0]])
    y = torch.tensor([[1.0, 1.0], [0.0, 0.0]])
    c = PointCloudCost(x, y).materialize()
    assert torch.allclose(c, torch.tensor([[2.0, 0.0], [1.0, 1.0], [2.0, 4.0]], dtype=torch.float64))
    assert PointCloudCost(x, y).dim == 2
    assert PointCloudCost(x, y).packed("cpu").shape == (5, 2)
    mu, nu = torch.full((4, 3), 1 / 3), torch.full((4, 2), 0.5)
    assert _check_shapes(mu, nu, PointCloudCost(x, y)) == (4, 3, 2)
    with pytest.raises(ShapeMismatch):
        _check_shapes(mu, nu, PointCloudCost(x, y[:1]))
    with pytest.raises(ShapeMismatch):
        _check_shapes(mu, nu, PointCloudCost(x, torch.zeros(2, 3)))
