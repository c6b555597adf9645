"""Odd shapes on every solver path against the float64 oracle.

Degenerate and ragged extents (1, 7, 129, 1023, 1025, 2049 -- not multiples
of the tiles, vectors, chunks or lane groups the kernels use), B above one
64-lane tensor-core tile, one-row and one-column problems.  A ragged-extent
fault in the tiled sweeps went unnoticed through round 1; this sweep is the
guard.  Tolerances are the north star's (conftest.py).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import GRAD_ATOL, LOSS_RTOL

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

SHAPES = [(1, 1, 1), (1, 1, 7), (3, 7, 1), (2, 5, 129), (5, 129, 5), (1, 1025, 3), (4, 63, 65),
          (2, 257, 1023), (3, 1030, 70), (65, 33, 31), (2, 2049, 17), (3, 300, 1500),
          (2, 130, 2048), (2, 64, 2052), (5, 40, 3001), (2, 33, 4096), (1, 20, 4097),
          (2, 9, 8192), (1, 5, 8193), (2, 6, 12000), (1, 4, 16384), (1, 3, 16385)]
SHARED_PATHS = {"auto": {}, "tiled": {"tiled_only": True, "fused": False, "gemm": False},
                "fused": {"tiled_only": True}, "gemm": {"tiled_only": True, "gemm": True}}
PER_SAMPLE_PATHS = {"auto": {}, "lane": {"fused": False}}


def _inputs(B, d1, d2, seed, per_sample):
    from oracle import sinkhorn_oracle as orc

    rng = np.random.default_rng(seed)
    mu = orc.fp32_exact(orc.random_histogram_batch(B, d1, rng))
    nu = orc.fp32_exact(orc.random_histogram_batch(B, d2, rng))
    shape = (B, d1, d2) if per_sample else (d1, d2)
    c = orc.fp32_exact(rng.random(shape))
    return mu, nu, c


def _check(res, ref, lam, cuda):
    import paper_1907_01729_b200 as skb

    got = res.cost_e0.double().cpu().numpy()
    rel = np.abs(got - ref.cost_e0) / np.abs(ref.cost_e0)
    assert rel.max() <= LOSS_RTOL, (rel.max(), res.path)
    B = got.shape[0]
    gm, gn = skb.potentials_backward(res.log_u, res.log_v, lam, torch.ones(B, device=cuda))
    from oracle import sinkhorn_oracle as orc

    gm_ref, gn_ref = orc.batch_backward(ref.log_u, ref.log_v, lam, np.ones(B))
    assert np.abs(gm.double().cpu().numpy() - gm_ref).max() <= GRAD_ATOL, res.path
    assert np.abs(gn.double().cpu().numpy() - gn_ref).max() <= GRAD_ATOL, res.path


@pytest.mark.parametrize("B,d1,d2", SHAPES)
def test_shared_cost_shapes(B, d1, d2, cuda):
    import paper_1907_01729_b200 as skb
    from oracle import sinkhorn_oracle as orc

    lam, iters = 0.1, 20
    mu, nu, c = _inputs(B, d1, d2, d1 * 7 + d2, per_sample=False)
    ref = orc.batch_forward(mu, nu, c, lam, iters, 0.0, workers=4)
    t = lambda a: torch.tensor(a, dtype=torch.float32, device=cuda)   # noqa: E731
    for name, kw in SHARED_PATHS.items():
        res = skb.solve(t(mu), t(nu), t(c), lam, iters, 0.0, **kw)
        assert res.iterations_run == iters, name
        _check(res, ref, lam, cuda)


@pytest.mark.parametrize("B,d1,d2", SHAPES)
def test_per_sample_cost_shapes(B, d1, d2, cuda):
    import paper_1907_01729_b200 as skb
    from oracle import sinkhorn_oracle as orc

    lam, iters = 0.1, 20
    mu, nu, c = _inputs(B, d1, d2, d1 * 5 + d2, per_sample=True)
    ref = orc.per_sample_forward(mu, nu, c, lam, iters, 0.0)
    t = lambda a: torch.tensor(a, dtype=torch.float32, device=cuda)   # noqa: E731
    for name, kw in PER_SAMPLE_PATHS.items():
        res = skb.solve(t(mu), t(nu), t(c), lam, iters, 0.0, **kw)
        assert res.iterations_run == iters, name
        _check(res, ref, lam, cuda)


BIG_B_PATHS = [pytest.param("shared", {}, id="fused"),
               pytest.param("shared", {"tiled_only": True, "fused": False, "gemm": False},
                            id="tiled"),
               pytest.param("shared", {"tiled_only": True, "gemm": True}, id="gemm"),
               pytest.param("per_sample", {}, id="per_sample_fused"),
               pytest.param("per_sample", {"fused": False}, id="per_sample_lane"),
               pytest.param("grid", {}, id="separable"),
               pytest.param("shared", {"fp64": True}, id="fp64")]


@pytest.mark.parametrize("kind,kw", BIG_B_PATHS)
def test_batches_above_the_grid_y_limit(kind, kw, cuda):
    """B = 70000 lanes (> 65535, the grid.y limit of the kernels with one grid
    row per lane; they launch in lane slices): lanes at both ends and across
    the slice boundary equal their single-lane solves."""
    import paper_1907_01729_b200 as skb

    B, d = 70000, 16
    gen = torch.Generator(device=cuda)
    gen.manual_seed(5)
    m = torch.rand(B, d, generator=gen, device=cuda, dtype=torch.float64) + 0.5
    mu = (m / m.sum(1, keepdim=True)).float()
    nu = mu.flip(0).contiguous()
    if kind == "shared":
        c = torch.rand(d, d, generator=gen, device=cuda)
    elif kind == "per_sample":
        c = torch.rand(B, d, d, generator=gen, device=cuda)
    else:
        c = skb.GridCost(4, 4)
    res = skb.solve(mu, nu, c, 0.1, 20, 0.0, **kw)
    for b in (0, 65534, 65535, 65536, B - 1):
        cb = c[b:b + 1] if kind == "per_sample" else c
        one = skb.solve(mu[b:b + 1], nu[b:b + 1], cb, 0.1, 20, 0.0, **kw)
        assert abs(float(one.cost_e0[0]) - float(res.cost_e0[b])) <= 1e-5 * float(one.cost_e0[0])
        assert float((one.log_u[0] - res.log_u[b]).abs().max()) <= 1e-4


@pytest.mark.parametrize("nx,ny", [(3, 300), (300, 3), (33, 257), (256, 64)])
def test_grid_costs_of_any_aspect(nx, ny, cuda):
    """Grid costs whose separable sweep does not fit shared memory (a long ny
    axis) fall back to the dense on-the-fly sweeps; either way the result
    equals the materialised stored cost on the tiled path."""
    import paper_1907_01729_b200 as skb

    B, d = 4, nx * ny
    gen = torch.Generator(device=cuda)
    gen.manual_seed(nx * 1000 + ny)
    m = torch.rand(B, d, generator=gen, device=cuda, dtype=torch.float64) + 0.5
    mu = (m / m.sum(1, keepdim=True)).float()
    nu = mu.flip(0).contiguous()
    gc = skb.GridCost(nx, ny)
    res = skb.solve(mu, nu, gc, 0.01, 10, 0.0)
    assert res.path in ("separable", "tiled")
    ref = skb.solve(mu, nu, gc.materialize(device=cuda).float(), 0.01, 10, 0.0, tiled_only=True,
                    fused=False, gemm=False)
    rel = ((res.cost_e0.double() - ref.cost_e0.double()).abs() / ref.cost_e0.double()).max()
    assert float(rel) <= 2e-6
    assert float((res.log_u - ref.log_u).abs().max()) <= 1e-4


@pytest.mark.parametrize("nx,ny", [(150, 160), (200, 96), (64, 420)])
def test_large_grids_take_the_split_separable_sweeps(nx, ny, cuda):
    """Grids too large for the one-kernel separable sweep run the two-kernel
    split (T through global memory) instead of the dense sweeps: equal to the
    dense on-the-fly path, with a lockstep stop."""
    import paper_1907_01729_b200 as skb

    B, d = 3, nx * ny
    gen = torch.Generator(device=cuda)
    gen.manual_seed(nx + ny)
    m = torch.rand(B, d, generator=gen, device=cuda, dtype=torch.float64) + 0.5
    mu = (m / m.sum(1, keepdim=True)).float()
    nu = mu.flip(0).contiguous()
    gc = skb.GridCost(nx, ny)
    for iters, tol in ((12, 0.0), (300, 1e-4)):
        res = skb.solve(mu, nu, gc, 0.01, iters, tol)
        assert res.path == "separable"
        ref = skb.solve(mu, nu, gc, 0.01, iters, tol, dense_grid=True)
        assert res.iterations_run == ref.iterations_run
        rel = ((res.cost_e0.double() - ref.cost_e0.double()).abs() / ref.cost_e0.double()).max()
        assert float(rel) <= 2e-6
        assert float((res.log_u - ref.log_u).abs().max()) <= 1e-4
