"""GPU tests beyond the forward/backward parity: dC through the transport plan
 and the distributed drivers on one device.

dC is checked against the oracle's transport_plan (core.py:363-368) evaluated
on the reference's own final potentials; the sharded drivers run with a
one-rank NCCL group, which exercises their collectives and the CUDA shard
backend (half-sweep C ABI) end to end against the reference fixtures.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from conftest import GRAD_ATOL, LOSS_RTOL, golden_cost, load_golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _skb():
    import paper_1907_01729_b200 as skb

    return skb


def _plan_grad_ref(g, c):
    from oracle import sinkhorn_oracle as orc

    up = g["upstream"]
    if c.ndim == 2:
        return sum(up[b] * orc.transport_plan(g["log_u"][b], g["log_v"][b], c, float(g["lam"]))
                   for b in range(len(up)))
    return np.stack([up[b] * orc.transport_plan(g["log_u"][b], g["log_v"][b], c[b], float(g["lam"]))
                     for b in range(len(up))])


@pytest.mark.parametrize("name", ["config1", "rect_37x53", "config4_subset"])
def test_plan_gradient_matches_transport_plan(name, cuda):
    """dC = sum_b up_b P_b (shared) / up_b P_b (per-sample) from the final potentials."""
    skb = _skb()
    g = load_golden(name)
    c = golden_cost(g)
    want = _plan_grad_ref(g, c)
    got = skb.plan_gradient(torch.tensor(g["log_u"], dtype=torch.float32, device=cuda),
                            torch.tensor(g["log_v"], dtype=torch.float32, device=cuda),
                            torch.tensor(c, dtype=torch.float32, device=cuda), float(g["lam"]),
                            torch.tensor(g["upstream"], dtype=torch.float32, device=cuda))
    got = got.double().cpu().numpy()
    scale = np.abs(want).max()
    assert np.abs(got - want).max() <= 1e-4 * scale


def test_autograd_reaches_the_cost(cuda):
    """sinkhorn_loss(..., cost.requires_grad) returns dC through the plan."""
    skb = _skb()
    g = load_golden("config1")
    c = golden_cost(g)
    mu = torch.tensor(g["mu"], device=cuda)
    nu = torch.tensor(g["nu"], device=cuda)
    ct = torch.tensor(c, dtype=torch.float32, device=cuda, requires_grad=True)
    loss = skb.sinkhorn_loss(mu, nu, ct, float(g["lam"]), max_iters=int(g["max_iters"]))
    loss.backward(torch.tensor(g["upstream"], dtype=torch.float32, device=cuda))
    want = _plan_grad_ref(g, c)
    assert np.abs(ct.grad.double().cpu().numpy() - want).max() <= 1e-4 * np.abs(want).max()


@pytest.fixture(scope="module")
def nccl_world1(cuda):
    import torch.distributed as dist

    if not dist.is_initialized():
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("nccl", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


@pytest.mark.parametrize("backend", ["lse", "gemm"])
@pytest.mark.parametrize("name", ["config5_pin4096", "rect_37x53", "config1_tol", "stability"])
def test_row_sharded_solve_on_the_device(name, backend, nccl_world1, cuda):
    """row_sharded_solve (NCCL, one rank) with the log-domain half-sweep shards
    and with the library's row-sharded GEMM loop, against the reference."""
    from paper_1907_01729_b200 import distributed as D

    g = load_golden(name)
    c = torch.tensor(golden_cost(g), dtype=torch.float32, device=cuda)
    mu = torch.tensor(g["mu"], dtype=torch.float32, device=cuda)
    nu = torch.tensor(g["nu"], dtype=torch.float32, device=cuda)
    if backend == "gemm":   # the library's row-sharded loop (sinkhorn_forward_rows_device_v1)
        res = D.row_sharded_solve_device(mu, nu, c, float(g["lam"]), int(g["max_iters"]),
                                         float(g["tol"]), int(g["check_interval"]))
    else:
        res = D.row_sharded_solve(mu, nu, D.CudaShardBackend(c), float(g["lam"]),
                                  int(g["max_iters"]), float(g["tol"]), int(g["check_interval"]))
    assert res.iterations_run == int(g["iterations_run"])
    rel = np.abs(res.cost_e0.double().cpu().numpy() - g["cost_e0"]) / g["cost_e0"]
    assert rel.max() <= LOSS_RTOL
    gm, gn = D.row_sharded_backward(res.log_u, res.log_v, float(g["lam"]),
                                    torch.tensor(g["upstream"], device=cuda))
    assert np.abs(gm.double().cpu().numpy() - g["grad_mu"]).max() <= GRAD_ATOL
    assert np.abs(gn.double().cpu().numpy() - g["grad_nu"]).max() <= GRAD_ATOL


def test_batch_sharded_solve_on_the_device(nccl_world1, cuda):
    """batch_sharded_solve (NCCL, one rank): local solve + the final loss all-gather."""
    from paper_1907_01729_b200 import distributed as D

    g = load_golden("config1_tol")
    c = torch.tensor(golden_cost(g), dtype=torch.float32, device=cuda)
    res, all_costs = D.batch_sharded_solve(torch.tensor(g["mu"], device=cuda),
                                           torch.tensor(g["nu"], device=cuda), c,
                                           float(g["lam"]), int(g["max_iters"]), float(g["tol"]),
                                           int(g["check_interval"]))
    assert res.iterations_run == int(g["iterations_run"])
    rel = np.abs(all_costs.double().cpu().numpy() - g["cost_e0"]) / g["cost_e0"]
    assert rel.max() <= LOSS_RTOL


@pytest.mark.parametrize("case", ["small", "fused", "tiled", "separable", "per_sample",
                                  "per_sample_lane"])
def test_warm_start_continues_the_iteration(case, cuda):
    """k1 iterations, then k2 more from the returned log_u, equal one run of
    k1 + k2 iterations (the k-th iterate depends only on log_u_{k-1}), on every
    solver path; a warm start from a converged solution stays there."""
    skb = _skb()
    from oracle import sinkhorn_oracle as orc

    rng = np.random.default_rng(11)
    kw = {}
    if case.startswith("per_sample"):
        B, d = 6, 48
        cost = torch.rand(B, d, d, device=cuda)
        kw = {"fused": case == "per_sample"}
    elif case == "separable":
        B, d = 6, 12 * 7
        cost = skb.GridCost(12, 7)
        kw = {"tiled_only": True}
    else:
        B, d = 6, 60
        cost = torch.tensor(orc.fp32_exact(orc.index_grid_cost(d)), dtype=torch.float32,
                            device=cuda)
        kw = {"tiled_only": case != "small", "fused": case != "tiled"}
    mu = torch.tensor(orc.fp32_exact(orc.random_histogram_batch(B, d, rng)), device=cuda)
    nu = torch.tensor(orc.fp32_exact(orc.random_histogram_batch(B, d, rng)), device=cuda)
    mu[2, 5] = 0.0
    mu[2] /= mu[2].sum()
    lam = 0.1
    full = skb.solve(mu, nu, cost, lam, 40, 0.0, **kw)
    first = skb.solve(mu, nu, cost, lam, 25, 0.0, **kw)
    rest = skb.solve(mu, nu, cost, lam, 15, 0.0, init_log_u=first.log_u, **kw)
    rel = ((rest.cost_e0 - full.cost_e0).abs() / full.cost_e0).max()
    assert float(rel) <= 2e-6
    fin = torch.isfinite(full.log_u)
    assert torch.equal(fin, torch.isfinite(rest.log_u))
    assert float((rest.log_u[fin] - full.log_u[fin]).abs().max()) <= 1e-4
    assert bool(torch.isneginf(rest.log_u[2, 5]))


def test_config5_pin_at_d16384(cuda):
    """config 5's 1-D index-grid path pinned to the reference at d=16384
    (2 lanes x 20 iterations; d=65536 is infeasible for the reference)."""
    skb = _skb()
    g = load_golden("config5_pin16384")
    c = torch.tensor(golden_cost(g), dtype=torch.float32, device=cuda)
    res = skb.solve(torch.tensor(g["mu"], device=cuda), torch.tensor(g["nu"], device=cuda), c,
                    float(g["lam"]), int(g["max_iters"]), 0.0)
    rel = np.abs(res.cost_e0.double().cpu().numpy() - g["cost_e0"]) / g["cost_e0"]
    assert rel.max() <= LOSS_RTOL
    gm, gn = skb.potentials_backward(res.log_u, res.log_v, float(g["lam"]),
                                     torch.ones(2, device=cuda))
    assert np.abs(gm.double().cpu().numpy() - g["grad_mu"]).max() <= GRAD_ATOL
    assert np.abs(gn.double().cpu().numpy() - g["grad_nu"]).max() <= GRAD_ATOL


def test_config5_full_support_against_float64(nccl_world1, cuda):
    """the reference cannot run at config 5's d = 65536.  There the
    fp32 paths -- the GEMM iteration, the log-domain tiled half-sweeps and the
    row-sharded driver on both shard backends (one NCCL rank) -- are checked
    against the float64 mode, which matches the reference's fixtures to 1e-9."""
    skb = _skb()
    from paper_1907_01729_b200 import distributed as D
    from paper_1907_01729_b200 import loss as L

    d, B, lam, iters = 65536, 2, 0.05, 3
    gen = torch.Generator(device=cuda)
    gen.manual_seed(5)
    mu = torch.rand(B, d, generator=gen, device=cuda, dtype=torch.float64) + 0.5
    nu = torch.rand(B, d, generator=gen, device=cuda, dtype=torch.float64) + 0.5
    mu, nu = (mu / mu.sum(1, keepdim=True)).float(), (nu / nu.sum(1, keepdim=True)).float()
    c = torch.empty(d, d, device=cuda)
    j = torch.arange(d, device=cuda, dtype=torch.float64)
    for a in range(0, d, 4096):
        i = torch.arange(a, a + 4096, device=cuda, dtype=torch.float64)
        c[a:a + 4096] = (((i[:, None] - j[None, :]).abs() / (d - 1)) ** 2).float()

    def release():
        L._WS_CACHE.clear()
        torch.cuda.empty_cache()

    ref = skb.solve(mu.double(), nu.double(), c, lam, iters, 0.0, fp64=True)
    want_cost, want_u = ref.cost_e0.cpu(), ref.log_u.cpu()
    del ref
    release()
    runs = {}
    for name, kw in (("gemm", {}), ("tiled", {"gemm": False})):
        r = skb.solve(mu, nu, c, lam, iters, 0.0, **kw)
        runs[name] = (r.path, r.cost_e0.double().cpu(), r.log_u.double().cpu())
        del r
        release()
    r = D.row_sharded_solve(mu, nu, D.CudaShardBackend(c), lam, iters, 0.0, d1_total=d)
    runs["rows-lse"] = ("rows-lse", r.cost_e0.double().cpu(), r.log_u.double().cpu())
    del r
    release()
    r = D.row_sharded_solve_device(mu, nu, c, lam, iters, 0.0)
    runs["rows-gemm"] = ("rows-gemm", r.cost_e0.double().cpu(), r.log_u.double().cpu())
    del r
    release()
    assert runs["gemm"][0] == "gemm" and runs["tiled"][0] == "tiled"
    for name, (_, cost, log_u) in runs.items():
        rel = float(((cost - want_cost).abs() / want_cost).max())
        assert rel <= 1e-5, (name, rel)
        assert float((log_u - want_u).abs().max()) <= 1e-3, name


@pytest.mark.parametrize("B,d1,d2", [(256, 784, 784), (64, 300, 190), (5, 1000, 77)])
def test_plan_gradient_tensor_core_path_matches_direct_sum(B, d1, d2, cuda):
    """The shared-cost dC contraction on the tensor cores (sinkhorn_plan_grad_ws_device_v1)
    against the direct per-cell sum over lanes (sinkhorn_plan_grad_device_v1), with
    mixed-sign upstream and zero-mass rows (-inf potentials)."""
    import ctypes

    from paper_1907_01729_b200 import _lib

    skb = _skb()
    lib = _lib.load()
    gen = torch.Generator(device=cuda)
    gen.manual_seed(B + d1)
    m = torch.rand(B, d1, generator=gen, device=cuda, dtype=torch.float64) + 0.5
    mu = (m / m.sum(1, keepdim=True)).float()
    mu[0, :5] = 0.0
    mu[0] /= mu[0].sum()
    m = torch.rand(B, d2, generator=gen, device=cuda, dtype=torch.float64) + 0.5
    nu = (m / m.sum(1, keepdim=True)).float()
    c = torch.rand(d1, d2, generator=gen, device=cuda)
    res = skb.solve(mu, nu, c, 0.05, 30, 0.0)
    up = torch.randn(B, generator=gen, device=cuda)
    got = skb.plan_gradient(res.log_u, res.log_v, c, 0.05, up)
    want = torch.empty_like(c)
    pr = _lib.Problem()
    pr.B, pr.d1, pr.d2, pr.cost_kind = B, d1, d2, _lib.COST_SHARED
    st = lib.sinkhorn_plan_grad_device_v1(ctypes.byref(pr), 0.05, res.log_u.data_ptr(),
                                          res.log_v.data_ptr(), c.data_ptr(), up.data_ptr(),
                                          want.data_ptr(), torch.cuda.current_stream().cuda_stream)
    assert st == 0
    torch.cuda.synchronize()
    scale = float(want.abs().max())
    assert float((got - want).abs().max()) <= 1e-5 * scale
