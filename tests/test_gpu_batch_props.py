"""The reference's batch-engine properties restated on the GPU backend.

* identical lanes agree (pkg/tests/test_batch.py:34-43);
* a batch equals its lanes solved one by one (test_batch.py:46-63);
* forward memory does not depend on the iteration count
  (test_batch.py:211-225; pkg/frontend/test/loss.test.ts:76-102);
* non-finite state is refused with status 12 (batch.py:326-327;
  pkg/frontend/src/ffi.ts:124-128), on every solver path and through the
  host C ABI;
* a lambda sweep at config 2's cost stays within the parity bar on the
  linear-domain fast path, with the exact reruns it needs counted
  (where the linear-domain cliff starts).

Tolerances are the north star's fp32 bars (conftest.py) where the reference
states tighter fp64 ones (1e-14 / 1e-12).
"""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

from conftest import GRAD_ATOL, LOSS_RTOL

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _skb():
    import paper_1907_01729_b200 as skb

    return skb


def _hist(B, d, gen, dev):
    m = torch.rand(B, d, generator=gen, device=dev, dtype=torch.float64) + 0.5
    return (m / m.sum(1, keepdim=True)).float()


def _grid_cost(n, dev):
    from paper_1907_01729_b200 import GridCost

    return GridCost(n, n).materialize(device=dev).float()


# (cost kind, d, solve kwargs): every solver family
PATHS = [
    pytest.param("shared", 100, {}, id="small"),
    pytest.param("shared", 300, {"tiled_only": True}, id="fused"),
    pytest.param("shared", 300, {"tiled_only": True, "fused": False, "gemm": False}, id="tiled"),
    pytest.param("shared", 300, {"tiled_only": True, "gemm": True}, id="gemm"),
    pytest.param("grid", 256, {}, id="separable"),
    pytest.param("per_sample", 128, {}, id="per_sample_fused"),
    pytest.param("per_sample", 128, {"fused": False}, id="per_sample_lane"),
]


def _cost(kind, d, B, gen, dev):
    skb = _skb()
    if kind == "shared":
        i = torch.arange(d, device=dev, dtype=torch.float64)
        return (((i[:, None] - i[None, :]).abs() / (d - 1)) ** 2).float()
    if kind == "grid":
        n = int(round(d ** 0.5))
        return skb.GridCost(n, n)
    return torch.rand(B, d, d, generator=gen, device=dev)


@pytest.mark.parametrize("kind,d,kw", PATHS)
def test_identical_lanes_agree(kind, d, kw, cuda):
    """test_batch.py:34-43: B copies of one lane give the same cost and potentials."""
    skb = _skb()
    gen = torch.Generator(device=cuda)
    gen.manual_seed(3)
    B = 24
    mu = _hist(1, d, gen, cuda).expand(B, d).contiguous()
    nu = _hist(1, d, gen, cuda).expand(B, d).contiguous()
    c = _cost(kind, d, 1, gen, cuda)
    if kind == "per_sample":
        c = c.expand(B, d, d).contiguous()
    res = skb.solve(mu, nu, c, 0.05, 60, 0.0, **kw)
    ce = res.cost_e0.double()
    assert float(((ce - ce[0]).abs() / ce[0]).max()) <= 1e-6
    assert float((res.log_u - res.log_u[0]).abs().max()) <= 1e-5
    assert float((res.log_v - res.log_v[0]).abs().max()) <= 1e-5


@pytest.mark.parametrize("kind,d,kw", PATHS)
def test_batch_equals_independent_lanes(kind, d, kw, cuda):
    """test_batch.py:46-63: the batch solve equals per-lane solves (tolerance 0,
    so lanes are independent), on cost, potentials and residuals."""
    skb = _skb()
    gen = torch.Generator(device=cuda)
    gen.manual_seed(4)
    B = 20
    mu, nu = _hist(B, d, gen, cuda), _hist(B, d, gen, cuda)
    c = _cost(kind, d, B, gen, cuda)
    full = skb.solve(mu, nu, c, 0.05, 60, 0.0, **kw)
    for b in range(B):
        cb = c[b:b + 1] if kind == "per_sample" else c
        one = skb.solve(mu[b:b + 1], nu[b:b + 1], cb, 0.05, 60, 0.0, **kw)
        assert abs(float(one.cost_e0[0]) - float(full.cost_e0[b])) <= LOSS_RTOL * float(one.cost_e0[0])
        assert float((one.log_u[0] - full.log_u[b]).abs().max()) <= 1e-4
        assert float((one.log_v[0] - full.log_v[b]).abs().max()) <= 1e-4
        assert abs(float(one.residuals[0]) - float(full.residuals[b])) <= 1e-6


@pytest.mark.parametrize("kind,d,kw", PATHS)
def test_forward_memory_independent_of_iterations(kind, d, kw, cuda):
    """test_batch.py:211-225 / loss.test.ts:76-102: peak device memory of a
    forward (workspace + outputs) and the autograd node's saved state do not
    grow with max_iters -- no per-iteration history is kept."""
    skb = _skb()
    gen = torch.Generator(device=cuda)
    gen.manual_seed(5)
    B = 16
    mu = _hist(B, d, gen, cuda).requires_grad_(True)
    nu = _hist(B, d, gen, cuda)
    c = _cost(kind, d, B, gen, cuda)
    peaks, saved = [], []
    for iters in (5, 5, 200):   # the first call grows the cached workspace
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats(cuda)
        base = torch.cuda.memory_allocated(cuda)
        loss = skb.sinkhorn_loss(mu, nu, c, 0.05, max_iters=iters)
        torch.cuda.synchronize()
        peaks.append(torch.cuda.max_memory_allocated(cuda) - base)
        saved.append(sum(t.numel() for t in loss.grad_fn.saved_tensors))
        loss.sum().backward()
    assert peaks[1] == peaks[2]
    assert saved[1] == saved[2] == 2 * B * d   # log_u and log_v only (loss.ts:104)


@pytest.mark.parametrize("kw", [pytest.param({}, id="small"),
                                pytest.param({"tiled_only": True}, id="fused"),
                                pytest.param({"tiled_only": True, "fused": False, "gemm": False},
                                             id="tiled"),
                                pytest.param({"tiled_only": True, "gemm": True}, id="gemm")])
def test_nonfinite_state_is_status_12(kw, cuda):
    """batch.py:326-327 / ffi.ts:124-128.  With c / lambda beyond even float64's
    range the reference's A = -c/lambda is -inf everywhere, its state turns NaN
    and batch_forward raises NaNProduced (checked against the reference in
    tests/test_oracle_golden.py); every device path must refuse the same
    instance with status 12 (NaNProduced), not return garbage."""
    skb = _skb()
    gen = torch.Generator(device=cuda)
    gen.manual_seed(6)
    B, d = 3, 64
    mu, nu = _hist(B, d, gen, cuda), _hist(B, d, gen, cuda)
    c = torch.full((d, d), 1.0e30, device=cuda)
    with pytest.raises(skb.NaNProduced):
        skb.solve(mu, nu, c, 1e-300, 20, 0.0, **kw)


def test_nonfinite_state_is_status_12_through_the_host_abi(cuda):
    """The same refusal through the reference-facing sinkhorn_forward_v1
    (host float64 views, ffi.ts:80-134): status 12 and the outputs untouched."""
    from paper_1907_01729_b200 import _lib

    lib = _lib.load()
    B, d = 2, 32
    rng = np.random.default_rng(6)
    mu = rng.uniform(0.5, 1.5, (B, d))
    mu /= mu.sum(1, keepdims=True)
    nu = rng.uniform(0.5, 1.5, (B, d))
    nu /= nu.sum(1, keepdims=True)
    c = np.full((d, d), 1.0e30)
    out_cost = np.full(B, 7.0)
    out_lu, out_lv = np.full((B, d), 7.0), np.full((B, d), 7.0)

    def view(a):
        v = _lib.View()
        v.data = a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        v.ndim = a.ndim
        v.shape[0] = a.shape[0]
        v.shape[1] = a.shape[1] if a.ndim == 2 else 0
        v.length = a.size
        return v
    vs = [view(a) for a in (mu, nu, c, out_cost, out_lu, out_lv)]
    st = lib.sinkhorn_forward_v1(*(ctypes.byref(v) for v in vs[:3]), 1e-300, 20, 0.0,
                                 *(ctypes.byref(v) for v in vs[3:]))
    assert st == 12
    assert np.all(out_cost == 7.0) and np.all(out_lu == 7.0) and np.all(out_lv == 7.0)


@pytest.mark.parametrize("lam", [0.05, 0.02, 0.01, 0.005])
def test_lambda_sweep_at_config2_cost_stays_in_parity(lam, cuda):
    """Config 2's 28x28 grid cost with lambda down to 0.005: the default path
    (the fused block pass: linear-domain rows, K = 2^A2) must stay within the
    parity bar against the float64 oracle; below some lambda its range guards
    fire and the solve is redone exactly (counted by sinkhorn_exact_reruns_v1,
    recorded by tools/lambda_sweep.py)."""
    from oracle import sinkhorn_oracle as orc

    skb = _skb()
    from paper_1907_01729_b200 import _lib

    lib = _lib.load()
    rng = np.random.default_rng(0)
    B, iters = 4, 100
    mu = orc.fp32_exact(orc.random_histogram_batch(B, 784, rng))
    nu = orc.fp32_exact(orc.random_histogram_batch(B, 784, rng))
    c = orc.fp32_exact(orc.grid2d_cost(28))
    ref = orc.batch_forward(mu, nu, c, lam, iters, 0.0, workers=4)
    r0 = lib.sinkhorn_exact_reruns_v1()
    res = skb.solve(torch.tensor(mu, device=cuda), torch.tensor(nu, device=cuda),
                    torch.tensor(c, dtype=torch.float32, device=cuda), lam, iters, 0.0,
                    tiled_only=True)
    reruns = lib.sinkhorn_exact_reruns_v1() - r0
    assert res.path == "fused" or reruns > 0
    rel = np.abs(res.cost_e0.double().cpu().numpy() - ref.cost_e0) / ref.cost_e0
    assert rel.max() <= LOSS_RTOL, (lam, rel.max(), reruns)
    gm, gn = skb.potentials_backward(res.log_u, res.log_v, lam, torch.ones(B, device=cuda))
    gm_ref, gn_ref = orc.batch_backward(ref.log_u, ref.log_v, lam, np.ones(B))
    assert np.abs(gm.double().cpu().numpy() - gm_ref).max() <= GRAD_ATOL
    assert np.abs(gn.double().cpu().numpy() - gn_ref).max() <= GRAD_ATOL
