"""The reference-facing C ABI on the GPU: sinkhorn_forward_v1 / sinkhorn_backward_v1
over host float64 views (ffi.ts:80-191), statuses and outputs against the
oracle's restatement of the same FFI (oracle.forward_v1 / backward_v1) and the
reference's own fixtures.

The check order follows ffi.ts: shapes, B == 0, histograms (11, ffi.ts:111-115),
config (14), cost (15), run, non-finite output (12); the backward refuses any
-inf potential with 13 (ffi.ts:177-179).
"""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

from conftest import GRAD_ATOL, LOSS_RTOL, golden_cost, load_golden

pytestmark = pytest.mark.gpu


def _lib():
    from paper_1907_01729_b200 import _lib as L

    return L, L.load()


def _view(L, a):
    v = L.View()
    v.data = a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    v.ndim = a.ndim
    v.shape[0] = a.shape[0] if a.ndim >= 1 else 0
    v.shape[1] = a.shape[1] if a.ndim == 2 else 0
    v.length = a.size
    return v


def forward_v1(mu, nu, cost, lam, iters, tol):
    L, lib = _lib()
    mu, nu, cost = (np.ascontiguousarray(x, dtype=np.float64) for x in (mu, nu, cost))
    B, d1, d2 = mu.shape[0], mu.shape[1], nu.shape[1]
    out_cost = np.full(B, -7.0)
    out_u = np.full((B, d1), -7.0)
    out_v = np.full((B, d2), -7.0)
    vs = [_view(L, a) for a in (mu, nu, cost, out_cost, out_u, out_v)]
    st = lib.sinkhorn_forward_v1(ctypes.byref(vs[0]), ctypes.byref(vs[1]), ctypes.byref(vs[2]),
                                 float(lam), int(iters), float(tol), ctypes.byref(vs[3]),
                                 ctypes.byref(vs[4]), ctypes.byref(vs[5]))
    return st, out_cost, out_u, out_v


def backward_v1(log_u, log_v, lam, up):
    L, lib = _lib()
    log_u, log_v, up = (np.ascontiguousarray(x, dtype=np.float64) for x in (log_u, log_v, up))
    g_mu = np.full(log_u.shape, -7.0)
    g_nu = np.full(log_v.shape, -7.0)
    vs = [_view(L, a) for a in (log_u, log_v, up, g_mu, g_nu)]
    st = lib.sinkhorn_backward_v1(ctypes.byref(vs[0]), ctypes.byref(vs[1]), float(lam),
                                  ctypes.byref(vs[2]), ctypes.byref(vs[3]), ctypes.byref(vs[4]))
    return st, g_mu, g_nu


@pytest.mark.parametrize("name", ["config1", "rect_37x53", "config1_tol", "closed_form_2x2"])
def test_host_forward_backward_match_reference(name, cuda):
    g = load_golden(name)
    c = golden_cost(g)
    st, cost, lu, lv = forward_v1(g["mu"], g["nu"], c, float(g["lam"]), int(g["max_iters"]),
                                  float(g["tol"]))
    assert st == 0
    assert np.max(np.abs(cost - g["cost_e0"]) / g["cost_e0"]) <= LOSS_RTOL
    scale = max(1.0, np.abs(g["log_u"]).max())
    assert np.abs(lu - g["log_u"]).max() <= 1e-4 * scale
    st, gm, gn = backward_v1(g["log_u"], g["log_v"], float(g["lam"]), g["upstream"])
    assert st == 0
    assert np.abs(gm - g["grad_mu"]).max() <= GRAD_ATOL
    assert np.abs(gn - g["grad_nu"]).max() <= GRAD_ATOL


def _base():
    from oracle import sinkhorn_oracle as orc

    rng = np.random.default_rng(3)
    mu = orc.random_histogram_batch(4, 12, rng)
    nu = orc.random_histogram_batch(4, 9, rng)
    c = orc.fp32_exact(rng.random((12, 9)))
    return mu, nu, c


def _bad(kind):
    mu, nu, c = _base()
    lam, iters = 0.1, 20
    if kind == "sum":
        mu[1, 3] += 1e-3                     # |sum - 1| > 1e-6
    elif kind == "negative":
        nu[2, 0] = -nu[2, 0]
    elif kind == "nan_hist":
        mu[0, 0] = np.nan
    elif kind == "lam0":
        lam = 0.0
    elif kind == "lam_inf":
        lam = np.inf
    elif kind == "iters0":
        iters = 0
    elif kind == "neg_cost":
        c[2, 2] = -0.5
    elif kind == "nan_cost":
        c[0, 1] = np.nan
    elif kind == "hist_and_lam":             # histograms are checked first (ffi.ts order)
        mu[1, 3] += 1e-3
        lam = -1.0
    return mu, nu, c, lam, iters


@pytest.mark.parametrize("kind,status", [("sum", 11), ("negative", 11), ("nan_hist", 11),
                                         ("lam0", 14), ("lam_inf", 14), ("iters0", 14),
                                         ("neg_cost", 15), ("nan_cost", 15),
                                         ("hist_and_lam", 11)])
def test_host_forward_statuses_match_the_ffi(kind, status, cuda):
    from oracle import sinkhorn_oracle as orc

    mu, nu, c, lam, iters = _bad(kind)
    want = orc.forward_v1(mu, nu, c, lam, iters, 0.0)[0]
    st, cost, lu, lv = forward_v1(mu, nu, c, lam, iters, 0.0)
    assert st == want == status
    # nothing is written on error (ffi.ts returns before filling the outputs)
    assert np.all(cost == -7.0) and np.all(lu == -7.0) and np.all(lv == -7.0)


def test_host_forward_empty_batch_and_shape_mismatch(cuda):
    mu, nu, c = _base()
    st, *_ = forward_v1(mu[:0], nu[:0], c, 0.1, 10, 0.0)
    assert st == 0                            # ffi.ts:107-109
    st, *_ = forward_v1(mu, nu, c[:, :5], 0.1, 10, 0.0)
    assert st == 10


def test_host_backward_refuses_minus_inf(cuda):
    from oracle import sinkhorn_oracle as orc

    g = load_golden("zero_mass")
    st, gm, gn = backward_v1(g["log_u"], g["log_v"], float(g["lam"]), np.ones(3))
    assert st == orc.backward_v1(g["log_u"], g["log_v"], float(g["lam"]), np.ones(3))[0] == 13
    assert np.all(gm == -7.0) and np.all(gn == -7.0)


def test_device_api_raises_the_reference_exceptions(cuda):
    """The torch layer maps device statuses to the reference's exception types."""
    import torch

    import paper_1907_01729_b200 as skb

    mu, nu, c = _base()
    bad = mu.copy()
    bad[2, 5] += 1e-3
    t = lambda a: torch.tensor(a, dtype=torch.float32, device=cuda)   # noqa: E731
    with pytest.raises(skb.InvalidHistogram) as exc:
        skb.solve(t(bad), t(nu), t(c), 0.1, 10)
    assert "row 2" in str(exc.value)
    c_bad = c.copy()
    c_bad[1, 1] = -1.0
    with pytest.raises(skb.InvalidCost):
        skb.solve(t(mu), t(nu), t(c_bad), 0.1, 10)


@pytest.mark.parametrize("path", ["fused", "gemm", "per_sample", "per_sample_fused", "fp64"])
def test_every_path_reports_invalid_inputs(path, cuda):
    """Status 11 (histogram) and 15 (cost) on the fused block pass, the GEMM
    iteration, the fused per-sample pass and the float64 mode, each raised as
    the reference's exception type before any result is returned."""
    import torch

    import paper_1907_01729_b200 as skb

    mu, nu, c = _base()
    if path == "per_sample_fused":   # d2 = 12: rows of whole 16-byte units (the fused pass)
        from oracle import sinkhorn_oracle as orc

        nu = orc.random_histogram_batch(4, 12, np.random.default_rng(9))
        c = orc.fp32_exact(np.random.default_rng(9).random((12, 12)))
    B, d1, d2 = mu.shape[0], mu.shape[1], nu.shape[1]
    dt = torch.float64 if path == "fp64" else torch.float32
    t = lambda a: torch.tensor(a, dtype=dt, device=cuda)   # noqa: E731
    kw = {"tiled_only": True, "gemm": path == "gemm", "fp64": path == "fp64"}
    if path == "per_sample":
        kw["fused"] = False   # the lane half-sweeps
    cost = np.repeat(c[None], B, axis=0) if path.startswith("per_sample") else c
    res = skb.solve(t(mu), t(nu), t(cost), 0.1, 20, **kw)
    assert res.path == {"per_sample": "lane", "per_sample_fused": "fused"}.get(path, path)
    bad = mu.copy()
    bad[1, 3] += 1e-3
    with pytest.raises(skb.InvalidHistogram):
        skb.solve(t(bad), t(nu), t(cost), 0.1, 20, **kw)
    c_bad = cost.copy()
    c_bad[..., 2, 2] = -1.0
    with pytest.raises(skb.InvalidCost):
        skb.solve(t(mu), t(nu), t(c_bad), 0.1, 20, **kw)


@pytest.mark.parametrize("offset", [0, 1, 2, 3])
def test_cost_validation_covers_every_element(offset, cuda):
    """validate_cost_kernel reads float4s after a scalar head: a bad element in
    the head, the vector body or the tail is found for every 16-byte
    misalignment of the caller's pointer, and a valid cost passes."""
    import torch

    import paper_1907_01729_b200 as skb

    B, d = 3, 13   # B*d*d = 507: head, body and tail all non-empty
    gen = torch.Generator(device=cuda)
    gen.manual_seed(offset)
    m = torch.rand(B, d, generator=gen, device=cuda) + 0.5
    mu = m / m.sum(1, keepdim=True)
    nu = mu.flip(0).contiguous()
    n = B * d * d
    flat = torch.rand(n + 8, generator=gen, device=cuda)
    cost = flat[offset:offset + n].view(B, d, d)
    skb.solve(mu, nu, cost, 0.1, 5)
    for k in (0, 1, 2, 3, 4, n // 2, n - 4, n - 3, n - 2, n - 1):
        for v in (-1.0, float("nan"), float("inf")):
            saved = float(flat[offset + k])
            flat[offset + k] = v
            with pytest.raises(skb.InvalidCost):
                skb.solve(mu, nu, cost, 0.1, 5)
            flat[offset + k] = saved
