"""Parity of the sm_100a path against the reference, on the GPU.

Every case runs the reference's own outputs (tests/golden, produced by
oracle/gen_golden.py from /root/reference) through the C ABI:
loss within 1e-5 relative, gradients within 1e-4, identical iterations_run
(BASELINE.json north_star).  The structure follows the reference's tests
(pkg/tests/test_batch.py, test_reduction.py, frontend/test/ffi.test.ts).
"""

from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import GRAD_ATOL, LOSS_RTOL, golden_cost, load_golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _skb():
    import paper_1907_01729_b200 as skb

    return skb


def _run_golden(name, cuda, cost=None, **kw):
    skb = _skb()
    g = load_golden(name)
    if cost is None:
        c = golden_cost(g)
        cost = torch.tensor(c, dtype=torch.float32, device=cuda)
    res = skb.solve(torch.tensor(g["mu"], device=cuda), torch.tensor(g["nu"], device=cuda), cost,
                    float(g["lam"]), int(g["max_iters"]), float(g["tol"]),
                    int(g["check_interval"]), **kw)
    return g, res


# Small shared/grid problems take the single-launch solver (sweep_small.cuh)
# unless tiled_only forces the sweeps: the fused row->column passes
# (sweep_fused.cuh, shared costs with d <= 1024) or, with fused=False, the
# stream-K tiled half-sweeps.  All of them must match.
PATHS = [pytest.param({}, id="auto"),
         pytest.param({"tiled_only": True, "fused": False, "gemm": False}, id="tiled"),
         pytest.param({"tiled_only": True}, id="fused"),
         pytest.param({"tiled_only": True, "gemm": True}, id="gemm")]


def _check_loss_and_grads(g, res, loss_rtol=LOSS_RTOL, grad_atol=GRAD_ATOL):
    skb = _skb()
    got = res.cost_e0.double().cpu().numpy()
    want = g["cost_e0"]
    rel = np.abs(got - want) / np.abs(want)
    assert rel.max() <= loss_rtol, (rel.max(), got[:4], want[:4])
    assert res.iterations_run == int(g["iterations_run"])
    if int(g["zero_mass_lane"]) < 0:
        up = torch.tensor(g["upstream"], dtype=torch.float32, device=res.cost_e0.device)
        gm, gn = skb.potentials_backward(res.log_u, res.log_v, res.lam, up)
        assert np.abs(gm.double().cpu().numpy() - g["grad_mu"]).max() <= grad_atol
        assert np.abs(gn.double().cpu().numpy() - g["grad_nu"]).max() <= grad_atol
    return rel.max()


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("name", ["config1", "rect_37x53", "stability", "config2_subset",
                                  "config5_pin4096"])
def test_shared_cost_matches_reference(name, path, cuda):
    g, res = _run_golden(name, cuda, **path)
    _check_loss_and_grads(g, res)
    # potentials agree up to fp32 rounding of O(c/lambda) values
    lu = res.log_u.double().cpu().numpy()
    scale = max(1.0, np.abs(g["log_u"][np.isfinite(g["log_u"])]).max())
    assert np.nanmax(np.abs(lu - g["log_u"])) <= 1e-4 * scale
    # residuals: the reference's fp64 values vs ours at the fp32 floor
    assert np.all(np.abs(res.residuals.double().cpu().numpy() - g["residuals"]) <= 1e-5)


@pytest.mark.parametrize("path", PATHS)
def test_closed_form_2x2(path, cuda):
    """conftest.py:9-24 / ffi.test.ts:101-116: E0 = e^-1/(1+e^-1) +- 1e-6."""
    g, res = _run_golden("closed_form_2x2", cuda, **path)
    k = math.exp(-1.0)
    assert abs(float(res.cost_e0[0]) - k / (1 + k)) <= 1e-6
    _check_loss_and_grads(g, res)


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("name", ["config1_tol", "lockstep"])
def test_early_stopping_iteration_count(name, path, cuda):
    """Lockstep stopping: identical iterations_run (batch.py:314-324, test_batch.py:77-90)."""
    g, res = _run_golden(name, cuda, **path)
    assert res.iterations_run == int(g["iterations_run"])
    assert float(res.residuals.max()) <= float(g["tol"])
    _check_loss_and_grads(g, res)


@pytest.mark.parametrize("path", PATHS)
def test_zero_mass_lanes(path, cuda):
    """-inf exactly where mass is 0; backward refuses the lane (test_batch.py:185-198)."""
    skb = _skb()
    g, res = _run_golden("zero_mass", cuda, **path)
    lu = res.log_u.double().cpu().numpy()
    lv = res.log_v.double().cpu().numpy()
    assert np.array_equal(np.isneginf(lu), np.isneginf(g["log_u"]))
    assert np.array_equal(np.isneginf(lv), np.isneginf(g["log_v"]))
    rel = np.abs(res.cost_e0.double().cpu().numpy() - g["cost_e0"]) / g["cost_e0"]
    assert rel.max() <= LOSS_RTOL
    with pytest.raises(skb.ZeroMassGradient) as exc:
        skb.batch_backward(res, torch.ones(3, device=cuda))
    assert exc.value.lane == int(g["zero_mass_lane"])


@pytest.mark.parametrize("dense_grid", [pytest.param(False, id="separable"),
                                        pytest.param(True, id="dense")])
def test_grid_cost_on_the_fly(dense_grid, cuda):
    """BASELINE config 3 subset: 64x64 grid, lambda 1e-3, cost never materialised,
    through the separable nested LSE (default) and the dense on-the-fly tiles."""
    skb = _skb()
    g, res = _run_golden("config3_subset", cuda, cost=skb.GridCost(64, 64),
                         dense_grid=dense_grid)
    assert res.path == ("tiled" if dense_grid else "separable")
    _check_loss_and_grads(g, res)


@pytest.mark.parametrize("nx,ny,tol", [(12, 7, 0.0), (40, 20, 0.0), (33, 70, 1e-4),
                                       (5, 1, 0.0)])
def test_separable_grid_ragged_shapes(nx, ny, tol, cuda):
    """Separable sweeps on ragged grids (partial jx blocks, ny > one m tile,
    1-D grids) against the oracle's dense float64 cost, incl. lockstep stops."""
    skb = _skb()
    from oracle import sinkhorn_oracle as orc

    rng = np.random.default_rng(nx * 100 + ny)
    B, d = 3, nx * ny
    mu = orc.fp32_exact(orc.random_histogram_batch(B, d, rng))
    nu = orc.fp32_exact(orc.random_histogram_batch(B, d, rng))
    lam = 0.05
    c = orc.grid2d_cost(nx, ny)
    ref = orc.batch_forward(mu, nu, c, lam, max_iters=60, tolerance=tol, check_interval=5)
    res = skb.solve(torch.tensor(mu, device=cuda), torch.tensor(nu, device=cuda),
                    skb.GridCost(nx, ny), lam, 60, tol, 5, tiled_only=True)
    assert res.path == "separable"
    assert res.iterations_run == ref.iterations_run
    rel = np.abs(res.cost_e0.double().cpu().numpy() - ref.cost_e0) / ref.cost_e0
    assert rel.max() <= LOSS_RTOL
    lu = res.log_u.double().cpu().numpy()
    assert np.abs(lu - ref.log_u).max() <= 1e-4 * max(1.0, np.abs(ref.log_u).max())
    assert np.all(np.abs(res.residuals.double().cpu().numpy() - ref.residuals) <= 1e-5)


@pytest.mark.parametrize("fused", [pytest.param(True, id="fused"), pytest.param(False, id="lane")])
def test_per_sample_cost(fused, cuda):
    """BASELINE config 4 subset: per-lane U[0,1) costs, d=1024, streamed from HBM,
    through the fused per-sample pass (one read of C_b per iteration) and the
    two-half-sweep lane kernels."""
    g, res = _run_golden("config4_subset", cuda, fused=fused)
    assert res.path == ("fused" if fused else "lane")
    _check_loss_and_grads(g, res)


@pytest.mark.parametrize("B,d1,d2,tol", [(37, 50, 68, 1e-5), (16, 64, 64, 0.0), (5, 300, 1024, 0.0),
                                         (20, 1000, 36, 1e-4), (9, 40, 67, 1e-5),
                                         (7, 33, 1999, 0.0), (3, 100, 1537, 1e-5),
                                         (3, 20, 3001, 1e-5), (5, 12, 5000, 0.0)])
def test_fused_per_sample_ragged_shapes_against_oracle(B, d1, d2, tol, cuda):
    """Per-sample costs through the fused pass: ragged lane groups, d2 not a
    multiple of 64 (zeroed ring tails) nor of 4 (the zero-padded copy), rows
    above 1024 columns, zero-mass bins, lockstep stops."""
    skb = _skb()
    from oracle import sinkhorn_oracle as orc

    rng = np.random.default_rng(B * 11 + d2)
    mu = orc.fp32_exact(orc.random_histogram_batch(B, d1, rng))
    nu = orc.fp32_exact(orc.random_histogram_batch(B, d2, rng))
    mu[1 % B, 3] = 0.0
    mu[1 % B] = orc.fp32_exact(mu[1 % B] / mu[1 % B].sum())
    nu[0, d2 - 1] = 0.0
    nu[0] = orc.fp32_exact(nu[0] / nu[0].sum())
    c = orc.fp32_exact(rng.random((B, d1, d2)) * 2.0)
    lam, iters = 0.1, 40
    refs = [orc.batch_forward(mu[b:b + 1], nu[b:b + 1], c[b], lam, max_iters=iters,
                              tolerance=0.0, check_interval=10) for b in range(B)]
    res = skb.solve(torch.tensor(mu, device=cuda), torch.tensor(nu, device=cuda),
                    torch.tensor(c, dtype=torch.float32, device=cuda), lam, iters, 0.0, 10,
                    tiled_only=True)   # (small lanes would take the single-launch solver)
    assert res.path == "fused"
    want = np.array([r.cost_e0[0] for r in refs])
    rel = np.abs(res.cost_e0.double().cpu().numpy() - want) / want
    assert rel.max() <= LOSS_RTOL
    lu = res.log_u.double().cpu().numpy()
    ref_lu = np.concatenate([r.log_u for r in refs])
    assert np.array_equal(np.isneginf(lu), np.isneginf(ref_lu))
    fu = np.isfinite(ref_lu)
    assert np.abs(lu[fu] - ref_lu[fu]).max() <= 1e-3 * max(1.0, np.abs(ref_lu[fu]).max())
    if tol > 0:   # lockstep stop: the same iteration count as the unfused lane kernels
        a = skb.solve(torch.tensor(mu, device=cuda), torch.tensor(nu, device=cuda),
                      torch.tensor(c, dtype=torch.float32, device=cuda), lam, 400, tol, 10,
                      tiled_only=True)
        b_ = skb.solve(torch.tensor(mu, device=cuda), torch.tensor(nu, device=cuda),
                       torch.tensor(c, dtype=torch.float32, device=cuda), lam, 400, tol, 10,
                       fused=False, tiled_only=True)
        assert a.path == "fused" and b_.path == "lane"
        assert a.iterations_run == b_.iterations_run


def test_half_sweep_matches_fused_log_reduction(cuda):
    """fused_log_reduction (batch.py:208-230) incl. a -inf target (test_reduction.py:207-216)."""
    skb = _skb()
    g = load_golden("half_sweep")
    with np.errstate(divide="ignore"):
        log_nu = np.log(g["nu"].astype(np.float64))
    out = skb.fused_log_reduction(torch.tensor(g["log_u"], device=cuda),
                                  torch.tensor(g["c"], device=cuda), float(g["lam"]),
                                  torch.tensor(log_nu, dtype=torch.float32, device=cuda))
    got = out.double().cpu().numpy()
    want = g["out"]
    assert np.array_equal(np.isneginf(got), np.isneginf(want))
    fin = np.isfinite(want)
    assert np.abs(got[fin] - want[fin]).max() <= 2e-5 * max(1.0, np.abs(want[fin]).max())


def test_partial_reduction_merges_like_accumulator(cuda):
    """Row-sharded building block: partial (max, sum) over row blocks merged with
    OnlineLseAccumulator.merge equals the full reduction (batch.py:116-130)."""
    skb = _skb()
    g = load_golden("half_sweep")
    lu = torch.tensor(g["log_u"], device=cuda)
    c = torch.tensor(g["c"], device=cuda)
    lam = float(g["lam"])
    m1, s1 = skb.partial_log_reduction(lu[:, :17], c[:17], lam)
    m2, s2 = skb.partial_log_reduction(lu[:, 17:], c[17:], lam)
    m = torch.maximum(m1, m2)
    s = s1 * torch.exp2(m1 - m) + s2 * torch.exp2(m2 - m)
    lse = (m + torch.log2(s)) * math.log(2.0)
    mf, sf = skb.partial_log_reduction(lu, c, lam)
    full = (mf + torch.log2(sf)) * math.log(2.0)
    assert torch.allclose(lse, full, rtol=0, atol=2e-5)


def test_autograd_node_matches_reference_gradients(cuda):
    """sinkhorn_loss as a torch.autograd.Function (loss.ts:59-131)."""
    skb = _skb()
    g = load_golden("config1")
    mu = torch.tensor(g["mu"], device=cuda, requires_grad=True)
    nu = torch.tensor(g["nu"], device=cuda, requires_grad=True)
    c = torch.tensor(g["cost"], device=cuda)
    loss = skb.sinkhorn_loss(mu, nu, c, float(g["lam"]), max_iters=int(g["max_iters"]),
                             tolerance=0.0)
    assert loss.shape == (mu.shape[0],)
    loss.backward(torch.tensor(g["upstream"], dtype=torch.float32, device=cuda))
    assert np.abs(mu.grad.double().cpu().numpy() - g["grad_mu"]).max() <= GRAD_ATOL
    assert np.abs(nu.grad.double().cpu().numpy() - g["grad_nu"]).max() <= GRAD_ATOL
    # each lane's gradient is mean-zero (loss.test.ts:124-151)
    assert torch.allclose(mu.grad.sum(dim=1), torch.zeros(mu.shape[0], device=cuda), atol=1e-5)


@pytest.mark.parametrize("name", ["config2_subset", "stability", "zero_mass"])
def test_estimate_mode_matches_exact_two_pass(name, cuda):
    """The one-pass chunks seeded by the previous lse (estimate mode) and the
    exact two-pass chunks agree to fp32 rounding."""
    skb = _skb()
    g = load_golden(name)
    c = torch.tensor(golden_cost(g), dtype=torch.float32, device=cuda)
    args = (torch.tensor(g["mu"], device=cuda), torch.tensor(g["nu"], device=cuda), c,
            float(g["lam"]), int(g["max_iters"]), float(g["tol"]), int(g["check_interval"]))
    fast = skb.solve(*args, tiled_only=True, fused=False, gemm=False)
    exact = skb.solve(*args, exact_max=True, tiled_only=True, fused=False, gemm=False)
    assert fast.iterations_run == exact.iterations_run
    rel = (fast.cost_e0.double() - exact.cost_e0.double()).abs() / exact.cost_e0.double().abs()
    assert float(rel.max()) <= 2e-6
    fin = torch.isfinite(exact.log_u)
    assert torch.equal(fin, torch.isfinite(fast.log_u))
    scale = max(1.0, float(exact.log_u[fin].abs().max()))
    assert float((fast.log_u[fin] - exact.log_u[fin]).abs().max()) <= 2e-5 * scale


@pytest.mark.parametrize("name", ["config2_subset", "config5_pin4096"])
def test_polynomial_exp2_share_matches_mufu_only(name, cuda):
    """Part of the exponentials run as an FMA-pipe polynomial (ex2_poly2); the
    result must match the all-MUFU path to fp32 rounding."""
    skb = _skb()
    g = load_golden(name)
    c = torch.tensor(golden_cost(g), dtype=torch.float32, device=cuda)
    args = (torch.tensor(g["mu"], device=cuda), torch.tensor(g["nu"], device=cuda), c,
            float(g["lam"]), int(g["max_iters"]), float(g["tol"]), int(g["check_interval"]))
    poly = skb.solve(*args)
    mufu = skb.solve(*args, mufu_only=True)
    rel = (poly.cost_e0.double() - mufu.cost_e0.double()).abs() / mufu.cost_e0.double().abs()
    assert float(rel.max()) <= 2e-6
    _check_loss_and_grads(g, poly)


@pytest.mark.parametrize("name", ["config1", "config1_tol", "lockstep", "zero_mass"])
def test_persistent_loop_matches_reference(name, cuda):
    """Opt-in cooperative whole-loop kernel: same results and iteration counts,
    with the stopping test decided on the device."""
    skb = _skb()
    g = load_golden(name)
    c = torch.tensor(golden_cost(g), dtype=torch.float32, device=cuda)
    res = skb.solve(torch.tensor(g["mu"], device=cuda), torch.tensor(g["nu"], device=cuda), c,
                    float(g["lam"]), int(g["max_iters"]), float(g["tol"]),
                    int(g["check_interval"]), persistent=True, tiled_only=True, fused=False)
    ref = skb.solve(torch.tensor(g["mu"], device=cuda), torch.tensor(g["nu"], device=cuda), c,
                    float(g["lam"]), int(g["max_iters"]), float(g["tol"]),
                    int(g["check_interval"]))
    assert res.iterations_run == int(g["iterations_run"]) == ref.iterations_run
    rel = np.abs(res.cost_e0.double().cpu().numpy() - g["cost_e0"]) / g["cost_e0"]
    assert rel.max() <= LOSS_RTOL
    assert torch.equal(torch.isneginf(res.log_u), torch.isneginf(ref.log_u))


def test_small_problem_runs_in_one_solver_launch(cuda):
    """Config 1 shape: the whole lockstep loop is one kernel launch (plus setup)."""
    skb = _skb()
    from paper_1907_01729_b200 import _lib

    lib = _lib.load()
    g = load_golden("config1")
    args = (torch.tensor(g["mu"], device=cuda), torch.tensor(g["nu"], device=cuda),
            torch.tensor(g["cost"], dtype=torch.float32, device=cuda), float(g["lam"]),
            int(g["max_iters"]), 0.0, 10)
    n0 = lib.sinkhorn_launch_count_v1()
    skb.solve(*args)
    small = lib.sinkhorn_launch_count_v1() - n0
    n0 = lib.sinkhorn_launch_count_v1()
    skb.solve(*args, tiled_only=True, fused=False)
    tiled = lib.sinkhorn_launch_count_v1() - n0
    assert small <= 8 < 200 <= tiled, (small, tiled)


@pytest.mark.parametrize("kind", ["shared", "grid"])
def test_small_solver_many_lanes_per_cta_lockstep(kind, cuda):
    """Several lanes per CTA and a cross-CTA lockstep stop, against the oracle."""
    skb = _skb()
    from oracle import sinkhorn_oracle as orc

    rng = np.random.default_rng(7)
    if kind == "shared":
        B, d1, d2 = 700, 40, 56
        c = orc.fp32_exact(rng.random((d1, d2)))
        cost = torch.tensor(c, dtype=torch.float32, device=cuda)
        lam = 0.2
    else:
        B, d1, d2 = 400, 64, 64
        c = orc.grid2d_cost(8, 8)
        cost = skb.GridCost(8, 8)
        lam = 0.5
    mu = orc.fp32_exact(orc.random_histogram_batch(B, d1, rng))
    nu = orc.fp32_exact(orc.random_histogram_batch(B, d2, rng))
    ref = orc.batch_forward(mu, nu, c, lam, max_iters=400, tolerance=1e-5, check_interval=5)
    res = skb.solve(torch.tensor(mu, device=cuda), torch.tensor(nu, device=cuda), cost, lam,
                    400, 1e-5, 5)
    assert res.iterations_run == ref.iterations_run
    rel = np.abs(res.cost_e0.double().cpu().numpy() - ref.cost_e0) / ref.cost_e0
    assert rel.max() <= LOSS_RTOL
    tiled = skb.solve(torch.tensor(mu, device=cuda), torch.tensor(nu, device=cuda), cost, lam,
                      400, 1e-5, 5, tiled_only=True)
    assert tiled.iterations_run == res.iterations_run


def test_fused_pass_is_the_shared_cost_path_and_matches_tiled(cuda):
    """Shared costs with d <= 1024 run one fused row->column pass per
    iteration (sweep_fused.cuh); it agrees with the two-half-sweep tiled path
    and with the reference."""
    skb = _skb()
    g = load_golden("config2_subset")
    c = torch.tensor(golden_cost(g), dtype=torch.float32, device=cuda)
    args = (torch.tensor(g["mu"], device=cuda), torch.tensor(g["nu"], device=cuda), c,
            float(g["lam"]), int(g["max_iters"]), float(g["tol"]), int(g["check_interval"]))
    fused = skb.solve(*args, tiled_only=True)
    tiled = skb.solve(*args, tiled_only=True, fused=False, gemm=False)
    assert fused.path == "fused" and tiled.path == "tiled"
    _check_loss_and_grads(g, fused)
    rel = (fused.cost_e0.double() - tiled.cost_e0.double()).abs() / tiled.cost_e0.double()
    assert float(rel.max()) <= 2e-6
    fin = torch.isfinite(tiled.log_v)
    assert torch.equal(fin, torch.isfinite(fused.log_v))
    scale = max(1.0, float(tiled.log_v[fin].abs().max()))
    assert float((fused.log_v[fin] - tiled.log_v[fin]).abs().max()) <= 2e-5 * scale


@pytest.mark.parametrize("B,d1,d2,tol", [(37, 50, 70, 1e-5), (16, 64, 64, 0.0), (130, 130, 97, 0.0),
                                         (300, 200, 1000, 0.0), (5, 1000, 33, 1e-4)])
def test_fused_pass_ragged_shapes_against_oracle(B, d1, d2, tol, cuda):
    """Ragged lane groups (B not a multiple of 16), rectangular costs, padded
    rows and lockstep stops through the fused passes."""
    skb = _skb()
    from oracle import sinkhorn_oracle as orc

    rng = np.random.default_rng(B * 7 + d1)
    mu = orc.fp32_exact(orc.random_histogram_batch(B, d1, rng))
    nu = orc.fp32_exact(orc.random_histogram_batch(B, d2, rng))
    mu[1 % B, 3] = 0.0           # a zero-mass bin on each side
    mu[1 % B] = orc.fp32_exact(mu[1 % B] / mu[1 % B].sum())
    nu[0, d2 - 1] = 0.0
    nu[0] = orc.fp32_exact(nu[0] / nu[0].sum())
    c = orc.fp32_exact(rng.random((d1, d2)) * 2.0)
    lam, iters = 0.1, 60
    ref = orc.batch_forward(mu, nu, c, lam, max_iters=iters, tolerance=tol, check_interval=10)
    res = skb.solve(torch.tensor(mu, device=cuda), torch.tensor(nu, device=cuda),
                    torch.tensor(c, dtype=torch.float32, device=cuda), lam, iters, tol, 10,
                    tiled_only=True)
    assert res.path == "fused"
    assert res.iterations_run == ref.iterations_run
    rel = np.abs(res.cost_e0.double().cpu().numpy() - ref.cost_e0) / ref.cost_e0
    assert rel.max() <= LOSS_RTOL
    lu, lv = res.log_u.double().cpu().numpy(), res.log_v.double().cpu().numpy()
    assert np.array_equal(np.isneginf(lu), np.isneginf(ref.log_u))
    assert np.array_equal(np.isneginf(lv), np.isneginf(ref.log_v))
    fu = np.isfinite(ref.log_u)
    assert np.abs(lu[fu] - ref.log_u[fu]).max() <= 1e-3 * max(1.0, np.abs(ref.log_u[fu]).max())
    res_r = res.residuals.double().cpu().numpy()
    assert np.allclose(res_r, ref.residuals, atol=2e-6), (res_r[:4], ref.residuals[:4])


@pytest.mark.parametrize("kind", ["shared", "per_sample"])
def test_repeated_fused_solve_replays_the_same_result(kind, cuda):
    """Tolerance-0 fused solves: the first runs eagerly, the second captures the
    iteration loop as a CUDA graph and replays it, the third replays it again.
    All three give bitwise the same potentials and costs."""
    skb = _skb()
    from oracle import sinkhorn_oracle as orc

    rng = np.random.default_rng(5)
    B, d = 40, 96
    mu = torch.tensor(orc.fp32_exact(orc.random_histogram_batch(B, d, rng)), device=cuda)
    nu = torch.tensor(orc.fp32_exact(orc.random_histogram_batch(B, d, rng)), device=cuda)
    shape = (d, d) if kind == "shared" else (B, d, d)
    cost = torch.tensor(orc.fp32_exact(rng.random(shape)), dtype=torch.float32, device=cuda)
    runs = [skb.solve(mu, nu, cost, 0.1, 30, 0.0, 10, tiled_only=True) for _ in range(3)]
    assert all(r.path == "fused" for r in runs)
    for r in runs[1:]:
        assert torch.equal(r.cost_e0, runs[0].cost_e0)
        assert torch.equal(r.log_u, runs[0].log_u) and torch.equal(r.log_v, runs[0].log_v)
        assert r.iterations_run == runs[0].iterations_run == 30
    # the input changes between replays: the graph reads the current buffers
    mu2 = torch.tensor(orc.fp32_exact(orc.random_histogram_batch(B, d, rng)), device=cuda)
    a = skb.solve(mu2, nu, cost, 0.1, 30, 0.0, 10, tiled_only=True)
    ref = skb.solve(mu2, nu, cost, 0.1, 30, 0.0, 10, tiled_only=True, fused=False)
    rel = ((a.cost_e0 - ref.cost_e0).abs() / ref.cost_e0).max().item()
    assert rel <= 2e-6


# ---------------------------------------------------------------------------
# float64 parity mode

@pytest.mark.parametrize("name", ["closed_form_2x2", "config1", "config1_tol", "lockstep",
                                  "zero_mass", "rect_37x53", "stability", "config4_subset"])
def test_fp64_mode_matches_reference_to_float64_precision(name, cuda):
    """solve(fp64=True) runs the reference's float64 iteration on the device:
    costs to 1e-9 relative, potentials to 1e-8 (relative to their scale),
    identical iteration counts and -inf patterns."""
    skb = _skb()
    g = load_golden(name)
    c = torch.tensor(golden_cost(g), dtype=torch.float64, device=cuda)
    res = skb.solve(torch.tensor(g["mu"], device=cuda), torch.tensor(g["nu"], device=cuda), c,
                    float(g["lam"]), int(g["max_iters"]), float(g["tol"]),
                    int(g["check_interval"]), fp64=True)
    assert res.path == "fp64" and res.cost_e0.dtype == torch.float64
    assert res.iterations_run == int(g["iterations_run"])
    rel = np.abs(res.cost_e0.cpu().numpy() - g["cost_e0"]) / np.abs(g["cost_e0"])
    assert rel.max() <= 1e-9, rel.max()
    for got, want in ((res.log_u, g["log_u"]), (res.log_v, g["log_v"])):
        got = got.cpu().numpy()
        assert np.array_equal(np.isneginf(got), np.isneginf(want))
        fin = np.isfinite(want)
        scale = max(1.0, np.abs(want[fin]).max())
        assert np.abs(got[fin] - want[fin]).max() <= 1e-8 * scale
    assert np.abs(res.residuals.cpu().numpy() - g["residuals"]).max() <= 1e-10


def test_fp64_mode_reaches_the_reference_default_tolerance(cuda):
    """tolerance 1e-9 (core.py:85): the fp64 mode stops at the reference's
    iteration with residuals <= 1e-9, and its backward matches in float64."""
    skb = _skb()
    from oracle import sinkhorn_oracle as orc

    rng = np.random.default_rng(21)
    B, d1, d2, lam = 6, 30, 41, 0.2
    mu = orc.random_histogram_batch(B, d1, rng)
    nu = orc.random_histogram_batch(B, d2, rng)
    c = rng.random((d1, d2))
    ref = orc.batch_forward(mu, nu, c, lam, max_iters=2000, tolerance=1e-9, check_interval=10)
    res = skb.solve(torch.tensor(mu, device=cuda), torch.tensor(nu, device=cuda),
                    torch.tensor(c, device=cuda), lam, 2000, 1e-9, 10, fp64=True)
    assert res.iterations_run == ref.iterations_run < 2000
    assert float(res.residuals.max()) <= 1e-9
    assert np.abs(res.cost_e0.cpu().numpy() - ref.cost_e0).max() <= 1e-12
    up = rng.normal(size=B)
    gm_ref, gn_ref = orc.batch_backward(ref.log_u, ref.log_v, lam, up)
    gm, gn = skb.potentials_backward(res.log_u, res.log_v, lam, torch.tensor(up, device=cuda))
    assert gm.dtype == torch.float64
    assert np.abs(gm.cpu().numpy() - gm_ref).max() <= 1e-10
    assert np.abs(gn.cpu().numpy() - gn_ref).max() <= 1e-10


@pytest.mark.parametrize("name", ["config2_subset", "config5_pin4096", "config5_pin16384"])
def test_gemm_path_matches_reference_and_tiled(name, cuda):
    """Large shared costs run as two fp32 GEMMs per iteration (sweep_gemm.cuh):
    parity with the reference and with the log-domain tiled half-sweeps."""
    skb = _skb()
    g = load_golden(name)
    c = torch.tensor(golden_cost(g), dtype=torch.float32, device=cuda)
    args = (torch.tensor(g["mu"], device=cuda), torch.tensor(g["nu"], device=cuda), c,
            float(g["lam"]), int(g["max_iters"]), float(g["tol"]), int(g["check_interval"]))
    res = skb.solve(*args, tiled_only=True, gemm=True)
    assert res.path == "gemm"
    _check_loss_and_grads(g, res)
    tiled = skb.solve(*args, tiled_only=True, fused=False, gemm=False)
    rel = ((res.cost_e0.double() - tiled.cost_e0.double()).abs() / tiled.cost_e0.double()).max()
    assert float(rel) <= 2e-6


def test_gemm_path_underflowing_rows_fall_back_exactly(cuda):
    """c/lambda >= 5000 (test_acceptance.py:175-201): K = 2^A2 underflows, so
    rows fall back to the log domain (or the solve reruns exactly); the result
    still matches the reference."""
    skb = _skb()
    g = load_golden("stability")
    c = torch.tensor(golden_cost(g), dtype=torch.float32, device=cuda)
    res = skb.solve(torch.tensor(g["mu"], device=cuda), torch.tensor(g["nu"], device=cuda), c,
                    float(g["lam"]), int(g["max_iters"]), float(g["tol"]),
                    int(g["check_interval"]), tiled_only=True, gemm=True)
    _check_loss_and_grads(g, res)


@pytest.mark.parametrize("d1,d2", [(190, 190), (257, 190), (190, 257), (255, 131)])
def test_tiled_sweeps_with_ragged_extents(d1, d2, cuda):
    """The stream-K tiled half-sweeps (also the exact-rerun path of every shared
    cost) with output extents that are not multiples of 4 or 64: the last tile
    is shifted to end at the extent on a float4 boundary (an unaligned shift
    faulted in round 1).  Against the float64 oracle."""
    from oracle import sinkhorn_oracle as orc

    skb = pytest.importorskip("paper_1907_01729_b200")
    rng = np.random.default_rng(d1 + d2)
    mu = orc.fp32_exact(orc.random_histogram_batch(5, d1, rng))
    nu = orc.fp32_exact(orc.random_histogram_batch(5, d2, rng))
    c = orc.fp32_exact(rng.random((d1, d2)))
    ref = orc.batch_forward(mu, nu, c, 0.1, 40, 0.0, workers=2)
    res = skb.solve(torch.tensor(mu, device=cuda), torch.tensor(nu, device=cuda),
                    torch.tensor(c, dtype=torch.float32, device=cuda), 0.1, 40, 0.0,
                    tiled_only=True, fused=False, gemm=False)
    assert res.path == "tiled"
    rel = np.abs(res.cost_e0.double().cpu().numpy() - ref.cost_e0) / ref.cost_e0
    assert rel.max() <= LOSS_RTOL
    assert np.abs(res.log_v.double().cpu().numpy() - ref.log_v).max() <= 1e-4


@pytest.mark.parametrize("B,d1,d2", [(70, 1300, 2100), (130, 2049, 1031)])
def test_gemm_path_ragged_tiles_match_tiled(B, d1, d2, cuda):
    """The tcgen05 contractions with ragged M tiles (d not a multiple of 128),
    a ragged reduction chunk (not a multiple of 64) and more than one 64-lane
    N tile (the last one partial): equal to the log-domain tiled half-sweeps."""
    skb = _skb()
    gen = torch.Generator(device=cuda)
    gen.manual_seed(B)

    def hist(d):
        m = torch.rand(B, d, generator=gen, device=cuda, dtype=torch.float64) + 0.5
        return (m / m.sum(1, keepdim=True)).float()
    mu, nu = hist(d1), hist(d2)
    i = torch.arange(d1, device=cuda, dtype=torch.float64)[:, None] / (d1 - 1)
    j = torch.arange(d2, device=cuda, dtype=torch.float64)[None, :] / (d2 - 1)
    c = ((i - j) ** 2 + 0.1 * torch.rand(d1, d2, generator=gen, device=cuda,
                                          dtype=torch.float64)).float()
    args = (mu, nu, c, 0.05, 40, 0.0)
    res = skb.solve(*args, tiled_only=True, gemm=True)
    assert res.path == "gemm"
    tiled = skb.solve(*args, tiled_only=True, fused=False, gemm=False)
    rel = ((res.cost_e0.double() - tiled.cost_e0.double()).abs() / tiled.cost_e0.double()).max()
    assert float(rel) <= 2e-6
    assert float((res.log_u - tiled.log_u).abs().max()) <= 1e-4
    assert float((res.log_v - tiled.log_v).abs().max()) <= 1e-4
    gm, gn = skb.potentials_backward(res.log_u, res.log_v, 0.05, torch.ones(B, device=cuda))
    tm, tn = skb.potentials_backward(tiled.log_u, tiled.log_v, 0.05, torch.ones(B, device=cuda))
    assert float((gm - tm).abs().max()) <= GRAD_ATOL
    assert float((gn - tn).abs().max()) <= GRAD_ATOL


@pytest.mark.parametrize("B,d1,d2", [(8, 256, 256), (4, 300, 210), (6, 181, 333)])
def test_small_solver_clusters_match_tiled(B, d1, d2, cuda):
    """Problems large enough for the single-launch solver to spread each lane
    over a thread-block cluster (slices exchanged through distributed shared
    memory, ragged slices when C does not divide d): equal to the tiled
    half-sweeps, including a lockstep tolerance stop."""
    skb = _skb()
    gen = torch.Generator(device=cuda)
    gen.manual_seed(d1 + d2)

    def hist(d):
        m = torch.rand(B, d, generator=gen, device=cuda, dtype=torch.float64) + 0.5
        return (m / m.sum(1, keepdim=True)).float()
    mu, nu = hist(d1), hist(d2)
    c = torch.rand(d1, d2, generator=gen, device=cuda)
    for iters, tol in ((60, 0.0), (400, 1e-5)):
        res = skb.solve(mu, nu, c, 0.05, iters, tol)
        assert res.path == "small"
        ref = skb.solve(mu, nu, c, 0.05, iters, tol, tiled_only=True, fused=False, gemm=False)
        assert res.iterations_run == ref.iterations_run
        rel = ((res.cost_e0.double() - ref.cost_e0.double()).abs() / ref.cost_e0.double()).max()
        assert float(rel) <= 2e-6
        assert float((res.log_u - ref.log_u).abs().max()) <= 1e-4
        assert float((res.log_v - ref.log_v).abs().max()) <= 1e-4


@pytest.mark.parametrize("kind,d,kw", [("shared", 300, {"tiled_only": True}),
                                       ("shared", 1100, {"tiled_only": True, "gemm": True}),
                                       ("per_sample", 256, {}),
                                       ("per_sample", 3000, {})])
def test_graph_replay_equals_eager(kind, d, kw, cuda):
    """Tolerance-0 solves repeated on the same workspace and cost are captured
    as one CUDA graph on the second call and replayed from the third (fused
    passes and the GEMM iteration): every call returns the same numbers."""
    skb = _skb()
    gen = torch.Generator(device=cuda)
    gen.manual_seed(d)
    B = 6

    def hist():
        m = torch.rand(B, d, generator=gen, device=cuda, dtype=torch.float64) + 0.5
        return (m / m.sum(1, keepdim=True)).float()
    mu, nu = hist(), hist()
    if kind == "shared":
        c = torch.rand(d, d, generator=gen, device=cuda)
    else:
        c = torch.rand(B, d, d, generator=gen, device=cuda)
    runs = [skb.solve(mu, nu, c, 0.05, 30, 0.0, **kw) for _ in range(4)]
    for r in runs[1:]:
        assert r.path == runs[0].path
        assert torch.equal(r.cost_e0, runs[0].cost_e0)
        assert torch.equal(r.log_u, runs[0].log_u)
        assert torch.equal(r.log_v, runs[0].log_v)



@pytest.mark.parametrize("B,d1,d2,tol", [(37, 50, 68, 0.0), (300, 16, 20, 1e-5), (5, 64, 64, 0.0),
                                         (2000, 7, 9, 0.0)])
def test_small_solver_per_sample_against_oracle(B, d1, d2, tol, cuda):
    """Per-sample costs of <= 64 x 64 cells per lane take the single-launch
    solver (each lane's cost staged once, validated there): against the
    reference lane by lane, zero-mass bins and lockstep stops included."""
    skb = _skb()
    from oracle import sinkhorn_oracle as orc

    rng = np.random.default_rng(B + d1 * 3 + d2)
    mu = orc.fp32_exact(orc.random_histogram_batch(B, d1, rng))
    nu = orc.fp32_exact(orc.random_histogram_batch(B, d2, rng))
    mu[1 % B, 3 % d1] = 0.0
    mu[1 % B] = orc.fp32_exact(mu[1 % B] / mu[1 % B].sum())
    c = orc.fp32_exact(rng.random((B, d1, d2)) * 2.0)
    lam, iters = 0.1, 400 if tol > 0 else 40
    t = lambda a: torch.tensor(a, dtype=torch.float32, device=cuda)   # noqa: E731
    res = skb.solve(t(mu), t(nu), t(c), lam, iters, tol, 10)
    assert res.path == "small"
    ref = orc.per_sample_forward(mu, nu, c, lam, iters, tol, 10)
    assert res.iterations_run == ref.iterations_run
    rel = np.abs(res.cost_e0.double().cpu().numpy() - ref.cost_e0) / ref.cost_e0
    assert rel.max() <= LOSS_RTOL
    fused = skb.solve(t(mu), t(nu), t(c), lam, iters, tol, 10, tiled_only=True)
    assert fused.iterations_run == res.iterations_run
    bad = c.copy()
    bad[B - 1, d1 - 1, d2 - 1] = -1.0
    with pytest.raises(skb.InvalidCost):
        skb.solve(t(mu), t(nu), t(bad), lam, iters, tol, 10)
