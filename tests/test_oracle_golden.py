"""Pin the CPU oracle (oracle/sinkhorn_oracle.py) to the reference.

The fixtures in tests/golden were produced by running the reference package
itself (oracle/gen_golden.py); the oracle must reproduce them to the
reference's own tolerances (test_batch.py:46-63 uses 1e-12), plus the
reference's closed-form known answers.  Runs on CPU.
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np
import pytest

from conftest import golden_cost, load_golden
from oracle import sinkhorn_oracle as orc


def _forward(g, cost=None, workers=1):
    c = golden_cost(g) if cost is None else cost
    return orc.batch_forward(g["mu"].astype(np.float64), g["nu"].astype(np.float64), c,
                             float(g["lam"]), int(g["max_iters"]), float(g["tol"]),
                             int(g["check_interval"]), workers=workers)


@pytest.mark.parametrize("name", ["closed_form_2x2", "config1", "config1_tol", "rect_37x53",
                                  "zero_mass", "lockstep", "stability"])
def test_oracle_reproduces_reference_batch_forward(name):
    g = load_golden(name)
    r = _forward(g)
    assert r.iterations_run == int(g["iterations_run"])
    np.testing.assert_allclose(r.cost_e0, g["cost_e0"], rtol=1e-12, atol=0)
    np.testing.assert_array_equal(np.isneginf(r.log_u), np.isneginf(g["log_u"]))
    fin = np.isfinite(g["log_u"])
    assert np.abs(r.log_u[fin] - g["log_u"][fin]).max() <= 1e-9
    np.testing.assert_allclose(r.residuals, g["residuals"], rtol=1e-6, atol=1e-15)
    if int(g["zero_mass_lane"]) < 0:
        gm, gn = orc.batch_backward(r.log_u, r.log_v, r.lam, g["upstream"])
        assert np.abs(gm - g["grad_mu"]).max() <= 1e-11
        assert np.abs(gn - g["grad_nu"]).max() <= 1e-11
    else:
        with pytest.raises(orc.OracleError) as exc:
            orc.batch_backward(r.log_u, r.log_v, r.lam, g["upstream"])
        assert exc.value.lane == int(g["zero_mass_lane"])


def test_closed_form_known_answer():
    """conftest.py:9-24: symmetric 2x2 at lambda=1 gives e^-1/(1+e^-1)."""
    g = load_golden("closed_form_2x2")
    r = _forward(g)
    k = math.exp(-1.0)
    assert abs(r.cost_e0[0] - k / (1 + k)) <= 1e-6
    assert abs(g["cost_e0"][0] - 0.2689414213699951) <= 1e-6


@pytest.mark.slow
def test_oracle_config2_subset():
    g = load_golden("config2_subset")
    r = _forward(g)
    np.testing.assert_allclose(r.cost_e0, g["cost_e0"], rtol=1e-12)
    assert np.abs(r.log_v - g["log_v"]).max() <= 1e-9


def test_oracle_per_sample_lane():
    """Per-sample extension: lane-by-lane reference algorithm (config 4 subset, 1 lane)."""
    g = load_golden("config4_subset")
    cost = orc.per_sample_cost(1, 0, 1024, 1024).astype(np.float64)
    r = orc.batch_forward(g["mu"][:1].astype(np.float64), g["nu"][:1].astype(np.float64), cost,
                          float(g["lam"]), 4, 0.0, workers=1)
    # 4 iterations only (speed); compare against a dense restatement of run_sinkhorn
    d = orc.dense_forward(g["mu"][0].astype(np.float64), g["nu"][0].astype(np.float64), cost,
                          float(g["lam"]), 4)
    np.testing.assert_allclose(r.cost_e0[0], d.cost_e0[0], rtol=1e-12)
    full = orc.dense_forward(g["mu"][0].astype(np.float64), g["nu"][0].astype(np.float64), cost,
                             float(g["lam"]), int(g["max_iters"]))
    np.testing.assert_allclose(full.cost_e0[0], g["cost_e0"][0], rtol=1e-12)
    assert np.abs(full.log_u[0] - g["log_u"][0]).max() <= 1e-9


def test_per_sample_cost_digest_matches_fixture():
    import hashlib

    g = load_golden("config4_subset")
    digests = str(g["cost_digest"]).split(",")
    for b in range(2):
        c = orc.per_sample_cost(1, b, 1024, 1024).astype(np.float64)
        assert hashlib.sha256(c.tobytes()).hexdigest()[:16] == digests[b]


def test_grid_cost_digest_matches_fixture():
    import hashlib

    g = load_golden("config3_subset")
    c = orc.grid2d_cost(64, 64)
    assert hashlib.sha256(c.tobytes()).hexdigest()[:16] == str(g["cost_digest"]).split(",")[0]


@pytest.mark.slow
def test_oracle_config3_lane_dense():
    """64x64 grid, lambda 1e-3, 100 iterations: dense restatement of run_sinkhorn."""
    g = load_golden("config3_subset")
    r = orc.dense_forward(g["mu"][0].astype(np.float64), g["nu"][0].astype(np.float64),
                          orc.grid2d_cost(64, 64), float(g["lam"]), int(g["max_iters"]))
    np.testing.assert_allclose(r.cost_e0[0], g["cost_e0"][0], rtol=1e-10)
    assert np.abs(r.log_u[0] - g["log_u"][0]).max() <= 1e-7


def test_half_sweep_and_transposed_roles():
    g = load_golden("half_sweep")
    with np.errstate(divide="ignore"):
        log_nu = np.log(g["nu"].astype(np.float64))
    out = orc.fused_log_reduction(g["log_u"].astype(np.float64), g["c"].astype(np.float64),
                                  float(g["lam"]), log_nu)
    assert np.array_equal(np.isneginf(out), np.isneginf(g["out"]))
    fin = np.isfinite(g["out"])
    assert np.abs(out[fin] - g["out"][fin]).max() <= 1e-13


@pytest.mark.parametrize("workers", [2, 8])
def test_worker_count_does_not_change_results(workers):
    """test_reduction.py:195-204 / test_acceptance.py:98-113: partition determinism."""
    rng = np.random.default_rng(8)
    B, d1, d2 = 4, 33, 29
    c = rng.uniform(0.0, 1.0, (d1, d2))
    log_u = rng.normal(size=(B, d1))
    log_nu = np.log(orc.random_histogram_batch(B, d2, rng))
    base = orc.fused_log_reduction(log_u, c, 0.5, log_nu, workers=1)
    got = orc.fused_log_reduction(log_u, c, 0.5, log_nu, workers=workers)
    assert np.abs(got - base).max() <= 1e-13


def test_lse_monoid_against_reference_splits():
    """test_reduction.py:351-358: exhaustive split points, merge law <= 1e-13."""
    g = load_golden("lse_monoid")
    xs = g["xs"]
    for k in range(65):
        a = orc.lse_empty(())
        for x in xs[:k]:
            a = orc.lse_consume(a, np.float64(x))
        b = orc.lse_empty(())
        for x in xs[k:]:
            b = orc.lse_consume(b, np.float64(x))
        got = float(orc.lse_finalise(orc.lse_merge(a, b)))
        assert abs(got - g["splits"][k]) <= 1e-13


def test_lse_edge_cases():
    """test_reduction.py:289-304."""
    assert orc.lse_of([0.0, 0.0]) == pytest.approx(math.log(2.0), rel=1e-15)
    assert orc.lse_of([1000.0, 1000.0]) == pytest.approx(1000.0 + math.log(2.0), rel=1e-15)
    assert orc.lse_of([-np.inf, 0.0]) == 0.0
    assert orc.lse_of([]) == -np.inf
    assert orc.lse_of([-np.inf, -np.inf]) == -np.inf


def test_ffi_status_semantics():
    """ffi.ts:80-191 restated: statuses 0/10/11/12/13 and the B=0 no-op."""
    c2 = np.array([[0.0, 1.0], [1.0, 0.0]])
    st, *_ = orc.forward_v1(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros((3, 3)), 0.1, 10, 0)
    assert st == orc.STATUS_OK
    st, *_ = orc.forward_v1([[0.5, 0.5]], [[0.3, 0.3, 0.4]], c2, 0.1, 10, 0)
    assert st == orc.STATUS_SHAPE_MISMATCH
    st, *_ = orc.forward_v1([[0.5, 0.4]], [[0.5, 0.5]], c2, 0.1, 10, 0)
    assert st == orc.STATUS_INVALID_HISTOGRAM
    st, cost, lu, lv = orc.forward_v1([[0.0, 1.0]], [[0.5, 0.5]], c2, 0.5, 100, 0)
    assert st == orc.STATUS_OK and lu[0, 0] == -np.inf
    st, *_ = orc.backward_v1(lu, lv, 0.5, [1.0])
    assert st == orc.STATUS_ZERO_MASS_LANE
    st, *_ = orc.backward_v1(np.zeros((2, 2)), np.zeros((2, 2)), 0.5, np.zeros(3))
    assert st == orc.STATUS_SHAPE_MISMATCH
    st, *_ = orc.forward_v1([[0.5, 0.5]], [[0.5, 0.5]], c2, -1.0, 10, 0)
    assert st == orc.STATUS_INVALID_CONFIG
    st, *_ = orc.forward_v1([[0.5, 0.5]], [[0.5, 0.5]], -c2, 0.5, 10, 0)
    assert st == orc.STATUS_INVALID_COST


def test_nan_state_instance_raises_in_reference_and_oracle():
    """The status-12 instance of tests/test_gpu_batch_props.py: c = 1e30,
    lambda = 1e-300 makes A = -c/lambda = -inf, the state turns NaN and the
    reference raises NaNProduced (batch.py:326-327); the oracle agrees."""
    import warnings

    from oracle import sinkhorn_oracle as orc

    rng = np.random.default_rng(6)
    mu = orc.random_histogram_batch(3, 64, rng)
    nu = orc.random_histogram_batch(3, 64, rng)
    c = np.full((64, 64), 1.0e30)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        with pytest.raises(orc.OracleError, match="NaNProduced"):
            orc.batch_forward(mu, nu, c, 1e-300, 20, 0.0)
        ref_dir = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                               "baseline", "_ref")
        if os.path.isfile(os.path.join(ref_dir, "sinkloss", "batch.py")):
            sys.path.insert(0, ref_dir)
            import sinkloss as sk

            with pytest.raises(sk.NaNProduced):
                sk.batch_forward(sk.HistogramBatch(mu), sk.HistogramBatch(nu), sk.CostMatrix(c),
                                 sk.SinkhornConfig(lam=1e-300, max_iters=20, tolerance=0.0))
