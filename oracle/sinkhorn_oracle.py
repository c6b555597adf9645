"""CPU oracle for the batched log-domain Sinkhorn loss -- TEST INFRASTRUCTURE ONLY.

This module is the parity checker and the CPU baseline (``bench.py``'s
``cpu_baseline`` leg and ``--impl reference`` arm).  It is never imported by
the product package ``paper_1907_01729_b200``; only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` may use it.

It restates, in float64 NumPy, the algorithm of the reference package
``sinkloss`` (``/root/reference/pkg/src/sinkloss``); every function cites the
reference lines it follows.  It is *pinned*: ``tests/test_oracle_golden.py``
checks it against fixtures produced by running the reference itself
(``oracle/gen_golden.py`` -> ``tests/golden/*.npz``) and against the
reference's closed-form known answers (2x2 instance, ``conftest.py:9-24``).

Structure (same reduction structure as the reference, not the same code):

* the online log-sum-exp monoid on (running max, running sum) grids
  (``batch.py:59-146``);
* contiguous span partition of the reduction index with an ascending-order
  merge so results do not depend on the worker count (``batch.py:153-201``);
* the lockstep batched iteration, v first then u, with the residual check
  every ``check_interval`` iterations (``batch.py:264-349``);
* the stable E0 evaluation through the same fused reduction
  (``batch.py:329-337``);
* the history-free analytic backward (``batch.py:352-375``);
* the C-ABI status semantics of the FFI boundary (``ffi.ts:21-25,80-191``).

Extensions the reference lacks (per-sample cost, on-the-fly grid cost) are
expressed here by materialising the cost in float64 and running the same
algorithm lane by lane, which is what SURVEY.md section 8(c) prescribes.
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

NEG_INF = -np.inf

# core.py:29 -- |sum - 1| tolerance of a valid histogram
MASS_TOLERANCE = 1e-6

# ffi.ts:21-25 status codes, plus the extensions documented in include/sinkhorn_b200.h
STATUS_OK = 0
STATUS_SHAPE_MISMATCH = 10
STATUS_INVALID_HISTOGRAM = 11
STATUS_NON_FINITE_OUTPUT = 12
STATUS_ZERO_MASS_LANE = 13
STATUS_INVALID_CONFIG = 14
STATUS_INVALID_COST = 15

# batch.py:182 -- below this many cell-rows a span reduction runs serially
SERIAL_WORK_LIMIT = 10_000_000


class OracleError(Exception):
    """Raised where the reference raises a SinklossError subclass."""

    def __init__(self, kind: str, message: str = "", lane: int | None = None):
        self.kind = kind
        self.lane = lane
        super().__init__(f"{kind}: {message}" if message else kind)


# ---------------------------------------------------------------------------
# online log-sum-exp monoid (batch.py:59-146)


def lse_empty(shape) -> tuple[np.ndarray, np.ndarray]:
    """Empty accumulator: max -inf, sum 0 (batch.py:74-75)."""
    return np.full(shape, NEG_INF), np.zeros(shape)


def lse_consume(state, term: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Fold one slice into (m, s) (batch.py:91-114).

    m' = max(m, x); s' = s * exp(m - m') + exp(x - m').  Cells whose new max
    is -inf have seen nothing finite and keep s = 0 (batch.py:106-110).
    """
    m, s = state
    m_new = np.maximum(m, term)
    with np.errstate(invalid="ignore"):
        rescale = np.exp(m - m_new)
        inc = np.exp(term - m_new)
    dead = np.isneginf(m_new)
    if dead.any():
        rescale = np.where(dead, 0.0, rescale)
        inc = np.where(dead, 0.0, inc)
    return m_new, s * rescale + inc


def lse_merge(a, b) -> tuple[np.ndarray, np.ndarray]:
    """Accumulator of the union of two element sets (batch.py:116-130)."""
    ma, sa = a
    mb, sb = b
    m = np.maximum(ma, mb)
    dead = np.isneginf(m)
    with np.errstate(invalid="ignore"):
        wa = np.where(dead, 0.0, np.exp(ma - m))
        wb = np.where(dead, 0.0, np.exp(mb - m))
    return m, sa * wa + sb * wb


def lse_finalise(state) -> np.ndarray:
    """m + log(s); empty cells give -inf (batch.py:132-138)."""
    m, s = state
    with np.errstate(divide="ignore", invalid="ignore"):
        return m + np.log(s)


def lse_of(values) -> float:
    """Scalar accumulator fed element by element (batch.py:83-89)."""
    st = lse_empty(())
    for x in np.asarray(values, dtype=float).ravel():
        st = lse_consume(st, np.float64(x))
    return float(lse_finalise(st))


# ---------------------------------------------------------------------------
# span-partitioned fused reduction (batch.py:153-201)


def span_bounds(d: int, workers: int) -> list[tuple[int, int]]:
    """At most `workers` contiguous ascending spans of range(d) (batch.py:153-164)."""
    n = max(1, min(workers, d))
    q, r = divmod(d, n)
    out, lo = [], 0
    for w in range(n):
        hi = lo + q + (1 if w < r else 0)
        if hi > lo:
            out.append((lo, hi))
        lo = hi
    return out


def _span_reduce(log_x: np.ndarray, A: np.ndarray, lo: int, hi: int):
    """One cost row at a time into a (B, d2) accumulator (batch.py:167-176)."""
    st = lse_empty((log_x.shape[0], A.shape[1]))
    for i in range(lo, hi):
        st = lse_consume(st, log_x[:, i, None] + A[i][None, :])
    return st


def fused_lse(log_x: np.ndarray, A: np.ndarray, workers: int = 1, pool=None) -> np.ndarray:
    """out[b, j] = logsumexp_i(A[i, j] + log_x[b, i]) (batch.py:185-201)."""
    spans = span_bounds(A.shape[0], workers)
    if len(spans) == 1:
        return lse_finalise(_span_reduce(log_x, A, *spans[0]))
    work = log_x.shape[0] * A.shape[0] * A.shape[1]
    if work < SERIAL_WORK_LIMIT or pool is None and workers <= 1:
        parts = [_span_reduce(log_x, A, lo, hi) for lo, hi in spans]
    elif pool is None:
        with ThreadPoolExecutor(max_workers=len(spans)) as ex:
            parts = list(ex.map(lambda sp: _span_reduce(log_x, A, *sp), spans))
    else:
        parts = list(pool.map(lambda sp: _span_reduce(log_x, A, *sp), spans))
    acc = parts[0]
    for p in parts[1:]:  # ascending span order (batch.py:198-201)
        acc = lse_merge(acc, p)
    return lse_finalise(acc)


def fused_log_reduction(log_u, c, lam: float, log_nu, workers: int = 1) -> np.ndarray:
    """log_nu - logsumexp_i(-c/lam + log_u) : one half-sweep (batch.py:208-230)."""
    log_u = np.asarray(log_u, dtype=float)
    log_nu = np.asarray(log_nu, dtype=float)
    c = np.asarray(c, dtype=float)
    if log_u.ndim != 2 or log_nu.ndim != 2:
        raise OracleError("ShapeMismatch", "log_u and log_nu must be 2-D")
    if log_u.shape[0] != log_nu.shape[0]:
        raise OracleError("ShapeMismatch", "batch sizes differ")
    if log_u.shape[1] != c.shape[0] or log_nu.shape[1] != c.shape[1]:
        raise OracleError("ShapeMismatch", "cost does not match potentials")
    return log_nu - fused_lse(log_u, -c / lam, workers=workers)


# ---------------------------------------------------------------------------
# validation (core.py:47-96,143-160; batch.py:45-56; ffi.ts:53-63)


def histogram_rows_valid(mass: np.ndarray) -> np.ndarray:
    """Per-row validity: finite, >= 0, |sum - 1| <= 1e-6 (core.py:143-160)."""
    mass = np.asarray(mass, dtype=float)
    finite = np.isfinite(mass).all(axis=1)
    nonneg = (np.where(np.isfinite(mass), mass, 0.0) >= 0).all(axis=1)
    with np.errstate(invalid="ignore"):
        normed = np.abs(mass.sum(axis=1) - 1.0) <= MASS_TOLERANCE
    return finite & nonneg & normed


def config_valid(lam, max_iters, tolerance, check_interval) -> bool:
    """SinkhornConfig.__post_init__ (core.py:88-96)."""
    return (
        math.isfinite(lam) and lam > 0 and max_iters >= 1
        and math.isfinite(tolerance) and tolerance >= 0 and check_interval >= 1
    )


def cost_valid(c: np.ndarray) -> bool:
    """CostMatrix.__post_init__: finite and non-negative (core.py:53-63)."""
    c = np.asarray(c, dtype=float)
    return bool(np.isfinite(c).all() and (c >= 0).all())


# ---------------------------------------------------------------------------
# forward / backward (batch.py:237-375)


@dataclass(frozen=True)
class OracleResult:
    """Mirror of BatchLossResult (batch.py:237-253)."""

    cost_e0: np.ndarray
    log_u: np.ndarray
    log_v: np.ndarray
    lam: float
    iterations_run: int
    residuals: np.ndarray


def _resolve_workers(workers) -> int:
    # batch.py:256-261
    return (os.cpu_count() or 1) if workers is None else max(1, int(workers))


def batch_forward(mu, nu, c, lam: float, max_iters: int = 1000, tolerance: float = 1e-9,
                  check_interval: int = 10, workers: int | None = 1) -> OracleResult:
    """Lockstep log-domain iteration over B lanes sharing one cost (batch.py:264-349)."""
    mu = np.asarray(mu, dtype=float)
    nu = np.asarray(nu, dtype=float)
    c = np.asarray(c, dtype=float)
    if mu.shape[0] != nu.shape[0] or c.shape != (mu.shape[1], nu.shape[1]):
        raise OracleError("ShapeMismatch", "batch / cost shapes disagree")
    if not config_valid(lam, max_iters, tolerance, check_interval):
        raise OracleError("ValueError", "invalid SinkhornConfig")
    workers = _resolve_workers(workers)
    A = -c / lam                                   # batch.py:289
    At = np.ascontiguousarray(A.T)                 # batch.py:290
    with np.errstate(divide="ignore"):
        log_mu, log_nu = np.log(mu), np.log(nu)    # batch.py:291-293
    log_u = np.where(mu > 0, 0.0, NEG_INF)         # batch.py:295
    log_v = np.full_like(log_nu, NEG_INF)          # batch.py:296

    pool = ThreadPoolExecutor(max_workers=workers) if workers > 1 else None
    try:
        def lse(x, M):
            return fused_lse(x, M, workers=workers, pool=pool)

        def residuals_of(lu, lv):  # batch.py:303-309
            row = np.exp(lu + lse(lv, At))
            col = np.exp(lv + lse(lu, A))
            return np.maximum(np.abs(row - mu).max(axis=1), np.abs(col - nu).max(axis=1))

        k_run, res, converged = 0, None, False
        for k in range(1, max_iters + 1):          # batch.py:314-322
            log_v = log_nu - lse(log_u, A)
            log_u = log_mu - lse(log_v, At)
            k_run = k
            if tolerance > 0 and k % check_interval == 0:
                res = residuals_of(log_u, log_v)
                if res.max() <= tolerance:
                    converged = True
                    break
        if res is None or not converged:           # batch.py:323-324
            res = residuals_of(log_u, log_v)
        if np.isnan(log_u).any() or np.isnan(log_v).any():  # batch.py:326-327
            raise OracleError("NaNProduced", "NaN in batched solver state")
        with np.errstate(divide="ignore"):
            G = A + np.log(c)                      # batch.py:332
        S = lse(log_u, G)                          # batch.py:333
        st = lse_empty((mu.shape[0],))
        for j in range(nu.shape[1]):               # batch.py:334-336
            st = lse_consume(st, S[:, j] + log_v[:, j])
        cost_e0 = np.exp(lse_finalise(st))         # batch.py:337
    finally:
        if pool is not None:
            pool.shutdown(wait=False)
    return OracleResult(cost_e0, log_u, log_v, float(lam), k_run, res)


def batch_backward(log_u, log_v, lam: float, upstream) -> tuple[np.ndarray, np.ndarray]:
    """grad_x = up * lam * (log_x - mean log_x); refuses -inf lanes (batch.py:352-375)."""
    log_u = np.asarray(log_u, dtype=float)
    log_v = np.asarray(log_v, dtype=float)
    up = np.asarray(upstream, dtype=float)
    if up.shape != (log_u.shape[0],):
        raise OracleError("ShapeMismatch", "upstream shape")
    dead = np.isneginf(log_u).any(axis=1) | np.isneginf(log_v).any(axis=1)
    if dead.any():
        raise OracleError("ZeroMassGradient", lane=int(np.argmax(dead)))
    g_mu = up[:, None] * (lam * (log_u - log_u.mean(axis=1, keepdims=True)))
    g_nu = up[:, None] * (lam * (log_v - log_v.mean(axis=1, keepdims=True)))
    return g_mu, g_nu


def per_sample_forward(mu, nu, costs, lam: float, max_iters: int, tolerance: float = 0.0,
                       check_interval: int = 10) -> OracleResult:
    """Per-lane cost matrices (B, d1, d2): the reference algorithm run lane by lane.

    The reference has no per-sample API; with tolerance 0 the
    lanes are independent (test_batch.py:46-63), so lane-by-lane B=1
    ``batch_forward`` calls equal the batched semantics.  With tolerance > 0
    the lockstep count is the worst lane's (test_batch.py:77-90); this is
    reproduced by re-running every lane at the common iteration count.
    """
    mu = np.asarray(mu, dtype=float)
    nu = np.asarray(nu, dtype=float)
    B = mu.shape[0]
    runs = [batch_forward(mu[b:b + 1], nu[b:b + 1], costs[b], lam, max_iters, tolerance,
                          check_interval, workers=1) for b in range(B)]
    if tolerance > 0:
        k = max(r.iterations_run for r in runs)
        if any(r.iterations_run != k for r in runs):
            runs = [batch_forward(mu[b:b + 1], nu[b:b + 1], costs[b], lam, k, 0.0,
                                  check_interval, workers=1) for b in range(B)]
            runs = [OracleResult(r.cost_e0, r.log_u, r.log_v, r.lam, k, r.residuals)
                    for r in runs]
    return OracleResult(
        np.concatenate([r.cost_e0 for r in runs]),
        np.concatenate([r.log_u for r in runs]),
        np.concatenate([r.log_v for r in runs]),
        float(lam), runs[0].iterations_run if runs else 0,
        np.concatenate([r.residuals for r in runs]),
    )


def _dense_lse(arr: np.ndarray, axis: int) -> np.ndarray:
    """Max-extracted logsumexp along one axis; -inf slices stay -inf (core.py:191-199)."""
    m = arr.max(axis=axis)
    with np.errstate(invalid="ignore"):
        out = m + np.log(np.exp(arr - np.expand_dims(m, axis)).sum(axis=axis))
    return np.where(np.isneginf(m), NEG_INF, out)


def dense_forward(mu_row, nu_row, c, lam: float, max_iters: int) -> OracleResult:
    """Single-pair dense solve with tolerance 0: run_sinkhorn (core.py:305-357)
    with _update_log_v/_u (core.py:246-268), the residual (core.py:296-302) and
    primal_cost (core.py:378-391).  Equal to a batch lane to 1e-12
    (test_batch.py:46-63); used where the streaming port is too slow (d >= 1024)."""
    mu_row = np.asarray(mu_row, dtype=float)
    nu_row = np.asarray(nu_row, dtype=float)
    A = -np.asarray(c, dtype=float) / lam
    with np.errstate(divide="ignore"):
        log_mu, log_nu = np.log(mu_row), np.log(nu_row)
    log_u = np.where(mu_row > 0, 0.0, NEG_INF)
    log_v = np.full(nu_row.shape[0], NEG_INF)
    for _ in range(max_iters):
        log_v = log_nu - _dense_lse(A + log_u[:, None], axis=0)
        log_u = log_mu - _dense_lse(A + log_v[None, :], axis=1)
    row = np.exp(log_u + _dense_lse(A + log_v[None, :], axis=1))
    col = np.exp(log_v + _dense_lse(A + log_u[:, None], axis=0))
    res = max(np.abs(row - mu_row).max(), np.abs(col - nu_row).max())
    with np.errstate(divide="ignore"):
        terms = log_u[:, None] + A + np.log(np.asarray(c, dtype=float)) + log_v[None, :]
    m = terms.max()
    e0 = float(np.exp(m + np.log(np.exp(terms - m).sum()))) if np.isfinite(m) else 0.0
    return OracleResult(np.array([e0]), log_u[None, :], log_v[None, :], float(lam), max_iters,
                        np.array([res]))


def transport_plan(log_u_row, log_v_row, c, lam: float) -> np.ndarray:
    """P = exp(log_u[i] - c/lam + log_v[j]) (core.py:363-368)."""
    return np.exp(np.asarray(log_u_row)[:, None] - np.asarray(c) / lam
                  + np.asarray(log_v_row)[None, :])


# ---------------------------------------------------------------------------
# C-ABI restatement (ffi.ts:80-191): statuses instead of exceptions


def forward_v1(mu, nu, cost, lam, max_iters, tolerance, check_interval: int = 10):
    """Returns (status, cost_e0, log_u, log_v) as ffi.ts:80-134 would fill them."""
    mu = np.asarray(mu, dtype=float)
    nu = np.asarray(nu, dtype=float)
    cost = np.asarray(cost, dtype=float)
    if mu.ndim != 2 or nu.ndim != 2 or cost.ndim != 2:
        return STATUS_SHAPE_MISMATCH, None, None, None
    B, d1 = mu.shape
    d2 = nu.shape[1]
    if nu.shape[0] != B or cost.shape != (d1, d2):
        return STATUS_SHAPE_MISMATCH, None, None, None
    if B == 0:
        return STATUS_OK, np.zeros(0), np.zeros((0, d1)), np.zeros((0, d2))
    if not (histogram_rows_valid(mu).all() and histogram_rows_valid(nu).all()):
        return STATUS_INVALID_HISTOGRAM, None, None, None
    if not config_valid(lam, max_iters, tolerance, check_interval):
        return STATUS_INVALID_CONFIG, None, None, None
    if not cost_valid(cost):
        return STATUS_INVALID_COST, None, None, None
    r = batch_forward(mu, nu, cost, lam, max_iters, tolerance, check_interval, workers=1)
    if not np.isfinite(r.cost_e0).all():
        return STATUS_NON_FINITE_OUTPUT, None, None, None
    return STATUS_OK, r.cost_e0, r.log_u, r.log_v


def backward_v1(log_u, log_v, lam, upstream):
    """Returns (status, grad_mu, grad_nu) per ffi.ts:143-191."""
    log_u = np.asarray(log_u, dtype=float)
    log_v = np.asarray(log_v, dtype=float)
    up = np.asarray(upstream, dtype=float)
    if log_u.ndim != 2 or log_v.ndim != 2 or log_v.shape[0] != log_u.shape[0] \
            or up.shape != (log_u.shape[0],):
        return STATUS_SHAPE_MISMATCH, None, None
    if np.isneginf(log_u).any() or np.isneginf(log_v).any():
        return STATUS_ZERO_MASS_LANE, None, None
    g_mu, g_nu = batch_backward(log_u, log_v, lam, up)
    return STATUS_OK, g_mu, g_nu


# ---------------------------------------------------------------------------
# seeded instance families (oracle.py:152-165, conftest.py:27-34)


def random_histogram_batch(B: int, d: int, rng: np.random.Generator,
                           lo: float = 0.5, hi: float = 1.5) -> np.ndarray:
    """B rows of U(lo, hi) normalised (oracle.py:152-155)."""
    rows = [rng.uniform(lo, hi, d) for _ in range(B)]
    return np.stack([r / r.sum() for r in rows]) if B else np.zeros((0, d))


def fp32_exact(x: np.ndarray) -> np.ndarray:
    """Round to float32 and back so the CUDA path and the oracle see identical inputs."""
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def index_grid_cost(d1: int, d2: int | None = None, power: int = 2) -> np.ndarray:
    """|i - j|^p / (d - 1)^p (oracle.py:158-165)."""
    d2 = d1 if d2 is None else d2
    denom = max(max(d1, d2) - 1, 1)
    i = np.arange(d1, dtype=float)[:, None]
    j = np.arange(d2, dtype=float)[None, :]
    return (np.abs(i - j) / denom) ** power


def grid2d_cost(nx: int, ny: int | None = None) -> np.ndarray:
    """Squared Euclidean cost on an nx x ny grid with coordinates (col, row)/(n-1).

    Point k sits at (k % nx, k // nx) scaled by 1/(nx-1), 1/(ny-1)
    (BASELINE.md section 3, configs 2 and 3).
    """
    ny = nx if ny is None else ny
    k = np.arange(nx * ny)
    x = (k % nx) / max(nx - 1, 1)
    y = (k // nx) / max(ny - 1, 1)
    return (x[:, None] - x[None, :]) ** 2 + (y[:, None] - y[None, :]) ** 2


def per_sample_cost(seed: int, lane: int, d1: int, d2: int) -> np.ndarray:
    """Lane `lane`'s U[0,1) float32 cost, reproducible lane by lane (config 4)."""
    rng = np.random.default_rng([seed, lane])
    return rng.random((d1, d2), dtype=np.float32)
