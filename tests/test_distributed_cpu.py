"""Multi-process (gloo, world_size 2) tests of the sharded drivers on CPU.

The collective logic of paper_1907_01729_b200.distributed is exercised with
the CPU oracle as the per-shard backend and compared against the unsharded
oracle (which is pinned to the reference by test_oracle_golden.py)."""

from __future__ import annotations

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import sinkhorn_oracle as orc

LOG2E = 1.0 / math.log(2.0)


class OracleShardBackend:
    """Per-shard arithmetic restated with the oracle (test-only backend)."""

    def __init__(self, c_local: np.ndarray):
        self.c = np.asarray(c_local, dtype=np.float64)

    def col_partial(self, log_u_l, lam):
        if self.c.shape[0] == 0:
            B = log_u_l.shape[0]
            return (torch.full((B, self.c.shape[1]), -1e30, dtype=torch.float64),
                    torch.zeros(B, self.c.shape[1], dtype=torch.float64))
        lse = orc.fused_lse(log_u_l.numpy(), -self.c / lam)
        fin = np.isfinite(lse)
        m = np.where(fin, lse * LOG2E, -1e30)
        s = np.where(fin, 1.0, 0.0)
        return torch.from_numpy(m), torch.from_numpy(s)

    def row_update(self, log_v, lam, log_mu_l):
        return torch.from_numpy(orc.fused_log_reduction(log_v.numpy(), self.c.T, lam,
                                                        log_mu_l.numpy()))

    def e0_partial(self, log_u_l, log_v, lam):
        with np.errstate(divide="ignore"):
            t = (log_u_l.numpy()[:, :, None] - self.c[None] / lam + np.log(self.c)[None]
                 + log_v.numpy()[:, None, :])
        B = t.shape[0]
        flat = t.reshape(B, -1)
        m = flat.max(axis=1)
        out = m + np.log(np.exp(flat - m[:, None]).sum(axis=1))
        return torch.from_numpy(out * LOG2E)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    finally:
        dist.destroy_process_group()


def _spawn(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def _problem(seed=3, B=3, d1=20, d2=15):
    rng = np.random.default_rng(seed)
    mu = orc.random_histogram_batch(B, d1, rng)
    nu = orc.random_histogram_batch(B, d2, rng)
    c = rng.uniform(0.0, 1.0, (d1, d2))
    return mu, nu, c


def _row_sharded(rank, world, tol=0.0, iters=40, lam=0.3, zero=False, gemm=False):
    from paper_1907_01729_b200 import distributed as D

    mu, nu, c = _problem()
    if zero:
        mu[1, :3] = 0.0
        mu[1] /= mu[1].sum()
    d1 = mu.shape[1]
    lo, hi = rank * d1 // world, (rank + 1) * d1 // world
    res = D.row_sharded_solve(torch.from_numpy(mu[:, lo:hi].copy()), torch.from_numpy(nu),
                              D.CudaGemmShardBackend(torch.from_numpy(c[lo:hi].copy())) if gemm
                              else OracleShardBackend(c[lo:hi]), lam, iters, tol, 10)
    out = {"cost": res.cost_e0.numpy(), "log_u": res.log_u.numpy(), "log_v": res.log_v.numpy(),
           "iters": res.iterations_run, "res": res.residuals.numpy(), "lo": lo}
    up = torch.from_numpy(np.array([0.5, -1.0, 2.0]))
    try:
        gm, gn = D.row_sharded_backward(res.log_u, res.log_v, lam, up)
        out["gm"], out["gn"] = gm.numpy(), gn.numpy()
    except Exception as err:  # ZeroMassGradient
        out["err"] = (type(err).__name__, getattr(err, "lane", None))
    return out


def _assemble(outs):
    r0, r1 = outs[0], outs[1]
    return np.concatenate([r0["log_u"], r1["log_u"]], axis=1), r0, r1


def test_row_sharded_matches_unsharded_oracle():
    outs = _spawn(_row_sharded)
    mu, nu, c = _problem()
    ref = orc.batch_forward(mu, nu, c, 0.3, 40, 0.0)
    log_u, r0, r1 = _assemble(outs)
    np.testing.assert_allclose(r0["cost"], ref.cost_e0, rtol=1e-12)
    np.testing.assert_allclose(r1["cost"], ref.cost_e0, rtol=1e-12)
    np.testing.assert_allclose(log_u, ref.log_u, atol=1e-11)
    np.testing.assert_allclose(r0["log_v"], ref.log_v, atol=1e-11)
    np.testing.assert_allclose(r0["res"], ref.residuals, rtol=1e-6, atol=1e-15)
    gm_ref, gn_ref = orc.batch_backward(ref.log_u, ref.log_v, 0.3, [0.5, -1.0, 2.0])
    np.testing.assert_allclose(np.concatenate([r0["gm"], r1["gm"]], axis=1), gm_ref, atol=1e-12)
    np.testing.assert_allclose(r0["gn"], gn_ref, atol=1e-12)


def _row_sharded_tol(rank, world):
    return _row_sharded(rank, world, tol=1e-7, iters=2000, lam=0.2)


def test_row_sharded_lockstep_iteration_count():
    outs = _spawn(_row_sharded_tol)
    mu, nu, c = _problem()
    ref = orc.batch_forward(mu, nu, c, 0.2, 2000, 1e-7, 10)
    assert outs[0]["iters"] == outs[1]["iters"] == ref.iterations_run
    np.testing.assert_allclose(outs[0]["cost"], ref.cost_e0, rtol=1e-12)


def _row_sharded_zero(rank, world):
    return _row_sharded(rank, world, zero=True)


def test_row_sharded_zero_mass_refused_on_every_rank():
    outs = _spawn(_row_sharded_zero)
    assert outs[0]["err"] == ("ZeroMassGradient", 1)
    assert outs[1]["err"] == ("ZeroMassGradient", 1)


def _gather_ragged(rank, world):
    from paper_1907_01729_b200 import distributed as D

    local = torch.arange(3 + rank, dtype=torch.float32) + 10 * rank
    return D.gather_lane_values(local).numpy(), D.global_max(float(rank) + 0.5), \
        D.global_max(float("nan") if rank == 0 else 1.0)


def test_batch_sharded_collectives():
    """Final loss gather (ragged lane counts) and the lockstep residual max."""
    outs = _spawn(_gather_ragged)
    for r in (0, 1):
        vals, gmax, nanmax = outs[r]
        np.testing.assert_array_equal(vals, [0, 1, 2, 10, 11, 12, 13])
        assert gmax == 1.5
        assert nanmax == math.inf     # NaN on any rank never converges


def _row_sharded_linear(rank, world):
    """The device row-sharded iteration's collective structure, restated in
    float64 NumPy per rank (sweep_gemm.cuh): K_r = exp(-c_r/lam), X = exp(v -
    vmax), S_r = K_r X, a_r = mu_r / S_r, and the column sums T = sum_r K_r^T
    a_r merged by ONE all-reduce(SUM) -- the (max, sum-exp) merge with the max
    known in advance (every rank holds the same vmax) -- through the library's
    allreduce callback (_SumOverRanks) on host buffers."""
    from paper_1907_01729_b200 import distributed as D

    mu, nu, c = _problem()
    lam, iters = 0.3, 40
    d1 = mu.shape[1]
    lo, hi = rank * d1 // world, (rank + 1) * d1 // world
    K = np.exp(-c[lo:hi] / lam)
    mu_r = mu[:, lo:hi]
    summer = D._SumOverRanks(None, torch.device("cpu"))

    def col_sums(a):
        T = np.ascontiguousarray((a @ K).astype(np.float32))    # (B, d2) partial
        t = torch.from_numpy(T)
        summer._call(t.data_ptr(), t.numel(), 0, None, None)
        assert summer.error is None
        return t.numpy().astype(np.float64)

    log_v = np.log(nu) - np.log(col_sums(np.where(mu_r > 0, 1.0, 0.0)))   # u0 = 0 on the support
    for _ in range(iters):
        vmax = log_v.max(axis=1, keepdims=True)
        X = np.exp(log_v - vmax)
        S = X @ K.T                                   # (B, d1_r): local rows
        log_u = np.log(mu_r) - (vmax + np.log(S))
        a = mu_r / S                                  # = exp(u + vmax)
        log_v = np.log(nu) + vmax - np.log(col_sums(a))
    return {"log_u": log_u, "log_v": log_v, "calls": summer.calls}


def test_row_sharded_linear_sum_merge_matches_unsharded_oracle():
    """The single SUM collective per column sweep reproduces the unsharded
    lockstep iteration (fp32 collectives, so fp32 tolerances)."""
    outs = _spawn(_row_sharded_linear)
    mu, nu, c = _problem()
    ref = orc.batch_forward(mu, nu, c, 0.3, 40, 0.0)
    log_u = np.concatenate([outs[0]["log_u"], outs[1]["log_u"]], axis=1)
    # log_u after 40 iterations is computed from log_v of the 40th column sweep
    np.testing.assert_allclose(log_u, ref.log_u, atol=2e-5)
    assert outs[0]["calls"] == outs[1]["calls"] == 41


