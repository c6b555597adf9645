"""Multi-GPU drivers: batch-sharded and row-sharded solves.

One process per GPU with ``torch.distributed`` (NCCL on GPUs; the same code
runs on gloo/CPU tensors in the tests).

* Batch sharding -- lanes are independent (test_batch.py:46-63) and coupled
  only by the lockstep stopping rule (batch.py:318-322).  Each rank solves its
  own lanes with the single-GPU library; with tolerance > 0 the library calls
  back at every convergence check and the ranks agree on the global max
  residual with one 8-byte all-reduce(MAX), so ``iterations_run`` is global.
  The only other collective is the final all-gather of the per-lane losses.

* Row sharding -- for supports too large for one GPU, rank r owns rows
  I_r of the cost and of mu / log_u.  The column sweep becomes a local
  partial (max, sum) reduction over I_r followed by the cross-GPU merge of
  OnlineLseAccumulator.merge (batch.py:116-130): all-reduce(MAX) of the maxima,
  local rescale, all-reduce(SUM) of the sums.  The row sweep is local.  E0 and
  the backward's means merge the same way.

The per-shard arithmetic goes through a *backend* (the CUDA library in
production; tests inject the CPU oracle) so the collective logic is the same
code in both.
"""

from __future__ import annotations

import ctypes
import math
from contextlib import contextmanager

import torch
import torch.distributed as dist

from . import _lib
from .loss import SolveResult, potentials_backward, solve

LN2 = math.log(2.0)
NEG_BIG = -1.0e30


# ---------------------------------------------------------------------------
# batch sharding


def global_max(local: float, group=None) -> float:
    """Max over ranks of a per-rank residual; NaN never converges (batch.py:320)."""
    v = local if local == local else math.inf
    dev = torch.device("cuda", torch.cuda.current_device()) \
        if dist.get_backend(group) == "nccl" else torch.device("cpu")
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def gather_lane_values(local: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather per-lane values from ranks holding different lane counts."""
    ws = dist.get_world_size(group)
    dev = local.device
    sizes = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(ws)]
    dist.all_gather(sizes, torch.tensor([local.numel()], device=dev), group=group)
    n = max(int(x.item()) for x in sizes)
    buf = torch.full((n,), float("nan"), device=dev, dtype=local.dtype)
    buf[: local.numel()] = local
    parts = [torch.empty_like(buf) for _ in range(ws)]
    dist.all_gather(parts, buf, group=group)
    return torch.cat([p[: int(x.item())] for p, x in zip(parts, sizes)])


@contextmanager
def global_residual_reducer(group=None):
    """Make the library's convergence test use the max residual over all ranks."""
    lib = _lib.load()

    def reduce(local: float, _user) -> float:
        return global_max(local, group)

    cb = _lib.REDUCER(reduce)
    lib.sinkhorn_set_residual_reducer_v1(cb, None)
    try:
        yield
    finally:
        lib.sinkhorn_set_residual_reducer_v1(_lib.REDUCER(0), None)
        del cb


def batch_sharded_solve(mu_local, nu_local, cost, lam: float, max_iters: int = 1000,
                        tolerance: float = 0.0, check_interval: int = 10, group=None):
    """Solve this rank's lanes; returns (local SolveResult, all lanes' E0 costs)."""
    if tolerance > 0 and dist.get_world_size(group) > 1:
        with global_residual_reducer(group):
            res = solve(mu_local, nu_local, cost, lam, max_iters, tolerance, check_interval)
    else:
        res = solve(mu_local, nu_local, cost, lam, max_iters, tolerance, check_interval)
    return res, gather_lane_values(res.cost_e0, group)


# ---------------------------------------------------------------------------
# row sharding


class CudaShardBackend:
    """Per-shard arithmetic on the sm_100a library (half-sweep C ABI)."""

    def __init__(self, cost_local: torch.Tensor):
        from . import batch

        self._batch = batch
        self.c = cost_local.float().contiguous()
        self.ct = self.c.t().contiguous()

    def col_partial(self, log_u_l, lam):
        """(max, sum) over local rows of 2^(-c/lam*log2e + log2 u): both (B, d2), log base 2."""
        return self._batch.partial_log_reduction(log_u_l, self.c, lam)

    def row_update(self, log_v, lam, log_mu_l):
        """log_mu - LSE_j(-c/lam + log_v) for the local rows (batch.py:316)."""
        return self._batch.fused_log_reduction(log_v, self.ct, lam, log_mu_l)

    def e0_partial(self, log_u_l, log_v, lam):
        """Per lane log2 sum_{i local, j} P_ij c_ij (batch.py:331-337 restricted to I_r)."""
        return self._batch.e0_partial_log2(log_u_l, log_v, self.c, lam)


class CudaGemmShardBackend:
    """Per-shard arithmetic as fp32 GEMMs on the local rows' kernel matrix
    (the GEMM iteration of csrc/sweep_gemm.cuh, restricted to rows I_r).

    K_r = 2^(-c_r log2e / lam) <= 1 and, per lane, X_j = 2^(v_j - vmax):
      row update:   u_i = log_mu_i - (vmax + log2 (K_r X)_i)          (local)
      col partial:  (max, sum) = (umax_r, (K_r^T 2^(u - umax_r))_j)   (per lane shift)
    so the cross-rank merge of the column sums is the same (max, sum-exp)
    merge as the log-domain shards, with the max agreed once per lane.  A
    call whose sums fall below 2^-60 (terms may have flushed) is redone by the
    exact log-domain backend.  The GEMMs are cuBLAS SGEMMs through torch.
    """

    MIN = 2.0 ** -60

    def __init__(self, cost_local: torch.Tensor):
        self.c = cost_local.float().contiguous()
        self._lam = None
        self._exact = None

    def _kernel(self, lam):
        if self._lam != lam:
            self.K = torch.exp2(self.c * (-1.0 / (lam * LN2)))
            self.KC = self.K * self.c
            self._lam = lam
        return self.K

    def exact(self):
        if self._exact is None:
            self._exact = CudaShardBackend(self.c)
        return self._exact

    def col_partial(self, log_u_l, lam):
        K = self._kernel(lam)
        u2 = log_u_l.float() / LN2
        umax = torch.clamp(u2.amax(dim=1, keepdim=True), min=NEG_BIG)
        a = torch.exp2(u2 - umax)
        T = a @ K                                   # (B, d2) = sum_i a_i K_ij
        if bool((T < self.MIN).any()):
            return self.exact().col_partial(log_u_l, lam)
        return umax.expand_as(T), T

    def row_update(self, log_v, lam, log_mu_l):
        K = self._kernel(lam)
        v2 = log_v.float() / LN2
        vmax = torch.clamp(v2.amax(dim=1, keepdim=True), min=NEG_BIG)
        X = torch.exp2(v2 - vmax)
        S = X @ K.t()                               # (B, d1_r) = sum_j K_ij X_j
        if bool(((S < self.MIN) & ~torch.isneginf(log_mu_l)).any()):
            return self.exact().row_update(log_v, lam, log_mu_l)
        lse = (vmax + torch.log2(S)) * LN2
        return torch.where(torch.isneginf(log_mu_l), log_mu_l, log_mu_l - lse)

    def e0_partial(self, log_u_l, log_v, lam):
        """Per lane log2 sum_{i local, j} P_ij c_ij = log2 sum_i a_i (KC X)_i."""
        K = self._kernel(lam)
        v2 = log_v.float() / LN2
        vmax = torch.clamp(v2.amax(dim=1, keepdim=True), min=NEG_BIG)
        X = torch.exp2(v2 - vmax)
        # rows whose terms may have flushed: the exact log-domain partial
        if bool(((X @ K.t() < self.MIN) & ~torch.isneginf(log_u_l)).any()):
            return self.exact().e0_partial(log_u_l, log_v, lam)
        SE = X @ self.KC.t()                        # (B, d1_r)
        w = torch.exp2(log_u_l.float() / LN2 + vmax)  # a_i = 2^(u_i + vmax)
        tot = (w * SE).double().sum(dim=1)
        return torch.where(tot > 0, torch.log2(tot), torch.full_like(tot, -math.inf)).float()


def _merge_lse(m: torch.Tensor, s: torch.Tensor, group) -> torch.Tensor:
    """All-rank OnlineLseAccumulator.merge of (max, sum) pairs in log base 2 -> natural LSE."""
    M = m.clone()
    dist.all_reduce(M, op=dist.ReduceOp.MAX, group=group)
    scaled = s * torch.exp2(torch.clamp(m - M, max=0.0))
    scaled = torch.where(M <= NEG_BIG, torch.zeros_like(scaled), scaled)
    dist.all_reduce(scaled, op=dist.ReduceOp.SUM, group=group)
    with torch.no_grad():
        lse2 = torch.where(scaled > 0, M + torch.log2(scaled),
                           torch.full_like(M, -math.inf))
    return lse2 * LN2


def row_sharded_solve(mu_local, nu, backend, lam: float, max_iters: int,
                      tolerance: float = 0.0, check_interval: int = 10, group=None,
                      d1_total: int | None = None) -> SolveResult:
    """Lockstep log-domain iteration with the cost's rows sharded over ranks.

    mu_local (B, d1_r): this rank's columns of mu (rows I_r of the cost);
    nu (B, d2) replicated.  Returns log_u for the local rows, the full log_v,
    global E0 per lane, iterations and residuals (batch.py:264-349 semantics).
    """
    # float32 on the device; float64 when a CPU backend drives the same logic (tests)
    dt = torch.float64 if mu_local.dtype == torch.float64 else torch.float32
    mu_local = mu_local.to(dt)
    nu = nu.to(dt)
    log_mu = torch.log(mu_local)
    log_nu = torch.log(nu)
    log_u = torch.where(mu_local > 0, torch.zeros_like(mu_local),
                        torch.full_like(mu_local, -math.inf))
    log_v = torch.full_like(nu, -math.inf)

    def col_update(lu):
        m, s = backend.col_partial(lu, lam)
        lse = _merge_lse(m, s, group)
        return torch.where(torch.isneginf(log_nu), log_nu, log_nu - lse), lse

    def residuals(lu, lv):
        # row term over local rows, column term from the merged column sums (batch.py:303-309)
        zeros = torch.zeros_like(lu)
        row_lse = -backend.row_update(lv, lam, zeros)
        row = torch.exp(lu + row_lse)
        r_row = (row - mu_local).abs().amax(dim=1) if lu.shape[1] else torch.zeros(lu.shape[0])
        dist.all_reduce(r_row, op=dist.ReduceOp.MAX, group=group)
        _, col_lse = col_update(lu)
        col = torch.exp(lv + col_lse)
        r_col = (col - nu).abs().amax(dim=1)
        return torch.maximum(r_row, r_col)

    iters, res, converged = 0, None, False
    for k in range(1, max_iters + 1):
        log_v, _ = col_update(log_u)
        log_u = backend.row_update(log_v, lam, log_mu)
        iters = k
        if tolerance > 0 and k % check_interval == 0:
            res = residuals(log_u, log_v)
            if float(res.max()) <= tolerance:
                converged = True
                break
    if res is None or not converged:
        res = residuals(log_u, log_v)
    # E0: per-lane partial log2 sums merged across ranks
    e_loc = backend.e0_partial(log_u, log_v, lam)
    e_nat = _merge_lse(e_loc, torch.ones_like(e_loc), group)
    cost = torch.exp(e_nat)
    return SolveResult(cost, log_u, log_v, float(lam), iters, res)


def row_sharded_backward(log_u_local, log_v, lam: float, upstream, group=None,
                         d1_total: int | None = None):
    """batch_backward (batch.py:352-375) with log_u's rows sharded: the lane
    means of log_u need one all-reduce(SUM) of B partial sums (and a MAX of the
    zero-mass flags, ffi.ts:177-179)."""
    from .errors import ZeroMassGradient

    up = torch.as_tensor(upstream, dtype=torch.float64, device=log_u_local.device)
    dead = (torch.isneginf(log_u_local).any(dim=1) | torch.isneginf(log_v).any(dim=1)).to(
        torch.float64)
    dist.all_reduce(dead, op=dist.ReduceOp.MAX, group=group)
    if bool(dead.any()):
        raise ZeroMassGradient(int(torch.nonzero(dead)[0]))
    part = log_u_local.to(torch.float64).sum(dim=1)
    cnt = torch.tensor([float(log_u_local.shape[1])], dtype=torch.float64,
                       device=log_u_local.device)
    dist.all_reduce(part, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(cnt, op=dist.ReduceOp.SUM, group=group)
    mean_u = part / cnt
    g_mu = up[:, None] * lam * (log_u_local.to(torch.float64) - mean_u[:, None])
    g_nu = up[:, None] * lam * (log_v.to(torch.float64) - log_v.to(torch.float64).mean(dim=1,
                                                                                        keepdim=True))
    return g_mu.to(log_u_local.dtype), g_nu.to(log_v.dtype)


__all__ = [
    "CudaGemmShardBackend", "CudaShardBackend", "batch_sharded_solve", "gather_lane_values", "global_max",
    "global_residual_reducer",
    "row_sharded_backward", "row_sharded_solve",
]

_ = (ctypes, potentials_backward)
