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
  I_r of the cost and of mu / log_u.  ``row_sharded_solve_device`` runs the
  whole lockstep loop in the library (sinkhorn_forward_rows_device_v1: the
  GEMM iteration on the tensor cores over the rank's rows) and only hands
  back a stream-ordered collective: per column sweep one all-reduce(SUM) of
  the B x d2 column sums.  That sum *is* the (max, sum-exp) merge of
  OnlineLseAccumulator.merge (batch.py:116-130): every rank's partial sums
  carry the same per-lane shift vmax_b (all ranks hold the full log v), so the
  max half of the merge is known in advance.  No host synchronisation per
  iteration (tolerance 0); checks all-reduce one MAX.  A range guard (sums
  below 2^-60) makes every rank rerun through ``row_sharded_solve`` with the
  exact log-domain half-sweep shards (``CudaShardBackend``).

``row_sharded_solve`` is the backend-driven restatement used for that exact
fallback and, with the CPU oracle as backend, by the gloo tests; there the
column merge is all-reduce(MAX) of the maxima, a local rescale and
all-reduce(SUM) of the sums.
"""

from __future__ import annotations

import ctypes
import math
from contextlib import contextmanager

import torch
import torch.distributed as dist

from . import _lib
from .loss import SolveResult, solve

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


class _CudaArrayView:
    """A raw float32 device buffer as a zero-copy torch tensor (CUDA array interface)."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": "<f4",
                                         "data": (int(ptr), False), "version": 3}


class _SumOverRanks:
    """The library's allreduce callback: sum a float32 buffer over the group on
    the current stream (NCCL enqueues; nothing waits on the host)."""

    def __init__(self, group, device):
        self.group, self.device = group, device
        self.error = None
        self.calls = 0
        self.fn = _lib.ALLREDUCE(self._call)

    def _call(self, ptr, count, op, stream, user):
        try:
            if op != _lib.REDUCE_SUM:
                raise ValueError(f"unsupported reduction {op}")
            self.calls += 1
            if count == 0:
                return
            if self.device.type == "cuda":
                t = torch.as_tensor(_CudaArrayView(ptr, count), device=self.device)
            else:   # host buffers (the gloo tests drive the callback directly)
                import numpy as np

                t = torch.from_numpy(np.ctypeslib.as_array(
                    (ctypes.c_float * int(count)).from_address(int(ptr))))
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        except Exception as err:   # never unwind through the C ABI
            self.error = err


def _check_row_histograms(mu_local, nu, group):
    """validate_histogram (core.py:143-160) on row-sharded mu: finite and >= 0
    per shard, |sum - 1| <= 1e-6 over the shards' partial sums (ffi.ts:111-115)."""
    from .errors import InvalidHistogram

    part = mu_local.double().sum(dim=1)
    bad = (~torch.isfinite(mu_local).all(dim=1) | (mu_local < 0).any(dim=1)).double()
    dist.all_reduce(part, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(bad, op=dist.ReduceOp.MAX, group=group)
    badnu = ~torch.isfinite(nu).all(dim=1) | (nu < 0).any(dim=1) | \
        ((nu.double().sum(dim=1) - 1.0).abs() > 1e-6)
    rows = (bad > 0) | ((part - 1.0).abs() > 1e-6) | badnu
    if bool(rows.any()):
        raise InvalidHistogram(f"invalid histogram in row {int(torch.nonzero(rows)[0])}")


def row_sharded_solve_device(mu_local, nu, cost_local, lam: float, max_iters: int,
                             tolerance: float = 0.0, check_interval: int = 10, group=None,
                             validate: bool = True, time_loop: bool = False,
                             time_kernel: bool = False) -> SolveResult:
    """Row-sharded lockstep solve with the whole loop in the library.

    mu_local (B, d1_r) and cost_local (d1_r, d2): this rank's rows; nu (B, d2)
    replicated.  Returns log_u for the local rows, the full log_v, the global
    E0 per lane, the global iteration count and residuals -- batch.py:264-349
    semantics, sharded.  Falls back to the exact log-domain shards when the
    library reports a fired range guard (status 18, on every rank together).
    """
    from .errors import raise_for_status
    from .loss import _as_f32_cuda, _problem, _stream_handle, _workspace

    mu_local = _as_f32_cuda(mu_local)
    dev = mu_local.device
    nu = _as_f32_cuda(nu, dev)
    cost_local = _as_f32_cuda(cost_local, dev)
    B, d1 = mu_local.shape
    d2 = nu.shape[1]
    if nu.shape[0] != B or tuple(cost_local.shape) != (d1, d2):
        from .errors import ShapeMismatch

        raise ShapeMismatch(f"mu rows {tuple(mu_local.shape)}, nu {tuple(nu.shape)}, "
                            f"cost rows {tuple(cost_local.shape)}")
    if validate:
        _check_row_histograms(mu_local, nu, group)
    lib = _lib.load()
    pr = _problem(B, d1, d2, cost_local)
    op = _lib.Options()
    op.lam, op.max_iters, op.check_interval, op.tolerance = float(lam), int(max_iters), \
        int(check_interval), float(tolerance)
    op.flags = (_lib.FLAG_TIME_LOOP if time_loop else 0) | \
        (_lib.FLAG_TIME_KERNEL if time_kernel else 0)
    out_cost = torch.empty(B, device=dev, dtype=torch.float32)
    log_u = torch.empty(B, d1, device=dev, dtype=torch.float32)
    log_v = torch.empty(B, d2, device=dev, dtype=torch.float32)
    residuals = torch.empty(B, device=dev, dtype=torch.float32)
    iters = ctypes.c_int32(0)
    summer = _SumOverRanks(group, dev)
    with torch.cuda.device(dev), global_residual_reducer(group):
        ws = _workspace(dev, lib.sinkhorn_workspace_bytes_v1(ctypes.byref(pr)))
        st = lib.sinkhorn_forward_rows_device_v1(
            ctypes.byref(pr), ctypes.byref(op), mu_local.data_ptr(), nu.data_ptr(),
            cost_local.data_ptr(), out_cost.data_ptr(), log_u.data_ptr(), log_v.data_ptr(),
            ctypes.byref(iters), residuals.data_ptr(), summer.fn, None, ws.data_ptr(),
            ws.numel(), _stream_handle(dev))
    if summer.error is not None:
        raise summer.error
    if st == _lib.STATUS_EXACT_NEEDED:
        return row_sharded_solve(mu_local, nu, CudaShardBackend(cost_local), lam, max_iters,
                                 tolerance, check_interval, group)
    raise_for_status(st, "sinkhorn_forward_rows_device_v1")
    # row residuals are per shard: the lane maximum over the ranks
    dist.all_reduce(residuals, op=dist.ReduceOp.MAX, group=group)
    kms, kn = -1.0, 0
    if time_kernel:
        n = ctypes.c_int32(0)
        kms, kn = float(lib.sinkhorn_last_kernel_ms_v1(ctypes.byref(n))), int(n.value)
    return SolveResult(out_cost, log_u, log_v, float(lam), int(iters.value), residuals,
                       float(lib.sinkhorn_last_loop_ms_v1()) if time_loop else -1.0,
                       "row-sharded-gemm", kms, kn)


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
    "CudaShardBackend", "batch_sharded_solve", "gather_lane_values", "global_max",
    "global_residual_reducer", "row_sharded_backward", "row_sharded_solve",
    "row_sharded_solve_device",
]
