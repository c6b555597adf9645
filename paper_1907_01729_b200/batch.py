"""Mirror of the reference batch engine's public API (pkg/src/sinkloss/batch.py).

Same names, argument meaning and error behaviour as ``sinkloss``'s
``batch_forward`` / ``batch_backward`` / ``fused_log_reduction`` /
``SinkhornConfig``, executed by the sm_100a kernels.  Results are float32
CUDA tensors; ``workers`` is accepted for signature compatibility (the
reference's span threads, batch.py:256-261, have no GPU counterpart: the
reduction split is the kernel's stream-K schedule).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import torch

from . import _lib
from .errors import InvalidConfig, ShapeMismatch, ZeroMassGradient, raise_for_status
from .loss import GridCost, SolveResult, _as_f32_cuda, _ptr, _stream_handle, \
    potentials_backward, solve


@dataclass(frozen=True)
class SinkhornConfig:
    """Solver parameters with the reference's defaults and validation (core.py:74-96)."""

    lam: float
    max_iters: int = 1000
    tolerance: float = 1e-9
    check_interval: int = 10

    def __post_init__(self):
        if not (math.isfinite(self.lam) and self.lam > 0):
            raise InvalidConfig(f"lam must be positive and finite, got {self.lam}")
        if self.max_iters < 1:
            raise InvalidConfig(f"max_iters must be >= 1, got {self.max_iters}")
        if not (math.isfinite(self.tolerance) and self.tolerance >= 0):
            raise InvalidConfig(f"tolerance must be >= 0, got {self.tolerance}")
        if self.check_interval < 1:
            raise InvalidConfig(f"check_interval must be >= 1, got {self.check_interval}")


BatchLossResult = SolveResult


def _mass(x):
    return getattr(x, "mass", x)


def _cost(c):
    if isinstance(c, GridCost):
        return c
    return getattr(c, "cost", c)


def batch_forward(mu, nu, c, config: SinkhornConfig, workers: int | None = None,
                  validate: bool = True) -> BatchLossResult:
    """All lanes in lockstep (batch.py:264-349): per-lane E0, final potentials,
    the common iteration count and per-lane residuals."""
    if workers is not None and workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    return solve(_mass(mu), _mass(nu), _cost(c), config.lam, config.max_iters,
                 config.tolerance, config.check_interval, validate=validate)


def batch_backward(result: BatchLossResult, upstream):
    """Mean-zero gradients scaled by the upstream cotangent (batch.py:352-375)."""
    up = torch.as_tensor(upstream)
    B = result.cost_e0.shape[0]
    if tuple(up.shape) != (B,):
        raise ShapeMismatch(f"upstream must have shape ({B},), got {tuple(up.shape)}")
    return potentials_backward(result.log_u, result.log_v, result.lam, up)


def fused_log_reduction(log_u, c, lam: float, log_nu, workers: int = 1) -> torch.Tensor:
    """out[b, j] = log_nu[b, j] - logsumexp_i(-c[i, j]/lam + log_u[b, i]) (batch.py:208-230)."""
    log_u = _as_f32_cuda(log_u)
    dev = log_u.device
    log_nu = _as_f32_cuda(log_nu, dev)
    c = _as_f32_cuda(_cost(c), dev)
    _check_half(log_u, c, log_nu)
    B, d1 = log_u.shape
    d2 = c.shape[1]
    out = torch.empty(B, d2, device=dev, dtype=torch.float32)
    _half_sweep(log_u, c, lam, log_nu, out, None, None)
    return out


def partial_log_reduction(log_x, c, lam: float) -> tuple[torch.Tensor, torch.Tensor]:
    """The (max, sum) accumulator pairs of one half-sweep, log base 2:
    logsumexp_i(-c/lam + log_x) = ln2 * (max + log2(sum)).

    This is the partial state a row-sharded solve merges across GPUs with
    OnlineLseAccumulator.merge semantics (batch.py:116-130)."""
    log_x = _as_f32_cuda(log_x)
    dev = log_x.device
    c = _as_f32_cuda(_cost(c), dev)
    if log_x.dim() != 2 or c.dim() != 2 or log_x.shape[1] != c.shape[0]:
        raise ShapeMismatch("log_x (B, d1) must match cost (d1, d2)")
    B = log_x.shape[0]
    d2 = c.shape[1]
    m = torch.empty(B, d2, device=dev, dtype=torch.float32)
    s = torch.empty(B, d2, device=dev, dtype=torch.float32)
    _half_sweep(log_x, c, lam, None, None, m, s)
    return m, s


def e0_partial_log2(log_u, log_v, c, lam: float) -> torch.Tensor:
    """Per-lane log2 sum_{i,j} P_ij c_ij over the rows of `c` (a row shard);
    E0 = 2^(LSE over shards) (batch.py:331-337)."""
    log_u = _as_f32_cuda(log_u)
    dev = log_u.device
    log_v = _as_f32_cuda(log_v, dev)
    c = _as_f32_cuda(_cost(c), dev)
    if log_u.dim() != 2 or log_v.dim() != 2 or c.dim() != 2 or \
            tuple(c.shape) != (log_u.shape[1], log_v.shape[1]) or log_u.shape[0] != log_v.shape[0]:
        raise ShapeMismatch("e0_partial_log2: log_u (B,d1), log_v (B,d2), cost (d1,d2)")
    if not (math.isfinite(lam) and lam > 0):
        raise InvalidConfig(f"lam must be positive and finite, got {lam}")
    B, d1 = log_u.shape
    d2 = log_v.shape[1]
    out = torch.empty(B, device=dev, dtype=torch.float32)
    lib = _lib.load()
    with torch.cuda.device(dev):
        nbytes = lib.sinkhorn_half_sweep_workspace_bytes_v1(B, d1, d2)
        ws = torch.empty(max(nbytes, 256), device=dev, dtype=torch.uint8)
        st = lib.sinkhorn_e0_partial_device_v1(B, d1, d2, float(lam), _ptr(log_u), _ptr(log_v),
                                               _ptr(c), _ptr(out), _ptr(ws), ws.numel(),
                                               _stream_handle(dev))
    raise_for_status(st, "sinkhorn_e0_partial_device_v1")
    return out


def _check_half(log_u, c, log_nu):
    if log_u.dim() != 2 or log_nu.dim() != 2:
        raise ShapeMismatch("log_u and log_nu must be 2-D (batch, dim)")
    if log_u.shape[0] != log_nu.shape[0]:
        raise ShapeMismatch(f"batch sizes differ: {log_u.shape[0]} vs {log_nu.shape[0]}")
    if c.dim() != 2 or log_u.shape[1] != c.shape[0] or log_nu.shape[1] != c.shape[1]:
        raise ShapeMismatch(f"cost is {tuple(c.shape)} but potentials have "
                            f"d1={log_u.shape[1]}, d2={log_nu.shape[1]}")


def _half_sweep(log_x, c, lam, target, out, m, s):
    if not (math.isfinite(lam) and lam > 0):
        raise InvalidConfig(f"lam must be positive and finite, got {lam}")
    lib = _lib.load()
    dev = log_x.device
    B, d1 = log_x.shape
    d2 = c.shape[1]
    with torch.cuda.device(dev):
        nbytes = lib.sinkhorn_half_sweep_workspace_bytes_v1(B, d1, d2)
        ws = torch.empty(max(nbytes, 256), device=dev, dtype=torch.uint8)
        st = lib.sinkhorn_half_sweep_device_v1(B, d1, d2, float(lam), _ptr(log_x), _ptr(c),
                                               _ptr(target), _ptr(out), _ptr(m), _ptr(s),
                                               _ptr(ws), ws.numel(), _stream_handle(dev))
    raise_for_status(st, "sinkhorn_half_sweep_device_v1")


__all__ = [
    "BatchLossResult", "GridCost", "SinkhornConfig", "ZeroMassGradient", "batch_backward",
    "batch_forward", "fused_log_reduction", "partial_log_reduction",
]

_ = ctypes  # ctypes is used through _lib
