"""Adapters: the carrier type (``pkg/src/salr/residual.py:45-81``
``AdapterPair``), the truncated-SVD residual adapter that feeds ``fuse``
(``residual.py:138-173``) and its gradient-descent refinement
(``residual.py:231-349``), on the device.

The builder and the refinement are setup-time code:
E = W - W_hat is factored with cuSOLVER (``linalg.svd``, float64) instead of
the reference's Jacobi solver -- hours at 4096^2 in NumPy, seconds here --
and the refinement's products are float64 device GEMMs counted by
``linalg.matmul``.  Singular vectors are unique only up to sign, so parity
with the reference is on ``a @ b``, not on the factors."""

from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum

import torch

from .errors import ConfigError, DomainError, ShapeError, VerificationError
from .linalg import SvdResult, as_matrix, matmul, svd

__all__ = ["AdapterPair", "SV_CUTOFF_REL", "build_residual_adapter", "truncation_error_bound",
           "StepSizeMode", "ResidualTrainConfig", "lipschitz_constant", "power_iteration_sigma_max",
           "optimal_step_size", "residual_loss", "residual_gradient", "train_residual"]

SV_CUTOFF_REL = 1e-12  # residual.py:42


@dataclass(frozen=True)
class AdapterPair:
    """Low-rank factor pair; the effective update is ``scale * (a @ b)``.

    ``a`` is ``d_in x rank`` and ``b`` is ``rank x d_out`` (reference
    orientation), held as CUDA tensors: float64 when given float64 (the
    reference's precision, e.g. from :func:`build_residual_adapter`), else
    float32.  The linear kernel consumes them as bf16 operands (``fuse``).
    """

    a: torch.Tensor
    b: torch.Tensor
    rank: int
    scale: float = 1.0

    def __post_init__(self):
        a = as_matrix(self.a, "a")
        b = as_matrix(self.b, "b")
        dt = torch.float64 if (a.dtype == torch.float64 or b.dtype == torch.float64) else torch.float32
        a, b = a.to(dt), b.to(dt)
        object.__setattr__(self, "a", a)
        object.__setattr__(self, "b", b)
        if self.rank < 1:
            raise DomainError(f"rank must be >= 1, got {self.rank}")
        if a.shape[1] != self.rank or b.shape[0] != self.rank:
            raise ShapeError(f"factor shapes {tuple(a.shape)} x {tuple(b.shape)} do not match rank {self.rank}")
        if self.rank > min(a.shape[0], b.shape[1]):
            raise DomainError(f"rank {self.rank} exceeds min(d_in, d_out) = {min(a.shape[0], b.shape[1])}")

    @property
    def d_in(self) -> int:
        return int(self.a.shape[0])

    @property
    def d_out(self) -> int:
        return int(self.b.shape[1])

    def delta(self) -> torch.Tensor:
        """Dense update ``scale * a @ b`` (on the device)."""
        return self.scale * (self.a @ self.b)


# ---------------------------------------------------------------------------
# truncated-SVD residual adapter (residual.py:138-173)

def _checked_svd(e: torch.Tensor, svd_result: SvdResult | None) -> SvdResult:
    if svd_result is None:
        return svd(e)
    q = min(e.shape)
    u = as_matrix(svd_result.u, "svd_result.u", dtype=torch.float64)
    vt = as_matrix(svd_result.vt, "svd_result.vt", dtype=torch.float64)
    sv = torch.as_tensor(svd_result.s, dtype=torch.float64, device=e.device).reshape(-1)
    if tuple(u.shape) != (e.shape[0], q) or tuple(vt.shape) != (q, e.shape[1]):
        raise ShapeError("supplied svd_result does not match the matrix shape")
    return SvdResult(u=u, s=sv, vt=vt)


def build_residual_adapter(w, w_hat, rank: int, *, svd_result: SvdResult | None = None) -> AdapterPair:
    """Best rank-``rank`` factorization of ``E = w - w_hat`` (``residual.py:147-173``):
    ``a = U_r diag(s_r)``, ``b = Vt_r``; singular values below
    ``1e-12 * sigma_max`` are zeroed.  ``svd_result`` may carry a precomputed
    SVD of E (shape-checked, trusted otherwise)."""
    wm = as_matrix(w, "w", dtype=torch.float64)
    wh = as_matrix(w_hat, "w_hat", dtype=torch.float64)
    if wm.shape != wh.shape:
        raise ShapeError(f"w shape {tuple(wm.shape)} != w_hat shape {tuple(wh.shape)}")
    q = min(wm.shape)
    if not 1 <= rank <= q:
        raise DomainError(f"rank must be in [1, {q}], got {rank}")
    e = wm - wh
    res = _checked_svd(e, svd_result)
    sv = res.s[:rank].clone()
    cutoff = SV_CUTOFF_REL * (float(res.s[0]) if res.s.numel() else 0.0)
    sv[sv < cutoff] = 0.0
    a = res.u[:, :rank] * sv
    b = res.vt[:rank, :].clone()
    b[sv == 0.0, :] = 0.0
    return AdapterPair(a=a, b=b, rank=rank)


def truncation_error_bound(e, rank: int, *, svd_result: SvdResult | None = None) -> tuple[float, float]:
    """``(||E - E_r||_F^2 / dk, (1 - rank/q) ||E||_F^2 / dk)`` with the
    deterministic bound checked (``residual.py:176-205``)."""
    em = as_matrix(e, "e", dtype=torch.float64)
    q = min(em.shape)
    if not 1 <= rank <= q:
        raise DomainError(f"rank must be in [1, {q}], got {rank}")
    res = _checked_svd(em, svd_result)
    sq = res.s * res.s
    n = em.shape[0] * em.shape[1]
    lhs = float(sq[rank:].sum()) / n
    rhs = (1.0 - rank / q) * float(sq.sum()) / n
    if lhs > rhs * (1.0 + 1e-12) + 1e-300:
        raise VerificationError(f"rank-{rank} truncation error {lhs} exceeds bound {rhs}")
    return lhs, rhs


# ---------------------------------------------------------------------------
# gradient-descent refinement on the calibration loss (residual.py:98-136, 231-349)

class StepSizeMode(Enum):
    AUTO = "auto"
    AUTO_HALF = "auto-half"
    FIXED = "fixed"


@dataclass(frozen=True)
class ResidualTrainConfig:
    """Gradient-descent settings (``residual.py:104-135``)."""

    step_size_mode: StepSizeMode = StepSizeMode.AUTO_HALF
    step_size: float | None = None
    max_iters: int = 500
    grad_tol: float = 1e-8
    power_iters: int = 50

    def __post_init__(self):
        if self.step_size_mode is StepSizeMode.FIXED:
            if self.step_size is None or self.step_size <= 0.0:
                raise ConfigError("FIXED mode requires step_size > 0")
        elif self.step_size is not None:
            raise ConfigError("step_size is only meaningful in FIXED mode")
        if self.max_iters < 0:
            raise ConfigError("max_iters must be >= 0")
        if self.grad_tol < 0.0:
            raise ConfigError("grad_tol must be >= 0")
        if self.power_iters < 1:
            raise ConfigError("power_iters must be >= 1")


def lipschitz_constant(x) -> float:
    """``sigma_max(X)^2`` from the full SVD (``residual.py:231-235``)."""
    s = svd(as_matrix(x, "x", dtype=torch.float64)).s
    return float(s[0] * s[0])


def power_iteration_sigma_max(x, iters: int = 500, tol: float = 1e-13) -> float:
    """Largest singular value by power iteration on ``X^T X``
    (``linalg.py:252-281``); seeded start vector, deterministic."""
    a = as_matrix(x, "x", dtype=torch.float64)
    if iters < 1:
        raise DomainError("iters must be >= 1")
    g = torch.Generator(device="cpu").manual_seed(0x5EED)
    v = torch.randn(a.shape[1], generator=g, dtype=torch.float64).to(a.device)
    v = v / torch.linalg.vector_norm(v)
    sigma2 = 0.0
    for _ in range(iters):
        w = a.T @ (a @ v)
        nw = float(torch.linalg.vector_norm(w))
        if nw == 0.0:
            return 0.0
        sigma2_new = float(v @ w)
        v = w / nw
        if abs(sigma2_new - sigma2) <= tol * abs(sigma2_new):
            sigma2 = sigma2_new
            break
        sigma2 = sigma2_new
    return math.sqrt(max(sigma2, 0.0))


def optimal_step_size(x, power_iters: int = 50) -> float:
    """``1 / sigma_max(X)^2`` by power iteration (``residual.py:238-252``)."""
    if power_iters < 1:
        raise DomainError("power_iters must be >= 1")
    smax = power_iteration_sigma_max(x, iters=power_iters)
    if smax == 0.0:
        raise DomainError("step size undefined for zero X")
    return 1.0 / (smax * smax)


def _check_train_shapes(x, m, r_target):
    xm = as_matrix(x, "x", dtype=torch.float64)
    mm = as_matrix(m, "m", dtype=torch.float64)
    rm = as_matrix(r_target, "r_target", dtype=torch.float64)
    if xm.shape[1] != mm.shape[0]:
        raise ShapeError(f"x cols {xm.shape[1]} != m rows {mm.shape[0]}")
    if tuple(rm.shape) != (xm.shape[0], mm.shape[1]):
        raise ShapeError(f"r_target shape {tuple(rm.shape)} != expected {(xm.shape[0], mm.shape[1])}")
    return xm, mm, rm


def residual_loss(x, m, r_target) -> float:
    """``0.5 ||X M - R||_F^2`` (``residual.py:268-272``)."""
    xm, mm, rm = _check_train_shapes(x, m, r_target)
    diff = matmul(xm, mm) - rm
    return 0.5 * float((diff * diff).sum())


def residual_gradient(x, m, r_target) -> torch.Tensor:
    """``X^T (X M - R)`` (``residual.py:275-278``)."""
    xm, mm, rm = _check_train_shapes(x, m, r_target)
    return matmul(xm.T, matmul(xm, mm) - rm)


def train_residual(x, y, w_hat_dense, lora: AdapterPair, m0, cfg: ResidualTrainConfig,
                   final_rank: int | None = None):
    """Fit a dense correction M by gradient descent on the calibration loss
    (``residual.py:281-349``): target ``R = y - x @ (w_hat + lora.delta())``,
    ``M <- M - eta X^T (X M - R)`` until ``||grad||_F <= grad_tol`` or
    ``max_iters``.  Returns ``(m, loss_trace)`` (device tensor, host list);
    ``final_rank`` re-truncates M through :func:`build_residual_adapter`."""
    xm = as_matrix(x, "x", dtype=torch.float64)
    ym = as_matrix(y, "y", dtype=torch.float64)
    wh = as_matrix(w_hat_dense, "w_hat_dense", dtype=torch.float64)
    if lora.d_in != wh.shape[0] or lora.d_out != wh.shape[1]:
        raise ShapeError(f"adapter dims {(lora.d_in, lora.d_out)} != weight shape {tuple(wh.shape)}")
    r_target = ym - matmul(xm, wh + lora.scale * matmul(lora.a, lora.b))
    m = as_matrix(m0, "m0", dtype=torch.float64).clone()
    _check_train_shapes(xm, m, r_target)
    if cfg.step_size_mode is StepSizeMode.FIXED:
        lip = lipschitz_constant(xm)
        if lip > 0.0 and cfg.step_size >= 2.0 / lip:
            raise ConfigError(f"fixed step {cfg.step_size} >= divergence threshold {2.0 / lip}")
        eta = cfg.step_size
    else:
        smax = power_iteration_sigma_max(xm, iters=cfg.power_iters)
        if smax == 0.0:
            raise DomainError("step size undefined for zero X")
        eta = 1.0 / (smax * smax)
        if cfg.step_size_mode is StepSizeMode.AUTO_HALF:
            eta *= 0.5
    trace = [residual_loss(xm, m, r_target)]
    for _ in range(cfg.max_iters):
        grad = residual_gradient(xm, m, r_target)
        if float(torch.linalg.vector_norm(grad)) <= cfg.grad_tol:
            break
        m -= eta * grad
        trace.append(residual_loss(xm, m, r_target))
    if final_rank is not None:
        pair = build_residual_adapter(m, torch.zeros_like(m), final_rank)
        m = matmul(pair.a, pair.b)
    return m, trace
