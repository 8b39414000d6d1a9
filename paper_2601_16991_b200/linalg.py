"""Input coercion, the counted matrix product and the SVD hook, with the
reference's semantics (``pkg/src/salr/linalg.py``): ``as_matrix``
(``linalg.py:52-69``: 2-D, non-empty, finite, else ShapeError /
DomainError), ``matmul`` with its instrumentation counter
(``linalg.py:75-108``) and the ``SvdResult`` carrier (``linalg.py:116-126``).
Arrays become CUDA tensors; nothing is computed on the host.  Products run
in float64 on the device (cuBLAS DGEMM), the reference's arithmetic."""

from __future__ import annotations

import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import DomainError, ShapeError

__all__ = ["as_matrix", "to_cuda", "matmul", "matmul_call_count", "reset_matmul_count", "SvdResult", "svd"]


def to_cuda(x, dtype: torch.dtype | None = None) -> torch.Tensor:
    dev = _lib.require_cuda()
    if isinstance(x, torch.Tensor):
        t = x
    else:
        a = np.asarray(x)
        if a.dtype == np.float16 or a.dtype.kind not in "fiub":
            a = a.astype(np.float64)
        t = torch.from_numpy(np.ascontiguousarray(a))
    if t.dtype not in (torch.float32, torch.float64, torch.bfloat16):
        t = t.to(torch.float64)
    t = t.to(device=dev, dtype=dtype or t.dtype, non_blocking=True)
    return t.contiguous()


def as_matrix(x, name: str = "matrix", require_finite: bool = True,
              dtype: torch.dtype | None = None) -> torch.Tensor:
    """Coerce to a contiguous 2-D CUDA tensor (float64/float32/bf16 kept
    unless ``dtype`` is given).  Mirrors ``linalg.py:52-69``."""
    t = to_cuda(x, dtype)
    if t.dim() != 2:
        raise ShapeError(f"{name} must be 2-D, got ndim={t.dim()}")
    if t.shape[0] < 1 or t.shape[1] < 1:
        raise ShapeError(f"{name} must have at least one row and one column")
    if require_finite and not bool(torch.isfinite(t).all()):
        raise DomainError(f"{name} contains non-finite entries")
    return t


# ---------------------------------------------------------------------------
# matmul with an instrumentation counter (linalg.py:75-108)

_matmul_lock = threading.Lock()
_matmul_calls = 0


def matmul(a, b) -> torch.Tensor:
    """Matrix product in float64 on the device; increments the module-level
    product counter (:func:`matmul_call_count` / :func:`reset_matmul_count`),
    so a code path's product count can be asserted as in the reference."""
    global _matmul_calls
    am = as_matrix(a, "a", dtype=torch.float64)
    bm = as_matrix(b, "b", dtype=torch.float64)
    if am.shape[1] != bm.shape[0]:
        raise ShapeError(f"inner dimensions differ: a is {am.shape[0]}x{am.shape[1]}, "
                         f"b is {bm.shape[0]}x{bm.shape[1]}")
    with _matmul_lock:
        _matmul_calls += 1
    return am @ bm


def matmul_call_count() -> int:
    """Number of products issued through :func:`matmul` since the last reset."""
    with _matmul_lock:
        return _matmul_calls


def reset_matmul_count() -> None:
    global _matmul_calls
    with _matmul_lock:
        _matmul_calls = 0


# ---------------------------------------------------------------------------
# SVD (linalg.py:116-126 carrier; the reference's Jacobi solver is replaced by
# cuSOLVER through torch.linalg.svd -- setup code, not the hot path)

@dataclass(frozen=True)
class SvdResult:
    """Thin SVD ``m = u @ diag(s) @ vt`` with descending ``s``."""

    u: torch.Tensor
    s: torch.Tensor
    vt: torch.Tensor


def svd(m) -> SvdResult:
    """Thin SVD in float64 on the device (cuSOLVER); singular values
    descending, as the reference's ``svd`` returns them."""
    mm = as_matrix(m, "m", dtype=torch.float64)
    u, s, vt = torch.linalg.svd(mm, full_matrices=False)
    return SvdResult(u=u, s=s, vt=vt)
