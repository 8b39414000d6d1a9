"""Input coercion with the reference's validation semantics
(``pkg/src/salr/linalg.py:52-69`` ``as_matrix``): 2-D, non-empty, finite,
else ShapeError / DomainError.  Arrays become CUDA tensors; nothing is
computed on the host."""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .errors import DomainError, ShapeError

__all__ = ["as_matrix", "to_cuda"]


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
