"""Adapter carrier type (``pkg/src/salr/residual.py:45-81`` ``AdapterPair``).

The SVD-residual builder and the residual-training math of the reference
module are setup/offline code outside the hot path (SURVEY.md section 2,
rows 11-12) and are not part of this package."""

from __future__ import annotations

from dataclasses import dataclass

import torch

from .errors import DomainError, ShapeError
from .linalg import as_matrix

__all__ = ["AdapterPair"]


@dataclass(frozen=True)
class AdapterPair:
    """Low-rank factor pair; the effective update is ``scale * (a @ b)``.

    ``a`` is ``d_in x rank`` and ``b`` is ``rank x d_out`` (reference
    orientation); both are held as float32 CUDA tensors.
    """

    a: torch.Tensor
    b: torch.Tensor
    rank: int
    scale: float = 1.0

    def __post_init__(self):
        a = as_matrix(self.a, "a", dtype=torch.float32)
        b = as_matrix(self.b, "b", dtype=torch.float32)
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
        """Dense update ``scale * a @ b`` (float32, on the device)."""
        return self.scale * (self.a @ self.b)
