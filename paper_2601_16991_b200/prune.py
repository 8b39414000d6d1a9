"""Magnitude-prune masks on the B200, API-compatible with the reference
``pkg/src/salr/prune.py`` (``PruneMethod``, ``PruneConfig``, ``kept_count``,
``build_mask``: 145-255).

Global methods keep exactly ``kept_count(p, rows*cols)`` entries with the
reference's tie rule (equal magnitudes go to the lower row-major index);
the selection is the hand-written radix select of ``csrc/salr_prune.cu``
(``salr_topk_mask``), so masks are identical to the reference's stable
argsort, bit for bit.  N:M keeps the ``n`` largest of every contiguous group
of ``m`` columns (``salr_nm_mask``).  Scores are ``|W0|`` (static) or
``|W0 + Delta|`` (dynamic methods), in float64 like the reference."""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import torch

from . import _lib
from .bitmap import kept_count
from .errors import ConfigError, DomainError, ShapeError
from .linalg import as_matrix

__all__ = ["PruneMethod", "PruneConfig", "kept_count", "build_mask", "prune"]


class PruneMethod(Enum):
    """Masking strategy (``prune.py:58-64``); values double as CLI spellings."""

    STATIC_ON_W0 = "static"
    DYNAMIC_MASK_PRUNE_W0 = "dynamic-w0"
    DYNAMIC_ON_U = "dynamic-u"
    SEMI_STRUCTURED_NM = "nm"


@dataclass(frozen=True)
class PruneConfig:
    """Pruning parameters (``prune.py:67-100``), same validation."""

    sparsity: float
    method: PruneMethod = PruneMethod.STATIC_ON_W0
    nm: tuple | None = None
    sigma: float = 1.0
    tau: float = 0.0

    def __post_init__(self):
        if not 0.0 <= self.sparsity < 1.0:
            raise DomainError(f"sparsity must be in [0, 1), got {self.sparsity}")
        if self.sigma <= 0.0:
            raise DomainError(f"sigma must be > 0, got {self.sigma}")
        if self.tau < 0.0:
            raise DomainError(f"tau must be >= 0, got {self.tau}")
        if self.method is PruneMethod.SEMI_STRUCTURED_NM:
            if self.nm is None:
                raise ConfigError("SEMI_STRUCTURED_NM requires nm=(n, m)")
            n, m = self.nm
            if not 0 < n < m:
                raise ConfigError(f"nm requires 0 < n < m, got {self.nm}")
        elif self.nm is not None:
            raise ConfigError("nm is only meaningful with SEMI_STRUCTURED_NM")


def _scores_ptr(scores: torch.Tensor):
    code = {torch.float32: _lib.F32, torch.float64: _lib.F64}[scores.dtype]
    return _lib.ptr(scores), code


def build_mask(w0, delta, cfg: PruneConfig) -> torch.Tensor:
    """Boolean keep-mask (True = kept) on the device (``prune.py:224-255``)."""
    w0m = as_matrix(w0, "w0")
    dm = as_matrix(delta, "delta")
    if w0m.shape != dm.shape:
        raise ShapeError(f"w0 shape {tuple(w0m.shape)} != delta shape {tuple(dm.shape)}")
    rows, cols = (int(d) for d in w0m.shape)
    lib = _lib.load()
    st = _lib.stream_ptr()
    mask = torch.empty((rows, cols), dtype=torch.uint8, device=w0m.device)
    if cfg.method is PruneMethod.SEMI_STRUCTURED_NM:
        n, m = cfg.nm
        if cols % m != 0:
            raise ConfigError(f"group size m={m} must divide cols={cols}")
        if m > 64:
            raise ConfigError(f"group size m={m} above the device limit 64")
        scores = w0m.double().abs().contiguous()
        p, code = _scores_ptr(scores)
        _lib.check(lib.salr_nm_mask(p, code, rows, cols, int(n), int(m), _lib.ptr(mask), st))
        return mask.bool()
    if cfg.method is PruneMethod.STATIC_ON_W0:
        scores = w0m.double().abs()
    else:
        scores = (w0m.double() + dm.double()).abs()
    scores = scores.contiguous()
    keep = kept_count(cfg.sparsity, rows * cols)
    need = int(lib.salr_topk_mask_workspace_bytes(rows * cols))
    ws = torch.empty(need, dtype=torch.uint8, device=w0m.device)
    p, code = _scores_ptr(scores)
    _lib.check(lib.salr_topk_mask(p, code, rows * cols, keep, _lib.ptr(mask), _lib.ptr(ws), need, st))
    return mask.bool()


def prune(w0, cfg: PruneConfig, delta=None) -> torch.Tensor:
    """``W_hat``: the static mask applied to ``w0`` (zeros elsewhere), same dtype."""
    w = as_matrix(w0, "w0")
    d = torch.zeros_like(w) if delta is None else delta
    return torch.where(build_mask(w, d, cfg), w, torch.zeros_like(w))
