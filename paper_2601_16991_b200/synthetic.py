"""Seeded synthetic inputs for the SALR linear (harness helper, not the hot path).

Every tensor is generated on the CPU with ``torch.Generator().manual_seed``
and rounded to bf16-exact float32, so the same bits can be fed to the
reference/oracle (as float64) and to the B200 path (as bf16).  Distributions
follow SURVEY.md section 8(d): W ~ N(0, 0.02^2), X ~ N(0, 1), LoRA
A ~ N(0, 1/d_in), B ~ N(0, 0.02^2), scale 2.0.

Shapes use the reference orientation: a weight is (d_in, d_out) = (K, N) and
``y = x @ w`` (reference ``fusion.py:109-130``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch

__all__ = ["LLAMA3_8B_LINEARS", "bf16_exact", "gen_weight", "gen_x", "gen_lora",
           "gen_adapter_pair", "magnitude_prune_gpu", "LinearInputs", "gen_linear"]

# Llama3-8B per-layer linears, (d_in, d_out) reference orientation.
LLAMA3_8B_LINEARS = {
    "q": (4096, 4096),
    "k": (4096, 1024),
    "v": (4096, 1024),
    "o": (4096, 4096),
    "gate": (4096, 14336),
    "up": (4096, 14336),
    "down": (14336, 4096),
}


def bf16_exact(t: torch.Tensor) -> torch.Tensor:
    """Round to bf16 and back to float32 (every value exactly representable)."""
    return t.to(torch.bfloat16).to(torch.float32)


def _gen(seed: int) -> torch.Generator:
    return torch.Generator(device="cpu").manual_seed(int(seed))


def gen_weight(k: int, n: int, seed: int, std: float = 0.02) -> torch.Tensor:
    return bf16_exact(torch.randn(k, n, generator=_gen(seed)) * std)


def gen_x(m: int, k: int, seed: int = 7) -> torch.Tensor:
    return bf16_exact(torch.randn(m, k, generator=_gen(seed)))


def gen_lora(k: int, n: int, rank: int, seed: int):
    g = _gen(seed)
    a = bf16_exact(torch.randn(k, rank, generator=g) / math.sqrt(k))
    b = bf16_exact(torch.randn(rank, n, generator=g) * 0.02)
    return a, b


def gen_adapter_pair(k: int, n: int, rank: int, seed: int, std_b: float = 0.02):
    """Random stand-in for a residual adapter (bench only; parity uses real SVD)."""
    return gen_lora(k, n, rank, seed)


def magnitude_prune_gpu(w: torch.Tensor, sparsity: float) -> torch.Tensor:
    """Zero the smallest-|w| fraction ``sparsity`` of entries (bench helper).

    Threshold by ``kthvalue`` of |w| on the device.  Ties at the threshold are
    resolved arbitrarily, so the kept count can differ from the reference's
    stable top-k (``prune.py:215-255``) by the number of ties; parity tests use
    the oracle's exact ``build_mask`` instead.
    """
    flat = w.abs().flatten().float()
    n_drop = int(round(sparsity * flat.numel()))
    if n_drop <= 0:
        return w.clone()
    thr = torch.kthvalue(flat.cpu() if not flat.is_cuda else flat, n_drop).values
    return torch.where(w.abs() > thr.to(w.device), w, torch.zeros_like(w))


@dataclass
class LinearInputs:
    w_hat: torch.Tensor        # (K, N) float32, bf16-exact, pruned
    lora_a: torch.Tensor       # (K, r) float32
    lora_b: torch.Tensor       # (r, N) float32
    res_a: torch.Tensor        # (K, r) float32
    res_b: torch.Tensor        # (r, N) float32
    lora_scale: float


def gen_linear(k: int, n: int, seed: int, sparsity: float = 0.5, r_lora: int = 16,
               r_res: int = 16, device: str = "cpu") -> LinearInputs:
    """Bench-sized synthetic SALR linear: pruned base + LoRA + residual stand-in."""
    w = gen_weight(k, n, seed)
    w_dev = w.to(device)
    w_hat = magnitude_prune_gpu(w_dev, sparsity)
    la, lb = gen_lora(k, n, r_lora, seed + 100_000)
    ra, rb = gen_adapter_pair(k, n, r_res, seed + 200_000)
    return LinearInputs(w_hat, la.to(device), lb.to(device), ra.to(device), rb.to(device), 2.0)
