"""Column sharding of SALR linears across the GPUs of one node.

Output columns of a linear are independent (bitmap bits run along N,
reference ``bitmap.py:4-6``), so rank ``r`` of ``world`` owns a contiguous,
128-column-aligned stripe of every weight and decodes only its own TB tiles;
X and A_cat are replicated, B_cat is split with the columns.  The stripes are
all-gathered at layer boundaries.  Stripes can be unequal (e.g. 1024 columns
= 8 tiles over 3 ranks); the gather pads every stripe to the widest one.
"""

from __future__ import annotations

import torch

TILE_N = 128

__all__ = ["shard_cols", "stripe_widths", "gather_columns"]


def shard_cols(n: int, world: int, rank: int) -> tuple[int, int]:
    """Column range [c0, c1) of rank ``rank``: whole 128-column tiles split as
    evenly as possible, in rank order."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    tiles = (n + TILE_N - 1) // TILE_N
    t0 = tiles * rank // world
    t1 = tiles * (rank + 1) // world
    return min(TILE_N * t0, n), min(TILE_N * t1, n)


def stripe_widths(n: int, world: int) -> list[int]:
    return [c1 - c0 for c0, c1 in (shard_cols(n, world, r) for r in range(world))]


def gather_columns(local: torch.Tensor, n: int, group=None) -> torch.Tensor:
    """All-gather the column stripes of an (M x width_r) tensor into (M x n).

    One collective (``all_gather_into_tensor``) over stripes padded to the
    widest; the reassembly is a view + copy on the device."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    widths = stripe_widths(n, world)
    wmax = max(widths)
    m = local.shape[0]
    if local.shape[1] != widths[dist.get_rank(group)]:
        raise ValueError(f"local stripe width {local.shape[1]} != {widths[dist.get_rank(group)]}")
    if local.shape[1] != wmax:
        padded = local.new_zeros((m, wmax))
        padded[:, : local.shape[1]] = local
    else:
        padded = local.contiguous()
    flat = local.new_empty((world * m, wmax))  # dim-0 concatenation (NCCL and gloo)
    dist.all_gather_into_tensor(flat, padded, group=group)
    buf = flat.view(world, m, wmax)
    if all(w == wmax for w in widths):
        return buf.permute(1, 0, 2).reshape(m, world * wmax)[:, :n]
    return torch.cat([buf[r, :, : widths[r]] for r in range(world)], dim=1)
