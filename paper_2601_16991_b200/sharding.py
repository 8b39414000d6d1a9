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

__all__ = ["shard_cols", "stripe_widths", "gather_columns", "shard_adapters", "ShardedLinear", "ShardedStack"]


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


def gather_columns(local: torch.Tensor, n: int, group=None, keep: tuple[int, int] | None = None) -> torch.Tensor:
    """All-gather the column stripes of an (M x width_r) tensor into (M x n),
    or only the consumed columns ``keep = (a, b)`` into (M x (b - a)): every
    rank sends just its stripe's intersection with [a, b), so a consumer of
    part of a fused output (o reads the q columns of q|k|v) moves no more.

    One collective (``all_gather_into_tensor``) over pieces padded to the
    widest; the reassembly is a view + copy on the device."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    widths = stripe_widths(n, world)
    if local.shape[1] != widths[rank]:
        raise ValueError(f"local stripe width {local.shape[1]} != {widths[rank]}")
    if keep is not None:
        a, b = keep
        if not 0 <= a < b <= n:
            raise ValueError(f"keep range {keep} outside [0, {n})")
        ranges = [shard_cols(n, world, r) for r in range(world)]
        cuts = [(max(c0, a), min(c1, b)) for c0, c1 in ranges]
        c0 = ranges[rank][0]
        lo, hi = cuts[rank]
        piece = local[:, max(lo - c0, 0):max(hi - c0, 0)] if hi > lo else local[:, :0]
        pw = [max(h - l, 0) for l, h in cuts]
        return _gather_pieces(piece, pw, group)
    return _gather_pieces(local, widths, group)


def _gather_pieces(local: torch.Tensor, widths: list[int], group) -> torch.Tensor:
    import torch.distributed as dist

    world = len(widths)
    n = sum(widths)
    wmax = max(widths)
    m = local.shape[0]
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


def shard_adapters(fused, c0: int, c1: int):
    """The adapter factors of output columns [c0, c1): A_cat replicated,
    B_cat (scales folded in) cut with the columns."""
    from .fusion import FusedAdapters
    if fused is None:
        return None
    return FusedAdapters(a_cat=fused.a_cat, b_cat=fused.b_cat[:, c0:c1].contiguous(), offsets=fused.offsets,
                         ranks=fused.ranks)


class ShardedLinear:
    """One SALR linear column-sharded over the ranks of a process group:
    this rank's stripe of the weight (whole 128-column tiles, decoded only
    here) and of the adapters, plus the full output width for the gather."""

    def __init__(self, shard, fused_shard, n_full: int, world: int, rank: int):
        self.s, self.f, self.n, self.world, self.rank = shard, fused_shard, int(n_full), world, rank
        self.c0, self.c1 = shard_cols(self.n, world, rank)
        if shard.cols != self.c1 - self.c0:
            raise ValueError(f"shard has {shard.cols} columns, stripe is {self.c1 - self.c0}")

    @classmethod
    def from_full(cls, s, fused, world: int, rank: int):
        """Cut this rank's stripe out of a full matrix (``column_shard``)."""
        c0, c1 = shard_cols(s.cols, world, rank)
        return cls(s.column_shard(c0, c1), shard_adapters(fused, c0, c1), s.cols, world, rank)

    def local(self, x, out=None, pdl=False):
        from .pipeline import salr_linear
        return salr_linear(x, self.s, self.f, out=out, out_dtype=torch.bfloat16, check_finite=False, pdl=pdl)


class ShardedStack:
    """Decode-step forward of a column-sharded linear stack.

    ``layers`` is a list of ``{name: ShardedLinear}``; ``plan`` the chain of
    ``(name, input columns consumed from the previous output)`` per layer,
    e.g. ``[("qkv", None), ("o", (0, 4096)), ("gateup", None), ("down",
    (0, 14336))]`` for the Llama linear-only block: every rank runs its
    stripe with the fused kernel, then the stripes are all-gathered --
    only the columns the next linear consumes (o reads the q columns of
    q|k|v, down the gate columns of gate|up).  Everything runs on the
    current stream, so a whole step can be captured in one CUDA graph (NCCL
    collectives are graph-capturable); ``world == 1`` skips the gathers."""

    def __init__(self, layers, plan, world: int = 1, rank: int = 0, group=None, tokens: int = 1,
                 chain: bool | None = None):
        self.layers, self.plan, self.world, self.rank, self.group = layers, list(plan), world, rank, group
        # chain=True runs a layer as one persistent launch (salr_chain; single
        # GPU, decode-size M, each linear reading leading columns of the
        # previous output).  Off by default: measured slower than per-linear
        # launches (DESIGN.md 4.4 -- the split-K tails become L2 round trips
        # under the next linear's weight stream and gate every CTA).
        ok = world == 1 and tokens <= 256 and len(self.plan) <= 4 and all(
            keep is None or keep[0] == 0 for _, keep in self.plan[1:])
        self.chain = bool(chain) and ok
        first = layers[0][self.plan[0][0]]
        dev = first.s.device
        self.x_in = torch.zeros(tokens, first.s.rows, dtype=torch.bfloat16, device=dev)
        self.bufs = {name: [torch.empty(tokens, layers[0][name].s.cols, dtype=torch.bfloat16, device=dev)
                            for _ in range(2)] for name, _ in self.plan}
        self.launches_per_step = 0

    def _next_input(self, y, lin, keep):
        """The next linear's input: the consumed columns of this output."""
        if self.world == 1:
            return y if keep is None else y[:, keep[0]:keep[1]]
        return gather_columns(y, lin.n, group=self.group, keep=keep)

    def step(self, x):
        if self.chain:
            return self._step_chain(x)
        h = x
        launches = 0
        for li, layer in enumerate(self.layers):
            for j, (name, _) in enumerate(self.plan):
                lin = layer[name]
                y = lin.local(h, out=self.bufs[name][li & 1], pdl=self.world == 1)
                launches += 1
                keep = self.plan[j + 1][1] if j + 1 < len(self.plan) else self.plan[0][1]
                h = self._next_input(y, lin, keep)
        self.launches_per_step = launches
        return h

    def _step_chain(self, x):
        from .pipeline import salr_chain
        h = x
        for li, layer in enumerate(self.layers):
            outs = [self.bufs[name][li & 1] for name, _ in self.plan]
            salr_chain(h, [(layer[name].s, layer[name].f) for name, _ in self.plan], outs, pdl=True)
            last = outs[-1]
            keep = self.plan[0][1]
            h = last if keep is None else last[:, keep[0]:keep[1]]
        self.launches_per_step = len(self.layers)
        return h
