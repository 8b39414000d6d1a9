"""Multi-rank host logic of the column-sharded stack, on CPU with gloo
(world sizes 2 and 3): stripe math, padded all-gather reassembly, and that a
column-sharded linear chain equals the unsharded one (dense fp64 stand-in for
the per-rank linear -- the CUDA kernel itself is covered by the GPU tests)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2601_16991_b200.sharding import gather_columns, shard_cols, stripe_widths


def test_stripes_cover_columns_in_tile_units():
    for n in (1024, 4096, 6144, 14336, 130, 1):
        for world in (1, 2, 3, 4, 8):
            ranges = [shard_cols(n, world, r) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            for (a0, a1), (b0, b1) in zip(ranges, ranges[1:]):
                assert a1 == b0
            for c0, c1 in ranges[:-1]:
                assert c0 % 128 == 0 and c1 % 128 == 0
            assert sum(stripe_widths(n, world)) == n
    # k/v at 8 GPUs: exactly one 128-column tile each
    assert stripe_widths(1024, 8) == [128] * 8
    with pytest.raises(ValueError):
        shard_cols(128, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        g = torch.Generator().manual_seed(0)
        m = 5
        # a 3-linear chain with layer-boundary gathers: 256 -> 1024 -> 384 -> 256
        dims = [256, 1024, 384, 256]
        ws = [torch.randn(dims[i], dims[i + 1], generator=g, dtype=torch.float64) for i in range(3)]
        x = torch.randn(m, dims[0], generator=g, dtype=torch.float64)
        ref = x
        for w in ws:
            ref = ref @ w
        h = x
        for w in ws:
            n = w.shape[1]
            c0, c1 = shard_cols(n, world, rank)
            local = h @ w[:, c0:c1]            # the rank decodes only its stripe
            h = gather_columns(local, n)       # NCCL on the GPU path, gloo here
        ok = torch.allclose(h, ref, rtol=1e-12, atol=1e-12) and h.shape == ref.shape
        dist.destroy_process_group()
        q.put((rank, bool(ok), None))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, False, repr(e)))


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_chain_matches_unsharded(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, err in results:
        assert ok, (rank, err)
