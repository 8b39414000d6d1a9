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


# ---------------------------------------------------------------- product shard slicing (TB2 records on CPU)

def _bf16_exact(a):
    return torch.from_numpy(a).bfloat16().float().numpy()


def _tb2_matrix(dense):
    from paper_2601_16991_b200 import BitmapSparseMatrix
    from tb2_cpu import tb2_records
    rec, off = tb2_records(dense)
    return BitmapSparseMatrix.from_compute_format(dense.shape[0], dense.shape[1], torch.from_numpy(rec),
                                                  torch.from_numpy(off))


@pytest.mark.parametrize("cols,c0,c1", [(384, 128, 384), (300, 256, 300), (300, 0, 128), (512, 128, 256)])
def test_column_shard_is_bit_exact(cols, c0, c1):
    """column_shard of the TB2 records == TB2 records of the sliced matrix,
    byte for byte (offsets rebased, nnz from the tile headers)."""
    import numpy as np
    from tb2_cpu import tb2_records
    rng = np.random.default_rng(cols + c0)
    w = _bf16_exact(rng.normal(scale=0.02, size=(130, cols)).astype(np.float32))
    w[rng.random(w.shape) < 0.5] = 0.0
    s = _tb2_matrix(w)
    assert s.nnz == int((w != 0).sum())
    sh = s.column_shard(c0, c1)
    rec, off = tb2_records(np.ascontiguousarray(w[:, c0:c1]))
    r2, o2, mx = sh.compute_format()
    assert torch.equal(r2, torch.from_numpy(rec)) and torch.equal(o2, torch.from_numpy(off))
    assert sh.nnz == int((w[:, c0:c1] != 0).sum()) and (sh.rows, sh.cols) == (130, c1 - c0)
    from paper_2601_16991_b200.errors import ShapeError
    with pytest.raises(ShapeError):
        s.column_shard(64, 128)  # not a whole-tile stripe


def _shard_worker(rank, world, port, q):
    try:
        import numpy as np
        from tb2_cpu import tb2_decode
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        rng = np.random.default_rng(5)
        k, n, m = 96, 640, 3
        w = _bf16_exact(rng.normal(scale=0.02, size=(k, n)).astype(np.float32))
        w[rng.random(w.shape) < 0.5] = 0.0
        x = rng.normal(size=(m, k))
        full = _tb2_matrix(w)  # every rank holds the encoded matrix; decodes only its stripe
        c0, c1 = shard_cols(n, world, rank)
        sh = full.column_shard(c0, c1)
        r2, o2, _ = sh.compute_format()
        local = torch.from_numpy(x @ tb2_decode(r2.numpy(), o2.numpy(), k, c1 - c0).astype(np.float64))
        y = gather_columns(local, n)
        part = gather_columns(local, n, keep=(100, 530))  # consumed columns only
        ref = torch.from_numpy(x @ w.astype(np.float64))
        ok = torch.allclose(y, ref, rtol=1e-12, atol=1e-12) and torch.equal(part, y[:, 100:530])
        dist.destroy_process_group()
        q.put((rank, bool(ok), None))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, False, traceback.format_exc()))


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_tb2_linear_matches_unsharded(world):
    """Each rank cuts its stripe out of the encoded matrix (column_shard),
    expands only that stripe, and the all-gathered outputs (full, and the
    consumed-columns gather) equal the unsharded product."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, err in results:
        assert ok, (rank, err)
