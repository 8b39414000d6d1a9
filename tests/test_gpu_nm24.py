"""NM24: the 2:4 compute format.  Matrices pruned with the
reference's N:M rule (prune.py:238-248, device mask pinned by the prune
goldens) are re-encoded as fixed 9216-byte tiles; the codec matches the CPU
restatement byte for byte, and the linear kernel's NM24 decoder produces the
same dense tiles as the bitmap decoder, so every forward is BIT-IDENTICAL to
the TB2 path (itself pinned to the reference's pipelined_forward)."""

import numpy as np
import pytest
import torch

from nm24_cpu import nm24_records

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    import paper_2601_16991_b200 as S
    return S


def _w24(S, k, n, seed, zero_frac=0.02):
    g = torch.Generator().manual_seed(seed)
    w = (torch.randn(k, n, generator=g, dtype=torch.float64) * 0.02).float().bfloat16().float().cuda()
    cfg = S.PruneConfig(0.5, S.PruneMethod.SEMI_STRUCTURED_NM, nm=(2, 4))
    w = S.prune(w, cfg)
    w[torch.rand(k, n, generator=g).cuda() < zero_frac] = 0  # kept entries that are exactly zero
    return w


def _adapters(S, k, n, seed, r=16):
    g = torch.Generator().manual_seed(seed)
    return S.fuse([S.AdapterPair((torch.randn(k, r, generator=g) / 64).bfloat16().float(),
                                 (torch.randn(r, n, generator=g) * 0.02).bfloat16().float(), r, sc)
                   for sc in (1.0, 0.5)])


@pytest.mark.parametrize("shape", [(64, 128), (200, 300), (1000, 1500)])
def test_codec_matches_cpu_restatement(S, shape):
    w = _w24(S, *shape, seed=sum(shape))
    s = S.encode(w, value_dtype="bf16")
    assert not s.is_nm24()
    s.use_nm24()
    assert s.is_nm24() and s.records is None and s._tb2 is None  # the one resident format
    want = nm24_records(w.cpu().numpy())
    assert np.array_equal(s._nm24.cpu().numpy(), want)
    assert torch.equal(s._nm24_dense().float(), w)
    assert torch.equal(S.decode(s), w)           # TB rebuilt on demand
    t = S.encode(w, value_dtype="bf16")
    assert torch.equal(s.bitmap, t.bitmap) and torch.equal(s.values, t.values) and s.nnz == t.nnz
    assert s.device_bytes == 9216 * s.n_tiles


def test_rejects_unstructured(S):
    g = torch.Generator().manual_seed(3)
    w = torch.randn(128, 256, generator=g).bfloat16().float().cuda()
    w[torch.rand(128, 256, generator=g).cuda() < 0.5] = 0
    s = S.encode(w, value_dtype="bf16")
    with pytest.raises(S.FormatError):
        s.use_nm24()
    assert not s.is_nm24() and torch.equal(S.decode(s), w)  # unchanged


def test_f32_matrix_keeps_reference_values(S):
    w = _w24(S, 256, 512, 5)
    s = S.encode(w)  # float32 values
    s.use_nm24()
    assert s.is_nm24() and s.records is not None
    assert torch.equal(S.decode(s), w)


@pytest.mark.parametrize("M", [1, 8, 16, 32, 100, 300])
@pytest.mark.parametrize("adapters", [True, False])
def test_forward_bitwise_equal_tb2(S, M, adapters):
    k, n = 1000, 1500  # ragged: partial K and N tiles
    w = _w24(S, k, n, 11)
    f = _adapters(S, k, n, 12) if adapters else None
    a = S.encode(w, value_dtype="bf16")
    b = S.encode(w, value_dtype="bf16").use_nm24()
    x = torch.randn(M, k, generator=torch.Generator().manual_seed(M)).bfloat16().cuda()
    for dt in (torch.float32, torch.bfloat16):
        ya = S.salr_linear(x, a, f, out_dtype=dt)
        yb = S.salr_linear(x, b, f, out_dtype=dt)
        assert torch.equal(ya, yb), (M, dt)
    ref = x.double() @ w.double()
    if f is not None:
        ref = ref + (x.double() @ f.a_cat.double()) @ f.b_cat.double()
    rel = float((S.salr_linear(x, b, f).double() - ref).norm() / ref.norm())
    print(f"nm24 M={M} rel_frob={rel:.3e}")
    assert rel < 5e-4


@pytest.mark.parametrize("name,k,n", [("q", 4096, 4096), ("gate", 4096, 14336), ("down", 14336, 4096)])
@pytest.mark.parametrize("M", [1, 32])
def test_llama_shapes_bitwise(S, name, k, n, M):
    w = _w24(S, k, n, 21, zero_frac=0.0)
    f = _adapters(S, k, n, 22)
    a = S.encode(w, value_dtype="bf16")
    b = S.encode(w, value_dtype="bf16").use_nm24()
    assert b.device_bytes < a.compute_format()[0].numel()  # 1.125 B/weight vs TB2
    x = torch.randn(M, k, generator=torch.Generator().manual_seed(1)).bfloat16().cuda()
    assert torch.equal(S.salr_linear(x, a, f, out_dtype=torch.bfloat16),
                       S.salr_linear(x, b, f, out_dtype=torch.bfloat16))


@pytest.mark.parametrize("stages", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("ctas", [0, 1, 5, 300])
def test_schedule_independence(S, stages, ctas):
    k, n = 640, 896
    w = _w24(S, k, n, 31)
    a = S.encode(w, value_dtype="bf16")
    b = S.encode(w, value_dtype="bf16").use_nm24()
    x = torch.randn(8, k, generator=torch.Generator().manual_seed(2)).bfloat16().cuda()
    ya = S.salr_linear(x, a, stages=stages, num_ctas=ctas)
    yb = S.salr_linear(x, b, stages=stages, num_ctas=ctas)
    assert torch.equal(ya, yb)


def test_column_shard_and_probe(S):
    k, n = 512, 700
    w = _w24(S, k, n, 41)
    b = S.encode(w, value_dtype="bf16").use_nm24()
    x = torch.randn(4, k, generator=torch.Generator().manual_seed(3)).bfloat16().cuda()
    full = S.salr_linear(x, b)
    sh = b.column_shard(256, 700)
    assert sh.is_nm24() and sh.nnz == int((w[:, 256:] != 0).sum())
    ysh = S.salr_linear(x, sh)
    # same stripe in TB2: bit-identical (same grid); vs the unsharded
    # product: a different split-K schedule, so to rounding
    tb = S.encode(w, value_dtype="bf16").column_shard(256, 700)
    assert torch.equal(ysh, S.salr_linear(x, tb))
    ref = full[:, 256:].double()
    assert float((ysh.double() - ref).norm() / ref.norm()) < 1e-5
    probe = S.PipelineProbe(decode_delay=200, compute_delay=200, record=True, seed=5)
    y = S.pipelined_matmul(x, b, S.PipelineConfig(ring_capacity=2), probe=probe)
    assert torch.equal(y, full)
    assert probe.produced == probe.consumed > 0
    S.validate_transitions(probe, probe.capacity)


def test_chain_rejects_nm24(S):
    w = _w24(S, 256, 256, 51)
    b = S.encode(w, value_dtype="bf16").use_nm24()
    x = torch.randn(2, 256).bfloat16().cuda()
    with pytest.raises(S.ConfigError):
        S.salr_chain(x, [(b, None)], [torch.empty(2, 256, dtype=torch.bfloat16, device="cuda")])
