"""GPU parity of the fused SALR linear (tcgen05 decode+GEMM + adapter
epilogue) against the reference's pipelined_forward outputs
(tests/golden/forward.npz, config1.npz -- produced by the real reference) and
against the oracle at Llama3-8B shapes.

Tolerance (SURVEY.md 8(a), fp32-output parity mode, bf16 inputs, fp32
accumulation, U = X @ A_cat split hi/lo):
    rel_frob = ||y - ref||_F / ||ref||_F <= 5e-4  and
    max_abs  <= 2.5e-4 * max|ref|
Both numbers are printed for every case."""

import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

REL_FROB_TOL = 5e-4
MAX_ABS_TOL = 2.5e-4


@pytest.fixture(scope="module")
def S():
    import paper_2601_16991_b200 as S
    return S


def errors(y, ref):
    y = np.asarray(y, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    rel = np.linalg.norm(y - ref) / max(np.linalg.norm(ref), 1e-30)
    mabs = np.abs(y - ref).max() / max(np.abs(ref).max(), 1e-30)
    return rel, mabs


def assert_close(y, ref, tag=""):
    rel, mabs = errors(y, ref)
    print(f"{tag}: rel_frob={rel:.3e} max_abs/max|ref|={mabs:.3e}")
    assert rel <= REL_FROB_TOL and mabs <= MAX_ABS_TOL, (tag, rel, mabs)


def test_forward_goldens(S):
    z = np.load(os.path.join(GOLDEN, "forward.npz"))
    for i in range(int(z["n"])):
        ads = [S.AdapterPair(z[f"a{j}_{i}"], z[f"b{j}_{i}"], z[f"a{j}_{i}"].shape[1], float(z[f"scale{j}_{i}"]))
               for j in range(2)]
        s = S.encode(z[f"w_{i}"])
        y = S.pipelined_forward(z[f"x_{i}"], s, S.fuse(ads), S.PipelineConfig())
        assert_close(y.cpu().numpy(), z[f"y_{i}"], f"golden {i} {z[f'w_{i}'].shape} M={z[f'x_{i}'].shape[0]}")
        y2 = S.forward(z[f"x_{i}"], s, ads)
        assert torch.equal(y, y2)


def test_schedule_independence_bitwise(S):
    """serial (1-slot ring) == overlapped == every ring capacity, bit for bit
    (reference test_pipeline.py:90-112)."""
    g = torch.Generator().manual_seed(1)
    w = torch.randn(700, 900, generator=g)
    w[torch.rand(700, 900, generator=g) < 0.5] = 0
    x = torch.randn(13, 700, generator=g)
    s = S.encode(w, value_dtype="bf16")
    ref = S.pipelined_matmul(x, s, S.PipelineConfig(overlap=False, ring_capacity=1))
    for cap in (2, 3, 4, 8, 12):
        got = S.pipelined_matmul(x, s, S.PipelineConfig(ring_capacity=cap))
        assert torch.equal(ref, got), cap
    for st in (1, 2, 3, 4, 5, 6, 7, 8, 12, 16):  # every device ring depth
        assert torch.equal(ref, S.salr_linear(x, s, None, stages=st)), st
    for _ in range(3):  # run-to-run determinism of the split-K fixup
        assert torch.equal(ref, S.pipelined_matmul(x, s, S.PipelineConfig()))


def _dense_ref(x, w, fused=None):
    xd = x.double()
    y = xd @ w.double()
    if fused is not None:
        y = y + (xd @ fused.a_cat.double()) @ fused.b_cat.double()
    return y


@pytest.mark.parametrize("M", [1, 2, 8, 16, 32, 48, 64, 100, 128, 200, 256, 300])
def test_token_counts(S, M):
    g = torch.Generator().manual_seed(100 + M)
    K, N = 1024, 768
    w = (torch.randn(K, N, generator=g) * 0.02).bfloat16().float()
    w[torch.rand(K, N, generator=g) < 0.5] = 0
    x = torch.randn(M, K, generator=g).bfloat16().float()
    ads = [S.AdapterPair((torch.randn(K, 16, generator=g) / 32).bfloat16().float(),
                         (torch.randn(16, N, generator=g) * 0.02).bfloat16().float(), 16, 2.0),
           S.AdapterPair((torch.randn(K, 16, generator=g) / 32).bfloat16().float(),
                         (torch.randn(16, N, generator=g) * 0.02).bfloat16().float(), 16)]
    fused = S.fuse(ads)
    s = S.encode(w.cuda(), value_dtype="bf16")
    y = S.pipelined_forward(x, s, fused, S.PipelineConfig())
    assert_close(y.cpu().numpy(), _dense_ref(x.cuda(), w.cuda(), fused).cpu().numpy(), f"M={M}")


@pytest.mark.parametrize("shape", [(37, 53), (64, 128), (65, 129), (130, 260), (1000, 96), (96, 1000), (4096, 1024)])
@pytest.mark.parametrize("ctas", [0, 1, 5, 300])
def test_shapes_and_split_k(S, shape, ctas):
    K, N = shape
    g = torch.Generator().manual_seed(K * 7 + N)
    w = torch.randn(K, N, generator=g)
    w[torch.rand(K, N, generator=g) < 0.6] = 0
    w = w.bfloat16().float()
    x = torch.randn(9, K, generator=g).bfloat16().float()
    s = S.encode(w, value_dtype="bf16")
    y = S.salr_linear(x, s, None, num_ctas=ctas)
    assert_close(y.cpu().numpy(), (x.double() @ w.double()).numpy(), f"{shape} ctas={ctas}")


def test_bf16_output_and_zero_matrix(S):
    g = torch.Generator().manual_seed(9)
    w = torch.zeros(256, 384)
    x = torch.randn(4, 256, generator=g)
    y = S.pipelined_matmul(x, S.encode(w), S.PipelineConfig())
    assert not y.any()
    w = torch.randn(256, 384, generator=g).bfloat16().float()
    w[torch.rand(256, 384, generator=g) < 0.5] = 0
    s = S.encode(w)
    yb = S.salr_linear(x, s, out_dtype=torch.bfloat16)
    ref = x.bfloat16().double() @ w.double()
    assert yb.dtype == torch.bfloat16
    diff = (yb.double().cpu() - ref).abs()
    assert (diff <= 2.0 ** -8 * ref.abs() + 1e-3 * ref.abs().max()).all()


def test_config1_vs_reference(S):
    """BASELINE configs[0]: 4096x4096, p=0.5, LoRA r16 + SVD residual r16, M=16,
    compared with the real reference's pipelined_forward output."""
    import hashlib
    from test_oracle import config1_inputs
    z, w_hat, x, ads_o = config1_inputs()
    s = S.encode(w_hat)
    assert s.nnz == int(z["nnz"])
    assert hashlib.sha256(s.bitmap.cpu().numpy().tobytes()).hexdigest() == str(z["bitmap_sha256"])
    assert hashlib.sha256(s.values.cpu().numpy().tobytes()).hexdigest() == str(z["values_sha256"])
    ads = [S.AdapterPair(a.a, a.b, a.rank, a.scale) for a in ads_o]
    y = S.pipelined_forward(x, s, S.fuse(ads), S.PipelineConfig())
    assert_close(y.cpu().numpy(), z["y"], "config1 4096^2 M=16")


@pytest.mark.parametrize("name", ["q", "k", "down"])
@pytest.mark.parametrize("M", [1, 8, 32, 2048])
def test_llama_shapes(S, name, M):
    from paper_2601_16991_b200 import synthetic
    K, N = synthetic.LLAMA3_8B_LINEARS[name]
    li = synthetic.gen_linear(K, N, seed=1000 + M, device="cuda")
    x = synthetic.gen_x(M, K, seed=7).cuda()
    ads = [S.AdapterPair(li.res_a, li.res_b, 16), S.AdapterPair(li.lora_a, li.lora_b, 16, li.lora_scale)]
    fused = S.fuse(ads)
    s = S.encode(li.w_hat, value_dtype="bf16")
    y = S.pipelined_forward(x, s, fused, S.PipelineConfig())
    assert_close(y.cpu().numpy(), _dense_ref(x, li.w_hat, fused).cpu().numpy(), f"{name} M={M}")


def _last_launch():
    import ctypes
    from paper_2601_16991_b200 import _lib
    info = (ctypes.c_int32 * 12)()
    assert _lib.load().salr_debug_last_launch(ctypes.addressof(info)) == 0
    keys = ("ctas", "stages", "bm", "groups", "u_mode", "coop", "cluster", "pdl", "cluster_req", "cluster_max",
            "smem", "cooperative")
    return dict(zip(keys, list(info)))


@pytest.mark.parametrize("M", [8, 16, 32, 100])
@pytest.mark.parametrize("adapters", [False, True])
def test_split_k_reduction_modes(S, M, adapters):
    """The three split-K reductions give the same answer: DSMEM within a
    thread-block cluster (tiles split over exactly np CTAs of one cluster),
    cooperative global, last-CTA global.  K=4096 (64 k-tiles) x 4096 columns:
    128 CTAs x 16 units -> clusters of 4 where the cooperative reduction is
    off (M < 16)."""
    g = torch.Generator().manual_seed(77 + M)
    K, N = 4096, 4096
    w = (torch.randn(K, N, generator=g) * 0.02).bfloat16().float()
    w[torch.rand(K, N, generator=g) < 0.5] = 0
    x = torch.randn(M, K, generator=g).bfloat16().float().cuda()
    fused = None
    if adapters:
        fused = S.fuse([S.AdapterPair((torch.randn(K, 16, generator=g) / 64).bfloat16().float(),
                                      (torch.randn(16, N, generator=g) * 0.02).bfloat16().float(), 16)])
    s = S.encode(w.cuda(), value_dtype="bf16")
    ref = _dense_ref(x, w.cuda(), fused).cpu().numpy()
    n_mc = (M + 127) // 128 if M > 64 else 1
    seen = set()
    for ctas in (0, 128 * n_mc, 127, 37):
        y = S.salr_linear(x, s, fused, num_ctas=ctas)
        info = _last_launch()
        seen.add(info["cluster"])
        if (info["u_mode"] == 1 or info["coop"]) and not info["pdl"]:
            # CTAs wait on each other: the launch must be co-scheduled
            assert info["cooperative"] == 1, info
        assert_close(y.cpu().numpy(), ref, f"M={M} ctas={ctas} {info}")
        y2 = S.salr_linear(x, s, fused, num_ctas=ctas)
        assert torch.equal(y, y2)  # run-to-run determinism of every mode
    assert 0 in seen, seen
    if M < 16:
        assert max(seen) >= 2, seen


@pytest.mark.parametrize("rank", [16, 64])
@pytest.mark.parametrize("out_dtype", ["f32", "bf16"])
def test_prefill_kernel_ragged(S, rank, out_dtype):
    """The prefill kernel (M > 256 with >= 3/4 of the SMs worth of 512-token x
    128-column items): ragged M (partial 128-token chunk), K (partial k-tile)
    and N (partial last column tile), adapters with one and two 64-rank
    blocks, fp32 and bf16 output."""
    g = torch.Generator().manual_seed(4242 + rank)
    M, K, N = 300, 200, 14300
    w = (torch.randn(K, N, generator=g) * 0.05).bfloat16().float()
    w[torch.rand(K, N, generator=g) < 0.5] = 0
    x = torch.randn(M, K, generator=g).bfloat16().float().cuda()
    fused = S.fuse([S.AdapterPair((torch.randn(K, rank, generator=g) / 16).bfloat16().float(),
                                  (torch.randn(rank, N, generator=g) * 0.05).bfloat16().float(), rank),
                    S.AdapterPair((torch.randn(K, rank, generator=g) / 16).bfloat16().float(),
                                  (torch.randn(rank, N, generator=g) * 0.05).bfloat16().float(), rank, 2.0)])
    s = S.encode(w.cuda(), value_dtype="bf16")
    ref = _dense_ref(x, w.cuda(), fused).cpu().numpy()
    dt = torch.float32 if out_dtype == "f32" else torch.bfloat16
    y = S.salr_linear(x, s, fused, out_dtype=dt, dense_prefill=False)
    info = _last_launch()
    assert info["smem"] > 0 and info["groups"] == -1, info  # the prefill kernel ran
    if out_dtype == "f32":
        assert_close(y.cpu().numpy(), ref, f"prefill r={rank}")
    else:
        yb = y.double().cpu().numpy()
        err = np.abs(yb - ref)
        assert (err <= 2.0 ** -8 * np.abs(ref) + 2e-3 * np.abs(ref).max()).all(), err.max()
    assert torch.equal(y, S.salr_linear(x, s, fused, out_dtype=dt, dense_prefill=False))


@pytest.mark.parametrize("M", [1, 8, 32])
def test_pdl_chain_matches_serial(S, M):
    """Programmatic-dependent chains (as in the stack): every linear reads the
    previous one's output and the launches overlap; the in-kernel U epochs,
    split-K tickets and alternating workspaces must give exactly the serial
    results, eagerly and replayed from a CUDA graph."""
    g = torch.Generator().manual_seed(900 + M)
    K = 1024
    mats, fus = [], []
    for i in range(4):
        w = (torch.randn(K, K, generator=g) * 0.03).bfloat16().float()
        w[torch.rand(K, K, generator=g) < 0.5] = 0
        s = S.encode(w.cuda(), value_dtype="bf16")
        s.compute_format()
        mats.append(s)
        fus.append(S.fuse([S.AdapterPair((torch.randn(K, 16, generator=g) / 32).bfloat16().float(),
                                         (torch.randn(16, K, generator=g) * 0.03).bfloat16().float(), 16)]))
        fus[-1].device_operands()
    x = torch.randn(M, K, generator=g).bfloat16().cuda()

    def chain(pdl, outs):
        h = x
        for i in range(12):
            h = S.salr_linear(h, mats[i % 4], fus[i % 4], out=outs[i], out_dtype=torch.bfloat16,
                              check_finite=False, pdl=pdl)
        return outs

    ref = chain(False, [torch.empty(M, K, device="cuda", dtype=torch.bfloat16) for _ in range(12)])
    got = chain(True, [torch.empty(M, K, device="cuda", dtype=torch.bfloat16) for _ in range(12)])
    torch.cuda.synchronize()
    for i in range(12):
        assert torch.equal(ref[i], got[i]), i
    outs = [torch.empty(M, K, device="cuda", dtype=torch.bfloat16) for _ in range(12)]
    chain(True, outs)  # warm-up outside capture (workspaces, formats)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        chain(True, outs)
    for _ in range(3):
        graph.replay()
        torch.cuda.synchronize()
        for i in range(12):
            assert torch.equal(ref[i], outs[i]), i


@pytest.mark.parametrize("M", [1, 8, 32, 100, 300])
@pytest.mark.parametrize("adapters", [True, False])
def test_strided_input_no_copy(S, M, adapters):
    """The leading columns of a wider bf16 output (the stack's o / down
    inputs) go to the kernel as they are, with their row stride: same result
    as the contiguous copy, in-kernel U included, and no copy kernel."""
    g = torch.Generator().manual_seed(77 + M)
    K, N, W = 1024, 768, 1536
    w = (torch.randn(K, N, generator=g) * 0.03).bfloat16().float()
    w[torch.rand(K, N, generator=g) < 0.5] = 0
    s = S.encode(w.cuda(), value_dtype="bf16")
    s.compute_format()
    f = None
    if adapters:
        f = S.fuse([S.AdapterPair((torch.randn(K, 16, generator=g) / 32).bfloat16().float(),
                                  (torch.randn(16, N, generator=g) * 0.03).bfloat16().float(), 16)])
    wide = torch.randn(M, W, generator=g).bfloat16().cuda()
    view = wide[:, 256:256 + K]  # 512-byte offset: rows stay 16-byte aligned
    from paper_2601_16991_b200.pipeline import _prep_x
    xb, _, ldx = _prep_x(view, K, False)
    assert xb.data_ptr() == view.data_ptr() and ldx == W
    for dt in (torch.float32, torch.bfloat16):
        assert torch.equal(S.salr_linear(view, s, f, out_dtype=dt), S.salr_linear(view.contiguous(), s, f, out_dtype=dt))
    # unaligned or non-bf16 views still work through the copy
    odd = wide[:, 3:3 + K]
    assert _prep_x(odd, K, False)[0].data_ptr() != odd.data_ptr()
    assert torch.equal(S.salr_linear(odd, s, f), S.salr_linear(odd.contiguous(), s, f))


def test_strided_input_prefill(S):
    """A strided bf16 view through the prefill kernel and the dense prefill
    path (M=2048): same result as its contiguous copy (the X tensor map /
    the GEMM carry the row stride)."""
    g = torch.Generator().manual_seed(5)
    K, N, M = 1024, 4096, 2048
    w = (torch.randn(K, N, generator=g) * 0.03).bfloat16().float()
    w[torch.rand(K, N, generator=g) < 0.5] = 0
    s = S.encode(w.cuda(), value_dtype="bf16")
    s.compute_format()
    f = S.fuse([S.AdapterPair((torch.randn(K, 16, generator=g) / 32).bfloat16().float(),
                              (torch.randn(16, N, generator=g) * 0.03).bfloat16().float(), 16)])
    wide = torch.randn(M, 2 * K, generator=g).bfloat16().cuda()
    view = wide[:, K:]
    ref = _dense_ref(view.float(), w.cuda(), f)
    for dense in (False, True):  # the fused prefill kernel and the dense path
        y = S.salr_linear(view, s, f, dense_prefill=dense)
        assert torch.equal(y, S.salr_linear(view.contiguous(), s, f, dense_prefill=dense))
        assert float((y.double() - ref.double()).norm() / ref.double().norm()) < 5e-4


@pytest.mark.parametrize("shape", [(200, 300), (1000, 1500), (64, 128)])
def test_tb2_dense_decode(S, shape):
    """salr_tb2_decode (the dense scratch of prefill-size products) equals
    decode() of the same matrix bit for bit, ragged shapes included."""
    from paper_2601_16991_b200 import _lib
    g = torch.Generator().manual_seed(sum(shape))
    w = (torch.randn(*shape, generator=g) * 0.05).bfloat16().float()
    w[torch.rand(*shape, generator=g) < 0.5] = 0
    s = S.encode(w.cuda(), value_dtype="bf16")
    rec2, off2, _ = s.compute_format()
    K, N = shape
    out = torch.full((K, N + 8), 7.0, dtype=torch.bfloat16, device="cuda")
    _lib.check(_lib.load().salr_tb2_decode(_lib.ptr(rec2), _lib.ptr(off2), K, N, _lib.ptr(out), N + 8,
                                           _lib.stream_ptr()))
    assert torch.equal(out[:, :N].float(), w.cuda())
    assert bool((out[:, N:] == 7.0).all())  # nothing written past cols


@pytest.mark.parametrize("M", [300, 512, 2048])
@pytest.mark.parametrize("rank", [0, 16, 64, 96])
@pytest.mark.parametrize("fmt", ["tb2", "nm24"])
def test_dense_prefill_path(S, M, rank, fmt):
    """Prefill-size products (decode to a dense scratch + tensor-core GEMM,
    adapters folded along K) against fp64, ragged K/N, R up to 192 (tail),
    both compute formats; fp32 and bf16 outputs."""
    g = torch.Generator().manual_seed(M + rank)
    K, N = 1000, 1500
    w = (torch.randn(K, N, generator=g) * 0.05).bfloat16().float()
    if fmt == "nm24":
        w = S.prune(w.cuda(), S.PruneConfig(0.5, S.PruneMethod.SEMI_STRUCTURED_NM, nm=(2, 4))).cpu()
    else:
        w[torch.rand(K, N, generator=g) < 0.5] = 0
    fused = None
    if rank:
        fused = S.fuse([S.AdapterPair((torch.randn(K, rank, generator=g) / 16).bfloat16().float(),
                                      (torch.randn(rank, N, generator=g) * 0.05).bfloat16().float(), rank, sc)
                        for sc in (1.0, 2.0)])
    s = S.encode(w.cuda(), value_dtype="bf16")
    if fmt == "nm24":
        s.use_nm24()
    x = torch.randn(M, K, generator=g).bfloat16().float().cuda()
    ref = _dense_ref(x, w.cuda(), fused).cpu().numpy()
    y = S.salr_linear(x, s, fused)
    assert_close(y.cpu().numpy(), ref, f"dense prefill M={M} r={rank} {fmt}")
    yb = S.salr_linear(x, s, fused, out_dtype=torch.bfloat16)
    assert float((yb.double() - y.double()).norm() / y.double().norm()) < 4e-3
    assert torch.equal(y, S.salr_linear(x, s, fused))  # deterministic
