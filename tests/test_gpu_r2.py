"""Round-2 GPU parity: pruning masks, residual adapters, fusion contracts,
reference-written containers, storage, workspace contract, and the parity
gaps of round 1 (full Llama3-8B shapes incl. the stack's fused q|k|v and
gate|up, two rank blocks, other sparsities, scale invariance).

Goldens come from the real reference (tests/golden/make_golden_r2.py); the
tolerances are the ones of tests/test_gpu_linear.py (fp32-output parity mode)
or the reference's own (f64 paths)."""

import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    import paper_2601_16991_b200 as S
    return S


def _np(t):
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


# ---------------------------------------------------------------------------
# 8(f)-3: exact magnitude-prune masks

def test_prune_masks_match_reference(S):
    z = np.load(os.path.join(GOLDEN, "prune.npz"))
    for i in range(int(z["n"])):
        meth = str(z[f"method_{i}"])
        nm = tuple(int(v) for v in z[f"nm_{i}"])
        cfg = S.PruneConfig(float(z[f"p_{i}"]), method=S.PruneMethod(meth), nm=nm if meth == "nm" else None)
        got = _np(S.build_mask(z[f"w_{i}"], z[f"d_{i}"], cfg))
        want = z[f"mask_{i}"]
        assert got.dtype == np.bool_ and np.array_equal(got, want), (i, meth, int((got != want).sum()))
        if meth != "nm":
            assert int(got.sum()) == S.kept_count(float(z[f"p_{i}"]), got.size)


def test_prune_mask_config1_4096(S):
    """BASELINE configs[0]'s mask (reference build_mask on a 4096^2 Gaussian)
    -> the same bitmap, pinned by the reference's SHA-256."""
    import hashlib
    from paper_2601_16991_b200 import synthetic
    z = np.load(os.path.join(GOLDEN, "config1.npz"))
    w = synthetic.gen_weight(4096, 4096, int(z["seed_w"])).double().cuda()
    mask = S.build_mask(w, torch.zeros_like(w), S.PruneConfig(float(z["sparsity"])))
    w_hat = torch.where(mask, w, torch.zeros_like(w))
    s = S.encode(w_hat)
    assert s.nnz == int(z["nnz"])
    assert hashlib.sha256(_np(s.bitmap).tobytes()).hexdigest() == str(z["bitmap_sha256"])


def test_prune_mask_ties_large(S):
    """Many exact ties across blocks of the selector: a column of equal
    magnitudes must keep the lowest flat indices (stable argsort)."""
    g = torch.Generator().manual_seed(5)
    w = (torch.randint(-4, 5, (1000, 777), generator=g).double() * 0.5).cuda()
    for p in (0.1, 0.5, 0.93):
        mask = S.build_mask(w, torch.zeros_like(w), S.PruneConfig(p))
        flat = w.abs().flatten().cpu().numpy()
        order = np.argsort(-flat, kind="stable")
        keep = S.kept_count(p, flat.size)
        want = np.zeros(flat.size, dtype=bool)
        want[order[:keep]] = True
        assert np.array_equal(_np(mask).ravel(), want), p


# ---------------------------------------------------------------------------
# 8(f)-4 / a19: residual adapters and their refinement

def test_residual_adapter_matches_reference(S):
    z = np.load(os.path.join(GOLDEN, "residual.npz"))
    for i in range(int(z["n"])):
        w, wh, r = z[f"w_{i}"], z[f"wh_{i}"], int(z[f"rank_{i}"])
        pair = S.build_residual_adapter(w, wh, r)
        ab = _np(pair.a.double() @ pair.b.double())
        np.testing.assert_allclose(ab, z[f"ab_{i}"], rtol=0, atol=1e-10 * max(1.0, np.abs(z[f"ab_{i}"]).max()))
        u, s, vt = np.linalg.svd(w - wh, full_matrices=False)
        pair2 = S.build_residual_adapter(w, wh, r, svd_result=S.SvdResult(u, s, vt))
        np.testing.assert_allclose(_np(pair2.a @ pair2.b), z[f"ab2_{i}"], rtol=0, atol=1e-12)
        lhs, rhs = S.truncation_error_bound(w - wh, r)
        np.testing.assert_allclose([lhs, rhs], z[f"bound_{i}"], rtol=1e-10)
    with pytest.raises(S.ShapeError):
        S.build_residual_adapter(np.ones((4, 5)), np.ones((5, 4)), 2)
    with pytest.raises(S.DomainError):
        S.build_residual_adapter(np.ones((4, 5)), np.zeros((4, 5)), 5)


def test_train_residual_matches_reference(S):
    z = np.load(os.path.join(GOLDEN, "residual.npz"))
    for i in range(int(z["tn"])):
        mode = str(z[f"tmode_{i}"])
        step = float(z[f"tstep_{i}"]) or None
        cfg = S.ResidualTrainConfig(step_size_mode=S.StepSizeMode(mode), step_size=step,
                                    max_iters=int(z[f"titers_{i}"]))
        lora = S.AdapterPair(z[f"tla_{i}"], z[f"tlb_{i}"], int(z[f"tr_{i}"]), float(z[f"tls_{i}"]))
        d, k = z[f"twh_{i}"].shape
        m, trace = S.train_residual(z[f"tx_{i}"], z[f"ty_{i}"], z[f"twh_{i}"], lora, np.zeros((d, k)), cfg)
        want = z[f"ttrace_{i}"]
        # AUTO modes estimate sigma_max by power iteration from a seeded start
        # vector (a different stream than the reference's): step sizes agree
        # to the iteration tolerance, traces to ~1e-9 relative
        assert len(trace) == len(want)
        np.testing.assert_allclose(trace, want, rtol=1e-7, atol=1e-12)
        np.testing.assert_allclose(_np(m), z[f"tm_{i}"], rtol=1e-6, atol=1e-9)
        m2, _ = S.train_residual(z[f"tx_{i}"], z[f"ty_{i}"], z[f"twh_{i}"], lora, np.zeros((d, k)), cfg,
                                 final_rank=int(z[f"tr_{i}"]))
        np.testing.assert_allclose(_np(m2), z[f"tm2_{i}"], rtol=1e-6, atol=1e-9)


# ---------------------------------------------------------------------------
# a8-a10, a17: fusion contracts (reference test_fusion.py)

def test_fusion_layout_and_apply_match_reference(S):
    z = np.load(os.path.join(GOLDEN, "fusion.npz"))
    for i in range(int(z["n"])):
        ads = [S.AdapterPair(z[f"a_{i}_{j}"], z[f"b_{i}_{j}"], int(z[f"r_{i}_{j}"]), float(z[f"s_{i}_{j}"]))
               for j in range(int(z[f"nad_{i}"]))]
        f = S.fuse(ads)
        assert np.array_equal(_np(f.a_cat), z[f"acat_{i}"])
        assert np.array_equal(_np(f.b_cat), z[f"bcat_{i}"])
        assert np.array_equal(_np(f.offsets), z[f"offsets_{i}"]) and np.array_equal(_np(f.ranks), z[f"ranks_{i}"])
        assert f.total_rank == int(z[f"ranks_{i}"].sum())
        for j, ad in enumerate(ads):
            a, b = f.extract(j)
            assert torch.equal(a, ad.a) and torch.equal(b, ad.scale * ad.b)
        scale = max(1.0, float(np.abs(z[f"seq_{i}"]).max()))
        np.testing.assert_allclose(_np(S.apply_fused(z[f"x_{i}"], f)), z[f"fused_{i}"], rtol=0, atol=1e-12 * scale)
        np.testing.assert_allclose(_np(S.apply_sequential(z[f"x_{i}"], ads)), z[f"seq_{i}"], rtol=0,
                                   atol=1e-12 * scale)
    with pytest.raises(S.DomainError):
        S.fuse([])
    with pytest.raises(S.DomainError):
        f.extract(99)


def test_fused_equals_sequential_many(S):
    """fused == sequential on 100 random instances (test_fusion.py:103-115)."""
    rng = np.random.default_rng(12)
    for _ in range(100):
        n_ad, d_in, d_out, rows = (int(rng.integers(1, 6)), int(rng.integers(2, 10)), int(rng.integers(2, 10)),
                                   int(rng.integers(1, 8)))
        ads = []
        for _ in range(n_ad):
            r = int(rng.integers(1, min(4, d_in, d_out) + 1))
            ads.append(S.AdapterPair(rng.normal(size=(d_in, r)), rng.normal(size=(r, d_out)), r,
                                     scale=float(rng.uniform(0.2, 2.0))))
        x = rng.normal(size=(rows, d_in))
        fy, sy = _np(S.apply_fused(x, S.fuse(ads))), _np(S.apply_sequential(x, ads))
        np.testing.assert_allclose(fy, sy, rtol=0, atol=1e-12 * max(1.0, np.abs(sy).max()))


@pytest.mark.parametrize("n_adapters", [1, 2, 5, 16, 40])
def test_exactly_two_products(S, n_adapters):
    """apply_fused issues exactly two counted products; apply_sequential two
    per adapter (test_fusion.py:117-133, test_acceptance.py:308-319)."""
    rng = np.random.default_rng(13)
    ads = [S.AdapterPair(rng.normal(size=(6, 1)), rng.normal(size=(1, 6)), 1) for _ in range(n_adapters)]
    f = S.fuse(ads)
    x = rng.normal(size=(3, 6))
    S.reset_matmul_count()
    S.apply_fused(x, f)
    assert S.matmul_call_count() == 2
    S.reset_matmul_count()
    S.apply_sequential(x, ads)
    assert S.matmul_call_count() == 2 * n_adapters


def test_fused_forward_is_one_launch(S):
    """The device analog of "exactly two products": the encoded forward is ONE
    kernel launch (X A_cat and (X A_cat) B_cat both inside it) for M <= 256."""
    g = torch.Generator().manual_seed(3)
    bx = lambda t: t.bfloat16().float()  # noqa: E731  (bf16-exact: the kernel's input precision)
    w = bx(torch.randn(512, 384, generator=g))
    w[torch.rand(512, 384, generator=g) < 0.5] = 0
    ads = [S.AdapterPair(bx(torch.randn(512, 8, generator=g) / 16), bx(torch.randn(8, 384, generator=g) * 0.1), 8),
           S.AdapterPair(bx(torch.randn(512, 4, generator=g) / 16), bx(torch.randn(4, 384, generator=g) * 0.1), 4,
                         2.0)]
    s = S.encode(w)
    x = bx(torch.randn(16, 512, generator=g))
    S.forward(x, s, ads)  # formats built
    S.reset_launch_count()
    S.reset_matmul_count()
    y = S.forward(x, s, ads)
    assert S.launch_count() == 1 and S.matmul_call_count() == 0
    ref = S.forward(x, S.decode(s), ads)  # dense branch, float64 device GEMMs
    err = (y.double() - ref.double()).abs().max() / ref.abs().max()
    assert float(err) < 2.5e-4, float(err)


def test_forward_dense_branch(S):
    rng = np.random.default_rng(21)
    w = rng.normal(size=(10, 7))
    x = rng.normal(size=(4, 10))
    ads = [S.AdapterPair(rng.normal(size=(10, 2)), rng.normal(size=(2, 7)), 2, 0.5)]
    y = _np(S.forward(x, w, ads, out_dtype=torch.float64))
    np.testing.assert_allclose(y, x @ w + 0.5 * (x @ ads[0].a.cpu().numpy()) @ ads[0].b.cpu().numpy(), atol=1e-12)
    np.testing.assert_allclose(_np(S.forward(x, w, [], out_dtype=torch.float64)), x @ w, atol=1e-12)
    with pytest.raises(S.ShapeError):
        S.forward(x, rng.normal(size=(9, 7)), ads)


def test_fuse_cache_sees_in_place_edits(S):
    g = torch.Generator().manual_seed(8)
    w = torch.randn(256, 256, generator=g)
    w[torch.rand(256, 256, generator=g) < 0.5] = 0
    s = S.encode(w)
    ad = S.AdapterPair(torch.randn(256, 4, generator=g), torch.randn(4, 256, generator=g), 4)
    x = torch.randn(8, 256, generator=g)
    y1 = S.forward(x, s, [ad])
    ad.b.mul_(2.0)  # in-place edit of a factor
    y2 = S.forward(x, s, [ad])
    base = S.forward(x, s, [])
    np.testing.assert_allclose(_np(y2 - base), 2.0 * _np(y1 - base), rtol=2e-2, atol=2e-3)


def test_rank_above_128(S):
    """R > 128: 128 ranks in the kernel, the rest by two device GEMMs."""
    g = torch.Generator().manual_seed(31)
    K, N = 1024, 640
    w = (torch.randn(K, N, generator=g) * 0.02).bfloat16().float()
    w[torch.rand(K, N, generator=g) < 0.5] = 0
    ads = [S.AdapterPair((torch.randn(K, 100, generator=g) / 32).bfloat16().float(),
                         (torch.randn(100, N, generator=g) * 0.02).bfloat16().float(), 100),
           S.AdapterPair((torch.randn(K, 60, generator=g) / 32).bfloat16().float(),
                         (torch.randn(60, N, generator=g) * 0.02).bfloat16().float(), 60, 2.0)]
    f = S.fuse(ads)
    x = torch.randn(8, K, generator=g).bfloat16().float()
    y = S.pipelined_forward(x, S.encode(w), f, S.PipelineConfig())
    ref = x.double() @ w.double() + S.apply_fused(x, f).cpu()
    rel = float((y.double().cpu() - ref).norm() / ref.norm())
    assert rel < 5e-4, rel


# ---------------------------------------------------------------------------
# 8(f)-1: containers written by the reference

def test_reference_written_container(S, tmp_path):
    path = os.path.join(GOLDEN, "ref_written.salr")
    meta = np.load(os.path.join(GOLDEN, "ref_written_meta.npz"))
    s, ads = S.read_container(path)
    ref_s = S.encode(meta["w"])
    assert torch.equal(s.bitmap, ref_s.bitmap) and torch.equal(s.values, ref_s.values)
    assert len(ads) == 3
    for i, ad in enumerate(ads):
        assert ad.rank == int(meta["ranks"][i]) and ad.scale == pytest.approx(float(meta["scales"][i]))
        assert np.array_equal(_np(ad.a), meta[f"a{i}"].astype(np.float32))
        assert np.array_equal(_np(ad.b), meta[f"b{i}"].astype(np.float32))
    out = tmp_path / "rewrite.salr"
    n = S.write_container(str(out), s, ads)
    assert n == int(meta["nbytes"]) == S.container_size_bytes(s.rows, s.cols, s.nnz, [a.rank for a in ads])
    assert out.read_bytes() == open(path, "rb").read()  # byte-identical rewrite


# ---------------------------------------------------------------------------
# storage: one resident compute format

def test_tb2_only_storage_roundtrip(S):
    g = torch.Generator().manual_seed(41)
    w = (torch.randn(300, 700, generator=g) * 0.1).bfloat16()
    w[torch.rand(300, 700, generator=g) < 0.5] = 0
    s = S.encode(w.cuda(), value_dtype="bf16")
    bm0, v0, d0 = s.bitmap.clone(), s.values.clone(), S.decode(s)
    win0 = S.decode_block(s, (7, 250), (3, 60))
    s.compute_format()
    assert s.records is None  # the TB records were released
    algo = s.compressed_bytes
    assert s.device_bytes <= 1.2 * algo, (s.device_bytes, algo)
    assert torch.equal(s.bitmap, bm0) and torch.equal(s.values, v0)
    assert torch.equal(S.decode(s), d0) and torch.equal(S.decode_block(s, (7, 250), (3, 60)), win0)
    x = torch.randn(5, 300, generator=g)
    y = S.pipelined_matmul(x, s, S.PipelineConfig())
    ref = x.bfloat16().double() @ w.double()
    assert float((y.double().cpu() - ref).norm() / ref.norm()) < 5e-4


# ---------------------------------------------------------------------------
# workspace contract (include/salr_b200.h): only the documented prefix zeroed

def test_workspace_documented_zero_prefix(S):
    from paper_2601_16991_b200 import _lib
    lib = _lib.load()
    zb = int(lib.salr_linear_workspace_zero_bytes())
    assert zb == 768 * 1024
    g = torch.Generator().manual_seed(55)
    K, N, M = 2048, 1024, 16
    w = (torch.randn(K, N, generator=g) * 0.02).bfloat16().float()
    w[torch.rand(K, N, generator=g) < 0.5] = 0
    s = S.encode(w.cuda(), value_dtype="bf16")
    f = S.fuse([S.AdapterPair((torch.randn(K, 16, generator=g) / 32).bfloat16().float(),
                              (torch.randn(16, N, generator=g) * 0.02).bfloat16().float(), 16)])
    x = torch.randn(M, K, generator=g).bfloat16().cuda()
    ref = S.salr_linear(x, s, f)
    need = int(lib.salr_linear_workspace_bytes(M, N, K, 64, 0))
    ws = torch.randint(0, 255, (need,), dtype=torch.uint8, device="cuda")  # garbage
    ws[:zb].zero_()
    for _ in range(3):  # both U parity buffers, then reuse
        y = S.salr_linear(x, s, f, workspace=ws)
        assert torch.equal(y, ref)


# ---------------------------------------------------------------------------
# round-1 parity gaps: full shapes, fused stack shapes, two rank blocks,
# sparsities, scale invariance

REL_FROB_TOL, MAX_ABS_TOL = 5e-4, 2.5e-4


def _check(y, ref, tag):
    y, ref = y.double(), ref.double()
    rel = float((y - ref).norm() / ref.norm())
    mabs = float((y - ref).abs().max() / ref.abs().max())
    print(f"{tag}: rel_frob={rel:.3e} max_abs/max|ref|={mabs:.3e}")
    assert rel <= REL_FROB_TOL and mabs <= MAX_ABS_TOL, (tag, rel, mabs)


def _linear(S, K, N, seed, p=0.5, ranks=(16, 16)):
    from paper_2601_16991_b200 import synthetic
    w = synthetic.gen_weight(K, N, seed).cuda()
    w_hat = S.prune(w, S.PruneConfig(p))
    ads = []
    for i, r in enumerate(ranks):
        a, b = synthetic.gen_lora(K, N, r, seed + 7 * i + 1)
        ads.append(S.AdapterPair(a, b, r, 2.0 if i else 1.0))
    return w_hat, S.fuse(ads)


@pytest.mark.parametrize("shape", [(4096, 14336), (4096, 6144), (4096, 28672)])
@pytest.mark.parametrize("M", [1, 8, 32])
def test_full_llama_shapes(S, shape, M):
    """gate/up 4096x14336, and the stack's fused q|k|v (4096x6144) and
    gate|up (4096x28672) launches, vs the fp64 dense product."""
    K, N = shape
    w_hat, f = _linear(S, K, N, 3000 + N + M)
    s = S.encode(w_hat, value_dtype="bf16")
    x = torch.randn(M, K, generator=torch.Generator().manual_seed(M)).bfloat16().cuda()
    y = S.salr_linear(x, s, f)
    ref = x.double() @ w_hat.double() + (x.double() @ f.a_cat.double()) @ f.b_cat.double()
    _check(y, ref, f"{shape} M={M}")


@pytest.mark.parametrize("M", [1, 8, 32])
def test_two_rank_blocks_decode_kernel(S, M):
    """R = 128 (two 64-rank adapter blocks, ra = 2) in the decode-size kernel
    (the r = 64 sweep of configs[4])."""
    w_hat, f = _linear(S, 4096, 14336, 5000 + M, ranks=(64, 64))
    assert f.r_pad == 128
    s = S.encode(w_hat, value_dtype="bf16")
    x = torch.randn(M, 4096, generator=torch.Generator().manual_seed(M)).bfloat16().cuda()
    y = S.salr_linear(x, s, f)
    ref = x.double() @ w_hat.double() + (x.double() @ f.a_cat.double()) @ f.b_cat.double()
    _check(y, ref, f"R=128 M={M}")


@pytest.mark.parametrize("p", [0.3, 0.7])
@pytest.mark.parametrize("M", [1, 32])
def test_other_sparsities(S, p, M):
    w_hat, f = _linear(S, 4096, 4096, 6000 + int(10 * p) + M, p=p)
    s = S.encode(w_hat, value_dtype="bf16")
    assert s.nnz == S.kept_count(p, 4096 * 4096)
    x = torch.randn(M, 4096, generator=torch.Generator().manual_seed(M)).bfloat16().cuda()
    y = S.salr_linear(x, s, f)
    ref = x.double() @ w_hat.double() + (x.double() @ f.a_cat.double()) @ f.b_cat.double()
    _check(y, ref, f"p={p} M={M}")


@pytest.mark.parametrize("e", [-40, 40])
def test_scale_invariance(S, e):
    """X scaled by 2^e (exact in bf16): Y and U = X A_cat scale by 2^e.  U then
    leaves the in-kernel fixed-point window (|U| < 2^37, resolution 2^-26), so
    the public API must switch to the fp32 U pre-kernel; the adapter term is
    ~10 % of Y, so a lost or overflowed U fails the tolerance."""
    g = torch.Generator().manual_seed(60)
    K, N, M = 4096, 1024, 16
    w = (torch.randn(K, N, generator=g) * 0.02).bfloat16().float()
    w[torch.rand(K, N, generator=g) < 0.5] = 0
    a = (torch.randn(K, 16, generator=g) / 64).bfloat16().float()
    b = (torch.randn(16, N, generator=g) * 0.02).bfloat16().float()
    x = torch.randn(M, K, generator=g).bfloat16().float()
    s = S.encode(w.cuda(), value_dtype="bf16")
    f = S.fuse([S.AdapterPair(a, b, 16)])
    sc = 2.0 ** e
    base = x.double() @ w.double()
    delta = (x.double() @ a.double()) @ b.double()
    assert float(delta.norm() / base.norm()) > 0.05
    y1 = S.salr_linear(x.cuda(), s, f)
    _check(y1.cpu(), base + delta, "scale 1 (fixed-point U)")
    ys = S.salr_linear((x * sc).cuda(), s, f)
    _check(ys.cpu(), sc * (base + delta), f"scale 2^{e} (fp32 U)")
