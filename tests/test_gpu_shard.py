"""GPU side of the column-sharded path: a matrix's stripe
(``column_shard``) runs through the fused kernel and equals those columns of
the unsharded product; the package's ShardedStack at world 1 equals the same
chain of linears run one by one."""

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    import paper_2601_16991_b200 as S
    return S


def _mat(S, k, n, seed):
    g = torch.Generator().manual_seed(seed)
    w = (torch.randn(k, n, generator=g) * 0.02).bfloat16().float()
    w[torch.rand(k, n, generator=g) < 0.5] = 0
    ads = [S.AdapterPair((torch.randn(k, 16, generator=g) / 64).bfloat16().float(),
                         (torch.randn(16, n, generator=g) * 0.02).bfloat16().float(), 16, sc) for sc in (1.0, 2.0)]
    return w.cuda(), S.fuse(ads)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_column_shard_matches_full_columns(S, world):
    from paper_2601_16991_b200.sharding import ShardedLinear, shard_cols
    k, n, m = 1024, 1408, 8
    w, f = _mat(S, k, n, 3 + world)
    s = S.encode(w, value_dtype="bf16")
    s.compute_format()
    x = torch.randn(m, k, generator=torch.Generator().manual_seed(9)).bfloat16().cuda()
    full = S.salr_linear(x, s, f, out_dtype=torch.float32).double()
    for r in range(world):
        lin = ShardedLinear.from_full(s, f, world, r)
        c0, c1 = shard_cols(n, world, r)
        assert lin.s.nnz == int((w[:, c0:c1] != 0).sum())
        y = S.salr_linear(x, lin.s, lin.f, out_dtype=torch.float32).double()
        ref = full[:, c0:c1]
        rel = float((y - ref).norm() / ref.norm())
        assert rel < 1e-5, (r, rel)
        # the shard's codec view is the slice of the full matrix
        assert torch.equal(S.decode(lin.s), S.decode(s)[:, c0:c1])


def test_sharded_stack_world1_equals_chain(S):
    from paper_2601_16991_b200.sharding import ShardedLinear, ShardedStack
    m = 4
    dims = {"a": (512, 768), "b": (512, 512), "c": (512, 1024)}
    mats = {nm: _mat(S, kk, nn, i) for i, (nm, (kk, nn)) in enumerate(dims.items())}
    enc = {}
    for nm, (w, f) in mats.items():
        s = S.encode(w, value_dtype="bf16")
        s.compute_format()
        enc[nm] = (s, f)
    plan = [("a", None), ("b", (0, 512)), ("c", None)]  # b consumes the first 512 columns of a
    layers = [{nm: ShardedLinear(s, f, s.cols, 1, 0) for nm, (s, f) in enc.items()}]
    st = ShardedStack(layers, plan, 1, 0, None, m, chain=False)  # per-linear launches
    x = torch.randn(m, 512, generator=torch.Generator().manual_seed(1)).bfloat16().cuda()
    y = st.step(x).clone()
    h = S.salr_linear(x, enc["a"][0], enc["a"][1], out_dtype=torch.bfloat16)
    h = S.salr_linear(h[:, :512], enc["b"][0], enc["b"][1], out_dtype=torch.bfloat16)
    h = S.salr_linear(h, enc["c"][0], enc["c"][1], out_dtype=torch.bfloat16)
    assert torch.equal(y, h)
    assert st.launches_per_step == 3


@pytest.mark.parametrize("M", [1, 8, 32, 100])
@pytest.mark.parametrize("adapters", [True, False])
def test_chain_equals_per_linear_launches(S, M, adapters):
    """One persistent launch over a chain of linears (salr_chain) equals the
    same linears launched one by one (each reading the previous bf16 output's
    leading columns), and both match an fp64 chain."""
    dims = [(1024, 1536), (1024, 1024), (1024, 2304), (2304, 640)]  # x -> a -> b(:1024 of a) -> c -> d
    lin = []
    for i, (k, n) in enumerate(dims):
        w, f = _mat(S, k, n, 40 + i)
        s = S.encode(w, value_dtype="bf16")
        s.compute_format()
        lin.append((s, f if adapters else None, w))
    x = torch.randn(M, 1024, generator=torch.Generator().manual_seed(2)).bfloat16().cuda()
    outs = [torch.empty(M, n, dtype=torch.bfloat16, device="cuda") for _, n in dims]
    S.salr_chain(x, [(s, f) for s, f, _ in lin], outs)
    for rep in range(2):  # counters and U buffers reset themselves between launches
        outs2 = [torch.empty_like(o) for o in outs]
        S.salr_chain(x, [(s, f) for s, f, _ in lin], outs2)
        for a, b in zip(outs, outs2):
            assert torch.equal(a, b)
    h = x
    ref = x.double()
    for (s, f, w), o, (k, n) in zip(lin, outs, dims):
        y = S.salr_linear(h[:, :k], s, f, out_dtype=torch.bfloat16)
        r = ref[:, :k] @ w.double()
        if f is not None:
            r = r + (ref[:, :k] @ f.a_cat.double()) @ f.b_cat.double()
        rel = float((o.double() - y.double()).norm() / y.double().norm())
        assert rel < 1e-2, rel  # bf16 outputs: one ulp of rounding apart at most
        relr = float((o.double() - r).norm() / r.norm())
        assert relr < 2e-2, relr
        h = o  # follow the chain's own activations
        ref = o.double()


def test_sharded_stack_chain_equals_unchained(S):
    """The chained step (one launch per layer) equals the per-linear step."""
    from paper_2601_16991_b200.sharding import ShardedLinear, ShardedStack
    m = 8
    dims = {"a": (512, 768), "b": (512, 512), "c": (512, 1024)}
    mats = {nm: _mat(S, kk, nn, 20 + i) for i, (nm, (kk, nn)) in enumerate(dims.items())}
    layers = []
    for _ in range(2):
        lay = {}
        for nm, (w, f) in mats.items():
            s = S.encode(w, value_dtype="bf16")
            s.compute_format()
            lay[nm] = ShardedLinear(s, f, s.cols, 1, 0)
        layers.append(lay)
    plan = [("a", (0, 512)), ("b", (0, 512)), ("c", (0, 512))]  # the next layer reads c[:, :512]
    x = torch.randn(m, 512, generator=torch.Generator().manual_seed(4)).bfloat16().cuda()
    ch = ShardedStack(layers, plan, 1, 0, None, m, chain=True)
    assert ch.chain
    y1 = ch.step(x).clone()
    assert ch.launches_per_step == 2
    un = ShardedStack(layers, plan, 1, 0, None, m)
    y2 = un.step(x).clone()
    rel = float((y1.double() - y2.double()).norm() / y2.double().norm())
    assert rel < 1e-2, rel
