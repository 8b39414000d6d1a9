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
    st = ShardedStack(layers, plan, 1, 0, None, m)
    x = torch.randn(m, 512, generator=torch.Generator().manual_seed(1)).bfloat16().cuda()
    y = st.step(x).clone()
    h = S.salr_linear(x, enc["a"][0], enc["a"][1], out_dtype=torch.bfloat16)
    h = S.salr_linear(h[:, :512], enc["b"][0], enc["b"][1], out_dtype=torch.bfloat16)
    h = S.salr_linear(h, enc["c"][0], enc["c"][1], out_dtype=torch.bfloat16)
    assert torch.equal(y, h)
    assert st.launches_per_step == 3
