"""Chain kernel vs per-linear launches on small cases (debug aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2601_16991_b200 as S

def mat(k, n, seed):
    g = torch.Generator().manual_seed(seed)
    w = (torch.randn(k, n, generator=g) * 0.02).bfloat16().float()
    w[torch.rand(k, n, generator=g) < 0.5] = 0
    ads = [S.AdapterPair((torch.randn(k, 16, generator=g) / 64).bfloat16().float(),
                         (torch.randn(16, n, generator=g) * 0.02).bfloat16().float(), 16, sc) for sc in (1.0, 2.0)]
    s = S.encode(w.cuda(), value_dtype="bf16"); s.compute_format()
    return s, S.fuse(ads), w.cuda()

for M in (1, 32):
    for ad in (False, True):
        for dims in ([(1024, 1536)], [(1024, 1536), (1024, 1024)]):
            lin = [mat(k, n, 7 + i) for i, (k, n) in enumerate(dims)]
            x = torch.randn(M, 1024, generator=torch.Generator().manual_seed(3)).bfloat16().cuda()
            outs = [torch.full((M, n), 7.0, dtype=torch.bfloat16, device="cuda") for _, n in dims]
            S.salr_chain(x, [(s, f if ad else None) for s, f, _ in lin], outs)
            torch.cuda.synchronize()
            h = x
            msg = []
            for (s, f, w), o, (k, n) in zip(lin, outs, dims):
                y = S.salr_linear(h[:, :k], s, f if ad else None, out_dtype=torch.bfloat16)
                diff = (o.float() - y.float()).abs()
                msg.append(f"max|d|={float(diff.max()):.3e} n7={int((o == 7).sum())} bad={int((diff > 1e-2).sum())}/{o.numel()}")
                h = o
            print(f"M={M} adapters={ad} L={len(dims)}: " + " | ".join(msg), flush=True)
