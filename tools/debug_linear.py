import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2601_16991_b200 as S
from paper_2601_16991_b200 import pipeline as P
torch.manual_seed(0)
for (K, N, M) in [(37, 53, 11), (256, 512, 32), (1024, 768, 8)]:
    w = torch.randn(K, N).bfloat16().float(); w[torch.rand(K, N) < 0.5] = 0
    x = torch.randn(M, K).bfloat16().float()
    s = S.encode(w.cuda(), value_dtype="bf16")
    y0 = S.salr_linear(x, s, None).cpu().double()
    ref0 = x.double() @ w.double()
    print(K, N, M, "no-adapter rel", ((y0 - ref0).norm() / ref0.norm()).item())
    a = torch.randn(K, 16).bfloat16().float() / 8; b = torch.randn(16, N).bfloat16().float() / 8
    f = S.fuse([S.AdapterPair(a, b, 16)])
    y1 = S.salr_linear(x, s, f).cpu().double()
    ref1 = ref0 + (x.double() @ a.double()) @ b.double()
    print(K, N, M, "adapter rel", ((y1 - ref1).norm() / ref1.norm()).item())
    ws = P._WS[torch.cuda.current_device()]
    u = ws[256 * 1024: 256 * 1024 + M * 64 * 4].view(torch.float32).view(M, 64)[:, :16].cpu().double()
    uref = x.double() @ a.double()
    print("   U rel", ((u - uref).norm() / uref.norm()).item())
    d = (y1 - ref1)
    print("   delta-only rel", ((y1 - y0) - (ref1 - ref0)).norm().item() / (ref1 - ref0).norm().item())
