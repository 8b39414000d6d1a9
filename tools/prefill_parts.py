"""Component times of the dense prefill path (decode, U chain, GEMM) at M=2048."""
import torch, json, sys, os
sys.path.insert(0, os.getcwd())
import paper_2601_16991_b200 as S
from paper_2601_16991_b200 import _lib, pipeline
def timed(fn, iters=20):
    fn(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream(); st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        fn()
        with torch.cuda.graph(g, stream=st):
            fn()
    torch.cuda.current_stream().wait_stream(st)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters): g.replay()
    e1.record(); torch.cuda.synchronize()
    return 1e3 * e0.elapsed_time(e1) / iters
for K, N in ((4096, 4096), (4096, 14336)):
    w = (torch.randn(K, N, device="cuda") * 0.02).bfloat16()
    w = torch.where(w.float().abs() < 0.0135, torch.zeros_like(w), w)
    s = S.encode(w, value_dtype="bf16"); rec, off, _ = s.compute_format()
    dense = torch.empty(K + 128, N, dtype=torch.bfloat16, device="cuda")
    lib = _lib.load()
    t_dec = timed(lambda: lib.salr_tb2_decode(_lib.ptr(rec), _lib.ptr(off), K, N, _lib.ptr(dense), N, _lib.stream_ptr()))
    M = 2048
    x = torch.randn(M, K, device="cuda").bfloat16()
    acat = torch.randn(K, 64, device="cuda").bfloat16()
    def uchain():
        u = torch.mm(x, acat, out_dtype=torch.float32)
        hi = u.to(torch.bfloat16); lo = (u - hi.float()).to(torch.bfloat16)
        return torch.cat([x, hi, lo], dim=1)
    t_u = timed(uchain)
    t_umm = timed(lambda: torch.mm(x, acat, out_dtype=torch.float32))
    xs = x.view(M, 8, K // 8).transpose(0, 1)
    as_ = acat.view(8, K // 8, 64)
    t_ubmm = timed(lambda: torch.bmm(xs, as_, out_dtype=torch.float32).sum(0))
    t_cat = timed(lambda: torch.cat([x, x[:, :128]], dim=1))
    xc = uchain()
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    t_mm = timed(lambda: torch.mm(xc, dense, out=out))
    t_mm0 = timed(lambda: torch.mm(x, dense[:K], out=out))
    print(json.dumps({"K": K, "N": N, "decode_us": round(t_dec, 1), "decode_GBps": round((rec.numel() + 2 * K * N) / t_dec / 1e3, 0), "u_cat_us": round(t_u, 1), "u_mm_us": round(t_umm, 1), "u_bmm_us": round(t_ubmm, 1), "cat_us": round(t_cat, 1), "mm_Kplus_us": round(t_mm, 1), "mm_us": round(t_mm0, 1)}))
