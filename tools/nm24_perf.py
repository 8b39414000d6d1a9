"""Per-linear kernel time, 2:4-pruned weights: TB2 (bitmap decoder) vs NM24
(permute decoder) vs cuBLAS dense bf16, graph-replayed over rotating weight
copies (> L2), adapters r16+r16.  Prints one JSON line per (shape, M).

    python tools/nm24_perf.py [--shapes q,gate,down,qkv,gateup] [--tokens 1,8,32]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2601_16991_b200 as S
from paper_2601_16991_b200 import synthetic

ap = argparse.ArgumentParser()
ap.add_argument("--shapes", default="q,k,gate,down,qkv,gateup")
ap.add_argument("--tokens", default="1,8,32")
ap.add_argument("--iters", type=int, default=60)
ap.add_argument("--stages", default="0", help="ring depths to sweep (0 = deepest that fits)")
ap.add_argument("--ncu", action="store_true", help="one eager launch per format (capture target)")
a = ap.parse_args()
SHAPES = dict(synthetic.LLAMA3_8B_LINEARS, qkv=(4096, 6144), gateup=(4096, 28672))
cfg = S.PruneConfig(0.5, S.PruneMethod.SEMI_STRUCTURED_NM, nm=(2, 4))


def timed(fn, iters):
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        for _ in range(3):
            fn()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            fn()
    torch.cuda.current_stream().wait_stream(st)
    for _ in range(3):
        g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(iters):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return 1e3 * e0.elapsed_time(e1) / iters


for name in a.shapes.split(","):
    K, N = SHAPES[name]
    copies = max(2, min(6, int(3 * 126e6 // (1.125 * K * N)) + 1))
    gen = torch.Generator(device="cuda").manual_seed(0)
    ws, tb2, nm = [], [], []
    for c in range(copies):
        w = (torch.randn(K, N, generator=gen, device="cuda") * 0.02).bfloat16()
        w = S.prune(w.float(), cfg).bfloat16()
        ws.append(w)
        t = S.encode(w, value_dtype="bf16")
        t.compute_format()
        tb2.append(t)
        nm.append(S.encode(w, value_dtype="bf16").use_nm24())
    f = S.fuse([S.AdapterPair(torch.randn(K, 16, device="cuda") / 64, torch.randn(16, N, device="cuda") * 0.02, 16),
                S.AdapterPair(torch.randn(K, 16, device="cuda") / 64, torch.randn(16, N, device="cuda") * 0.02, 16,
                              2.0)])
    for M in (int(t) for t in a.tokens.split(",")):
        x = torch.randn(M, K, device="cuda").bfloat16()
        out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        if a.ncu:
            S.salr_linear(x, tb2[0], f, out=out, check_finite=False)
            S.salr_linear(x, nm[0], f, out=out, check_finite=False)
            torch.cuda.synchronize()
            continue
        res = {"shape": name, "K": K, "N": N, "M": M, "copies": copies}
        for st in (int(v) for v in a.stages.split(",")):
            for key, mats in (("tb2", tb2), ("nm24", nm)):
                def run(mats=mats, st=st):
                    for s in mats:
                        S.salr_linear(x, s, f, out=out, check_finite=False, pdl=True, stages=st)
                res[key + "_us" + (f"_s{st}" if st else "")] = round(timed(run, a.iters) / copies, 2)
        if "nm24_us" not in res:
            print(json.dumps(res), flush=True)
            continue
        def dense():  # the merged dense weight (W + A_cat B_cat), one GEMM
            for w in ws:
                torch.matmul(x, w, out=out)
        res["cublas_us"] = round(timed(dense, a.iters) / copies, 2)
        nb = K * N / 8 + 2 * (K * N // 2)
        res["nm24_GBps"] = round(nb / (res["nm24_us"] * 1e-6) / 1e9, 1)
        res["nm24_vs_cublas"] = round(res["cublas_us"] / res["nm24_us"], 3)
        res["nm24_vs_tb2"] = round(res["tb2_us"] / res["nm24_us"], 3)
        print(json.dumps(res), flush=True)
