"""Prefill-size products: fused prefill kernel vs decode-to-dense + cuBLAS
(the default path above 256 tokens) vs cuBLAS on the merged
dense weight; graph-timed over rotating weight copies, adapters r16+r16.

    python tools/prefill_compare.py [--shapes q,gate,down] [--tokens 256,512,1024,2048]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2601_16991_b200 as S
from paper_2601_16991_b200 import pipeline, synthetic

ap = argparse.ArgumentParser()
ap.add_argument("--shapes", default="q,gate,down")
ap.add_argument("--tokens", default="256,512,1024,2048")
ap.add_argument("--iters", type=int, default=10)
a = ap.parse_args()
SHAPES = dict(synthetic.LLAMA3_8B_LINEARS, qkv=(4096, 6144), gateup=(4096, 28672))


def timed(fn, iters):
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        fn()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            fn()
    torch.cuda.current_stream().wait_stream(st)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return 1e3 * e0.elapsed_time(e1) / iters


for name in a.shapes.split(","):
    K, N = SHAPES[name]
    gen = torch.Generator(device="cuda").manual_seed(0)
    mats, dense = [], []
    for c in range(3):
        w = (torch.randn(K, N, generator=gen, device="cuda") * 0.02).bfloat16()
        w = torch.where(w.float().abs() < 0.02 * 0.6744897501960817, torch.zeros_like(w), w)
        s = S.encode(w, value_dtype="bf16")
        s.compute_format()
        mats.append(s)
        dense.append(w)
    f = S.fuse([S.AdapterPair(torch.randn(K, 16, device="cuda") / 64, torch.randn(16, N, device="cuda") * 0.02, 16),
                S.AdapterPair(torch.randn(K, 16, device="cuda") / 64, torch.randn(16, N, device="cuda") * 0.02, 16, 2.0)])
    for M in (int(t) for t in a.tokens.split(",")):
        x = torch.randn(M, K, device="cuda").bfloat16()
        out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        res = {"shape": name, "K": K, "N": N, "M": M}
        for key, use_dense in (("fused_us", False), ("dense_us", True)):
            def run(use_dense=use_dense):
                for s in mats:
                    S.salr_linear(x, s, f, out=out, check_finite=False, dense_prefill=use_dense)
            res[key] = round(timed(run, a.iters) / len(mats), 1)

        def blas():
            for w in dense:
                torch.mm(x, w, out=out)
        res["cublas_us"] = round(timed(blas, a.iters) / len(dense), 1)
        res["dense_vs_cublas"] = round(res["cublas_us"] / res["dense_us"], 3)
        res["fused_vs_cublas"] = round(res["cublas_us"] / res["fused_us"], 3)
        res["dense_tflops"] = round(2 * M * K * N / (res["dense_us"] * 1e-6) / 1e12, 1)
        print(json.dumps(res), flush=True)
