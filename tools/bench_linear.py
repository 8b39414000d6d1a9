"""Per-linear device timing of the fused SALR kernel vs cuBLAS dense bf16.

    python tools/bench_linear.py [--tokens 1,8,32] [--shapes q,k,gate,down] [--reps 30]

Each timed region is one CUDA-graph replay of --reps back-to-back launches
(host overhead excluded), rotating through --copies distinct encodings so the
big shapes stream from HBM.
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
ap.add_argument("--tokens", default="1,8,32")
ap.add_argument("--shapes", default="q,k,o,gate,down")
ap.add_argument("--reps", type=int, default=30)
ap.add_argument("--copies", type=int, default=6)
ap.add_argument("--no-adapters", action="store_true")
ap.add_argument("--ctas", type=int, default=0)
ap.add_argument("--stages", type=int, default=0)
ap.add_argument("--cublas", action="store_true")
ap.add_argument("--pdl", action="store_true", help="launch as in the stack (programmatic dependent launch)")
a = ap.parse_args()
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
try:
    peak = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    peak = 6650.0
g = torch.Generator(device="cuda").manual_seed(0)


def graph_time(fn, reps):
    fn(0)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for i in range(reps):
            fn(i)
    gr.replay()
    torch.cuda.synchronize()
    best = None
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gr.replay()
        e1.record()
        e1.synchronize()
        t = 1e3 * e0.elapsed_time(e1) / reps
        best = t if best is None else min(best, t)
    return best


for name in a.shapes.split(","):
    K, N = dict(synthetic.LLAMA3_8B_LINEARS, qkv=(4096, 6144), gateup=(4096, 28672))[name]
    mats, fus, dense = [], [], []
    for c in range(a.copies):
        w = (torch.randn(K, N, generator=g, device="cuda") * 0.02).bfloat16()
        w = torch.where(w.float().abs() < 0.02 * 0.6744897501960817, torch.zeros_like(w), w)
        mats.append(S.encode(w, value_dtype="bf16"))
        mats[-1].compute_format()
        f = None if a.no_adapters else S.fuse([
            S.AdapterPair(torch.randn(K, 16, device="cuda") / 64, torch.randn(16, N, device="cuda") * 0.02, 16),
            S.AdapterPair(torch.randn(K, 16, device="cuda") / 64, torch.randn(16, N, device="cuda") * 0.02, 16, 2.0)])
        fus.append(f)
        if a.cublas and c < 4:
            dense.append(w)
        del w
    for M in [int(t) for t in a.tokens.split(",")]:
        x = torch.randn(M, K, device="cuda").bfloat16()
        outs = [torch.empty(M, N, device="cuda", dtype=torch.bfloat16) for _ in range(2)]
        us = graph_time(lambda i: S.salr_linear(x, mats[i % a.copies], fus[i % a.copies], out=outs[i & 1],
                                                check_finite=False, num_ctas=a.ctas, stages=a.stages,
                                                pdl=a.pdl), a.reps)
        cb = mats[0].compressed_bytes
        row = {"linear": name, "M": M, "us": round(us, 2), "GBs": round(cb / us / 1e3, 1),
               "frac": round(cb / us / 1e3 / peak, 3)}
        if a.cublas:
            cus = graph_time(lambda i: torch.matmul(x, dense[i % len(dense)]), a.reps)
            row["cublas_us"] = round(cus, 2)
            row["speedup"] = round(cus / us, 3)
        print(json.dumps(row), flush=True)
