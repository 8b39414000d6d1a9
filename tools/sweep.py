"""BASELINE configs[4]: sparsity x adapter-rank sweep at 4096x14336 vs cuBLAS.

    python tools/sweep.py [--tokens 1,8,32] [--reps 24]

For p in {0.3, 0.5, 0.7} and r in {8, 16, 64} (LoRA r + residual r, R = 2r)
prints one JSON line per (p, r, M): the fused kernel's graph-timed device
time (programmatic dependent launch, as in the stack), compressed GB/s and
fraction of the measured HBM peak, the compressed/dense byte ratio, and
cuBLAS dense bf16 on the merged weight (W_hat + A B) for the speedup.
Weights rotate over --copies encodings (> L2) so launches stream from HBM.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2601_16991_b200 as S

ap = argparse.ArgumentParser()
ap.add_argument("--tokens", default="1,8,32")
ap.add_argument("--reps", type=int, default=24)
ap.add_argument("--copies", type=int, default=6)
a = ap.parse_args()
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
try:
    peak = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    peak = 6650.0
QUANT = {0.3: 0.3853204664075676, 0.5: 0.6744897501960817, 0.7: 1.0364333894937898}
K, N = 4096, 14336


def graph_time(fn, reps):
    fn(0)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(reps):
            fn(i)
    g.replay()
    torch.cuda.synchronize()
    best = None
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        e1.synchronize()
        t = 1e3 * e0.elapsed_time(e1) / reps
        best = t if best is None else min(best, t)
    return best


gen = torch.Generator(device="cuda").manual_seed(0)
for p in (0.3, 0.5, 0.7):
    for r in (8, 16, 64):
        mats, fus, dense = [], [], []
        for c in range(a.copies):
            w = (torch.randn(K, N, generator=gen, device="cuda") * 0.02).bfloat16()
            w = torch.where(w.float().abs() < 0.02 * QUANT[p], torch.zeros_like(w), w)
            s = S.encode(w, value_dtype="bf16")
            s.compute_format()
            f = S.fuse([S.AdapterPair(torch.randn(K, r, generator=gen, device="cuda") / 64,
                                      torch.randn(r, N, generator=gen, device="cuda") * 0.02, r),
                        S.AdapterPair(torch.randn(K, r, generator=gen, device="cuda") / 64,
                                      torch.randn(r, N, generator=gen, device="cuda") * 0.02, r, 2.0)])
            f.device_operands()
            mats.append(s)
            fus.append(f)
            if c < 4:
                dense.append((w.float() + f.a_cat @ f.b_cat).bfloat16())
            del w
        for M in [int(t) for t in a.tokens.split(",")]:
            x = torch.randn(M, K, device="cuda").bfloat16()
            outs = [torch.empty(M, N, device="cuda", dtype=torch.bfloat16) for _ in range(2)]
            us = graph_time(lambda i: S.salr_linear(x, mats[i % a.copies], fus[i % a.copies], out=outs[i & 1],
                                                    check_finite=False, pdl=True), a.reps)
            cus = graph_time(lambda i: torch.matmul(x, dense[i % len(dense)]), a.reps)
            cb = mats[0].compressed_bytes
            print(json.dumps({"sparsity": p, "rank": r, "R": 2 * r, "M": M, "us": round(us, 2),
                              "compressed_bytes": cb, "GBs": round(cb / us / 1e3, 1),
                              "frac_hbm": round(cb / us / 1e3 / peak, 3),
                              "bytes_vs_dense": round(cb / (2 * K * N), 3),
                              "cublas_us": round(cus, 2), "speedup_vs_cublas": round(cus / us, 3)}), flush=True)
        del mats, fus, dense
        torch.cuda.empty_cache()
