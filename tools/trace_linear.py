"""Device-side event timeline of the fused linear (globaltimer stamps per CTA).

    python tools/trace_linear.py --shape gate --tokens 1 [--no-adapters]

Prints, per event, min/median/max offset (us) from the earliest kernel-entry
stamp of the same launch, plus the gap between consecutive launches.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2601_16991_b200 as S
from paper_2601_16991_b200 import _lib, synthetic

EV = {10: "entry", 0: "setup done", 1: "tma first", 2: "tma last", 3: "head acc ready", 5: "head pass0 loaded", 12: "head pass0 stored",
      4: "dec first", 11: "dec last", 6: "mma acc_full(last seg)", 7: "epi first acc",
      8: "epi done", 9: "cta end", 19: "u start (epoch read)", 15: "u claim1 back", 16: "dec warp at setup bar", 17: "u compute1 done", 18: "u slice1 synced", 13: "u slices added", 14: "u ready seen", 20: "pub ticket added", 21: "barriers init", 22: "coop0 reduced", 23: "pre-issued S units", 24: "pdl_wait done", 25: "epi seg0 stored", 26: "final syncthreads", 27: "tmem alloc done", 28: "x tiles issued", 29: "head poll start", 30: "head ticket ok", 31: "head reduced"}
ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="gate")
ap.add_argument("--tokens", type=int, default=1)
ap.add_argument("--no-adapters", action="store_true")
ap.add_argument("--launches", type=int, default=4)
ap.add_argument("--detail", type=int, default=4, help="print the event sequence of the N latest CTAs")
ap.add_argument("--graph", action="store_true", help="capture the launches (PDL-chained) in one CUDA graph")
a = ap.parse_args()
K, N = dict(synthetic.LLAMA3_8B_LINEARS, qkv=(4096, 6144), gateup=(4096, 28672))[a.shape]
g = torch.Generator(device="cuda").manual_seed(0)
w = (torch.randn(K, N, generator=g, device="cuda") * 0.02).bfloat16()
w = torch.where(w.float().abs() < 0.02 * 0.6744897501960817, torch.zeros_like(w), w)
s = S.encode(w, value_dtype="bf16")
s.compute_format()
f = None if a.no_adapters else S.fuse([
    S.AdapterPair(torch.randn(K, 16, device="cuda") / 64, torch.randn(16, N, device="cuda") * 0.02, 16),
    S.AdapterPair(torch.randn(K, 16, device="cuda") / 64, torch.randn(16, N, device="cuda") * 0.02, 16, 2.0)])
x = torch.randn(a.tokens, K, device="cuda").bfloat16()
out = torch.empty(a.tokens, N, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    S.salr_linear(x, s, f, out=out, check_finite=False)
torch.cuda.synchronize()
bufs = [torch.zeros(148 * 32 + 16 * 64, dtype=torch.int64, device="cuda") for _ in range(a.launches)]
gr = torch.cuda.CUDAGraph()
lib = _lib.load()
outs = [out, torch.empty_like(out)]
if a.graph:
    # the trace pointer is a kernel argument: baked per captured launch
    with torch.cuda.graph(gr):
        for i, b in enumerate(bufs):
            lib.salr_debug_set_trace(_lib.ptr(b))
            S.salr_linear(x, s, f, out=outs[i & 1], check_finite=False, pdl=True)
    lib.salr_debug_set_trace(None)
    for _ in range(3):
        gr.replay()
    torch.cuda.synchronize()
else:
    # launches are recorded eagerly back to back (trace pointer is baked per launch)
    for b in bufs:
        lib.salr_debug_set_trace(_lib.ptr(b))
        S.salr_linear(x, s, f, out=out, check_finite=False)
    lib.salr_debug_set_trace(None)
    torch.cuda.synchronize()
prev_end = None
for i, b in enumerate(bufs):
    t = b[:148 * 32].view(148, 32).cpu()
    dd = b[148 * 32:].view(16, 64).cpu()
    t0 = int(t[:, 10][t[:, 10] > 0].min())
    if prev_end is None and i == 0 and a.graph:
        pass
    print(f"launch {i}: " + (f"gap from previous last cta end {(t0 - prev_end) / 1e3:.2f} us" if prev_end else ""))
    for ev, name in EV.items():
        col = t[:, ev]
        col = col[col > 0]
        if col.numel() == 0:
            continue
        d = (col - t0).double() / 1e3
        print(f"  {name:24s} min {d.min():8.2f}  med {d.median():8.2f}  max {d.max():8.2f} us  (n={col.numel()})")
    prev_end = int(t[:, 9].max())
    # the latest-finishing CTAs, event by event
    ends = t[:, 9].clone()
    for cta in torch.argsort(ends, descending=True)[:a.detail].tolist():
        evs = sorted((int(t[cta, e]), e) for e in EV if int(t[cta, e]) >= t0)
        print(f"  cta {cta:3d}: " + "  ".join(f"{EV[e]}@{(v - t0) / 1e3:.2f}" for v, e in evs))
    names = ["tma issue", "prep sees full", "prep done", "dec w4 done", "dec w19 done", "mma issued", "-", "-", "iss start", "iss shfl", "iss empty ok", "iss divmod"]
    print("  CTA0 per-unit (SM clock cycles from CTA entry):")
    print("   unit " + " ".join(f"{names[e]:>14s}" for e in (0, 1, 2, 3, 4, 5, 8, 9, 10, 11)))
    print("   epilogue seg: before tmem ld / after 1st ld / stored  (cycles)")
    for sg in range(4):
        if int(dd[12, sg]):
            print(f"   seg {sg}: " + " ".join(f"{int(dd[e, sg]) - int(dd[7, 0]):10d}" for e in (12, 13, 14)))
    for i in range(min(24, 64)):
        if int(dd[0, i]) == 0:
            break
        c0 = int(dd[7, 0])
        print(f"   {i:4d} " + " ".join(f"{(int(dd[e, i]) - c0):14d}" if int(dd[e, i]) else f"{'-':>14s}" for e in (0, 1, 2, 3, 4, 5, 8, 9, 10, 11)))
