"""Run one SALR linear a few times (target for ncu captures).

    python tools/profile_linear.py --shape gate --tokens 32 --reps 5
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2601_16991_b200 as S
from paper_2601_16991_b200 import synthetic

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="gate")
ap.add_argument("--tokens", type=int, default=32)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--no-adapters", action="store_true")
ap.add_argument("--nm24", action="store_true", help="2:4-pruned weights in the NM24 format")
a = ap.parse_args()
# the bench stack's fused launches too: q|k|v and gate|up share their input
SHAPES = dict(synthetic.LLAMA3_8B_LINEARS, qkv=(4096, 6144), gateup=(4096, 28672))
K, N = SHAPES[a.shape]
g = torch.Generator(device="cuda").manual_seed(0)
w = (torch.randn(K, N, generator=g, device="cuda") * 0.02).bfloat16()
if a.nm24:
    w = S.prune(w.float(), S.PruneConfig(0.5, S.PruneMethod.SEMI_STRUCTURED_NM, nm=(2, 4))).bfloat16()
    s = S.encode(w, value_dtype="bf16").use_nm24()
else:
    w = torch.where(w.float().abs() < 0.02 * 0.6744897501960817, torch.zeros_like(w), w)
    s = S.encode(w, value_dtype="bf16")
    s.compute_format()
fused = None
if not a.no_adapters:
    fused = S.fuse([S.AdapterPair(torch.randn(K, 16, device="cuda") / 64, torch.randn(16, N, device="cuda") * 0.02, 16),
                    S.AdapterPair(torch.randn(K, 16, device="cuda") / 64, torch.randn(16, N, device="cuda") * 0.02, 16, 2.0)])
x = torch.randn(a.tokens, K, device="cuda").bfloat16()
out = torch.empty(a.tokens, N, device="cuda", dtype=torch.bfloat16)
for _ in range(a.reps):
    S.salr_linear(x, s, fused, out=out, check_finite=False)
torch.cuda.synchronize()
print("compressed_bytes", s.compressed_bytes, "nnz", s.nnz, "device_bytes", s.device_bytes)
