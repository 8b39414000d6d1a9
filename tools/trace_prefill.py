"""Per-k-step timeline of salr_prefill_kernel, CTA 0 (tools only).

    python tools/trace_prefill.py --shape q --tokens 512
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2601_16991_b200 as S
from paper_2601_16991_b200 import _lib, synthetic

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="q")
ap.add_argument("--tokens", type=int, default=512)
a = ap.parse_args()
K, N = synthetic.LLAMA3_8B_LINEARS[a.shape]
g = torch.Generator(device="cuda").manual_seed(0)
w = (torch.randn(K, N, generator=g, device="cuda") * 0.02).bfloat16()
w = torch.where(w.float().abs() < 0.02 * 0.6744897501960817, torch.zeros_like(w), w)
s = S.encode(w, value_dtype="bf16")
s.compute_format()
x = torch.randn(a.tokens, K, device="cuda").bfloat16()
for _ in range(3):
    S.salr_linear(x, s, None, check_finite=False)
torch.cuda.synchronize()
buf = torch.zeros(4 * 64, dtype=torch.int64, device="cuda")
lib = _lib.load()
lib.salr_debug_set_trace(_lib.ptr(buf))
S.salr_linear(x, s, None, check_finite=False)
lib.salr_debug_set_trace(None)
torch.cuda.synchronize()
t = buf.view(4, 64).cpu()
t0 = int(t[0, 0])
print("step  rec_issued  dec_done  mma_w_full_seen  mma_step_issued   (us from first record issue)")
for k in range(64):
    if int(t[0, k]) == 0:
        break
    print(f"{k:4d} " + " ".join(f"{(int(t[e, k]) - t0) / 1e3:10.2f}" for e in (0, 1, 3, 2)))
