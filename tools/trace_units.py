"""Per-unit pipeline timeline of CTA 0 of the decode-size kernel (needs a
library built with -DSALR_UNIT_TRACE; load it via SALR_B200_DEBUG=1 SALR_B200_LIB_AB=...).

    SALR_B200_DEBUG=1 SALR_B200_LIB_AB=ab/libT.so python tools/trace_units.py --shape gate --tokens 32

Columns (us from CTA entry, SM clock / --mhz): producer issue of the record,
decoder group sees it (full), group decode done (first / last warp), MMA warp
sees decoded + X, MMA issued; then per-unit averages of the stage
life-cycle: wait-for-data, decode, decode->MMA, MMA->refill issue.
"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2601_16991_b200 as S
from paper_2601_16991_b200 import _lib, synthetic

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="gate")
ap.add_argument("--tokens", type=int, default=32)
ap.add_argument("--no-adapters", action="store_true")
ap.add_argument("--mhz", type=float, default=1965.0)
ap.add_argument("--units", type=int, default=48)
ap.add_argument("--nm24", action="store_true", help="2:4-pruned weights in the NM24 format")
a = ap.parse_args()
K, N = synthetic.LLAMA3_8B_LINEARS[a.shape]
g = torch.Generator(device="cuda").manual_seed(0)
w = (torch.randn(K, N, generator=g, device="cuda") * 0.02).bfloat16()
if a.nm24:
    w = S.prune(w.float(), S.PruneConfig(0.5, S.PruneMethod.SEMI_STRUCTURED_NM, nm=(2, 4))).bfloat16()
    s = S.encode(w, value_dtype="bf16").use_nm24()
else:
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
lib = _lib.load()
b = torch.zeros(148 * 32 + 16 * 64, dtype=torch.int64, device="cuda")
lib.salr_debug_set_trace(_lib.ptr(b))
S.salr_linear(x, s, f, out=out, check_finite=False)
lib.salr_debug_set_trace(None)
torch.cuda.synchronize()
dd = b[148 * 32:].view(16, 64).cpu()
c0 = int(dd[7, 0])
us = lambda v: (int(v) - c0) / a.mhz  # noqa: E731
cols = [(8, "iss in"), (9, "iss shfl"), (10, "iss empty"), (0, "issue"), (1, "full"), (3, "dec0"), (4, "dec3"),
        (2, "mma wait"), (6, "mma rdy"), (5, "mma iss")]
print("unit " + " ".join(f"{n:>8s}" for _, n in cols))
rows = []
for i in range(min(a.units, 64)):
    if int(dd[0, i]) == 0:
        break
    r = {e: (us(dd[e, i]) if int(dd[e, i]) else None) for e, _ in cols}
    rows.append(r)
    print(f"{i:4d} " + " ".join(f"{r[e]:8.2f}" if r[e] is not None else f"{'-':>8s}" for e, _ in cols))
S_ = lib.salr_debug_last_launch_stages() if hasattr(lib, "salr_debug_last_launch_stages") else None


def avg(xs):
    xs = [v for v in xs if v is not None]
    return statistics.mean(xs) if xs else float("nan")


n = len(rows)
print("stage life-cycle averages (us):")
print(f"  issue -> full seen by decoders : {avg([r[1] - r[0] for r in rows if r[1] and r[0]]):.3f}")
print(f"  decode (full -> last warp done): {avg([r[4] - r[1] for r in rows if r[4] and r[1]]):.3f}")
print(f"  decoded -> MMA ready           : {avg([r[6] - r[4] for r in rows if r[6] and r[4]]):.3f}")
ex = {e: [(us(dd[e, i]) if int(dd[e, i]) else None) for i in range(len(rows))] for e in (11, 13)}
print(f"  warp q0: full -> decode issued : {avg([ex[11][i] - rows[i][1] for i in range(len(rows)) if ex[11][i] and rows[i][1]]):.3f}")
print(f"  warp q0: tcgen05.wait::st      : {avg([ex[13][i] - ex[11][i] for i in range(len(rows)) if ex[13][i] and ex[11][i]]):.3f}")
print(f"  warp q0: stores done -> arrive : {avg([rows[i][3] - ex[13][i] for i in range(len(rows)) if ex[13][i] and rows[i][3]]):.3f}")
print(f"  MMA ready -> issued            : {avg([r[5] - r[6] for r in rows if r[5] and r[6]]):.3f}")
for S2 in (8, 4):
    print(f"  MMA issued -> issue of unit+{S2}   : {avg([rows[i + S2][0] - rows[i][5] for i in range(n - S2) if rows[i][5]]):.3f}")
if n > 1:
    print(f"  mean unit period (issue)       : {(rows[-1][0] - rows[0][0]) / (n - 1):.3f}")
    print(f"  mean unit period (mma issued)  : {(rows[n - 1][5] - rows[0][5]) / (n - 1):.3f}")
