"""Per-CTA event timeline of one chained layer launch (salr_chain, 4 linears
of the bench stack at M tokens): min/median/max of each event per linear.

    python tools/trace_chain.py --tokens 32
"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2601_16991_b200 as S
from paper_2601_16991_b200 import _lib
import bench as B

ap = argparse.ArgumentParser()
ap.add_argument("--tokens", type=int, default=32)
a = ap.parse_args()
dev = torch.device("cuda", 0)
stack = B.build_stack(2, 1, 0, 0.5, dev)
runner = B.make_runner(stack, a.tokens, 1, 0)
x = B.gen_x(a.tokens, dev)
for _ in range(3):
    runner.step(x)
torch.cuda.synchronize()
lib = _lib.load()
buf = torch.zeros(148 * 32, dtype=torch.int64, device="cuda")
lib.salr_debug_set_trace(_lib.ptr(buf))
runner.step(x)
lib.salr_debug_set_trace(None)
torch.cuda.synchronize()
t = buf.view(148, 32).cpu()
t0 = int(t[t > 0].min())
names = ["x past barrier", "mma first", "mma last", "tickets", "reduced", "epi first acc", "epi segs done", "Y done"]
for l, lname in enumerate(("qkv", "o", "gateup", "down")):
    print(f"linear {l} ({lname})")
    for k, nm in enumerate(names):
        col = t[:, 8 * l + k]
        col = col[col > 0]
        if col.numel() == 0:
            continue
        d = (col - t0).double() / 1e3
        print(f"   {nm:16s} min {d.min():8.2f} med {d.median():8.2f} max {d.max():8.2f} us (n={col.numel()})")
for l in range(4):
    gap = (t[:, 8 * l + 7] - t[:, 8 * l + 6]).double() / 1e3
    top = torch.argsort(gap, descending=True)[:4].tolist()
    print(f"linear {l}: largest tail (segs done -> Y done): " +
          ", ".join(f"cta {c} {gap[c]:.2f} us (segs@{(int(t[c, 8*l+6]) - t0) / 1e3:.2f} tickets@{(int(t[c, 8*l+3]) - t0) / 1e3:.2f} "
                    f"reduced@{(int(t[c, 8*l+4]) - t0) / 1e3:.2f} Y@{(int(t[c, 8 * l + 7]) - t0) / 1e3:.2f})" for c in top))
