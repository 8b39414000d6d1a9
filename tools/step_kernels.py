"""List every CUDA kernel one stack step launches (torch.profiler / CUPTI):
the step should consist of the fused SALR launches only (no copy kernels
between chained linears, which would break the programmatic-launch overlap).

    python tools/step_kernels.py [--tokens 32] [--layers 2]
"""
import argparse
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench

ap = argparse.ArgumentParser()
ap.add_argument("--tokens", type=int, default=32)
ap.add_argument("--layers", type=int, default=2)
a = ap.parse_args()
dev = torch.device("cuda", 0)
stack = bench.build_stack(a.layers, 1, 0, 0.5, dev)
r = bench.make_runner(stack, a.tokens, 1, 0)
r.x_in.copy_(bench.gen_x(a.tokens, dev))
for _ in range(2):
    r.step(r.x_in)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    r.step(r.x_in)
    torch.cuda.synchronize()
names = [e.name for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
c = collections.Counter(n[:100] for n in names)
print(f"{len(names)} kernels in one {a.layers}-layer step (M={a.tokens})")
for k, v in c.most_common():
    print(f"{v:4d}  {k}")
