"""Benchmark of the B200 SALR linear hot path (driver contract: see DESIGN.md
"Measurement").

Workload (one "step"): one decode token-batch (M tokens, default 32) through
the Llama3-8B SALR linear stack -- 32 layers x 7 linears (q, k, v, o, gate, up,
down; BASELINE configs[1] shapes, stacked as in configs[3]) at 50% magnitude
sparsity with LoRA r16 + residual r16 adapters fused (R = 32).  Weights are
synthetic random-init (no checkpoints offline).  At --gpus N the stack is
column-sharded: every rank decodes only its 128-column-aligned stripe of each
linear and the shards are all-gathered (NCCL) at the four layer boundaries
(after q|k|v, o, gate|up, down) -- SURVEY.md 8(e).

Output: one JSON line (rank 0) with value = whole-job tokens/s (device-timed,
CUDA events, max over ranks), e2e (host buffers in and out, public API),
roofline of the dominant kernel (compressed bytes / kernel time vs the
measured HBM copy bandwidth), cuBLAS dense-bf16 comparator, clocks (NVML
sampled during the timed region), and the CPU baseline (oracle port of the
reference pipelined_forward on the host cores, bounded sample).

``--impl reference`` times the reference's own CPU implementation instead:
the unmodified package installed offline into baseline/_ref (pure
Python/NumPy, its stock ``salr.pipeline.pipelined_forward``), on layer 0 of
the same stack (the same seeded weights, adapters and X as the GPU arm), one
layer per step, and prints the same metric with "impl": "reference".  Only
when baseline/_ref is missing does it fall back to the oracle port
(oracle/salr_oracle.py, kind "port").
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

LINEARS = ["q", "k", "v", "o", "gate", "up", "down"]
SHAPES = {"q": (4096, 4096), "k": (4096, 1024), "v": (4096, 1024), "o": (4096, 4096),
          "gate": (4096, 14336), "up": (4096, 14336), "down": (14336, 4096)}
METRIC = "SALR linear tokens/s & compressed-weight HBM GB/s, Llama3-8B shapes @50% sparsity"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["salr", "reference"], default="salr")
    ap.add_argument("--tokens", type=int, default=32)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--sparsity", type=float, default=0.5)
    ap.add_argument("--batches", default="1,8,32", help="extra decode batch sizes reported per-M")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cublas", action="store_true")
    ap.add_argument("--no-nm24", action="store_true", help="skip the 2:4 (NM24) stack leg")
    ap.add_argument("--chain", action="store_true",
                    help="one persistent launch per layer (salr_chain) instead of one launch per linear")
    return ap.parse_args()


def peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


# ---------------------------------------------------------------------------
# clocks: NVML sampled in a background thread during the timed region

class ClockSampler:
    def __init__(self, dev_index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    _REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self._REASONS.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception:
                break
            time.sleep(0.002)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        reasons = sorted(self.reasons - {"gpu_idle"})
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# distributed helpers

def dist_setup(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return world, rank, local


def shard_cols(n: int, world: int, rank: int):
    """128-column-aligned stripe of an output dimension."""
    from paper_2601_16991_b200.sharding import shard_cols as _sc
    return _sc(n, world, rank)


# ---------------------------------------------------------------------------
# reference arm: oracle (CPU) on a bounded sample

def _reference_pkg():
    """The unmodified reference package installed offline into baseline/_ref
    (pure Python/NumPy), or None."""
    ref = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "salr")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        import salr  # noqa: F401
        from salr import bitmap, fusion, pipeline, residual
        return bitmap, fusion, pipeline, residual
    except Exception:
        return None


def _blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max((i.get("num_threads", 1) for i in threadpool_info()), default=1)
    except Exception:
        return os.cpu_count()


class RefLayer:
    """Layer 0 of the bench stack prepared for the reference CPU path: the
    GPU arm's own seeded weights / adapters / X (generated with the same
    seeds on the GPU when one is present, then copied to host float64),
    encoded and fused by the reference package itself (baseline/_ref), or by
    the oracle port when that is absent."""

    def __init__(self, tokens, sparsity):
        import torch
        dev = torch.device("cuda", 0) if torch.cuda.is_available() else torch.device("cpu")
        self.rng_device = dev.type
        layer = gen_layer(0, 1, 0, sparsity, dev)
        self.x = gen_x(tokens, dev).double().cpu().numpy()
        self.ref = _reference_pkg()
        self.kind = "reference" if self.ref is not None else "port"
        self.linears = []
        self.comp = 0
        for name in STACK_ORDER:
            w, ads, (k, n), _ = layer[name]
            wn = w.double().cpu().numpy()
            if self.ref is not None:
                bitmap, fusion, pipeline, residual = self.ref
                sm = bitmap.encode(wn)
                fz = fusion.fuse([residual.AdapterPair(a.double().cpu().numpy(), b.double().cpu().numpy(), 16, sc)
                                  for a, b, sc in ads])
            else:
                from oracle import salr_oracle as O
                sm = O.encode(wn)
                fz = O.fuse([O.Adapter(a.double().cpu().numpy(), b.double().cpu().numpy(), 16, sc)
                             for a, b, sc in ads])
            self.linears.append((name, sm, fz, k))
            self.comp += sm.rows * ((sm.cols + 7) // 8) + 2 * sm.nnz  # algorithmic bytes, bf16 values
        del layer

    def forward(self, overlap=True):
        """One layer (q|k|v, o, gate|up, down) at M tokens through the stock
        reference pipelined_forward; o consumes the q columns and down the
        gate columns, as on the GPU."""
        h = self.x
        for name, sm, fz, k in self.linears:
            if self.ref is not None:
                pipeline = self.ref[2]
                y = pipeline.pipelined_forward(h[:, :k], sm, fz, pipeline.PipelineConfig(overlap=overlap))
            else:
                from oracle import salr_oracle as O
                y = O.pipelined_forward(h[:, :k], sm, fz)
            h = y
        return h


def cpu_sample(tokens: int, sparsity: float, budget_s: float = 20.0):
    """Bounded CPU baseline for the GPU arm's line: median of up to 3 passes
    of layer 0 through the reference path (stock overlap=True), x32 layers."""
    rl = RefLayer(tokens, sparsity)
    times = []
    t_start = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        rl.forward()
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start > budget_s or len(times) >= 3:
            break
    layer_s = statistics.median(times)
    step_s = layer_s * 32
    what = ("reference salr.pipeline.pipelined_forward (stock PipelineConfig(): overlap=True, decoder "
            "thread + ring, f64) from baseline/_ref" if rl.kind == "reference" else
            "oracle port of pipelined_forward (f64, 64x8-byte tiles, serial)")
    return {
        "value": tokens / step_s, "unit": "tokens/s", "cores": _blas_threads(), "kind": rl.kind,
        "sample": f"{what} over layer 0 of the bench stack (the same seeded weights as the GPU arm; 4 linears: "
                  f"q|k|v, o, gate|up, down) at M={tokens}, median of {len(times)} passes = {layer_s:.3f} s/layer, "
                  f"x32 layers; {os.cpu_count()} host cores visible, OpenBLAS threads={_blas_threads()}",
        "compressed_gbs": rl.comp * 32 / step_s / 1e9,
        "layer_s": layer_s,
    }


def stack_config(args, world, how):
    return {"workload": "llama3-8b 32-layer SALR linear stack (q,k,v,o,gate,up,down; configs[1] shapes x32 "
                        "layers = configs[3] at this N), one decode token-batch per step; q|k|v and gate|up "
                        "weights column-concatenated (4 SALR linears per layer, adapters per original linear)",
            "tokens": args.tokens, "layers": 32, "sparsity": args.sparsity, "adapters": "r16+r16 fused (R=32)",
            "parallelism": f"col-shard{world}" if world > 1 else "single",
            "l2": "working set 7.85 GB >> 126 MB L2 (inputs larger than L2)", "execution": how}


def run_reference(args):
    """Reference arm: the reference's own CPU implementation (baseline/_ref)
    on layer 0 of the same stack.  One step = one of the 32 identical-shape
    layers (4 linears); value = M / (32 x step time) tokens/s of the stack.
    Exactly --steps timed steps after --warmup untimed ones (all with the
    stock overlap=True configuration); overlap=False is timed once more after
    the timed region and reported beside it."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    rl = RefLayer(args.tokens, args.sparsity)
    for _ in range(args.warmup):
        rl.forward()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        rl.forward()
    total = time.perf_counter() - t0
    layer_s = total / args.steps
    t1 = time.perf_counter()
    rl.forward(overlap=False)
    serial_s = time.perf_counter() - t1
    value = args.tokens / (32 * layer_s)
    cores = _blas_threads()
    what = ("reference salr.pipeline.pipelined_forward from baseline/_ref (unmodified)" if rl.kind == "reference"
            else "oracle port of pipelined_forward (baseline/_ref missing)")
    line = {
        "metric": METRIC, "impl": "reference", "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * layer_s, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": dict(stack_config(args, world, "CPU (reference host path)"),
                       step="one of the 32 layers (q|k|v, o, gate|up, down at M tokens); value = M / (32 x step)",
                       weights=f"layer 0 of the GPU arm (same seeds; generated on {rl.rng_device})"),
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": rl.kind,
                         "sample": f"{what}, stock PipelineConfig() (overlap=True), {args.steps} timed layers "
                                   f"after {args.warmup} warm-up layers; {os.cpu_count()} host cores, "
                                   f"OpenBLAS threads={cores}"},
        "overlap_false": {"value": args.tokens / (32 * serial_s), "unit": "tokens/s", "ms_per_layer": 1e3 * serial_s,
                          "note": "PipelineConfig(overlap=False), one layer after the timed region"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "compressed_gbs": rl.comp / layer_s / 1e9,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# the B200 arm

# The stack runs the per-layer linears as four SALR linears: q|k|v and
# gate|up share their input, so their weights are concatenated along the
# output columns (one encode each; adapters keep their per-linear blocks,
# B_cat is block-structured) -- mathematically the same seven linears with
# one weight stream and one launch per shared input.
FUSED = {"qkv": (4096, [("q", 4096), ("k", 1024), ("v", 1024)]),
         "o": (4096, [("o", 4096)]),
         "gateup": (4096, [("gate", 14336), ("up", 14336)]),
         "down": (14336, [("down", 4096)])}
STACK_ORDER = ("qkv", "o", "gateup", "down")


def _prune_threshold(sparsity):
    q = {0.3: 0.3853204664075676, 0.5: 0.6744897501960817, 0.7: 1.0364333894937898}.get(sparsity)
    if q is None:
        raise SystemExit(f"unsupported sparsity {sparsity}")
    return 0.02 * q  # |w| quantile of N(0, 0.02^2): magnitude pruning at `sparsity`


def gen_layer(layer, world, rank, sparsity, device, pattern="magnitude"):
    """Dense inputs of one stack layer, seeded per (layer, rank) so any layer
    can be regenerated alone: {fused name: (W_hat bf16 (k x n_local),
    [(A, B, scale)] bf16-exact fp32 adapter factors, (k, n_local), (c0, c1))}.
    The reference arm regenerates layer 0 with the same seeds.  pattern
    "2:4": the reference's N:M mask (prune.py:238-248, 2 largest |w| of every
    4 consecutive columns) instead of global magnitude pruning."""
    import torch
    import paper_2601_16991_b200 as S
    g = torch.Generator(device=device).manual_seed(1234 + 7919 * layer + 17 * rank)
    thr = _prune_threshold(sparsity)
    nm = S.PruneConfig(0.5, S.PruneMethod.SEMI_STRUCTURED_NM, nm=(2, 4))
    out = {}
    for name in STACK_ORDER:
        k, parts = FUSED[name]
        n = sum(w for _, w in parts)
        c0, c1 = shard_cols(n, world, rank)
        nl = c1 - c0
        w = (torch.randn(k, nl, generator=g, device=device) * 0.02).to(torch.bfloat16)
        if pattern == "2:4":
            w = S.prune(w.float(), nm).to(torch.bfloat16)
        else:
            w = torch.where(w.float().abs() < thr, torch.zeros_like(w), w)
        ads = []
        p0 = 0
        for _, pw in parts:  # LoRA r16 + residual r16 per original linear, on its own columns
            lo, hi = max(p0, c0) - c0, min(p0 + pw, c1) - c0
            for scale in (1.0, 2.0):
                a = (torch.randn(k, 16, generator=g, device=device) / 64).bfloat16().float()
                bm = torch.zeros(16, nl, device=device)
                if hi > lo:
                    bm[:, lo:hi] = (torch.randn(16, hi - lo, generator=g, device=device) * 0.02).bfloat16().float()
                ads.append((a, bm, scale))
            p0 += pw
        out[name] = (w, ads, (k, nl), (c0, c1))
    return out


def gen_x(tokens, device):
    import torch
    g = torch.Generator(device=device).manual_seed(7)
    return torch.randn(tokens, 4096, generator=g, device=device).bfloat16()


def build_stack(layers, world, rank, sparsity, device, pattern="magnitude"):
    """Per layer: {fused name: (BitmapSparseMatrix shard, FusedAdapters shard, (k, n_local), col range)}."""
    import paper_2601_16991_b200 as S

    stack = []
    for layer in range(layers):
        lin = {}
        for name, (w, ads, kn, cols) in gen_layer(layer, world, rank, sparsity, device, pattern).items():
            s = S.encode(w, value_dtype="bf16")
            if pattern == "2:4":
                s.use_nm24()  # fixed-size 2:4 tiles: the compute format of this stack
            else:
                s.compute_format()  # the linear kernel's operand format, built once at load
            del w
            fused = S.fuse([S.AdapterPair(a, b, 16, sc) for a, b, sc in ads])
            fused.device_operands()
            lin[name] = (s, fused, kn, cols)
        stack.append(lin)
    return stack


def layer_check(lin, x, layer0):
    """End-of-run parity check: the 4 fused linears of one layer through the
    product path vs a float64 dense reference on the same bf16-exact inputs
    (X, W_hat, A, B): rel-Frobenius and max-abs of each output."""
    import torch
    import paper_2601_16991_b200 as S
    worst = {"rel_frob": 0.0, "max_abs_rel": 0.0}
    h = x
    for name in STACK_ORDER:
        s, f, (k, nl), _ = lin[name]
        w, ads, _, _ = layer0[name]
        xin = h[:, :k]
        y = S.salr_linear(xin, s, f, out_dtype=torch.float32, check_finite=False).double()
        ref = xin.double() @ w.double()
        for a, b, sc in ads:
            ref += sc * ((xin.double() @ a.double()) @ b.double())
        rel = float((y - ref).norm() / ref.norm())
        mabs = float((y - ref).abs().max() / ref.abs().max())
        worst["rel_frob"] = max(worst["rel_frob"], rel)
        worst["max_abs_rel"] = max(worst["max_abs_rel"], mabs)
        h = y.bfloat16()
    worst["tolerance"] = "rel_frob <= 5e-4 and max_abs <= 2.5e-4 * max|ref| (fp32 accumulate, bf16 operands)"
    worst["ok"] = worst["rel_frob"] <= 5e-4 and worst["max_abs_rel"] <= 2.5e-4
    return worst


PLAN = [("qkv", None), ("o", (0, 4096)), ("gateup", None), ("down", (0, 14336))]


def make_runner(stack, tokens, world, rank, group=None, chain=None):
    """The package's column-sharded stack over this rank's shards: o consumes
    the q columns of q|k|v and down the gate columns of gate|up (the stack is
    linears only; attention and the MLP nonlinearity are outside the path),
    and only those columns are gathered."""
    from paper_2601_16991_b200.sharding import ShardedLinear, ShardedStack
    layers = []
    for lin in stack:
        layers.append({name: ShardedLinear(s, f, sum(w for _, w in FUSED[name][1]), world, rank)
                       for name, (s, f, _, _) in lin.items()})
    return ShardedStack(layers, PLAN, world, rank, group, tokens, chain=chain)


def time_steps(fn, steps, warmup, world, sampler_dev):
    import torch
    import torch.distributed as dist
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(sampler_dev) as cs:
        e0.record()
        for _ in range(steps):
            fn()
        e1.record()
        e1.synchronize()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
        ms = float(t.item())
    return ms, cs.summary()


def graph_time_us(fn, reps):
    """Device time per call of `fn(i)`: one CUDA graph of `reps` back-to-back
    calls, best of 3 replays timed with CUDA events on the capture stream."""
    import torch
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
    del g
    return best


def per_linear_kernel_times(stack, tokens, reps=32):
    """Device time of each linear (the fused kernel; launched back to back
    with programmatic dependent launch as in the stack), layers rotated so
    every launch streams its weights from HBM."""
    import torch
    import paper_2601_16991_b200 as S
    res = {}
    x = {4096: torch.randn(tokens, 4096, device="cuda").bfloat16(),
         14336: torch.randn(tokens, 14336, device="cuda").bfloat16()}
    L = len(stack)
    for name in STACK_ORDER:
        k, nl = stack[0][name][2]
        outs = [torch.empty(tokens, nl, dtype=torch.bfloat16, device="cuda") for _ in range(2)]

        def call(i):
            s, f, _, _ = stack[i % L][name]
            S.salr_linear(x[k], s, f, out=outs[i & 1], check_finite=False, pdl=True)

        us = graph_time_us(call, reps)
        s0 = stack[0][name][0]
        res[name] = {"us": us, "compressed_bytes": s0.compressed_bytes, "nnz": s0.nnz, "shape": [k, nl]}
    return res


def cublas_times(stack, tokens, reps=20):
    """cuBLAS dense bf16 baseline: X @ W_merged (W_hat + A B densified), same rotation."""
    import torch
    import paper_2601_16991_b200 as S
    res = {}
    L = min(len(stack), 8)
    for name in STACK_ORDER:
        k, nl = stack[0][name][2]
        ws = []
        for i in range(L):
            s, f, _, _ = stack[i][name]
            ws.append((S.decode(s) + f.a_cat @ f.b_cat).bfloat16())
        x = torch.randn(tokens, k, device="cuda").bfloat16()
        us = graph_time_us(lambda i: torch.matmul(x, ws[i % L]), reps)
        res[name] = {"us": us, "dense_bytes": 2 * k * nl}
        del ws
        torch.cuda.empty_cache()
    return res


def nm24_leg(args, dev, local, cublas):
    """The paper's published configuration (2:4 semi-structured, PAPER.md
    Table inference): the same 32-layer stack with weights under the
    reference's 2:4 mask, held in the NM24 compute format.  Stack tokens/s per
    decode batch, per-linear kernel times at --tokens, roofline of the fused
    kernel on its own record bytes, layer-0 check.  cuBLAS dense bf16 times do
    not depend on the weight values: the main leg's are reused."""
    import torch
    M = args.tokens
    stack = build_stack(args.layers, 1, 0, 0.5, dev, pattern="2:4")
    torch.cuda.synchronize()
    per_m = {}
    for mb in [int(v) for v in args.batches.split(",") if v]:
        r = make_runner(stack, mb, 1, 0)
        r.x_in.copy_(gen_x(mb, dev))
        r.step(r.x_in)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            r.step(r.x_in)
        n = max(5, args.steps // 2)
        ms, clk = time_steps(g.replay, n, 3, 1, local)
        per_m[str(mb)] = {"tokens_per_s": mb / (ms / n / 1e3), "ms_per_step": ms / n, "clocks": clk}
        del g, r
    per = per_linear_kernel_times(stack, M)
    rec_bytes = sum(stack[0][n][0].device_bytes for n in per)  # the 9216-byte tiles each launch streams
    k_us = sum(v["us"] for v in per.values())
    alg = sum(v["compressed_bytes"] for v in per.values())
    hbm_peak = peaks()[0]
    out = {
        "format": "NM24 (fixed 9216-byte 64x128 tiles: 2 bf16 + a 4-bit column mask per row group of 4)",
        "mask": "reference N:M rule, n=2 m=4 along the columns (prune.py:238-248), device mask",
        "per_batch": per_m,
        "per_linear": per,
        "kernel_us_per_layer": k_us,
        "roofline": {"bound": "hbm", "achieved_record_bytes": rec_bytes / (k_us * 1e-6) / 1e9,
                     "achieved_algorithmic": alg / (k_us * 1e-6) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                     "frac": rec_bytes / (k_us * 1e-6) / 1e9 / hbm_peak},
        "resident_bytes_per_weight": sum(lin[n][0].device_bytes for lin in stack for n in STACK_ORDER)
        / sum(lin[n][2][0] * lin[n][2][1] for lin in stack for n in STACK_ORDER),
        "check": layer_check(stack[0], gen_x(M, dev), gen_layer(0, 1, 0, 0.5, dev, "2:4")),
    }
    if cublas is not None:
        out["cublas_dense_bf16_speedup"] = cublas["us_per_layer"] / k_us
    del stack
    torch.cuda.empty_cache()
    return out


def run_salr(args):
    import torch
    import torch.distributed as dist

    world, rank, local = dist_setup(args)
    if world != args.gpus and rank == 0:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    dev = torch.device("cuda", torch.cuda.current_device())
    hbm_peak, tf_peak, peak_src = peaks()
    t_setup = time.time()
    stack = build_stack(args.layers, world, rank, args.sparsity, dev)
    torch.cuda.synchronize()
    setup_s = time.time() - t_setup
    M = args.tokens

    # ---- device-timed steps (graph-captured stack)
    runner = make_runner(stack, M, world, rank, chain=args.chain)
    x0 = gen_x(M, dev)
    runner.x_in.copy_(x0)
    use_graph = True
    runner.step(runner.x_in)  # warm call; allocates workspaces
    torch.cuda.synchronize()
    try:  # one CUDA graph per step (NCCL all-gathers are captured too at N > 1)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            out_static = runner.step(runner.x_in)
        step_fn = graph.replay
    except Exception as e:  # pragma: no cover - capture unsupported by this NCCL build
        print(f"warning: step graph capture failed ({e}); timing eager steps", file=sys.stderr)
        use_graph = False
        torch.cuda.synchronize()
        step_fn = lambda: runner.step(runner.x_in)  # noqa: E731
    ms, clocks = time_steps(step_fn, args.steps, args.warmup, world, local)
    ms_per_step = ms / args.steps
    tokens_per_s = M / (ms_per_step / 1e3)  # every rank processes the same M tokens (sharded columns)

    comp_bytes_local = sum(lin[n][0].compressed_bytes for lin in stack for n in STACK_ORDER)
    comp_bytes = comp_bytes_local
    if world > 1:
        t = torch.tensor([float(comp_bytes_local)], device=dev)
        dist.all_reduce(t)
        comp_bytes = t.item()

    # ---- e2e: pinned host X in, host Y out, every step
    h_x = torch.empty(M, 4096, dtype=torch.bfloat16, pin_memory=True)
    h_x.copy_(x0.cpu())
    h_y = torch.empty(M, 4096, dtype=torch.bfloat16, pin_memory=True)

    def e2e_step():
        runner.x_in.copy_(h_x, non_blocking=True)
        if use_graph:
            graph.replay()
            y = out_static
        else:
            y = runner.step(runner.x_in)
        h_y.copy_(y, non_blocking=True)
        torch.cuda.current_stream().synchronize()

    e2e_steps = max(5, min(args.steps, 50))
    for _ in range(3):
        e2e_step()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = t.item()
    e2e_value = M * e2e_steps / e2e_s

    line = None
    if rank == 0:
        per = per_linear_kernel_times(stack, M)
        k_bytes = sum(v["compressed_bytes"] for v in per.values())
        k_us = sum(v["us"] for v in per.values())
        achieved = k_bytes / (k_us * 1e-6) / 1e9
        # DRAM bytes of the dominant launch (gate|up, the largest share of the
        # step) from one committed `ncu --set full` capture of the same launch
        # (tools/gpu_ncu_bench.sh); null when that capture is absent
        traffic, traffic_src = None, None
        prof = os.path.join(REPO, "profiles", "ncu_summary.json")
        if os.path.exists(prof):
            try:
                d = json.load(open(prof))
                if d.get("launch") == f"gateup M={M}":
                    traffic, traffic_src = d.get("traffic_bytes_per_launch"), d.get("source")
            except Exception:
                traffic = None
        dom = max(per, key=lambda n: per[n]["us"])
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "traffic": traffic, "traffic_source": traffic_src,
                "traffic_algorithmic_bytes": per["gateup"]["compressed_bytes"],
                "dominant_launch": dom, "peak_source": peak_src,
                "kernel": "salr_linear_kernel (+ adapter_u_kernel, PDL-overlapped)",
                "algorithmic_bytes": "K*ceil(N/8) + 2*nnz per linear (SURVEY.md 8(d))",
                "per_linear": per}
        extra = {}
        if not args.no_cublas and world == 1:
            cb = cublas_times(stack, M)
            cb_us = sum(v["us"] for v in cb.values())
            extra["cublas_dense_bf16"] = {"us_per_layer": cb_us, "salr_us_per_layer": k_us,
                                          "speedup": cb_us / k_us, "per_linear": cb}
        if world == 1 and not args.no_nm24:
            extra["two_four"] = None  # filled after the main per-batch runs (own stack)
        per_m = {}
        if world == 1:
            for mb in [int(v) for v in args.batches.split(",") if v]:
                if mb == M:
                    per_m[str(mb)] = {"tokens_per_s": tokens_per_s, "ms_per_step": ms_per_step, "clocks": clocks,
                                      "compressed_gbs": comp_bytes / (ms_per_step / 1e3) / 1e9}
                    continue
                r2 = make_runner(stack, mb, 1, 0, chain=args.chain)
                r2.x_in.copy_(torch.randn(mb, 4096, device=dev).bfloat16())
                r2.step(r2.x_in)
                torch.cuda.synchronize()
                g2 = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g2):
                    r2.step(r2.x_in)
                ms2, clk2 = time_steps(g2.replay, max(5, args.steps // 2), 3, 1, local)
                per_m[str(mb)] = {"clocks": clk2, "tokens_per_s": mb / (ms2 / max(5, args.steps // 2) / 1e3),
                                  "ms_per_step": ms2 / max(5, args.steps // 2),
                                  "compressed_gbs": comp_bytes / (ms2 / max(5, args.steps // 2) / 1e3) / 1e9}
                del g2, r2
        resident = sum(lin[n][0].device_bytes for lin in stack for n in STACK_ORDER)
        dense_bf16 = sum(2 * lin[n][2][0] * lin[n][2][1] for lin in stack for n in STACK_ORDER)
        memory = {"resident_weight_bytes": resident, "dense_bf16_bytes": dense_bf16,
                  "compression_vs_dense_bf16": dense_bf16 / resident,
                  "resident_bytes_per_weight": resident / (dense_bf16 / 2),
                  "format": "TB2 records + tile offsets only (the compute format; TB rebuilt on demand)"}
        check = layer_check(stack[0], x0, gen_layer(0, world, rank, args.sparsity, dev))
        if "two_four" in extra:
            extra["two_four"] = nm24_leg(args, dev, local, extra.get("cublas_dense_bf16"))
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            c = cpu_sample(M, args.sparsity)
            cpu = {k: c[k] for k in ("value", "unit", "cores", "kind", "sample")}
        line = {
            "metric": METRIC, "value": tokens_per_s, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic random-init weights/inputs",
            "config": stack_config(args, world, ("CUDA graph per step" + (" (NCCL all-gathers captured)" if world > 1 else ""))
                                  if use_graph else "eager (NCCL all-gathers)"),
            "compressed_gbs": comp_bytes / (ms_per_step / 1e3) / 1e9,
            "compressed_bytes_per_step": comp_bytes,
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "tokens/s", "h2d_bytes_per_step": int(h_x.numel() * 2),
                    "d2h_bytes_per_step": int(h_y.numel() * 2),
                    "how": "pinned host X -> device, stack forward (public salr_linear API, graph-replayed), "
                           "device Y -> pinned host, synchronize; wall clock"},
            "gpu_launches": runner.launches_per_step * args.steps,
            "clocks": clocks,
            "memory": memory,
            "check": check,
            "per_batch": per_m,
            "setup_s": setup_s,
            **extra,
        }
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if line is not None:
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_salr(args)


if __name__ == "__main__":
    main()
