"""Generate golden fixtures by running the REAL reference package.

Run in the authoring container only (``/root/reference`` does not exist on the
GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Outputs (committed, small):
  codec.npz     -- random / edge-case dense inputs with the reference's
                   encode() bitmap + values (bit-exact targets)
  blocks.npz    -- decode_block() tiles for a few (rows, bytes) windows
  forward.npz   -- small pipelined_forward() cases (bf16-exact inputs so the
                   GPU path sees the same numbers)
  config1.npz   -- BASELINE configs[0]: 4096x4096, p=0.5, LoRA r16 + SVD
                   residual r16, M=16.  Stores seeds, the residual factors
                   (bf16-exact), SHA-256 digests of the reference bitmap and
                   values, nnz, and the reference output y (f64).
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

import salr  # noqa: E402  (the reference, via PYTHONPATH)
from salr.bitmap import decode_block, encode  # noqa: E402
from salr.fusion import fuse  # noqa: E402
from salr.linalg import SvdResult  # noqa: E402
from salr.pipeline import PipelineConfig, pipelined_forward  # noqa: E402
from salr.prune import PruneConfig, build_mask  # noqa: E402
from salr.residual import AdapterPair, build_residual_adapter  # noqa: E402

from paper_2601_16991_b200 import synthetic  # noqa: E402

assert "/root/reference" in os.path.abspath(salr.__file__), salr.__file__


def bf16x(a: np.ndarray) -> np.ndarray:
    """Round float64/32 array to bf16-exact float64 (RNE)."""
    f = np.asarray(a, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def codec_cases():
    rng = np.random.default_rng(20260117)
    out = {}
    cases = []
    # edge cases pinned by the reference's own tests (test_bitmap.py:84-120)
    cases.append(np.array([[0.0, 1.5, 0.0, 0.0, -2.0, 0.0, 0.0, 3.0]]))
    cases.append(np.ones((3, 5)))
    cases.append(np.array([[-0.0, 1.0]]))
    cases.append(np.array([[1e-60, 1.0]]))
    cases.append(np.array([[1.0, 0.0, 2.0], [0.0, 3.0, 0.0]]))
    cases.append(np.zeros((4, 12)))
    cases.append(rng.normal(size=(6, 10)))
    for cols in (1, 7, 8, 9, 15, 16, 17, 31, 32, 33, 63, 64, 65, 127, 128, 129):
        w = rng.normal(size=(5, cols))
        w[rng.random(size=w.shape) < 0.5] = 0.0
        cases.append(w)
    for i in range(200):
        rows = int(rng.integers(1, 40))
        cols = int(rng.integers(1, 140))
        density = float(rng.uniform(0.0, 1.0))
        w = rng.normal(size=(rows, cols))
        w[rng.random(size=w.shape) >= density] = 0.0
        if rng.random() < 0.3:
            w[rng.random(size=w.shape) < 0.05] = -0.0
        # most random cases are stored as float32 (encode casts to f32 first,
        # bitmap.py:159); every 10th stays float64 to pin the cast itself
        cases.append(w if i % 10 == 0 else w.astype(np.float32))
    for i, w in enumerate(cases):
        s = encode(w)
        out[f"w_{i}"] = w
        out[f"bitmap_{i}"] = s.bitmap
        out[f"values_{i}"] = s.values
    out["n"] = np.array(len(cases))
    np.savez_compressed(os.path.join(HERE, "codec.npz"), **out)
    print("codec cases:", len(cases))


def block_cases():
    rng = np.random.default_rng(31)
    w = rng.normal(size=(70, 203))
    w[rng.random(size=w.shape) < 0.5] = 0.0
    s = encode(w)
    out = {"w": w}
    windows = [((0, 70), (0, s.bytes_per_row)), ((3, 40), (2, 9)), ((0, 1), (25, 26)),
               ((69, 70), (0, 26)), ((10, 10), (0, 3)), ((5, 9), (4, 4)), ((64, 70), (24, 26))]
    for i, (rr, bb) in enumerate(windows):
        out[f"rr_{i}"] = np.array(rr)
        out[f"bb_{i}"] = np.array(bb)
        out[f"tile_{i}"] = decode_block(s, rr, bb)
    out["n"] = np.array(len(windows))
    np.savez_compressed(os.path.join(HERE, "blocks.npz"), **out)


def forward_cases():
    rng = np.random.default_rng(5150)
    shapes = [(37, 53, 11), (64, 128, 16), (200, 300, 7), (130, 260, 1), (256, 512, 32),
              (512, 384, 8), (96, 1000, 3), (1000, 96, 5)]
    out = {}
    for i, (k, n, m) in enumerate(shapes):
        w = bf16x(rng.normal(scale=0.05, size=(k, n)))
        w[rng.random(size=w.shape) < 0.5] = 0.0
        x = bf16x(rng.normal(size=(m, k)))
        ads = []
        for j in range(2):
            r = int(rng.integers(1, 9))
            a = bf16x(rng.normal(size=(k, r)) / np.sqrt(k))
            b = bf16x(rng.normal(scale=0.05, size=(r, n)))
            ads.append(AdapterPair(a, b, r, scale=float([2.0, 1.0][j])))
            out[f"a{j}_{i}"] = a
            out[f"b{j}_{i}"] = b
            out[f"scale{j}_{i}"] = np.array(ads[-1].scale)
        y = pipelined_forward(x, encode(w), fuse(ads), PipelineConfig())
        out[f"w_{i}"] = w
        out[f"x_{i}"] = x
        out[f"y_{i}"] = y
    out["n"] = np.array(len(shapes))
    np.savez_compressed(os.path.join(HERE, "forward.npz"), **out)
    print("forward cases:", len(shapes))


def config1():
    k = n = 4096
    m = 16
    seed_w, seed_x, seed_lora = 1000, 7, 1000 + 100_000
    t0 = time.time()
    w = synthetic.gen_weight(k, n, seed_w).double().numpy()
    x = synthetic.gen_x(m, k, seed_x).double().numpy()
    la, lb = synthetic.gen_lora(k, n, 16, seed_lora)
    la, lb = la.double().numpy(), lb.double().numpy()
    mask = build_mask(w, np.zeros_like(w), PruneConfig(0.5))
    w_hat = np.where(mask, w, 0.0)
    print("mask", time.time() - t0)
    u, sv, vt = np.linalg.svd(w - w_hat, full_matrices=False)
    res = build_residual_adapter(w, w_hat, 16, svd_result=SvdResult(u, sv, vt))
    ra, rb = bf16x(res.a), bf16x(res.b)
    print("svd", time.time() - t0)
    adapters = [AdapterPair(ra, rb, 16), AdapterPair(la, lb, 16, scale=2.0)]
    s = encode(w_hat)
    y = pipelined_forward(x, s, fuse(adapters), PipelineConfig(overlap=False))
    print("forward", time.time() - t0)
    np.savez_compressed(
        os.path.join(HERE, "config1.npz"),
        k=k, n=n, m=m, seed_w=seed_w, seed_x=seed_x, seed_lora=seed_lora, sparsity=0.5,
        res_a_bf16=(ra.astype(np.float32).view(np.uint32) >> 16).astype(np.uint16),
        res_b_bf16=(rb.astype(np.float32).view(np.uint32) >> 16).astype(np.uint16),
        bitmap_sha256=np.array(hashlib.sha256(s.bitmap.tobytes()).hexdigest()),
        values_sha256=np.array(hashlib.sha256(s.values.tobytes()).hexdigest()),
        nnz=s.nnz,
        y=y,
    )


if __name__ == "__main__":
    which = sys.argv[1:] or ["codec", "blocks", "forward", "config1"]
    if "codec" in which:
        codec_cases()
    if "blocks" in which:
        block_cases()
    if "forward" in which:
        forward_cases()
    if "config1" in which:
        config1()
