"""Device pipeline probe (the reference's PipelineProbe, pipeline.py:89-103,
and its stress in pkg/tests/test_acceptance.py:405-422): every ring-slot
transition of the fused kernel is logged on the device and audited by
validate_transitions, under random per-tile jitter injected before decodes
and MMA issues; the results stay bit-identical to the unprobed run."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    import paper_2601_16991_b200 as S
    return S


def _bf16(a):
    return torch.from_numpy(a).bfloat16().float()


def test_probe_stress_small_10k(S):
    """10^4 runs of a one-tile matrix (reference stress sizes: 8 x 16, x 4 x 8)."""
    rng = np.random.default_rng(0)
    w = rng.normal(size=(8, 16))
    w[rng.random(size=w.shape) < 0.5] = 0.0
    s = S.encode(_bf16(w.astype(np.float32)).cuda(), value_dtype="bf16")
    x = _bf16(rng.normal(size=(4, 8)).astype(np.float32)).cuda()
    cfg = S.PipelineConfig(tile_rows=2, tile_col_bytes=1, ring_capacity=2)
    ref = S.pipelined_matmul(x, s, cfg)
    for run in range(10_000):
        probe = S.PipelineProbe(decode_delay=2000, compute_delay=2000, record=True, seed=run)
        out = S.pipelined_matmul(x, s, cfg, probe=probe)
        S.validate_transitions(probe, probe.capacity)
        assert probe.produced == probe.consumed == 1
        assert torch.equal(out, ref), f"delayed run {run} changed the result"


@pytest.mark.parametrize("ring", [1, 2, 4, 8])
def test_probe_multi_cta_ring(S, ring):
    """Many CTAs x many units per CTA, every ring depth, with jitter: the log
    is a legal cycle per slot, fills == consumes == units, results unchanged."""
    g = torch.Generator().manual_seed(ring)
    K, N, M = 1024, 1536, 8
    w = (torch.randn(K, N, generator=g) * 0.02).bfloat16().float()
    w[torch.rand(K, N, generator=g) < 0.5] = 0
    s = S.encode(w.cuda(), value_dtype="bf16")
    x = torch.randn(M, K, generator=g).bfloat16().cuda()
    cfg = S.PipelineConfig(ring_capacity=max(ring, 2), overlap=ring > 1)
    ref = S.pipelined_matmul(x, s, cfg)
    for run in range(20):
        probe = S.PipelineProbe(decode_delay=3000, compute_delay=3000, record=True, seed=1000 * ring + run)
        out = S.pipelined_matmul(x, s, cfg, probe=probe)
        S.validate_transitions(probe, probe.capacity)
        units = (K // 64) * (N // 128)
        assert probe.produced == probe.consumed == units
        assert torch.equal(out, ref)


def test_probe_rejects_host_callables(S):
    from paper_2601_16991_b200.errors import ConfigError
    s = S.encode(torch.ones(8, 16).cuda(), value_dtype="bf16")
    with pytest.raises(ConfigError):
        S.pipelined_matmul(torch.ones(2, 8).cuda(), s, S.PipelineConfig(),
                           probe=S.PipelineProbe(decode_delay=lambda: None))
