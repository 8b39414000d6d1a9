"""NM24 (2:4) compute format on CPU: the format restatement round-trips, and
the linear kernel's permute-based column selection (decode_tile_nm24,
restated in tests/nm24_cpu.py) equals the direct rule for every mask pair,
column and row pair."""

import itertools

import numpy as np
import pytest

from nm24_cpu import nm24_dense, nm24_records, nm24_select, nm24_tile_tmem

MASKS = [m for m in range(16) if bin(m).count("1") <= 2]  # 11 patterns


def _direct(mask: int, w: int, j: int) -> int:
    if not (mask >> j) & 1:
        return 0
    k = bin(mask & ((1 << j) - 1)).count("1")
    return (w >> (16 * k)) & 0xFFFF


def test_selector_exhaustive():
    rng = np.random.default_rng(0)
    for m_lo, m_hi in itertools.product(MASKS, MASKS):
        for pidx in range(4):
            others = [int(x) for x in rng.choice(MASKS, 8)]
            others[2 * pidx], others[2 * pidx + 1] = m_lo, m_hi
            word = sum(v << (4 * i) for i, v in enumerate(others))
            w_lo, w_hi = (int(x) for x in rng.integers(1, 1 << 32, 2, dtype=np.uint64))
            for j in range(4):
                got = nm24_select(word, w_lo, w_hi, j, pidx)
                want = _direct(m_lo, w_lo, j) | _direct(m_hi, w_hi, j) << 16
                assert got == want, (m_lo, m_hi, pidx, j)


def _two_of_four(rows, cols, seed):
    """bf16-exact matrix under the reference's 2:4 rule (prune.py:238-248:
    keep the 2 largest |w| of each group of 4 columns, ties to the lower
    offset), plus some kept entries that are exactly zero."""
    rng = np.random.default_rng(seed)
    w = rng.standard_normal((rows, cols)).astype(np.float32)
    w = (w.view(np.uint32) & 0xFFFF0000).view(np.float32)
    g = np.abs(w).reshape(rows, cols // 4, 4)
    order = np.argsort(-g, axis=2, kind="stable")
    keep = np.zeros_like(g, dtype=bool)
    np.put_along_axis(keep, order[:, :, :2], True, axis=2)
    w = np.where(keep.reshape(rows, cols), w, 0).astype(np.float32)
    w[rng.random((rows, cols)) < 0.05] = 0
    return w


@pytest.mark.parametrize("shape", [(64, 128), (70, 260), (130, 36)])
def test_records_round_trip(shape):
    w = _two_of_four(*shape, seed=sum(shape))
    rec = nm24_records(w)
    n_tiles = -(-shape[0] // 64) * -(-shape[1] // 128)
    assert rec.size == 9216 * n_tiles
    assert np.array_equal(nm24_dense(rec, *shape), w)


def test_rejects_three_of_four():
    w = _two_of_four(64, 128, 1)
    w[5, 8:11] = 1.0
    with pytest.raises(ValueError):
        nm24_records(w)


def test_kernel_addressing_matches_dense():
    """The decoder's per-lane loads and selections reproduce the tile."""
    w = _two_of_four(64, 128, 7)
    rec = nm24_records(w)
    img = nm24_tile_tmem(rec)
    bits = (w.view(np.uint32) >> 16).astype(np.uint32)  # 64 x 128
    want = (bits[0::2, :] | bits[1::2, :] << 16).T       # lane n, column c
    assert np.array_equal(img, want)
