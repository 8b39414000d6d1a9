"""CPU oracle for the SALR linear hot path -- TEST INFRASTRUCTURE ONLY.

This module restates, in NumPy, the reference algorithm of the three hot-path
operations that the B200 product implements in CUDA:

* bitmap encode / decode / decode_block      (reference ``pkg/src/salr/bitmap.py``)
* concatenated-adapter fusion                (reference ``pkg/src/salr/fusion.py``)
* the pipelined SALR linear forward          (reference ``pkg/src/salr/pipeline.py``)

plus the two setup helpers the harness needs to build inputs identical to the
reference's (magnitude-prune mask, ``prune.py``; SVD residual adapter,
``residual.py``).

Rules ("Oracle"):

* Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` leg may import this module, and only
  as the *checker* / CPU baseline.  The product package
  ``paper_2601_16991_b200`` never imports it and has no CPU fallback.
* Parity is pinned: ``tests/golden/make_golden.py`` ran the real reference
  package (``/root/reference/pkg/src/salr``) in the authoring container and
  committed its outputs under ``tests/golden/``; ``tests/test_oracle.py``
  checks this restatement against those fixtures before anything trusts it.

Numerics follow the reference exactly: values are stored float32, all forward
arithmetic is float64, tile products accumulate in ascending tile order.
"""

from __future__ import annotations

import math

import numpy as np

__all__ = [
    "OracleError",
    "popcount8",
    "build_lut",
    "bytes_per_row",
    "Encoded",
    "encode",
    "decode",
    "decode_block",
    "fuse",
    "apply_fused",
    "apply_sequential",
    "pipelined_matmul",
    "pipelined_forward",
    "kept_count",
    "build_mask",
    "residual_adapter",
    "compression_ratio",
]


class OracleError(Exception):
    """Raised for inputs the reference would reject (shape/bounds)."""


# ---------------------------------------------------------------------------
# a1/a2: popcount table and the 256 x 8 rank LUT  (bitmap.py:56-85)

def popcount8(m: int) -> int:
    """Set bits of one byte.  Restates ``bitmap.py:61-65`` (table lookup)."""
    if not 0 <= m <= 255:
        raise OracleError(f"byte value out of range: {m}")
    return bin(m).count("1")


def build_lut() -> np.ndarray:
    """``lut[m, t]`` = rank of bit t among set bits of m, -1 if clear.

    Restates ``bitmap.py:68-85`` as a prefix-popcount: the rank of bit t is
    popcount(m & ((1 << t) - 1)).
    """
    m = np.arange(256, dtype=np.int64)[:, None]
    t = np.arange(8, dtype=np.int64)[None, :]
    below = m & ((1 << t) - 1)
    rank = np.zeros((256, 8), dtype=np.int64)
    for b in range(8):
        rank += (below >> b) & 1
    set_bit = ((m >> t) & 1).astype(bool)
    return np.where(set_bit, rank, -1).astype(np.int8)


def bytes_per_row(cols: int) -> int:
    """``ceil(cols / 8)`` (``bitmap.py:146-147``)."""
    return (cols + 7) // 8


# ---------------------------------------------------------------------------
# a3/a4: the encoded matrix and encode  (bitmap.py:88-165)

class Encoded:
    """(rows, cols, bitmap u8 [rows, ceil(cols/8)], values f32 [nnz]).

    Mirrors the invariants of ``BitmapSparseMatrix.__post_init__``
    (``bitmap.py:105-126``): bitmap shape, zero padding bits, popcount ==
    len(values).
    """

    def __init__(self, rows, cols, bitmap, values):
        bitmap = np.ascontiguousarray(bitmap, dtype=np.uint8)
        values = np.ascontiguousarray(values, dtype=np.float32)
        if rows < 1 or cols < 1:
            raise OracleError(f"invalid dims {(rows, cols)}")
        if bitmap.shape != (rows, bytes_per_row(cols)):
            raise OracleError(f"bitmap shape {bitmap.shape}")
        pad = 8 * bytes_per_row(cols) - cols
        if pad and np.any(bitmap[:, -1] >> (8 - pad)):
            raise OracleError("padding bits beyond cols are not zero")
        if int(np.unpackbits(bitmap).sum()) != values.size:
            raise OracleError("popcount != len(values)")
        self.rows, self.cols = int(rows), int(cols)
        self.bitmap, self.values = bitmap, values
        self._starts = None

    @property
    def nnz(self) -> int:
        return int(self.values.size)

    @property
    def bytes_per_row(self) -> int:
        return int(self.bitmap.shape[1])

    def byte_starts(self) -> np.ndarray:
        """Exclusive prefix of per-byte popcounts, row-major, cached (``bitmap.py:136-143``)."""
        if self._starts is not None:
            return self._starts
        counts = np.unpackbits(self.bitmap[..., None], axis=-1).sum(-1).astype(np.int64)
        flat = counts.ravel()
        starts = np.concatenate(([0], np.cumsum(flat)[:-1])).astype(np.int64)
        self._starts = starts.reshape(self.bitmap.shape)
        return self._starts


def _as_f64_matrix(x, name="x") -> np.ndarray:
    """``linalg.as_matrix`` semantics (``linalg.py:52-69``): 2-D, f64, finite."""
    a = np.ascontiguousarray(x, dtype=np.float64)
    if a.ndim != 2 or a.shape[0] < 1 or a.shape[1] < 1:
        raise OracleError(f"{name} must be a non-empty 2-D array")
    if not np.all(np.isfinite(a)):
        raise OracleError(f"{name} contains non-finite entries")
    return a


def encode(m) -> Encoded:
    """Bitmap-encode a dense matrix (restates ``bitmap.py:150-165``).

    Cast to float32 first, canonicalise -0.0 to +0.0, keep entries that are
    non-zero *in float32*, pack the keep-mask LSB-first (bit t of byte b is
    column 8b+t), values in row-major order of set bits.
    """
    dense = _as_f64_matrix(m, "m")
    rows, cols = dense.shape
    m32 = dense.astype(np.float32) + np.float32(0.0)
    keep = m32 != 0
    bpr = bytes_per_row(cols)
    padded = np.zeros((rows, bpr * 8), dtype=np.uint8)
    padded[:, :cols] = keep
    weights = (1 << np.arange(8, dtype=np.uint16)).astype(np.uint16)
    bitmap = (padded.reshape(rows, bpr, 8).astype(np.uint16) * weights).sum(-1)
    return Encoded(rows, cols, bitmap.astype(np.uint8), m32[keep])


def _expand(bitmap: np.ndarray, cols_padded: int) -> np.ndarray:
    """Boolean presence matrix from an LSB-first packed bitmap."""
    return np.unpackbits(bitmap, axis=1, bitorder="little")[:, :cols_padded].astype(bool)


def decode(s: Encoded) -> np.ndarray:
    """Exact inverse of encode; float64 holding f32 values (``bitmap.py:168-180``).

    Restated as a boolean scatter: row-major set positions receive the value
    stream in order.
    """
    present = _expand(s.bitmap, 8 * s.bytes_per_row)
    out = np.zeros(present.shape, dtype=np.float64)
    out[present] = s.values.astype(np.float64)
    return out[:, : s.cols]


def decode_block(s: Encoded, row_range, byte_block_range) -> np.ndarray:
    """Dense tile rows [r0,r1) x byte blocks [b0,b1) (``bitmap.py:183-212``)."""
    r0, r1 = row_range
    b0, b1 = byte_block_range
    if not (0 <= r0 <= r1 <= s.rows and 0 <= b0 <= b1 <= s.bytes_per_row):
        raise OracleError(f"block rows {row_range} bytes {byte_block_range} out of bounds")
    col_hi = min(8 * b1, s.cols)
    n_cols = max(col_hi - 8 * b0, 0)
    if r1 == r0 or b1 == b0 or n_cols == 0:
        return np.zeros((r1 - r0, n_cols), dtype=np.float64)
    # value index of the first set bit of every byte in the block
    starts = s.byte_starts()[r0:r1, b0:b1]
    sub = s.bitmap[r0:r1, b0:b1]
    bits = np.unpackbits(sub[..., None], axis=-1, bitorder="little").astype(np.int64)
    rank = np.cumsum(bits, axis=-1) - bits          # exclusive in-byte rank
    idx = starts[..., None] + rank
    vals = np.where(bits.astype(bool), s.values[np.minimum(idx, max(s.nnz - 1, 0))] if s.nnz else 0.0, 0.0)
    tile = vals.reshape(r1 - r0, 8 * (b1 - b0)).astype(np.float64)
    return tile[:, :n_cols]


# ---------------------------------------------------------------------------
# a7/a8/a9/a10: adapters and fusion  (residual.py:45-81, fusion.py:27-106)

class Adapter:
    """(a d_in x r, b r x d_out, rank, scale); restates ``residual.py:45-81``."""

    def __init__(self, a, b, rank, scale=1.0):
        self.a = _as_f64_matrix(a, "a")
        self.b = _as_f64_matrix(b, "b")
        self.rank, self.scale = int(rank), float(scale)
        if self.a.shape[1] != self.rank or self.b.shape[0] != self.rank:
            raise OracleError("factor shapes do not match rank")


class Fused:
    def __init__(self, a_cat, b_cat, offsets, ranks):
        self.a_cat, self.b_cat, self.offsets, self.ranks = a_cat, b_cat, offsets, ranks

    @property
    def d_in(self):
        return self.a_cat.shape[0]

    @property
    def d_out(self):
        return self.b_cat.shape[1]

    @property
    def total_rank(self):
        return self.a_cat.shape[1]


def fuse(adapters) -> Fused:
    """Rank-concatenate adapters, fold each scale into its rows of b_cat.

    Restates ``fusion.py:58-84``.
    """
    if not adapters:
        raise OracleError("fuse requires at least one adapter")
    d_in, d_out = adapters[0].a.shape[0], adapters[0].b.shape[1]
    for ad in adapters:
        if ad.a.shape[0] != d_in or ad.b.shape[1] != d_out:
            raise OracleError("adapter outer dims disagree")
    ranks = np.array([ad.rank for ad in adapters], dtype=np.int64)
    offsets = np.cumsum(np.concatenate(([0], ranks)))[:-1]
    a_cat = np.hstack([ad.a for ad in adapters])
    b_cat = np.vstack([ad.b * ad.scale for ad in adapters])
    return Fused(a_cat, b_cat, offsets, ranks)


def apply_fused(x, fused: Fused) -> np.ndarray:
    """``(x @ a_cat) @ b_cat`` -- two f64 products (``fusion.py:87-92``)."""
    xm = _as_f64_matrix(x)
    if xm.shape[1] != fused.d_in:
        raise OracleError("x cols != adapter d_in")
    return (xm @ fused.a_cat) @ fused.b_cat


def apply_sequential(x, adapters) -> np.ndarray:
    """Sum of scale_i * (x @ a_i) @ b_i (``fusion.py:95-106``)."""
    xm = _as_f64_matrix(x)
    total = None
    for ad in adapters:
        term = ad.scale * ((xm @ ad.a) @ ad.b)
        total = term if total is None else total + term
    return total


# ---------------------------------------------------------------------------
# a11-a16: the two-stage engine, serial schedule  (pipeline.py:186-331)
#
# Overlap only changes *when* tiles are decoded, never the reduction order
# (pipeline.py:1-13, :403-404), so the serial schedule is the oracle for both.

def _tiles(s: Encoded, tile_rows: int, tile_col_bytes: int):
    """Row blocks outer, byte blocks inner (``pipeline.py:186-196``)."""
    for r0 in range(0, s.rows, tile_rows):
        r1 = min(r0 + tile_rows, s.rows)
        for b0 in range(0, s.bytes_per_row, tile_col_bytes):
            yield r0, r1, b0, min(b0 + tile_col_bytes, s.bytes_per_row)


def pipelined_matmul(x, s: Encoded, tile_rows=64, tile_col_bytes=8) -> np.ndarray:
    """``x @ decode(s)`` accumulated tile by tile (``pipeline.py:214-272``)."""
    xm = _as_f64_matrix(x)
    if xm.shape[1] != s.rows:
        raise OracleError("x cols != sparse rows")
    out = np.zeros((xm.shape[0], s.cols), dtype=np.float64)
    for r0, r1, b0, b1 in _tiles(s, tile_rows, tile_col_bytes):
        tile = decode_block(s, (r0, r1), (b0, b1))
        c0, c1 = 8 * b0, min(8 * b1, s.cols)
        out[:, c0:c1] += xm[:, r0:r1] @ tile
    return out


def pipelined_forward(x, s: Encoded, fused: Fused, tile_rows=64, tile_col_bytes=8) -> np.ndarray:
    """The SALR linear ``x @ decode(s) + (x @ a_cat) @ b_cat``.

    Restates ``pipeline.py:275-331``: the result is ``tiles + delta`` with the
    adapter delta formed by exactly two products.
    """
    xm = _as_f64_matrix(x)
    if fused.d_in != s.rows or fused.d_out != s.cols:
        raise OracleError("fused adapter dims != weight dims")
    delta = apply_fused(xm, fused)
    return pipelined_matmul(xm, s, tile_rows, tile_col_bytes) + delta


# ---------------------------------------------------------------------------
# setup helpers: prune mask and SVD residual  (prune.py:202-255, residual.py:138-173)

def kept_count(p: float, total: int) -> int:
    """``ceil((1-p)*total)`` nudged one ulp toward zero (``prune.py:202-212``)."""
    if not 0.0 <= p < 1.0 or total < 1:
        raise OracleError("bad sparsity/total")
    return int(math.ceil(np.nextafter((1.0 - p) * total, 0.0)))


def build_mask(w0, sparsity: float) -> np.ndarray:
    """Static magnitude mask: keep the kept_count largest |w|, ties to the
    lower flat index (``prune.py:215-255``, STATIC_ON_W0 branch)."""
    w = _as_f64_matrix(w0, "w0")
    keep = kept_count(sparsity, w.size)
    order = np.argsort(-np.abs(w).ravel(), kind="stable")
    mask = np.zeros(w.size, dtype=bool)
    mask[order[:keep]] = True
    return mask.reshape(w.shape)


def residual_adapter(w, w_hat, rank: int):
    """Best rank-r factorisation of E = w - w_hat via LAPACK SVD.

    Restates ``residual.py:147-173`` (a = U_r diag(s_r), b = Vt_r, singular
    values below 1e-12 * s_max zeroed) with ``np.linalg.svd`` standing in for
    the reference's Jacobi SVD, exactly as the reference allows through its
    ``svd_result=`` hook.
    """
    e = _as_f64_matrix(w) - _as_f64_matrix(w_hat)
    u, sv, vt = np.linalg.svd(e, full_matrices=False)
    s = sv[:rank].copy()
    s[s < 1e-12 * (sv[0] if sv.size else 0.0)] = 0.0
    a = u[:, :rank] * s
    b = vt[:rank, :].copy()
    b[s == 0.0, :] = 0.0
    return a, b


def compression_ratio(d: int, k: int, p: float, bytes_per_value: int,
                      adapter_params: int, n_adapters: int = 0) -> float:
    """Dense / compressed bytes incl. container header (``bitmap.py:358-378``)."""
    nnz = kept_count(p, d * k)
    header = 41 + 8 * n_adapters
    comp = nnz * bytes_per_value + d * bytes_per_row(k) + adapter_params * bytes_per_value + header
    return d * k * bytes_per_value / comp
