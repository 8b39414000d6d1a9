"""Bitmap codec on the B200: ``encode``/``decode``/``decode_block`` and the
GPU-resident :class:`BitmapSparseMatrix`, API-compatible with the reference
``pkg/src/salr/bitmap.py``.

Storage is the TB ("tiled bitmap") device format of ``include/salr_b200.h``:
64 x 128 tiles, each a 16-byte-aligned record of bitmap words and compacted
values.  The *logical* content is the reference's: the bitmap is bit-identical
(LSB-first, bit t of byte b = column 8b+t, ``bitmap.py:4-6``) and ``values``
come back in the reference's row-major set-bit order (``bitmap.py:114``).
Values are float32 (reference-exact, the default) or bf16 (the compute
format of the linear kernel; ``bf16 == rne(f32)`` of the reference values).
"""

from __future__ import annotations

import os
import struct

import numpy as np
import torch

from . import _lib
from .errors import BoundsError, CorruptionError, DomainError, FormatError, SalrError, ShapeError
from .linalg import as_matrix, to_cuda
from .residual import AdapterPair

__all__ = ["DTYPE_F32", "popcount8", "build_lut", "bytes_per_row", "BitmapSparseMatrix",
           "encode", "decode", "decode_block", "write_container", "read_container",
           "header_bytes", "container_size_bytes", "compression_ratio", "kept_count"]

NM24_RECORD_BYTES = 9216  # fixed NM24 tile record (csrc/salr_format.cuh)
DTYPE_F32 = 0  # the only stored precision of the container format (bitmap.py:48)

_MAGIC = b"SALR"
_VERSION = 1
_FIXED_HEADER = struct.Struct("<4sHIIBH")
_ADAPTER_HEADER = struct.Struct("<If")
_OFFSETS = struct.Struct("<QQQ")

_VALUE_DTYPES = {"f32": (_lib.F32, torch.float32, 4), "bf16": (_lib.BF16, torch.bfloat16, 2)}


def popcount8(m: int) -> int:
    """Set bits of one byte (``bitmap.py:61-65``)."""
    if not 0 <= m <= 255:
        raise BoundsError(f"byte value out of range: {m}")
    return bin(m).count("1")


def build_lut() -> np.ndarray:
    """256 x 8 int8 rank table (``bitmap.py:68-85``): rank of bit t among the
    set bits of m, -1 if clear.  The device decoder computes the same rank
    as ``popc(word & lanemask_lt)``."""
    lut = np.full((256, 8), -1, dtype=np.int8)
    for m in range(256):
        r = 0
        for t in range(8):
            if (m >> t) & 1:
                lut[m, t] = r
                r += 1
    return lut


def bytes_per_row(cols: int) -> int:
    return (cols + 7) // 8


def _popcount_table(device) -> torch.Tensor:
    return torch.tensor([bin(i).count("1") for i in range(256)], dtype=torch.int64, device=device)


def _u32(t: torch.Tensor):
    return _lib.ptr(t)


class BitmapSparseMatrix:
    """Bitmap + compact values of one pruned matrix, resident on the GPU.

    ``BitmapSparseMatrix(rows, cols, bitmap, values, dtype_code=0)`` accepts
    the reference layout (bitmap ``rows x ceil(cols/8)`` uint8, values in
    row-major set-bit order) from NumPy or torch and validates it exactly as
    ``bitmap.py:105-126`` does (ShapeError / FormatError / CorruptionError),
    then converts it to TB records on the device.
    """

    def __init__(self, rows: int, cols: int, bitmap, values, dtype_code: int = DTYPE_F32,
                 value_dtype: str = "f32"):
        if rows < 1 or cols < 1:
            raise ShapeError(f"invalid dims {(rows, cols)}")
        bpr = bytes_per_row(cols)
        bm = to_cuda(bitmap) if isinstance(bitmap, torch.Tensor) else to_cuda(np.asarray(bitmap, dtype=np.uint8))
        if bm.dtype != torch.uint8:
            bm = bm.to(torch.uint8)
        if tuple(bm.shape) != (rows, bpr):
            raise ShapeError(f"bitmap shape {tuple(bm.shape)} != expected {(rows, bpr)}")
        vals = to_cuda(values) if isinstance(values, torch.Tensor) else to_cuda(np.asarray(values, dtype=np.float32))
        if vals.dim() != 1:
            raise ShapeError("values must be one-dimensional")
        if dtype_code != DTYPE_F32:
            raise FormatError(f"unsupported dtype code {dtype_code}")
        if value_dtype not in _VALUE_DTYPES:
            raise FormatError(f"unsupported value dtype {value_dtype!r}")
        pad = 8 * bpr - cols
        if pad and bool((bm[:, -1] >> (8 - pad)).any()):
            raise CorruptionError("padding bits beyond cols are not zero")
        vals = vals.to(torch.bfloat16 if vals.dtype == torch.bfloat16 else torch.float32).contiguous()
        bm = bm.contiguous()
        self._init_geometry(rows, cols, value_dtype)
        self._from_reference(bm, vals)
        if self.nnz != int(vals.numel()):
            raise CorruptionError(f"bitmap popcount {self.nnz} != values length {int(vals.numel())}")
        # the reference-layout inputs are not kept: the TB records hold the
        # same content and .bitmap/.values rebuild it on request

    # ------------------------------------------------------------------ internals
    def _init_geometry(self, rows, cols, value_dtype):
        self.rows, self.cols = int(rows), int(cols)
        self.dtype_code = DTYPE_F32
        self.value_dtype = value_dtype
        self.n_kt, self.n_nt, self.n_tiles = _lib.geometry(self.rows, self.cols)
        self._byte_starts = None
        self._tb2 = None
        self._nm24 = None  # NM24 records (2:4 matrices, use_nm24())

    @classmethod
    def _wrap(cls, rows, cols, value_dtype, records, tile_off):
        obj = cls.__new__(cls)
        obj._init_geometry(rows, cols, value_dtype)
        obj.records, obj.tile_off = records, tile_off
        obj._max_rec = None
        obj.max_record_bytes  # computed eagerly (never inside a graph capture)
        obj.nnz = obj._count_nnz()
        return obj

    def _count_nnz(self) -> int:
        lib = _lib.load()
        out = torch.empty(1, dtype=torch.int64, device=self.records.device)
        _lib.check(lib.salr_tb_nnz(_lib.ptr(self.records), _u32(self.tile_off), self.n_tiles, _lib.ptr(out),
                                   _lib.stream_ptr()))
        return int(out.item())

    def _from_reference(self, bm: torch.Tensor, vals: torch.Tensor):
        lib = _lib.load()
        dev = bm.device
        vcode = _VALUE_DTYPES[self.value_dtype][0]
        rowtile_off = torch.empty(self.rows * self.n_nt + 1, dtype=torch.int32, device=dev)
        tile_cnt = torch.empty(4 * self.n_tiles, dtype=torch.int32, device=dev)
        tile_off = torch.empty(self.n_tiles + 1, dtype=torch.int32, device=dev)
        s = _lib.stream_ptr()
        _lib.check(lib.salr_from_reference_count(_lib.ptr(bm), self.rows, self.cols, vcode, _u32(rowtile_off),
                                                 _u32(tile_cnt), _u32(tile_off), s))
        total_nnz = int(rowtile_off[-1].item())
        if total_nnz != int(vals.numel()):
            raise CorruptionError(f"bitmap popcount {total_nnz} != values length {int(vals.numel())}")
        units = int(tile_off[-1].item()) & 0xFFFFFFFF
        records = torch.empty(16 * units, dtype=torch.uint8, device=dev)
        _lib.check(lib.salr_from_reference_write(_lib.ptr(bm), _lib.ptr(vals), _lib.dtype_code(vals.dtype),
                                                 self.rows, self.cols, vcode, _u32(rowtile_off), _u32(tile_cnt),
                                                 _u32(tile_off), _lib.ptr(records), s))
        self.records, self.tile_off = records, tile_off
        self._max_rec = None
        self.max_record_bytes  # computed eagerly (never inside a graph capture)
        self.nnz = total_nnz

    def _to_reference(self):
        lib = _lib.load()
        records, tile_off = self.tb()
        dev = records.device
        bpr = bytes_per_row(self.cols)
        rowtile_off = torch.empty(self.rows * self.n_nt + 1, dtype=torch.int32, device=dev)
        bm = torch.empty((self.rows, bpr), dtype=torch.uint8, device=dev)
        vals = torch.empty(max(self.nnz, 1), dtype=torch.float32, device=dev)
        _lib.check(lib.salr_to_reference(_lib.ptr(records), _u32(tile_off),
                                         _VALUE_DTYPES[self.value_dtype][0], self.rows, self.cols, _u32(rowtile_off),
                                         _lib.ptr(bm), _lib.ptr(vals), _lib.F32, _lib.stream_ptr()))
        return bm, vals[: self.nnz]

    def tb(self):
        """(records, tile_off) of the TB records: the resident ones, or -- when
        only the TB2 compute format is kept -- rebuilt from it (bit-exact,
        transient, not cached)."""
        if self.records is not None:
            return self.records, self.tile_off
        if self._tb2 is None:  # NM24 only: dense bf16 -> TB
            e = encode(self._nm24_dense(), "bf16")
            return e.records, e.tile_off
        rec2, off2, _ = self._tb2
        lib = _lib.load()
        st = _lib.stream_ptr()
        off = torch.empty(self.n_tiles + 1, dtype=torch.int32, device=rec2.device)
        _lib.check(lib.salr_tb_from_tb2_count(_lib.ptr(rec2), _u32(off2), self.rows, self.cols, _u32(off), st))
        units = int(off[-1].item()) & 0xFFFFFFFF
        rec = torch.empty(16 * units, dtype=torch.uint8, device=rec2.device)
        _lib.check(lib.salr_tb_from_tb2_write(_lib.ptr(rec2), _u32(off2), self.rows, self.cols, _u32(off),
                                              _lib.ptr(rec), st))
        return rec, off

    # ------------------------------------------------------------------ reference API
    @property
    def bitmap(self) -> torch.Tensor:
        """Reference-layout bitmap ``rows x ceil(cols/8)`` uint8, rebuilt on the
        device on every access (a fresh array, like the reference's copy)."""
        return self._to_reference()[0]

    @property
    def values(self) -> torch.Tensor:
        """Values in reference row-major set-bit order, float32 (fresh array)."""
        return self._to_reference()[1]

    @property
    def bytes_per_row(self) -> int:
        return bytes_per_row(self.cols)

    def byte_starts(self) -> torch.Tensor:
        """Exclusive running sum of per-byte popcounts, row-major, int64, cached
        (``bitmap.py:136-143``)."""
        if self._byte_starts is None:
            bm = self.bitmap
            counts = _popcount_table(bm.device)[bm.long()].reshape(-1)
            starts = torch.zeros_like(counts)
            if counts.numel() > 1:
                starts[1:] = torch.cumsum(counts[:-1], 0)
            self._byte_starts = starts.reshape(bm.shape)
        return self._byte_starts

    # ------------------------------------------------------------------ B200 extras
    @property
    def compressed_bytes(self) -> int:
        """Algorithmic bytes: bitmap ``rows*ceil(cols/8)`` + values."""
        return self.rows * self.bytes_per_row + _VALUE_DTYPES[self.value_dtype][2] * self.nnz

    @property
    def max_record_bytes(self) -> int:
        """Largest TB record (bytes); sizes the linear kernel's ring slots."""
        if getattr(self, "_max_rec", None) is None:
            if self.tile_off is None:
                return self._tb2[2] if self._tb2 is not None else NM24_RECORD_BYTES
            off = self.tile_off.to(torch.int64) & 0xFFFFFFFF
            self._max_rec = int(16 * (off[1:] - off[:-1]).max().item()) if off.numel() > 1 else 0
        return self._max_rec

    @property
    def device_bytes(self) -> int:
        """Bytes this matrix keeps resident in HBM: every stored format
        (TB records, the TB2 compute format, offsets; cached reference
        ``byte_starts`` if requested)."""
        n = 0
        if self.records is not None:
            n += int(self.records.numel()) + 4 * int(self.tile_off.numel())
        if self._tb2 is not None:
            n += int(self._tb2[0].numel()) + 4 * int(self._tb2[1].numel())
        if self._nm24 is not None:
            n += int(self._nm24.numel())
        if self._byte_starts is not None:
            n += 8 * int(self._byte_starts.numel())
        return n

    def compute_format(self):
        """(records2, tile_off2, max_record_bytes) of the TB2 compute format
        the linear kernel consumes; built once on the current stream and
        cached (never inside a CUDA-graph capture).

        One compute format stays resident: a bf16 matrix releases its TB
        records once TB2 exists (``tb()`` rebuilds them bit-exactly when the
        reference layout or a decode is requested), so a bf16 stack holds
        ~K*N/8 + 2*nnz bytes plus the per-tile headers.  A float32 matrix
        (reference-exact values) keeps its TB records; the bf16 records that
        feed TB2 are transient."""
        if self._tb2 is None:
            if torch.cuda.is_current_stream_capturing():
                raise SalrError("build the compute format (BitmapSparseMatrix.compute_format()) before "
                                "capturing a CUDA graph")
            sb = self.to_bf16()
            lib = _lib.load()
            st = _lib.stream_ptr()
            rec, toff = sb.tb()
            off2 = torch.empty(self.n_tiles + 1, dtype=torch.int32, device=rec.device)
            _lib.check(lib.salr_tb2_count(_lib.ptr(rec), _u32(toff), self.rows, self.cols, _u32(off2), st))
            units = int(off2[-1].item()) & 0xFFFFFFFF
            rec2 = torch.empty(16 * units, dtype=torch.uint8, device=rec.device)
            _lib.check(lib.salr_tb2_write(_lib.ptr(rec), _u32(toff), self.rows, self.cols, _u32(off2),
                                          _lib.ptr(rec2), st))
            del rec, toff
            o = off2.to(torch.int64) & 0xFFFFFFFF
            mx = int(16 * (o[1:] - o[:-1]).max().item()) if o.numel() > 1 else 0
            self._tb2 = (rec2, off2, mx)
            del sb
            if self.value_dtype == "bf16":
                self.records = self.tile_off = None  # TB2 is the one resident format
        return self._tb2

    # ------------------------------------------------------------------ NM24 (2:4)
    def is_nm24(self) -> bool:
        """True when NM24 is this matrix's compute format (``use_nm24``)."""
        return self._nm24 is not None

    def use_nm24(self) -> "BitmapSparseMatrix":
        """Make NM24 the compute format: for a matrix under the reference's
        2:4 mask (``prune.py:238-248``, at most 2 nonzeros in every group of
        4 consecutive columns of a row) the linear kernel then reads fixed
        9216-byte tiles (1.125 B/weight) and expands them with byte permutes
        instead of the bitmap decoder -- same dense tile, bit-identical
        results.  Raises FormatError (matrix unchanged) when some group holds
        more than 2 nonzeros.  A bf16 matrix then keeps only NM24 resident
        (``tb()`` / ``compute_format()`` rebuild the others on request);
        float32 values are rounded to bf16 as for TB2 and the TB records stay.
        Built once on the current stream, never inside a graph capture."""
        if self._nm24 is not None:
            return self
        if torch.cuda.is_current_stream_capturing():
            raise SalrError("build the compute format (use_nm24()) before capturing a CUDA graph")
        dense = _decode_window(self, 0, self.rows, 0, self.cols, torch.bfloat16)
        lib = _lib.load()
        rec = torch.empty(self.n_tiles * NM24_RECORD_BYTES, dtype=torch.uint8, device=dense.device)
        bad = torch.zeros(1, dtype=torch.int32, device=dense.device)
        _lib.check(lib.salr_nm24_write(_lib.ptr(dense), self.rows, self.cols, self.cols, _lib.ptr(rec),
                                       _lib.ptr(bad), _lib.stream_ptr()))
        nbad = int(bad.item())
        if nbad:
            raise FormatError(f"{nbad} groups of 4 columns hold more than 2 nonzeros: the matrix is not 2:4")
        self._nm24 = rec
        if self.value_dtype == "bf16":
            self.records = self.tile_off = None
            self._tb2 = None
        return self

    def _nm24_dense(self) -> torch.Tensor:
        out = torch.empty((self.rows, self.cols), dtype=torch.bfloat16, device=self._nm24.device)
        _lib.check(_lib.load().salr_nm24_decode(_lib.ptr(self._nm24), self.rows, self.cols, _lib.ptr(out),
                                                self.cols, _lib.stream_ptr()))
        return out

    def kernel_operand(self):
        """(records, tile_off, max_record_bytes, nm24) the linear kernel reads:
        NM24 when ``use_nm24`` made it the compute format, else TB2."""
        if self._nm24 is not None:
            return self._nm24, None, NM24_RECORD_BYTES, True
        rec2, off2, mx = self.compute_format()
        return rec2, off2, mx, False

    @classmethod
    def from_compute_format(cls, rows: int, cols: int, records2: torch.Tensor, tile_off2: torch.Tensor):
        """A bf16 matrix held only in the TB2 compute format (records built
        elsewhere: another rank, a file, ``column_shard``).  No kernel runs:
        the tile headers give nnz and the offsets the largest record."""
        if records2.dtype != torch.uint8 or records2.dim() != 1 or tile_off2.dim() != 1:
            raise FormatError("records2 must be a 1-D uint8 tensor and tile_off2 1-D")
        obj = cls.__new__(cls)
        obj._init_geometry(rows, cols, "bf16")
        if int(tile_off2.numel()) != obj.n_tiles + 1:
            raise ShapeError(f"tile_off2 has {int(tile_off2.numel())} entries, expected {obj.n_tiles + 1}")
        off = tile_off2.to(torch.int64) & 0xFFFFFFFF
        if int(off[0]) != 0 or 16 * int(off[-1]) > int(records2.numel()) or bool((off[1:] < off[:-1]).any()):
            raise CorruptionError("tile_off2 is not a monotone offset table within records2")
        obj.records = obj.tile_off = None
        obj._max_rec = None
        mx = int(16 * (off[1:] - off[:-1]).max()) if off.numel() > 1 else 0
        obj._tb2 = (records2, tile_off2.to(torch.int32), mx)
        obj.nnz = _tile_nnz_sum(records2, off[:-1])
        return obj

    def column_shard(self, c0: int, c1: int) -> "BitmapSparseMatrix":
        """Columns [c0, c1) as a matrix of their own (multi-GPU column
        sharding): tiles are stored n-tile-major, so a stripe
        of whole 128-column tiles is one contiguous run of records -- the
        shard is a byte-exact copy of that run plus rebased offsets, in every
        resident format.  c0 must be a multiple of 128 and c1 too unless it
        is ``cols``."""
        tn = _lib.TILE_N
        if not (0 <= c0 < c1 <= self.cols) or c0 % tn or (c1 % tn and c1 != self.cols):
            raise ShapeError(f"column range [{c0}, {c1}) of {self.cols} is not a whole-tile stripe")
        t0 = (c0 // tn) * self.n_kt
        t1 = ((c1 + tn - 1) // tn) * self.n_kt

        def cut(records, tile_off):
            off = tile_off.to(torch.int64) & 0xFFFFFFFF
            o0, o1 = int(off[t0]), int(off[t1])
            return records[16 * o0:16 * o1].clone(), (off[t0:t1 + 1] - o0).to(torch.int32)

        obj = self.__class__.__new__(self.__class__)
        obj._init_geometry(self.rows, c1 - c0, self.value_dtype)
        obj.records = obj.tile_off = None
        if self.records is not None:
            obj.records, obj.tile_off = cut(self.records, self.tile_off)
        if self._tb2 is not None:
            r2, o2 = cut(self._tb2[0], self._tb2[1])
            oo = o2.to(torch.int64)
            obj._tb2 = (r2, o2, int(16 * (oo[1:] - oo[:-1]).max()) if oo.numel() > 1 else 0)
        if self._nm24 is not None:  # fixed-size tiles: a plain byte range
            obj._nm24 = self._nm24[t0 * NM24_RECORD_BYTES:t1 * NM24_RECORD_BYTES].clone()
        obj._max_rec = None
        if obj.records is None and obj._tb2 is None:
            obj.nnz = int((obj._nm24_dense() != 0).sum())
        elif obj.records is not None:
            obj.max_record_bytes  # computed eagerly (never inside a graph capture)
            obj.nnz = _tile_nnz_sum(obj.records, obj.tile_off.to(torch.int64)[:-1])
        else:
            obj.nnz = _tile_nnz_sum(obj._tb2[0], obj._tb2[1].to(torch.int64)[:-1])
        return obj

    def to_bf16(self) -> "BitmapSparseMatrix":
        """The same matrix with bf16 values (the linear kernel's operand
        format); a new object (not cached) for a float32 matrix."""
        if self.value_dtype == "bf16":
            return self
        bm, vals = self._to_reference()
        return BitmapSparseMatrix(self.rows, self.cols, bm, vals, value_dtype="bf16")

    @property
    def device(self) -> torch.device:
        for t in (self.records, self._tb2[0] if self._tb2 is not None else None, self._nm24):
            if t is not None:
                return t.device
        raise SalrError("matrix holds no records")

    def __repr__(self):
        return (f"BitmapSparseMatrix(rows={self.rows}, cols={self.cols}, nnz={self.nnz}, "
                f"value_dtype={self.value_dtype!r}, device={self.device})")


def _tile_nnz_sum(records: torch.Tensor, starts16: torch.Tensor) -> int:
    """Sum of the per-tile nnz words (u32 header word 3 of every TB / TB2
    record starting at 16 * starts16) -- plain tensor indexing, any device."""
    if starts16.numel() == 0:
        return 0
    base = 16 * (starts16.to(records.device) & 0xFFFFFFFF) + 12
    idx = base.unsqueeze(1) + torch.arange(4, device=records.device)
    b = records[idx].to(torch.int64)
    return int((b[:, 0] | (b[:, 1] << 8) | (b[:, 2] << 16) | (b[:, 3] << 24)).sum())


def encode(m, value_dtype: str = "f32") -> BitmapSparseMatrix:
    """Encode a dense matrix on the GPU; exact zeros after the float32 cast are
    pruned and -0.0 normalises to +0.0 (``bitmap.py:150-165``).

    ``m`` may be float64/float32/bf16 (NumPy or torch); float64 inputs are
    cast to float32 on the device with round-to-nearest-even, as NumPy does.
    """
    if value_dtype not in _VALUE_DTYPES:
        raise FormatError(f"unsupported value dtype {value_dtype!r}")
    dense = as_matrix(m, "m")
    rows, cols = (int(d) for d in dense.shape)
    lib = _lib.load()
    s = BitmapSparseMatrix.__new__(BitmapSparseMatrix)
    s._init_geometry(rows, cols, value_dtype)
    vcode = _VALUE_DTYPES[value_dtype][0]
    dev = dense.device
    tile_cnt = torch.empty(4 * s.n_tiles, dtype=torch.int32, device=dev)
    tile_off = torch.empty(s.n_tiles + 1, dtype=torch.int32, device=dev)
    st = _lib.stream_ptr()
    icode = _lib.dtype_code(dense.dtype)
    _lib.check(lib.salr_encode_count(_lib.ptr(dense), icode, rows, cols, cols, vcode, _u32(tile_cnt),
                                     _u32(tile_off), st))
    units = int(tile_off[-1].item()) & 0xFFFFFFFF
    records = torch.empty(16 * units, dtype=torch.uint8, device=dev)
    _lib.check(lib.salr_encode_write(_lib.ptr(dense), icode, rows, cols, cols, vcode, _u32(tile_cnt),
                                     _u32(tile_off), _lib.ptr(records), st))
    s.records, s.tile_off = records, tile_off
    s._max_rec = None
    s.max_record_bytes  # computed eagerly (never inside a graph capture)
    s.nnz = int(tile_cnt.sum().item())
    return s


def _decode_window(s: BitmapSparseMatrix, r0, r1, c0, c1, dtype=torch.float32) -> torch.Tensor:
    out = torch.zeros((r1 - r0, c1 - c0), dtype=dtype, device=s.device)
    if r1 > r0 and c1 > c0:
        records, tile_off = s.tb()
        _lib.check(_lib.load().salr_decode(_lib.ptr(records), _u32(tile_off), _VALUE_DTYPES[s.value_dtype][0],
                                           s.rows, s.cols, r0, r1, c0, c1, _lib.ptr(out), _lib.dtype_code(dtype),
                                           c1 - c0, _lib.stream_ptr()))
    return out


def decode(s: BitmapSparseMatrix, dtype: torch.dtype = torch.float32) -> torch.Tensor:
    """Exact inverse of :func:`encode` (``bitmap.py:168-180``), on the GPU."""
    return _decode_window(s, 0, s.rows, 0, s.cols, dtype)


def decode_block(s: BitmapSparseMatrix, row_range, byte_block_range,
                 dtype: torch.dtype = torch.float32) -> torch.Tensor:
    """Dense tile for rows ``[r0, r1)`` and byte blocks ``[b0, b1)``
    (``bitmap.py:183-212``); BoundsError outside, empty ranges -> empty."""
    r0, r1 = (int(v) for v in row_range)
    b0, b1 = (int(v) for v in byte_block_range)
    bpr = s.bytes_per_row
    if not (0 <= r0 <= r1 <= s.rows and 0 <= b0 <= b1 <= bpr):
        raise BoundsError(f"block rows {tuple(row_range)} bytes {tuple(byte_block_range)} outside {(s.rows, bpr)}")
    col_hi = min(8 * b1, s.cols)
    n_cols = max(col_hi - 8 * b0, 0)
    if r1 == r0 or b1 == b0 or n_cols == 0:
        return torch.zeros((r1 - r0, n_cols), dtype=dtype, device=s.device)
    return _decode_window(s, r0, r1, 8 * b0, col_hi, dtype)


# ---------------------------------------------------------------------------
# container format (bitmap.py:215-355) -- host I/O around the device codec

def header_bytes(n_adapters: int) -> int:
    return _FIXED_HEADER.size + n_adapters * _ADAPTER_HEADER.size + _OFFSETS.size


def container_size_bytes(rows: int, cols: int, nnz: int, adapter_ranks) -> int:
    ranks = list(adapter_ranks)
    params = sum(r * (rows + cols) for r in ranks)
    return header_bytes(len(ranks)) + rows * bytes_per_row(cols) + 4 * nnz + 4 * params


def write_container(path, s: BitmapSparseMatrix, adapters) -> int:
    """Serialize to the reference ``.salr`` layout, byte-identical to the
    reference writer (``bitmap.py:236-270``)."""
    for i, ad in enumerate(adapters):
        if ad.d_in != s.rows or ad.d_out != s.cols:
            raise ShapeError(f"adapter {i} dims {(ad.d_in, ad.d_out)} != matrix {(s.rows, s.cols)}")
    bitmap_off = header_bytes(len(adapters))
    values_off = bitmap_off + s.rows * s.bytes_per_row
    adapters_off = values_off + 4 * s.nnz
    blob = bytearray(_FIXED_HEADER.pack(_MAGIC, _VERSION, s.rows, s.cols, s.dtype_code, len(adapters)))
    for ad in adapters:
        blob += _ADAPTER_HEADER.pack(ad.rank, ad.scale)
    blob += _OFFSETS.pack(bitmap_off, values_off, adapters_off)
    blob += s.bitmap.cpu().numpy().tobytes()
    blob += s.values.cpu().numpy().astype("<f4").tobytes()
    for ad in adapters:
        blob += ad.a.cpu().numpy().astype("<f4").tobytes()
        blob += ad.b.cpu().numpy().astype("<f4").tobytes()
    expect = container_size_bytes(s.rows, s.cols, s.nnz, [a.rank for a in adapters])
    if len(blob) != expect:
        raise FormatError(f"serialized size {len(blob)} != accounted {expect}")
    with open(path, "wb") as fh:
        fh.write(blob)
    return len(blob)


def _take(blob: bytes, off: int, n: int, section: str) -> bytes:
    if off + n > len(blob):
        raise FormatError(f"{section}: truncated (need {off + n}, have {len(blob)})")
    return blob[off:off + n]


def read_container(path):
    """Parse a ``.salr`` file (``bitmap.py:279-355``) straight into TB device form."""
    with open(path, "rb") as fh:
        blob = fh.read()
    magic, version, rows, cols, dtype_code, n_ad = _FIXED_HEADER.unpack(_take(blob, 0, _FIXED_HEADER.size,
                                                                              "fixed header"))
    if magic != _MAGIC:
        raise FormatError(f"magic: expected {_MAGIC!r}, got {magic!r}")
    if version != _VERSION:
        raise FormatError(f"version: expected {_VERSION}, got {version}")
    if dtype_code != DTYPE_F32:
        raise FormatError(f"dtype: code {dtype_code} not supported (0 = f32 only)")
    if rows < 1 or cols < 1:
        raise FormatError(f"dims: invalid {(rows, cols)}")
    pos = _FIXED_HEADER.size
    meta = []
    for i in range(n_ad):
        rank, scale = _ADAPTER_HEADER.unpack(_take(blob, pos, _ADAPTER_HEADER.size, f"adapter {i} header"))
        if not 1 <= rank <= min(rows, cols):
            raise FormatError(f"adapter {i} header: rank {rank} out of range")
        meta.append((rank, scale))
        pos += _ADAPTER_HEADER.size
    b_off, v_off, a_off = _OFFSETS.unpack(_take(blob, pos, _OFFSETS.size, "section offsets"))
    pos += _OFFSETS.size
    if b_off != pos or not b_off <= v_off <= a_off:
        raise FormatError(f"section offsets: non-monotone or misplaced ({b_off}, {v_off}, {a_off})")
    bpr = bytes_per_row(cols)
    if v_off - b_off != rows * bpr:
        raise FormatError(f"bitmap section: size {v_off - b_off} != {rows * bpr}")
    bitmap = np.frombuffer(_take(blob, b_off, rows * bpr, "bitmap section"), dtype=np.uint8).reshape(rows, bpr)
    nnz = int(np.unpackbits(bitmap).sum())
    if v_off + 4 * nnz != a_off:
        raise CorruptionError(f"values section size {a_off - v_off} != 4 * popcount {4 * nnz}")
    values = np.frombuffer(_take(blob, v_off, 4 * nnz, "values section"), dtype="<f4").astype(np.float32)
    s = BitmapSparseMatrix(rows, cols, bitmap.copy(), values)
    adapters = []
    pos = a_off
    for i, (rank, scale) in enumerate(meta):
        na, nb = 4 * rows * rank, 4 * rank * cols
        a = np.frombuffer(_take(blob, pos, na, f"adapter {i} A factor"), dtype="<f4").reshape(rows, rank)
        pos += na
        b = np.frombuffer(_take(blob, pos, nb, f"adapter {i} B factor"), dtype="<f4").reshape(rank, cols)
        pos += nb
        adapters.append(AdapterPair(a=a.astype(np.float32), b=b.astype(np.float32), rank=rank, scale=scale))
    if pos != len(blob):
        raise FormatError(f"trailing bytes: file has {len(blob) - pos} extra")
    return s, adapters


def kept_count(p: float, total: int) -> int:
    """``ceil((1 - p) * total)`` nudged one ulp toward zero (``prune.py:202-212``)."""
    import math
    if not 0.0 <= p < 1.0:
        raise DomainError(f"sparsity p must be in [0, 1), got {p}")
    if total < 1:
        raise DomainError("total must be >= 1")
    return int(math.ceil(np.nextafter((1.0 - p) * total, 0.0)))


def compression_ratio(d: int, k: int, p: float, bytes_per_value: int, adapter_params: int,
                      n_adapters: int = 0) -> float:
    """Dense over compressed size incl. header (``bitmap.py:358-378``)."""
    if d < 1 or k < 1:
        raise ShapeError(f"invalid dims {(d, k)}")
    nnz = kept_count(p, d * k)
    dense = d * k * bytes_per_value
    comp = nnz * bytes_per_value + d * bytes_per_row(k) + adapter_params * bytes_per_value + header_bytes(n_adapters)
    return dense / comp
