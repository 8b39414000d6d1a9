"""CPU restatement of the TB2 compute format (test infrastructure only).

Builds and expands TB2 records with NumPy exactly as ``tb2_write_kernel``
(salr_codec.cu) lays them out -- see salr_format.cuh / include/salr_b200.h:
per 64x128 tile, n-tile-major (t = nt * n_kt + kt), 16-byte aligned:
  u32 hdr[4]           value offsets of column groups 1,2,3 and the tile nnz
  u16 bandoff[4][16]   per 32-column group and 4-row band: offset of the
                       band's values from the group's first value
  u64 cmask[128]       cmask[n] bit r <=> element (row r, col n) nonzero
  bf16 values          group-major; band-major; column-major; ascending rows
so the multi-rank sharding tests can run without a GPU.
"""

from __future__ import annotations

import numpy as np

TILE_K, TILE_N = 64, 128
T2_BANDOFF, T2_MASK, T2_VAL = 16, 144, 1168


def _bf16_bits(a: np.ndarray) -> np.ndarray:
    """float32 -> bf16 bit patterns (inputs must be bf16-exact)."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    if np.any(u & 0xFFFF):
        raise ValueError("values are not bf16-exact")
    return (u >> 16).astype(np.uint16)


def tb2_records(dense: np.ndarray):
    """(records uint8, tile_off int32 in 16-byte units) of a bf16-exact matrix."""
    rows, cols = dense.shape
    n_kt, n_nt = -(-rows // TILE_K), -(-cols // TILE_N)
    bits = _bf16_bits(dense)
    out, off = [], [0]
    for nt in range(n_nt):
        for kt in range(n_kt):
            tile = np.zeros((TILE_K, TILE_N), dtype=np.uint16)
            blk = bits[kt * TILE_K:(kt + 1) * TILE_K, nt * TILE_N:(nt + 1) * TILE_N]
            tile[:blk.shape[0], :blk.shape[1]] = blk
            nz = tile != 0
            hdr = np.zeros(4, dtype=np.uint32)
            bandoff = np.zeros((4, 16), dtype=np.uint16)
            cmask = np.zeros(128, dtype=np.uint64)
            for n in range(128):
                cmask[n] = np.uint64(sum(1 << r for r in range(64) if nz[r, n]))
            vals = []
            for g in range(4):
                if g:
                    hdr[g - 1] = len(vals)
                g0 = len(vals)
                for b in range(16):
                    bandoff[g, b] = len(vals) - g0
                    for c in range(32 * g, 32 * g + 32):
                        for r in range(4 * b, 4 * b + 4):
                            if nz[r, c]:
                                vals.append(tile[r, c])
            hdr[3] = len(vals)
            rec = hdr.tobytes() + bandoff.tobytes() + cmask.tobytes() + np.array(vals, dtype=np.uint16).tobytes()
            rec += b"\0" * (-len(rec) % 16)
            out.append(rec)
            off.append(off[-1] + len(rec) // 16)
    return np.frombuffer(b"".join(out), dtype=np.uint8).copy(), np.array(off, dtype=np.int32)


def tb2_decode(records: np.ndarray, tile_off: np.ndarray, rows: int, cols: int) -> np.ndarray:
    """Dense float32 matrix of TB2 records (inverse of ``tb2_records``)."""
    n_kt, n_nt = -(-rows // TILE_K), -(-cols // TILE_N)
    out = np.zeros((n_kt * TILE_K, n_nt * TILE_N), dtype=np.float32)
    for nt in range(n_nt):
        for kt in range(n_kt):
            o = 16 * int(tile_off[nt * n_kt + kt])
            rec = records[o:]
            hdr = rec[:16].view(np.uint32)
            bandoff = rec[T2_BANDOFF:T2_MASK].view(np.uint16).reshape(4, 16)
            cmask = rec[T2_MASK:T2_VAL].view(np.uint64)
            vals = rec[T2_VAL:T2_VAL + 2 * int(hdr[3])].view(np.uint16)
            for g in range(4):
                gbase = int(hdr[g - 1]) if g else 0
                for b in range(16):
                    pos = gbase + int(bandoff[g, b])
                    for c in range(32 * g, 32 * g + 32):
                        m = int(cmask[c])
                        for r in range(4 * b, 4 * b + 4):
                            if (m >> r) & 1:
                                out[kt * TILE_K + r, nt * TILE_N + c] = \
                                    (np.uint32(vals[pos]) << np.uint32(16)).view(np.float32)
                                pos += 1
    return out[:rows, :cols]
