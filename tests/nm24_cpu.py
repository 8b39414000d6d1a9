"""CPU restatement of the NM24 compute format (test infrastructure only).

NM24 (csrc/salr_format.cuh) holds a matrix whose nonzeros are 2:4 along the
columns -- at most 2 in every group of 4 consecutive columns of a row, the
reference's N:M mask (prune.py:238-248).  Per 64x128 tile (n-tile-major,
t = nt * n_kt + kt), fixed 9216 bytes:
  values [16 bands][32 groups] x 16 B  u32 per band row: v0 | v1 << 16, the
                                       group's first / second nonzero (bf16)
  masks  [2 halves][32 groups] x 16 B  at 8192: word w of (h, g) = rows
                                       32h + 8w .. +7, row i's 4-bit column
                                       mask at bits 4i .. 4i+3
``nm24_select`` restates the linear kernel's permute-based decoder
(decode_tile_nm24 in salr_linear.cu) so its bit tricks are checked on CPU.
"""

from __future__ import annotations

import numpy as np

TILE_K, TILE_N, REC = 64, 128, 9216


def _bf16_bits(a: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    if np.any(u & 0xFFFF):
        raise ValueError("values are not bf16-exact")
    return (u >> 16).astype(np.uint32)


def nm24_records(dense: np.ndarray) -> np.ndarray:
    """uint8 NM24 records of a bf16-exact matrix (ValueError if not 2:4)."""
    rows, cols = dense.shape
    n_kt, n_nt = -(-rows // TILE_K), -(-cols // TILE_N)
    bits = np.zeros((n_kt * TILE_K, n_nt * TILE_N), dtype=np.uint32)
    bits[:rows, :cols] = _bf16_bits(dense)
    out = np.zeros((n_nt * n_kt, REC), dtype=np.uint8)
    for nt in range(n_nt):
        for kt in range(n_kt):
            tile = bits[kt * TILE_K:(kt + 1) * TILE_K, nt * TILE_N:(nt + 1) * TILE_N].reshape(TILE_K, 32, 4)
            nz = (tile & 0x7FFF) != 0
            if (nz.sum(axis=2) > 2).any():
                raise ValueError("not 2:4 along the columns")
            vals = np.zeros((TILE_K, 32), dtype=np.uint32)
            masks = np.zeros((TILE_K, 32), dtype=np.uint32)
            for r in range(TILE_K):
                for g in range(32):
                    v = [int(tile[r, g, j]) for j in range(4) if nz[r, g, j]]
                    v += [0] * (2 - len(v))
                    vals[r, g] = v[0] | v[1] << 16
                    masks[r, g] = sum(1 << j for j in range(4) if nz[r, g, j])
            rec = np.zeros(REC // 4, dtype=np.uint32)
            # values: band b, group g, row 4b + i -> u32 index 4 * (32 b + g) + i
            for b in range(16):
                for g in range(32):
                    rec[4 * (32 * b + g):4 * (32 * b + g) + 4] = vals[4 * b:4 * b + 4, g]
            # masks: half h, group g, word w: rows 32h + 8w + i at bits 4i
            for h in range(2):
                for g in range(32):
                    for w in range(4):
                        word = 0
                        for i in range(8):
                            word |= int(masks[32 * h + 8 * w + i, g]) << (4 * i)
                        rec[2048 + 4 * (32 * h + g) + w] = word
            out[nt * n_kt + kt] = rec.view(np.uint8)
    return out.reshape(-1)


def nm24_dense(records: np.ndarray, rows: int, cols: int) -> np.ndarray:
    """float32 matrix of NM24 records (direct rule: k-th set mask bit <- v_k)."""
    n_kt, n_nt = -(-rows // TILE_K), -(-cols // TILE_N)
    out = np.zeros((n_kt * TILE_K, n_nt * TILE_N), dtype=np.uint32)
    rec = records.reshape(n_nt * n_kt, REC // 4 * 4).view(np.uint32)
    for nt in range(n_nt):
        for kt in range(n_kt):
            r32 = rec[nt * n_kt + kt]
            for r in range(TILE_K):
                b, i = divmod(r, 4)
                h, rr = divmod(r, 32)
                w, ii = divmod(rr, 8)
                for g in range(32):
                    v = int(r32[4 * (32 * b + g) + i])
                    m = (int(r32[2048 + 4 * (32 * h + g) + w]) >> (4 * ii)) & 0xF
                    k = 0
                    for j in range(4):
                        if (m >> j) & 1:
                            out[kt * TILE_K + r, nt * TILE_N + 4 * g + j] = (v >> (16 * k)) & 0xFFFF if k < 2 else 0
                            k += 1
    return (out[:rows, :cols] << 16).view(np.float32)


def prmt(a: int, b: int, sel: int) -> int:
    """PTX prmt.b32 (default mode): byte i of the result from selector nibble i
    (bits 0-2 index bytes of {b, a}; bit 3 replicates that byte's sign)."""
    src = (a & 0xFFFFFFFF) | (b & 0xFFFFFFFF) << 32
    out = 0
    for i in range(4):
        n = (sel >> (4 * i)) & 0xF
        byte = (src >> (8 * (n & 7))) & 0xFF
        if n & 8:
            byte = 0xFF if byte & 0x80 else 0
        out |= byte << (8 * i)
    return out


def nm24_select(mask_word: int, w_lo: int, w_hi: int, j: int, pidx: int) -> int:
    """The kernel's packed (row 2p, row 2p+1) bf16 pair of column j of a group,
    from the 8-row mask word and the two rows' value words (decode_tile_nm24)."""
    m32 = 0xFFFFFFFF
    lower = (0x11111111 * ((1 << j) - 1)) & m32
    kx = ((mask_word << (3 - j)) & m32) & 0x88888888
    bx = (((mask_word & lower) + 0x77777777) & m32) & 0x88888888
    klo, blo = (kx << 4) & m32, (bx << 4) & m32
    sel = (0x8 | pidx) * 0x11 | ((0xC | pidx) * 0x11) << 8  # byte mask: halves
    vsel = (0x8 | pidx) | (0xC | pidx) << 4                   # selector: nibble pairs
    msk = prmt(klo, kx, sel)
    vs = (prmt(blo, bx, vsel) & 0x2222) | 0x5410
    return prmt(w_lo, w_hi, vs) & msk


def nm24_tile_tmem(rec_tile: np.ndarray) -> np.ndarray:
    """TMEM image (128 lanes x 32 u32 columns; column c = rows 2c | 2c+1 << 16)
    the kernel's decoder writes for one 9216-byte tile, with its addressing:
    lane 32q + l = column j = l & 3 of group g = 8q + (l >> 2); per 4 bands b0
    one 8-byte mask load at 8192 + 16 (32 (b0 >> 3) + g) + 4 ((b0 >> 1) & 3),
    per band one 16-byte value load at 16 (32 b + g)."""
    r8 = rec_tile.view(np.uint8)

    def u32(off):
        return int(r8[off:off + 4].view(np.uint32)[0])

    out = np.zeros((128, 32), dtype=np.uint32)
    for lane_all in range(128):
        q, lane = divmod(lane_all, 32)
        g, j = 8 * q + (lane >> 2), lane & 3
        for b0 in range(0, 16, 4):
            mo = 8192 + 16 * (32 * (b0 >> 3) + g) + 4 * ((b0 >> 1) & 3)
            mw = (u32(mo), u32(mo + 4))
            for h in range(2):
                for bb in range(2):
                    vo = 16 * (32 * (b0 + 2 * h + bb) + g)
                    w = [u32(vo + 4 * i) for i in range(4)]
                    for t in range(2):
                        col = 2 * b0 + 4 * h + 2 * bb + t
                        out[lane_all, col] = nm24_select(mw[h], w[2 * t], w[2 * t + 1], j, 2 * bb + t)
    return out
