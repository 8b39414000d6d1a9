/*
 * salr_b200.h -- C ABI of the B200-native SALR linear hot path.
 *
 * Drop-in boundary for the reference package's hot path (reference
 * pkg/src/salr/__init__.py:61-82 re-exports; there is no FFI in the
 * reference, so these entry points are what its Python API binds to through
 * ctypes -- see INTEGRATION.md).  Every entry point:
 *   - takes plain device pointers, sizes and a cudaStream_t (as void*);
 *   - is stream-ordered and CUDA-graph capturable;
 *   - never allocates device memory (workspaces come from the caller);
 *   - returns an int status that maps 1:1 onto the reference error tree
 *     (reference pkg/src/salr/errors.py:22-51).
 *
 * Matrix orientation follows the reference: a weight W is (rows=d_in=K,
 * cols=d_out=N) and the linear computes y = x @ W (reference
 * fusion.py:109-130, pipeline.py:405-461).
 *
 * TB ("tiled bitmap") device format -- the GPU-resident form of
 * BitmapSparseMatrix (reference bitmap.py:88-143):
 *   tiles of 64 rows x 128 cols, tile t = nt * n_kt + kt;
 *   record(t) at byte offset 16 * tile_off[t]:
 *     u32 hdr[4]        group value offsets G1, G2, G3 and tile nnz
 *     u32 bits[4][64]   bits[g][k] bit l  <=> element (k, 32 g + l)
 *     values            group-major, then row-major set-bit order
 *     zero pad to 16 B
 *   The logical bitmap is bit-identical to the reference's (LSB-first, bit
 *   t of byte b = column 8b+t, reference bitmap.py:4-6); salr_to_reference
 *   reproduces the reference row-major bitmap and value order exactly.
 */
#ifndef SALR_B200_H
#define SALR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes -> reference exceptions (errors.py:22-51) */
#define SALR_OK 0
#define SALR_ERR_SHAPE 1      /* ShapeError      */
#define SALR_ERR_DOMAIN 2     /* DomainError     */
#define SALR_ERR_BOUNDS 3     /* BoundsError     */
#define SALR_ERR_CONFIG 4     /* ConfigError     */
#define SALR_ERR_FORMAT 5     /* FormatError     */
#define SALR_ERR_CORRUPTION 6 /* CorruptionError */
#define SALR_ERR_CUDA 7       /* SalrError (device/runtime failure) */

/* element types */
#define SALR_F32 0
#define SALR_BF16 1
#define SALR_F64 2

#define SALR_TILE_K 64
#define SALR_TILE_N 128

/* ---- library ------------------------------------------------------------ */
int salr_version(void);
/* Message for the last non-OK status returned on this thread. */
const char* salr_last_error(void);

/* ---- geometry ------------------------------------------------------------ */
/* Tile grid of a rows x cols matrix.  Replaces bitmap.bytes_per_row /
 * BitmapSparseMatrix shape bookkeeping (reference bitmap.py:146-147). */
int salr_tb_geometry(int64_t rows, int64_t cols, int64_t* n_kt, int64_t* n_nt, int64_t* n_tiles);

/* ---- encode (reference bitmap.py:150-165) -------------------------------- */
/* Phase 1: count set bits per tile/group and write tile_off[n_tiles + 1]
 * (16-byte units).  tile_cnt is a caller workspace of 4 * n_tiles u32.  The
 * caller reads tile_off[n_tiles] to size the record buffer. */
int salr_encode_count(const void* dense, int in_dtype, int64_t rows, int64_t cols, int64_t ld,
                      int value_dtype, uint32_t* tile_cnt, uint32_t* tile_off, void* stream);
/* Phase 2: write the records (bitmap words + compacted values). */
int salr_encode_write(const void* dense, int in_dtype, int64_t rows, int64_t cols, int64_t ld,
                      int value_dtype, const uint32_t* tile_cnt, const uint32_t* tile_off,
                      uint8_t* records, void* stream);

/* ---- decode (reference bitmap.py:168-212: decode / decode_block) --------- */
/* Dense window rows [r0,r1) x cols [c0,c1) into out (row-major, ld_out). */
int salr_decode(const uint8_t* records, const uint32_t* tile_off, int value_dtype, int64_t rows,
                int64_t cols, int64_t r0, int64_t r1, int64_t c0, int64_t c1, void* out,
                int out_dtype, int64_t ld_out, void* stream);

/* nnz of the whole matrix (sum of record headers) -> *nnz_dev (u64, device). */
int salr_tb_nnz(const uint8_t* records, const uint32_t* tile_off, int64_t n_tiles,
                unsigned long long* nnz_dev, void* stream);

/* ---- reference layout <-> TB (reference bitmap.py:88-143 storage) -------- */
/* rowtile_off: workspace of rows * n_nt + 1 u32 (exclusive value offsets). */
int salr_to_reference(const uint8_t* records, const uint32_t* tile_off, int value_dtype, int64_t rows,
                      int64_t cols, uint32_t* rowtile_off, uint8_t* bitmap_out, void* values_out,
                      int values_dtype, void* stream);
/* Phase 1: from a reference row-major bitmap (rows x ceil(cols/8) u8),
 * compute rowtile_off (rows*n_nt+1), tile_cnt (4*n_tiles) and tile_off. */
int salr_from_reference_count(const uint8_t* bitmap, int64_t rows, int64_t cols, int value_dtype,
                              uint32_t* rowtile_off, uint32_t* tile_cnt, uint32_t* tile_off,
                              void* stream);
/* Phase 2: write TB records from the reference bitmap + values. */
int salr_from_reference_write(const uint8_t* bitmap, const void* values, int values_dtype,
                              int64_t rows, int64_t cols, int value_dtype,
                              const uint32_t* rowtile_off, const uint32_t* tile_cnt,
                              const uint32_t* tile_off, uint8_t* records, void* stream);

/* ---- TB2 compute format (linear kernel operand; built once per matrix) --- */
/* From bf16 TB records: tile_off2[n_tiles + 1] (16-byte units), then the
 * TB2 records (layout in csrc/salr_format.cuh: per tile the column masks,
 * band offsets and band-column-major values, so a decoder lane reads its
 * column's values contiguously).  Same logical bitmap and values. */
int salr_tb2_count(const uint8_t* records, const uint32_t* tile_off, int64_t rows, int64_t cols,
                   uint32_t* tile_off2, void* stream);
int salr_tb2_write(const uint8_t* records, const uint32_t* tile_off, int64_t rows, int64_t cols,
                   const uint32_t* tile_off2, uint8_t* records2, void* stream);
/* Dense bf16 matrix (row-major, leading dim ld >= cols) from TB2 records
 * (prefill-size products: decode once, tensor-core GEMM). */
int salr_tb2_decode(const uint8_t* records2, const uint32_t* tile_off2, int64_t rows, int64_t cols,
                    void* dense_bf16, int64_t ld, void* stream);
/* Inverse (bit-exact): bf16 TB records from TB2 records, so a matrix may keep
 * only the compute format resident and rebuild TB on demand (decode,
 * reference layout).  Count: tile_off[n_tiles + 1]; write: the records. */
int salr_tb_from_tb2_count(const uint8_t* records2, const uint32_t* tile_off2, int64_t rows, int64_t cols,
                          uint32_t* tile_off, void* stream);
int salr_tb_from_tb2_write(const uint8_t* records2, const uint32_t* tile_off2, int64_t rows, int64_t cols,
                          const uint32_t* tile_off, uint8_t* records, void* stream);

/* ---- NM24 compute format (2:4 along the columns; csrc/salr_format.cuh) -- */
/* For matrices under the reference's 2:4 mask (prune.py:238-248: at most 2
 * nonzeros in every group of 4 consecutive columns of a row).  Fixed 9216
 * bytes per 64x128 tile (n_tiles = n_nt * n_kt, n-tile-major), no offset
 * table.  Write: from a dense bf16 matrix (leading dim ld); groups with more
 * than 2 nonzeros are added to *bad_groups (device u32, zeroed by the caller)
 * and the records are then not a valid encoding.  Decode: dense bf16. */
int salr_nm24_write(const void* dense_bf16, int64_t rows, int64_t cols, int64_t ld, uint8_t* records,
                    uint32_t* bad_groups, void* stream);
int salr_nm24_decode(const uint8_t* records, int64_t rows, int64_t cols, void* dense_bf16, int64_t ld,
                     void* stream);

/* ---- exact magnitude-prune masks (reference prune.py:213-255) ----------- */
/* Global methods: mask[i] = 1 for exactly `keep` entries -- the largest
 * scores (non-negative, float32 dtype 0 or float64 dtype 2), ties broken
 * toward the lower flat index (the reference's stable argsort).  Radix
 * select + ordered tie scan, stream-ordered, no host sync; workspace of
 * salr_topk_mask_workspace_bytes(n) bytes (no initialisation needed). */
size_t salr_topk_mask_workspace_bytes(int64_t n);
int salr_topk_mask(const void* scores, int dtype, int64_t n, int64_t keep, uint8_t* mask, void* workspace,
                   size_t workspace_bytes, void* stream);
/* N:M: keep the n largest scores of every contiguous group of m columns of a
 * row-major rows x cols matrix, ties toward the lower column offset. */
int salr_nm_mask(const void* scores, int dtype, int64_t rows, int64_t cols, int n_keep, int m_group,
                 uint8_t* mask, void* stream);

/* ---- SALR linear forward (reference pipeline.py:405-461, fusion.py:87-130) */
/* Y (M x N) = X (M x K) @ decode(W) + (X @ A_cat) @ B_cat.
 *   records / tile_off  W in the TB2 compute format (salr_tb2_*)
 *   max_record_bytes  largest TB2 record of W (16 * max(tile_off[t+1]-tile_off[t])),
 *             sizes the shared-memory ring slots; <= 0 means the worst case
 *   x      bf16, row-major, leading dim ldx (ldx % 8 == 0, 16-byte aligned)
 *   acat   bf16 K x r_pad row-major (zero-padded rank columns) or NULL
 *   bcat_t bf16 (n_nt*128) x r_pad row-major = B_cat^T, zero padded, or NULL
 *   r_pad  64 (the fused rank R = sum r_i must be <= 64) or 0 without adapters
 *   y      f32 or bf16, row-major, leading dim ldy
 *   stages    shared-memory ring slots (PipelineConfig.ring_capacity;
 *             1 = serial decode/MMA schedule, <= 0 = deepest that fits)
 *   num_ctas  persistent CTAs (<= 0: one per SM)
 *   workspace >= salr_linear_workspace_bytes(M, N, K, r_pad, num_ctas); its
 *   first salr_linear_workspace_zero_bytes() bytes (ticket counters, adapter
 *   control words, in-kernel U accumulators at fixed offsets) must be zeroed
 *   once at allocation -- the kernels maintain them from then on, so the same
 *   workspace serves back-to-back / graph-replayed calls.  Split-K partials are summed in a fixed order: results are
 *   bit-identical from run to run for a given num_ctas. */
size_t salr_linear_workspace_bytes(int64_t M, int64_t N, int64_t K, int64_t r_pad, int num_ctas);
/* Bytes at the start of every workspace that must be zero before its first
 * use (ticket counters, adapter control words and the two parity buffers of
 * the in-kernel U fixed-point accumulator; 768 KiB).  The kernels maintain
 * the invariant from then on (counters self-reset; each launch clears the
 * U buffer the previous launch used), so zero it once, at allocation. */
size_t salr_linear_workspace_zero_bytes(void);
/* Instrumentation (tools only): when buf != NULL, subsequent linear launches
 * write per-CTA %globaltimer stamps of pipeline events into buf[cta][32]
 * (u64, device memory, >= 32 * 8 * num_ctas bytes).  NULL disables. */
int salr_debug_set_trace(void* buf);
/* Instrumentation (tests/tools): configuration of the most recent
 * salr_linear_forward launch on this host thread's process: {ctas, stages,
 * BM, decoder groups, u_mode (0 none, 1 in-kernel U, 2 U pre-kernel), coop,
 * cluster size (0 = global split-K reduction), pdl, cluster size requested,
 * max co-resident clusters (-1 = not queried), dynamic smem bytes,
 * cooperative (1 = launched co-scheduled: in-kernel U / cooperative split-K
 * wait on other CTAs, so the driver guarantees every CTA is resident)}. */
int salr_debug_last_launch(int32_t* info12);
/* Pipeline probe (tests / tools): the device form of the reference's
 * PipelineProbe (pipeline.py:89-103).  While log != NULL, decode-size linear
 * launches append every ring-slot transition (slot = cta * stages + stage,
 * EMPTY 0 -> FILLED 1 -> CONSUMED 2 -> EMPTY) to log[4 + i] as
 * slot << 8 | old << 4 | new, count entries in log[0], fills in log[1] and
 * consumes in log[2] (device u32, zeroed by the caller), and sleep a hashed
 * 0..max_delay_ns before every tile decode and MMA issue (jitter
 * injection).  NULL disables. */
int salr_debug_set_probe(void* log, size_t log_words, int max_delay_ns, uint32_t seed);
/* flags: SALR_FLAG_PDL launches the kernel as a programmatic dependent of the
 * preceding work on the stream: its weight-streaming prologue overlaps the
 * tail of that work and it waits for it (griddepcontrol.wait) before reading
 * x.  The caller must not let the preceding kernel still READ y, and must use
 * a workspace the preceding kernel does not use (alternate two).  Without the
 * flag, launches whose CTAs wait on each other (in-kernel U, cooperative
 * split-K) are co-scheduled (cooperative launch: the driver guarantees every
 * CTA resident).  With it they are not (co-scheduling would wait for the
 * preceding grid to drain): the grid is checked against occupancy, and the
 * caller must not run concurrent kernels that wait on this grid. */
#define SALR_FLAG_PDL 1
/* flags: SALR_FLAG_U_FP32 computes U = X @ A_cat in the fp32 pre-kernel
 * instead of the in-kernel int64 fixed-point accumulator (resolution 2^-26,
 * range |U| < 2^37).  The Python layer sets it when the bound
 * K * max|X| * max|A_cat| falls outside [2^-6, 2^34]. */
#define SALR_FLAG_U_FP32 2
/* flags: SALR_FLAG_NM24: records are NM24 (salr_nm24_write); tile_off and
 * max_record_bytes are ignored.  Decode-size kernel at every M. */
#define SALR_FLAG_NM24 4
int salr_linear_forward(const void* x, int64_t M, int64_t K, int64_t ldx, const uint8_t* records,
                        const uint32_t* tile_off, int64_t max_record_bytes, int64_t N, const void* acat, const void* bcat_t,
                        int64_t r_pad, void* y, int y_dtype, int64_t ldy, void* workspace,
                        size_t workspace_bytes, int stages, int num_ctas, int flags, void* stream);

/* ---- chained linears (one persistent launch; no reference counterpart:
 * the reference runs pipelined_forward once per linear, pipeline.py:275-331,
 * and this is L such calls fused for a decode step's linear chain).
 * Linear l computes y_l = x_l @ W_l [+ (x_l @ A_cat_l) @ B_cat_l] in bf16 out,
 * where x_0 = x0 (M x K_0, ld ldx0) and x_l = columns [0, K_l) of y_{l-1}
 * (ld ldy_{l-1}; K_l <= N_{l-1}).  Records are TB2 (salr_tb2_*), adapters
 * as in salr_linear_forward (r_pad 0 / 64 / 128).  1 <= L <= 4, M <= 256.
 * Results equal L salr_linear_forward calls with the same grid (the SM
 * count).  The workspace's first salr_chain_workspace_zero_bytes() bytes
 * must be zero once, at allocation (counters reset themselves). */
typedef struct {
  const uint8_t* records;
  const uint32_t* tile_off;
  int64_t max_record_bytes;
  int64_t K, N;
  const void* acat;
  const void* bcat_t;
  int64_t r_pad;
  void* y;
  int64_t ldy;
} salr_chain_linear_t;
size_t salr_chain_workspace_bytes(int64_t M, int L);
size_t salr_chain_workspace_zero_bytes(void);
int salr_chain_forward(const salr_chain_linear_t* lin, int L, const void* x0, int64_t M, int64_t ldx0,
                       void* workspace, size_t workspace_bytes, int flags, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SALR_B200_H */
