/*
 * dfss.h -- C ABI of libdfss_sm100a.so, the B200 (sm_100a) DFSS attention path.
 *
 * This is the drop-in boundary for the kernel-backend interface of the
 * reference package nmattn 0.1.0 (backend.kernels(), backend.py:63-67): the
 * numba kernels _kernels_numba.sddmm_compress / softmax_nonzeros /
 * spmm_gather are replaced by dfss_sddmm_prune / dfss_softmax_rows /
 * dfss_spmm, and pipeline.nm_attention (pipeline.py:15-32) by
 * dfss_nm_attention.  Citations are file:line into /root/reference/pkg/src/nmattn.
 *
 * Conventions (all entry points):
 *   - every pointer argument is DEVICE memory unless stated otherwise; the
 *     caller allocates every output (the reference kernels return fresh
 *     arrays, _kernels_numba.py:20,69,95,115; here the host layer allocates);
 *   - tensors are dense, row-major, batched over a leading "bh" dimension
 *     (flattened batch x heads); the reference ops have no batch dimension
 *     (SPEC.md:310), slice h of every argument is one reference call;
 *   - calls are asynchronous and stream-ordered on `stream` (a cudaStream_t
 *     passed as void*; NULL = legacy default stream);
 *   - the return value is a dfss_status; validation failures are reported
 *     before any launch (the reference validates before dispatch, fused.py:58-82);
 *   - no global state other than a per-device attribute cache.
 *
 * Sparse layouts on the device:
 *   nonzeros : [bh, rows, cols/2] in the nonzero dtype, row-major -- the
 *              reference's compressed nonzeros (codec.py:203-216), kept values
 *              of each group in ascending column order;
 *   meta_hw  : uint32 words, [bh, ceil(rows/128), ceil(groups/8), 128] where
 *              groups = cols/group_size.  Word (rb, c, L) with
 *              L = 16*m2 + 8*k1 + m0 (m0<8, k1<2, m2<8) packs the 4-bit nibbles
 *              (codec.py:72-76, value lo|hi<<2) of groups 8c+4k1 .. 8c+4k1+3:
 *              bits [0,16)  from row 128*rb + 16*m2 + m0   (nibble i at bits 4i),
 *              bits [16,32) from row 128*rb + 16*m2 + 8 + m0.
 *              This is the tcgen05.mma.sp metadata layout of one 128-lane TMEM
 *              column, so the SpMM moves words straight into TMEM.  Padding rows /
 *              groups hold nibble 0x4 with zero nonzeros.
 *   meta_logical : uint8 per group, [bh, rows, groups] -- the reference's
 *              LOGICAL metadata stream (codec.py:331-335), one nibble per byte.
 */
#ifndef DFSS_H_
#define DFSS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  DFSS_OK = 0,
  DFSS_ERR_INVALID = -1,      /* argument validation failed (reference: ValueError) */
  DFSS_ERR_UNSUPPORTED = -2,  /* valid request this build has no kernel for */
  DFSS_ERR_CUDA = -3,         /* CUDA runtime / driver error (reference: none; host raises RuntimeError) */
  DFSS_ERR_NO_DEVICE = -4     /* no sm_100 device or driver entry point */
} dfss_status;

/* group size doubles as the mode id: codec.py:34-50 */
enum { DFSS_MODE_1_2 = 2, DFSS_MODE_2_4 = 4 };

enum { DFSS_F32 = 0, DFSS_BF16 = 1, DFSS_F16 = 2 };

/* arithmetic for the QK^T contraction */
enum {
  DFSS_MATH_AUTO = 0, /* tcgen05 for 16-bit inputs, exact FP32 FFMA for fp32 inputs */
  DFSS_MATH_FFMA = 1, /* force SIMT FP32 FFMA (any dtype) */
  DFSS_MATH_TF32 = 2  /* fp32 inputs on tcgen05 kind::tf32 */
};

/* Words in a meta_hw buffer for [bh, rows, cols] under `mode`. */
int64_t dfss_meta_hw_words(int mode, int64_t bh, int64_t rows, int64_t cols);

/*
 * Fused score + prune: replaces _kernels_numba.sddmm_compress
 * (_kernels_numba.py:110-188) behind fused.sddmm_prune (fused.py:41-96).
 *   q [bh, n_q, d], k [bh, n_k, d] in `in_dtype`; scores = scale * q k^T
 *   accumulated in fp32; each group of `mode` consecutive scores of a row is
 *   pruned by signed value, ties to the lower index (codec.py:104-123),
 *   AFTER scaling (_kernels_numba.py:140-145).  Writes nonzeros [bh, n_q, n_k/2]
 *   in `nz_dtype` and meta_hw; never a dense score matrix unless `scores_dbg`
 *   (nullable, fp32 [bh, n_q, n_k]) is given -- the parity hook that dumps the
 *   exact post-scale scores the epilogue selected on.
 *   tile_keep (nullable): uint8 [ceil(n_q/tile_rows), ceil(n_k/tile_cols)] shared by
 *   all bh -- the BlockMask grid (codec.py:150-200); masked tiles are skipped
 *   and left as zero nonzeros / nibble 0x4 padding.
 *   FusedStats (fused.py:22-38) are structural and computed by the host layer
 *   from the tile grid; dense_elems_written is 0 unless scores_dbg is given.
 *   row_max (nullable, fp32 [bh, n_q, 4], tcgen05 path only): the four column-quarter
 *   partial maxima of every row's kept scores (max over a row = its max over the
 *   kept values, the row maximum always survives) -- the input that lets
 *   dfss_spmm apply the softmax on the fly.
 */
int dfss_sddmm_prune(const void* q, const void* k, void* nonzeros, uint32_t* meta_hw, float scale,
                     int mode, int in_dtype, int nz_dtype, int math, int64_t bh, int n_q, int n_k, int d,
                     const uint8_t* tile_keep, int tile_rows, int tile_cols, float* scores_dbg,
                     float* row_max, void* stream);

/*
 * Softmax over each row's present nonzeros: replaces
 * _kernels_numba.softmax_nonzeros (_kernels_numba.py:66-87) behind
 * sparse_ops.softmax_rows (sparse_ops.py:18-37).  nz_in [bh, rows, nz_cols]
 * in `in_dtype` -> p_out in `out_dtype` (may alias nz_in when dtypes match).
 * tile_keep/tile_rows/tile_cols: optional BlockMask grid in DENSE columns
 * (present nonzero j of row i <=> keep[i/tile_rows][2j/tile_cols]).
 * err_row (nullable, device int32[2], caller-initialised to INT32_MAX):
 * err_row[0] = 1 + first empty flattened row (bh*rows + row), err_row[1] =
 * 1 + first flattened row holding a NaN (sparse_ops.py:27-32); the host layer
 * turns them into the reference's ValueErrors.
 */
int dfss_softmax_rows(const void* nz_in, void* p_out, int in_dtype, int out_dtype, int64_t bh, int rows,
                      int nz_cols, const uint8_t* tile_keep, int tile_rows, int tile_cols, int32_t* err_row,
                      void* stream);

/*
 * Compressed SpMM out = decompress(P) . V: replaces _kernels_numba.spmm_gather
 * (_kernels_numba.py:91-103) behind sparse_ops.spmm (sparse_ops.py:40-68).
 *   p [bh, rows, n_k/2] in `p_dtype`, meta_hw for [bh, rows, n_k],
 *   v [bh, n_k, d] in `v_dtype`, out [bh, rows, d] in `out_dtype`, fp32 accumulation.
 *   16-bit P and V on aligned shapes run tcgen05.mma.sp with the metadata
 *   consumed straight from meta_hw; otherwise an FP32 FFMA gather kernel.
 *   tile_keep: optional BlockMask grid (masked tiles contribute zero).
 *   row_max (nullable, [bh, rows, 4] from dfss_sddmm_prune): p holds RAW kept
 *   scores and the softmax (sparse_ops.softmax_rows) is fused in: each staged
 *   P tile is rewritten as exp(s - max_row) in shared memory before the MMA and
 *   the output rows are divided by the row sums -- out = spmm(softmax_rows(p), v)
 *   without the softmax's HBM round trip (tcgen05 path only).
 */
int dfss_spmm(const void* p, const uint32_t* meta_hw, const void* v, void* out, int mode, int p_dtype,
              int v_dtype, int out_dtype, int64_t bh, int rows, int n_k, int d, const uint8_t* tile_keep,
              int tile_rows, int tile_cols, const float* row_max, void* stream);

/*
 * End-to-end DFSS attention: replaces pipeline.nm_attention (pipeline.py:15-32)
 * for [bh, n, d] q/k/v in `dtype`, scale = 1/sqrt(d) (fused.py:110).
 *   out [bh, n, d] in `dtype`.  `workspace` (device) must hold
 *   dfss_nm_attention_workspace_bytes(...) bytes for the compressed P, meta and
 *   row maxima.  16-bit 2:4 on tiled shapes runs two kernels (SDDMM+prune+row
 *   max, softmax-fused SpMM); everything else runs SDDMM -> softmax -> SpMM.
 */
int64_t dfss_nm_attention_workspace_bytes(int mode, int dtype, int64_t bh, int n, int d);
/* Exact workspace for the path dfss_nm_attention(_masked) will take with these arguments:
 * 0 for the fused 16-bit kernel (masked: the step / chunk liveness bitmaps and the
 * row-block schedule, a few KB), bh*n*d*4 (V^T) for the fused tf32 kernel (+ the same
 * bitmaps when masked), the staged bytes above otherwise.  masked != 0 when a tile_keep grid
 * will be passed. */
int64_t dfss_nm_attention_workspace_bytes_for(int mode, int dtype, int math, int64_t bh, int n, int d,
                                              int tile_rows, int tile_cols, int masked);
int dfss_nm_attention(const void* q, const void* k, const void* v, void* out, int mode, int dtype, int math,
                      int64_t bh, int n, int d, void* workspace, int64_t workspace_bytes, void* stream);

/*
 * nm_attention with a BlockMask (pipeline.py:15-32 with block_mask; mask threaded as in
 * fused.py:73-82 and sparse_ops.py:27-30,57-64): tile_keep is the DEVICE uint8 grid
 * [ceil(n/tile_rows)][ceil(n/tile_cols)] shared by every (batch, head); masked tiles are
 * structurally absent.  16-bit inputs (and fp32 with math = TF32) with tile_rows and
 * tile_cols multiples of 32 run the fused kernel: masked 32x32 chunks are absent, 128x128
 * steps with no kept tile are skipped entirely (no K/V load, no MMA), and the 256-row items
 * are scheduled heaviest-first; two small pre-kernels build the liveness bitmaps in the
 * workspace (dfss_nm_attention_workspace_bytes_for).  Other shapes run the staged kernels.  Rows whose
 * tiles are all masked are undefined here -- the host layer rejects them first, as the
 * reference's softmax_rows does ("empty row N").  tile_keep == NULL is dfss_nm_attention.
 */
int dfss_nm_attention_masked(const void* q, const void* k, const void* v, void* out, int mode, int dtype, int math,
                             int64_t bh, int n, int d, const uint8_t* tile_keep, int tile_rows, int tile_cols,
                             void* workspace, int64_t workspace_bytes, void* stream);

/*
 * Parity hook for the path dfss_nm_attention_masked takes (same arguments, same kernels, same
 * output), with the selection evidence of every prune: scores_dbg (device fp32 [bh, n, n]) gets
 * the post-scale scores each prune compared -- for the fused kernels the fp32 tcgen05
 * accumulators of Q K^T times the exact scale 1/sqrt(64) = 2^-3, in key order -- and meta_dbg
 * (device uint32, dfss_meta_hw_words(*meta_mode, bh, n, n) words) the metadata words handed to
 * tcgen05.mma.sp (fused) or written by the SDDMM (staged), in the meta_hw layout above.
 * *meta_mode (host int) is the group size of that layout: 4 for the fused 16-bit kernel, which
 * runs 1:2 as the 2:4 pattern "one survivor per pair" (nibble 8 + a + 4b: elements a and 2 + b),
 * and the call's mode otherwise.  Entries of 128 x 128 steps the fused kernels skip (fully
 * masked) are not written.  The selection test feeds scores_dbg to the reference
 * compress_logical / prune_dense (codec.py:324-335) and compares the decoded metadata bitwise.
 * Replaces: nothing in the reference (its fused path keeps no dense scores by design,
 * fused.py:22-38); this is the evidence channel for _kernels_numba.py:145-184 on the GPU path.
 */
int dfss_nm_attention_dump(const void* q, const void* k, const void* v, void* out, int mode, int dtype, int math,
                           int64_t bh, int n, int d, const uint8_t* tile_keep, int tile_rows, int tile_cols,
                           void* workspace, int64_t workspace_bytes, float* scores_dbg, uint32_t* meta_dbg,
                           int* meta_mode, void* stream);

/* Which path dfss_nm_attention(_masked) takes for these arguments (no launch): 1 fused 16-bit
 * (flash_tc.cu), 2 fused tf32 (flash_tf32.cu), 3 staged tcgen05 SDDMM + softmax-fused SpMM,
 * 4 staged exact-FP32 FFMA, 5 staged with a block mask, 6 staged exact-FP32 on tcgen05 as
 * 3xTF32 (sddmm_tf32.cu / spmm_tf32.cu: fp32 1:2, math auto, from ~1 M scores = bh * n^2);
 * a negative dfss_status if unsupported.  The _bh form takes the batch x heads count (the
 * 3xTF32 choice depends on it); the other assumes bh = 1. */
int dfss_nm_attention_path(int mode, int dtype, int math, int n, int d, int tile_rows, int tile_cols, int masked);
int dfss_nm_attention_path_bh(int mode, int dtype, int math, int64_t bh, int n, int d, int tile_rows, int tile_cols,
                              int masked);

/*
 * Parity hook: prune a given fp32 score tensor with the SAME device selection
 * routine the SDDMM epilogue uses (codec._select_rows, codec.py:289-313).
 *   scores [rows, cols] fp32 -> nonzeros [rows, cols/2] (nz_dtype),
 *   meta_logical uint8 [rows, cols/gs], kept uint8 [rows, cols] (prune_dense mask,
 *   codec.py:324-328).  Any output pointer may be NULL.
 */
int dfss_prune_scores(const float* scores, void* nonzeros, uint8_t* meta_logical, uint8_t* kept, int mode,
                      int nz_dtype, int64_t rows, int cols, void* stream);

/* The same selection on float64 scores (the reference's own dtype): scores [rows, cols] f64 ->
 * nonzeros f64 [rows, cols/2], meta_logical uint8 [rows, cols/gs], kept uint8 [rows, cols]
 * (any output NULL to skip).  Used by the codec for float64 matrices (compress_logical /
 * prune_dense on DenseMatrix data), so no value is rounded to fp32 before it is compared. */
int dfss_prune_scores_f64(const double* scores, double* nonzeros, uint8_t* meta_logical, uint8_t* kept, int mode,
                          int64_t rows, int cols, void* stream);

/* meta_hw <-> LOGICAL nibble stream (one nibble per byte), [bh, rows, cols/gs]. */
int dfss_meta_hw_to_logical(const uint32_t* meta_hw, uint8_t* meta_logical, int mode, int64_t bh, int rows,
                            int cols, void* stream);
int dfss_meta_logical_to_hw(const uint8_t* meta_logical, uint32_t* meta_hw, int mode, int64_t bh, int rows,
                            int cols, void* stream);

/*
 * The reference kernel module (backend.kernels(), backend.py:63-67) on the GPU, float64.
 * The reference's hot loops are five duck-typed functions (_kernels_numba.py:39,62,87,106,188);
 * these are the same five, on DEVICE float64 buffers, computed with the reference's arithmetic:
 * one running accumulator per output, ascending reduction index, separately rounded products
 * and sums (numba runs with fastmath off).  sddmm_compress, spmm_gather and gemm_abt are
 * therefore bitwise equal to the reference; the softmaxes differ only through exp (<= 1 ulp).
 * integration/_kernels_cuda.py wraps them with the reference's Python signatures.  Unlike the
 * production entry points above (tile masks, meta_hw words), these take the reference's
 * arbitrary per-nonzero `present` masks and decoded int64 column indices.
 */
/* sddmm_compress (_kernels_numba.py:110-188): q [n, d], k [m, d]; keep uint8 [ceil(n/tile_rows),
 * ceil(m/tile_cols)] (the reference always passes a grid); writes nonzeros [n, m/2] and logical
 * meta uint8 [n, m/group_size], zero in masked tiles.  peak / nnz / nib are structural (host). */
int dfss_kmod_sddmm_compress(const double* q, const double* k, double scale, int group_size, int n, int m, int d,
                             int tile_rows, int tile_cols, const uint8_t* keep, double* nonzeros, uint8_t* meta,
                             void* stream);
/* softmax_nonzeros (_kernels_numba.py:66-87): nz [rows, cols], present uint8 [rows, cols]
 * (nullable = all present) -> out [rows, cols], absent slots 0. */
int dfss_kmod_softmax_nonzeros(const double* nz, const uint8_t* present, double* out, int64_t rows, int cols,
                               void* stream);
/* spmm_gather (_kernels_numba.py:91-106): nz [rows, nz_cols], cols int64 [rows, nz_cols],
 * present uint8 [rows, nz_cols] (nullable), v [v_rows, d] -> out [rows, d].  err (nullable, device
 * int32, caller-initialised to INT32_MAX) receives the first row holding a column outside
 * [0, v_rows) -- such entries are skipped. */
int dfss_kmod_spmm_gather(const double* nz, const int64_t* cols, const uint8_t* present, const double* v,
                          double* out, int64_t rows, int nz_cols, int v_rows, int d, int32_t* err, void* stream);
/* gemm_abt (_kernels_numba.py:16-39): out [n, m] = scale * a [n, kdim] . b [m, kdim]^T (the
 * reference's tile / k-panel arguments only reorder traversal, never the per-element sum). */
int dfss_kmod_gemm_abt(const double* a, const double* b, double scale, int64_t n, int64_t m, int kdim, double* out,
                       void* stream);
/* row_softmax_dense (_kernels_numba.py:43-62): x [rows, cols] -> out [rows, cols]. */
int dfss_kmod_row_softmax_dense(const double* x, double* out, int64_t rows, int cols, void* stream);

/* Human-readable status; last CUDA error text for DFSS_ERR_CUDA. Never NULL. */
const char* dfss_status_string(int status);
const char* dfss_last_error(void);
/* 1 if the tcgen05 path can run on the current device (sm_100), else 0. */
int dfss_has_tcgen05(void);
int dfss_version(void);

#ifdef __cplusplus
}
#endif

#endif /* DFSS_H_ */
