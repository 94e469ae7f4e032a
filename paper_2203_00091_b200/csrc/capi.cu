// capi.cu -- extern "C" entry points of libdfss_sm100a.so (include/dfss.h).
//
// Validation happens here, before any launch, mirroring the reference's
// wrappers (fused.py:58-82, sparse_ops.py:25-32,50-64); dispatch picks the
// tcgen05 kernels for 16-bit inputs on shapes they tile and the FP32 FFMA
// kernels otherwise.  There is no CPU path.
#include <stdio.h>

#include <string>

#include "dfss_common.cuh"
#include "tc_common.cuh"

namespace {

thread_local std::string g_last_error;

int fail(int status, const char* what) {
  g_last_error = what;
  return status;
}

int cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return DFSS_OK;
  g_last_error = std::string(cudaGetErrorName(e)) + ": " + cudaGetErrorString(e);
  return DFSS_ERR_CUDA;
}

bool valid_mode(int mode) { return mode == DFSS_MODE_1_2 || mode == DFSS_MODE_2_4; }
bool valid_dtype(int dt) { return dt == DFSS_F32 || dt == DFSS_BF16 || dt == DFSS_F16; }

int check_keep(const uint8_t* keep, int tile_rows, int tile_cols, int gs) {
  if (!keep) return DFSS_OK;
  if (tile_rows < 1 || tile_cols < 1) return fail(DFSS_ERR_INVALID, "tile dimensions must be >= 1");
  if (tile_cols % gs != 0) return fail(DFSS_ERR_INVALID, "tile columns not divisible by the group size");
  return DFSS_OK;
}

}  // namespace

extern "C" {

int dfss_version(void) { return 100; }

const char* dfss_status_string(int status) {
  switch (status) {
    case DFSS_OK: return "ok";
    case DFSS_ERR_INVALID: return "invalid argument";
    case DFSS_ERR_UNSUPPORTED: return "unsupported configuration";
    case DFSS_ERR_CUDA: return "CUDA error";
    case DFSS_ERR_NO_DEVICE: return "no sm_100 device";
    default: return "unknown status";
  }
}

const char* dfss_last_error(void) { return g_last_error.c_str(); }

int dfss_has_tcgen05(void) { return dfss::device_cc(dfss::current_device()) == 100 ? 1 : 0; }

int64_t dfss_meta_hw_words(int mode, int64_t bh, int64_t rows, int64_t cols) {
  if (!valid_mode(mode) || rows < 0 || cols < 0 || bh < 0) return -1;
  dfss::MetaGeom geo((int)rows, (int)(cols / mode));
  return bh * geo.words_per_bh();
}

int dfss_sddmm_prune(const void* q, const void* k, void* nonzeros, uint32_t* meta_hw, float scale, int mode,
                     int in_dtype, int nz_dtype, int math, int64_t bh, int n_q, int n_k, int d,
                     const uint8_t* tile_keep, int tile_rows, int tile_cols, float* scores_dbg, float* row_max,
                     void* stream) {
  if (!valid_mode(mode)) return fail(DFSS_ERR_INVALID, "unknown sparsity mode (expected 2 or 4)");
  if (!valid_dtype(in_dtype) || !valid_dtype(nz_dtype)) return fail(DFSS_ERR_INVALID, "unknown dtype");
  if (bh < 0 || n_q < 1 || n_k < 1 || d < 1) return fail(DFSS_ERR_INVALID, "shape dimensions must be positive");
  if (n_k % mode != 0) return fail(DFSS_ERR_INVALID, "score columns not group-aligned for the mode");
  if (int st = check_keep(tile_keep, tile_rows, tile_cols, mode)) return st;
  if (!q || !k || !nonzeros || !meta_hw) return fail(DFSS_ERR_INVALID, "null tensor pointer");
  cudaStream_t s = (cudaStream_t)stream;
  // (block masks on tcgen05 too: masked groups written absent in the epilogue; row maxima unmasked only)
  const bool tc_ok = (!tile_keep || !row_max) && dfss::tc_sddmm_supported(mode, in_dtype, nz_dtype, n_q, n_k, d) &&
                     dfss_has_tcgen05();
  if (math == DFSS_MATH_TF32) {
    if (in_dtype != DFSS_F32 || !tc_ok) return fail(DFSS_ERR_UNSUPPORTED, "tf32 path needs fp32 inputs on a tiled shape");
    return cuda_status(dfss::launch_sddmm_tc(q, k, nonzeros, meta_hw, scale, mode, in_dtype, bh, n_q, n_k, d,
                                             scores_dbg, row_max, s, tile_keep, tile_rows, tile_cols));
  }
  if (math == DFSS_MATH_AUTO && in_dtype != DFSS_F32 && tc_ok)
    return cuda_status(dfss::launch_sddmm_tc(q, k, nonzeros, meta_hw, scale, mode, in_dtype, bh, n_q, n_k, d,
                                             scores_dbg, row_max, s, tile_keep, tile_rows, tile_cols));
  if (row_max) return fail(DFSS_ERR_UNSUPPORTED, "row_max is produced by the tcgen05 SDDMM only");
  return cuda_status(dfss::launch_sddmm_simt(q, k, nonzeros, meta_hw, scale, mode, in_dtype, nz_dtype, bh, n_q, n_k,
                                             d, tile_keep, tile_rows, tile_cols, scores_dbg, s));
}

int dfss_softmax_rows(const void* nz_in, void* p_out, int in_dtype, int out_dtype, int64_t bh, int rows, int nz_cols,
                      const uint8_t* tile_keep, int tile_rows, int tile_cols, int32_t* err_row, void* stream) {
  if (!valid_dtype(in_dtype) || !valid_dtype(out_dtype)) return fail(DFSS_ERR_INVALID, "unknown dtype");
  if (bh < 0 || rows < 1 || nz_cols < 1) return fail(DFSS_ERR_INVALID, "shape dimensions must be positive");
  if (tile_keep && (tile_rows < 1 || tile_cols < 2 || tile_cols % 2))
    return fail(DFSS_ERR_INVALID, "tile_cols must be even to map tiles onto nonzeros");
  if (nz_in == p_out && in_dtype != out_dtype) return fail(DFSS_ERR_INVALID, "in-place softmax needs equal dtypes");
  if (!nz_in || !p_out) return fail(DFSS_ERR_INVALID, "null tensor pointer");
  return cuda_status(dfss::launch_softmax(nz_in, p_out, in_dtype, out_dtype, bh, rows, nz_cols, tile_keep, tile_rows,
                                          tile_cols, err_row, (cudaStream_t)stream));
}

int dfss_spmm(const void* p, const uint32_t* meta_hw, const void* v, void* out, int mode, int p_dtype, int v_dtype,
              int out_dtype, int64_t bh, int rows, int n_k, int d, const uint8_t* tile_keep, int tile_rows,
              int tile_cols, const float* row_max, void* stream) {
  if (!valid_mode(mode)) return fail(DFSS_ERR_INVALID, "unknown sparsity mode (expected 2 or 4)");
  if (!valid_dtype(p_dtype) || !valid_dtype(v_dtype) || !valid_dtype(out_dtype))
    return fail(DFSS_ERR_INVALID, "unknown dtype");
  if (bh < 0 || rows < 1 || n_k < 1 || d < 1) return fail(DFSS_ERR_INVALID, "shape dimensions must be positive");
  if (n_k % mode != 0) return fail(DFSS_ERR_INVALID, "dense columns not divisible by the group size");
  if (int st = check_keep(tile_keep, tile_rows, tile_cols, mode)) return st;
  if (!p || !meta_hw || !v || !out) return fail(DFSS_ERR_INVALID, "null tensor pointer");
  cudaStream_t s = (cudaStream_t)stream;
  // block masks on the tcgen05 path too: its transform warps zero the absent nonzeros in shared memory
  if ((!tile_keep || !row_max) && dfss::tc_spmm_supported(mode, p_dtype, v_dtype, out_dtype, rows, n_k, d) &&
      dfss_has_tcgen05())
    return cuda_status(dfss::launch_spmm_tc(p, meta_hw, v, out, mode, p_dtype, out_dtype, bh, rows, n_k, d, row_max, s,
                                            tile_keep, tile_rows, tile_cols));
  if (row_max && tile_keep) return fail(DFSS_ERR_UNSUPPORTED, "fused softmax SpMM is unmasked-only");
  if (row_max) return fail(DFSS_ERR_UNSUPPORTED, "fused softmax SpMM needs the tcgen05 path (2:4 or 1:2, 16-bit, d=64)");
  if (d > 256) return fail(DFSS_ERR_UNSUPPORTED, "head dim > 256 not supported by the FFMA SpMM");
  return cuda_status(dfss::launch_spmm_simt(p, meta_hw, v, out, mode, p_dtype, v_dtype, out_dtype, bh, rows, n_k, d,
                                            tile_keep, tile_rows, tile_cols, s));
}

// exact-FP32 attention (math auto) with the SpMM on tcgen05 as 3xTF32: 1:2, d = 64, n % 128 == 0
// -- from ~1 M scores (bh * n^2) up: its four launches run as a programmatic-dependent chain
// (tools/time_f32_sizes.py / bench: c1, 12 x 384^2 = 1.8 M: 0.0275 vs 0.0375 ms with the FFMA pair;
// 24 x 384^2: 0.026 vs 0.049 ms; 96 x 384^2: 0.066 vs 0.156 ms); tiny problems keep the pair
#ifndef DFSS_X3_MIN_SCORES
#define DFSS_X3_MIN_SCORES (1 << 20)
#endif
static bool exact_f32_on_tc(int mode, int dtype, int math, int64_t bh, int n, int d) {
  return math == DFSS_MATH_AUTO && dtype == DFSS_F32 && mode == 2 && bh * (int64_t)n * n >= DFSS_X3_MIN_SCORES &&
         dfss::tc_spmm_tf32x3_supported(2, n, n, d) && dfss::tc_sddmm_tf32x3_supported(2, n, n, d) &&
         dfss_has_tcgen05();
}
// its workspace beyond the staged buffers: V^T hi / lo (SpMM), then Q / K hi / lo (SDDMM)
static int64_t exact_f32_tc_extra_bytes(int64_t bh, int n) {
  return dfss::spmm_tf32x3_workspace_bytes(bh, n) + dfss::sddmm_tf32x3_workspace_bytes(bh, n, n);
}

int64_t dfss_nm_attention_workspace_bytes_for(int mode, int dtype, int math, int64_t bh, int n, int d,
                                              int tile_rows, int tile_cols, int masked) {
  if (!valid_mode(mode) || !valid_dtype(dtype) || bh < 0 || n < 1 || d < 1) return -1;
  const bool mask_ok = !masked || dfss::tc_flash_mask_supported(tile_rows, tile_cols);
  if (math == DFSS_MATH_AUTO && dtype != DFSS_F32 && dfss::tc_flash_supported(mode, dtype, n, d) && mask_ok &&
      dfss_has_tcgen05())
    // fused: no n x n intermediate in HBM -- mask bitmaps, or the split last round's partial O
    return masked ? dfss::flash_mask_workspace_bytes(n) : dfss::flash_split_workspace_bytes(bh, n);
  if (math == DFSS_MATH_TF32 && dtype == DFSS_F32 && dfss::tc_flash_tf32_supported(mode, n, d) &&
      (!masked || (mask_ok && dfss::flash_mask_two_set_ok(n))) && dfss_has_tcgen05())
    return dfss::flash_tf32_workspace_bytes(bh, n, masked);  // V^T (K-major tf32 B) + mask bitmaps
  const int64_t staged = dfss_nm_attention_workspace_bytes(mode, dtype, bh, n, d);
  if (!masked && exact_f32_on_tc(mode, dtype, math, bh, n, d))
    return staged + exact_f32_tc_extra_bytes(bh, n);  // + the 3xTF32 kernels' split operands
  return staged;
}

int64_t dfss_nm_attention_workspace_bytes(int mode, int dtype, int64_t bh, int n, int d) {
  (void)d;
  if (!valid_mode(mode) || !valid_dtype(dtype) || bh < 0 || n < 1) return -1;
  const int64_t nz = bh * (int64_t)n * (n / 2) * dfss::dtype_bytes(dtype);
  const int64_t meta = dfss_meta_hw_words(mode, bh, n, n) * 4;
  return (nz + 255) / 256 * 256 + (meta + 255) / 256 * 256 + bh * (int64_t)n * 4 * 4 + 256;
}

int dfss_nm_attention(const void* q, const void* k, const void* v, void* out, int mode, int dtype, int math,
                      int64_t bh, int n, int d, void* workspace, int64_t workspace_bytes, void* stream) {
  return dfss_nm_attention_masked(q, k, v, out, mode, dtype, math, bh, n, d, nullptr, 0, 0, workspace,
                                  workspace_bytes, stream);
}

}  // extern "C"

namespace {

enum Path { kFused16 = 1, kFusedTf32 = 2, kStagedTc = 3, kStagedFfma = 4, kStagedMasked = 5, kStaged3xTf32 = 6 };

// The path dfss_nm_attention(_masked) takes (no launch).  Validation is the caller's.
int attention_path(int mode, int dtype, int math, int64_t bh, int n, int d, bool masked, int tile_rows, int tile_cols) {
  const bool tc = dfss_has_tcgen05() != 0;
  if (math == DFSS_MATH_AUTO && dtype != DFSS_F32 && dfss::tc_flash_supported(mode, dtype, n, d) &&
      (!masked || dfss::tc_flash_mask_supported(tile_rows, tile_cols)) && tc)
    return kFused16;
  if (math == DFSS_MATH_TF32 && dtype == DFSS_F32 && dfss::tc_flash_tf32_supported(mode, n, d) &&
      (!masked || (dfss::tc_flash_mask_supported(tile_rows, tile_cols) && dfss::flash_mask_two_set_ok(n))) && tc)
    return kFusedTf32;
  if (math == DFSS_MATH_TF32) return DFSS_ERR_UNSUPPORTED;
  if (masked) return kStagedMasked;
  if (math == DFSS_MATH_AUTO && dtype != DFSS_F32 && dfss::tc_sddmm_supported(mode, dtype, dtype, n, n, d) &&
      dfss::tc_spmm_supported(mode, dtype, dtype, dtype, n, n, d) && tc)
    return kStagedTc;
  if (exact_f32_on_tc(mode, dtype, math, bh, n, d)) return kStaged3xTf32;
  return kStagedFfma;
}

int nm_attention_impl(const void* q, const void* k, const void* v, void* out, int mode, int dtype, int math,
                      int64_t bh, int n, int d, const uint8_t* tile_keep, int tile_rows, int tile_cols,
                      void* workspace, int64_t workspace_bytes, void* stream, float* dump_s, uint32_t* dump_meta,
                      int* dump_meta_mode) {
  if (!valid_mode(mode)) return fail(DFSS_ERR_INVALID, "unknown sparsity mode (expected 2 or 4)");
  if (!valid_dtype(dtype)) return fail(DFSS_ERR_INVALID, "unknown dtype");
  if (bh < 0 || n < 1 || d < 1) return fail(DFSS_ERR_INVALID, "shape dimensions must be positive");
  if (n % mode != 0) return fail(DFSS_ERR_INVALID, "sequence length not group-aligned for the mode");
  if (int st = check_keep(tile_keep, tile_rows, tile_cols, mode)) return st;
  const int64_t need =
      dfss_nm_attention_workspace_bytes_for(mode, dtype, math, bh, n, d, tile_rows, tile_cols, tile_keep != nullptr);
  if (need > 0 && (!workspace || workspace_bytes < need)) return fail(DFSS_ERR_INVALID, "workspace too small");
  const int path = attention_path(mode, dtype, math, bh, n, d, tile_keep != nullptr, tile_rows, tile_cols);
  if (path < 0) return fail(DFSS_ERR_UNSUPPORTED, "tf32 attention needs fp32 inputs, mode 1:2, d = 64 and n % 128 == 0");
  const bool dumping = dump_s != nullptr;
  if (dumping && !dump_meta) return fail(DFSS_ERR_INVALID, "dump needs both score and metadata buffers");
  if (dump_meta_mode) *dump_meta_mode = path == kFused16 ? DFSS_MODE_2_4 : mode;
  if (bh == 0) return DFSS_OK;
  const int64_t nz_bytes = bh * (int64_t)n * (n / 2) * dfss::dtype_bytes(dtype);
  const int64_t meta_bytes = dfss_meta_hw_words(mode, bh, n, n) * 4;
  char* ws = (char*)workspace;
  void* nz = ws;
  uint32_t* meta = (uint32_t*)(ws + (nz_bytes + 255) / 256 * 256);
  float* row_max = (float*)(ws + (nz_bytes + 255) / 256 * 256 + (meta_bytes + 255) / 256 * 256);
  const float scale = 1.0f / sqrtf((float)d);
  cudaStream_t s = (cudaStream_t)stream;
  switch (path) {
    case kFused16:  // fully fused: one kernel, no n x n tensor in HBM (flash_tc.cu); 32-aligned block masks
      if (dumping)
        return cuda_status(dfss::launch_flash_tc_dump(q, k, v, out, scale, mode, dtype, bh, n, d, tile_keep,
                                                      tile_rows, tile_cols, workspace, dump_s, dump_meta, s));
      return cuda_status(dfss::launch_flash_tc(q, k, v, out, scale, mode, dtype, bh, n, d, tile_keep, tile_rows,
                                               tile_cols, workspace, s));
    case kFusedTf32:  // tf32 1:2 on fp32 inputs (configs[4] "1:2 tf32"); V^T in the workspace
      return cuda_status(dfss::launch_flash_tf32(q, k, v, out, scale, bh, n, d, tile_keep, tile_rows, tile_cols,
                                                 workspace, s, dump_s, dump_meta));
    default: break;
  }
  // staged: the dump is the SDDMM's post-scale score hook plus a copy of its metadata
  if (tile_keep) {
    // the mask threaded through every stage (fused.py:73-82, sparse_ops.py:27-30,57-64)
    int st = dfss_sddmm_prune(q, k, nz, meta, scale, mode, dtype, dtype, math, bh, n, n, d, tile_keep, tile_rows,
                              tile_cols, dump_s, nullptr, stream);
    if (!st && dumping) st = cuda_status(cudaMemcpyAsync(dump_meta, meta, meta_bytes, cudaMemcpyDeviceToDevice, s));
    if (st) return st;
    st = dfss_softmax_rows(nz, nz, dtype, dtype, bh, n, n / 2, tile_keep, tile_rows, tile_cols, nullptr, stream);
    if (st) return st;
    // the masked softmax wrote exact zeros for every absent nonzero and nm_attention's V is finite
    // (the reference's DenseMatrix rejects NaN / Inf, dense.py:34-35), so the unmasked tcgen05
    // SpMM gives what skipping them gives
    if (dfss::tc_spmm_supported(mode, dtype, dtype, dtype, n, n, d) && dfss_has_tcgen05())
      return cuda_status(dfss::launch_spmm_tc(nz, meta, v, out, mode, dtype, dtype, bh, n, n, d, nullptr, s));
    return dfss_spmm(nz, meta, v, out, mode, dtype, dtype, dtype, bh, n, n, d, tile_keep, tile_rows, tile_cols,
                     nullptr, stream);
  }
  const int64_t staged_bytes = dfss_nm_attention_workspace_bytes(mode, dtype, bh, n, d);
  const bool x3_aligned = (((uintptr_t)q | (uintptr_t)k | (uintptr_t)v | (uintptr_t)out) & 15) == 0;
  if (path == kStaged3xTf32 && x3_aligned) {  // (workspace checked above; unaligned views: the FFMA pair)
    // exact FP32 (math auto) on tcgen05 as 3xTF32: scores + 1:2 prune + row maxima (sddmm_tf32.cu), SpMM
    // with the row softmax fused (spmm_tf32.cu); fp32-accurate, selection bit-exact on the dumped scores
    char* x3 = ws + staged_bytes;
    char* x3_qk = x3 + dfss::spmm_tf32x3_workspace_bytes(bh, n);
    // split Q / K, split V^T (alongside), SDDMM, SpMM: each a programmatic dependent of the last
    int st = cuda_status(dfss::launch_split_tf32x3((const float*)q, (const float*)k, bh, n, n, x3_qk, s));
    if (!st) st = cuda_status(dfss::launch_vt_split_tf32x3((const float*)v, bh, n, x3, s));
    if (!st)
      st = cuda_status(dfss::launch_sddmm_tf32x3((const float*)q, (const float*)k, (float*)nz, meta, scale, bh, n, n,
                                                 dump_s, row_max, x3_qk, s));
    if (!st && dumping) st = cuda_status(cudaMemcpyAsync(dump_meta, meta, meta_bytes, cudaMemcpyDeviceToDevice, s));
    if (st) return st;
    // the row softmax fused into the SpMM: exp of (score - the SDDMM's row maximum), row sums divided out
    return cuda_status(
        dfss::launch_spmm_tf32x3((const float*)nz, meta, (const float*)v, (float*)out, bh, n, n, row_max, x3, s));
  }
  // SDDMM+prune (+row max) -> SpMM with the softmax applied to the staged P tiles
  const bool fused = path == kStagedTc;
  int st = dfss_sddmm_prune(q, k, nz, meta, scale, mode, dtype, dtype, math, bh, n, n, d, nullptr, 0, 0, dump_s,
                            fused ? row_max : nullptr, stream);
  if (!st && dumping) st = cuda_status(cudaMemcpyAsync(dump_meta, meta, meta_bytes, cudaMemcpyDeviceToDevice, s));
  if (st) return st;
  if (fused)
    return dfss_spmm(nz, meta, v, out, mode, dtype, dtype, dtype, bh, n, n, d, nullptr, 0, 0, row_max, stream);
  if (dtype == DFSS_F32 && d <= 64)  // exact FP32: softmax fused into the SIMT SpMM (one pass less)
    return cuda_status(dfss::launch_spmm_simt_softmax_f32(nz, meta, v, out, mode, bh, n, n, d, s));
  st = dfss_softmax_rows(nz, nz, dtype, dtype, bh, n, n / 2, nullptr, 0, 0, nullptr, stream);
  if (st) return st;
  return dfss_spmm(nz, meta, v, out, mode, dtype, dtype, dtype, bh, n, n, d, nullptr, 0, 0, nullptr, stream);
}

}  // namespace

extern "C" {

int dfss_nm_attention_masked(const void* q, const void* k, const void* v, void* out, int mode, int dtype, int math,
                             int64_t bh, int n, int d, const uint8_t* tile_keep, int tile_rows, int tile_cols,
                             void* workspace, int64_t workspace_bytes, void* stream) {
  return nm_attention_impl(q, k, v, out, mode, dtype, math, bh, n, d, tile_keep, tile_rows, tile_cols, workspace,
                           workspace_bytes, stream, nullptr, nullptr, nullptr);
}

int dfss_nm_attention_dump(const void* q, const void* k, const void* v, void* out, int mode, int dtype, int math,
                           int64_t bh, int n, int d, const uint8_t* tile_keep, int tile_rows, int tile_cols,
                           void* workspace, int64_t workspace_bytes, float* scores_dbg, uint32_t* meta_dbg,
                           int* meta_mode, void* stream) {
  if (!scores_dbg || !meta_dbg) return fail(DFSS_ERR_INVALID, "null dump buffer");
  return nm_attention_impl(q, k, v, out, mode, dtype, math, bh, n, d, tile_keep, tile_rows, tile_cols, workspace,
                           workspace_bytes, stream, scores_dbg, meta_dbg, meta_mode);
}

int dfss_nm_attention_path(int mode, int dtype, int math, int n, int d, int tile_rows, int tile_cols, int masked) {
  return dfss_nm_attention_path_bh(mode, dtype, math, 1, n, d, tile_rows, tile_cols, masked);
}

int dfss_nm_attention_path_bh(int mode, int dtype, int math, int64_t bh, int n, int d, int tile_rows, int tile_cols,
                              int masked) {
  if (!valid_mode(mode) || !valid_dtype(dtype) || bh < 0 || n < 1 || d < 1) return DFSS_ERR_INVALID;
  return attention_path(mode, dtype, math, bh, n, d, masked != 0, tile_rows, tile_cols);
}

int dfss_prune_scores(const float* scores, void* nonzeros, uint8_t* meta_logical, uint8_t* kept, int mode,
                      int nz_dtype, int64_t rows, int cols, void* stream) {
  if (!valid_mode(mode)) return fail(DFSS_ERR_INVALID, "unknown sparsity mode (expected 2 or 4)");
  if (!valid_dtype(nz_dtype)) return fail(DFSS_ERR_INVALID, "unknown dtype");
  if (rows < 0 || cols < 0 || cols % mode) return fail(DFSS_ERR_INVALID, "column count not divisible by group size");
  if (!scores) return fail(DFSS_ERR_INVALID, "null tensor pointer");
  return cuda_status(
      dfss::launch_prune_scores(scores, nonzeros, meta_logical, kept, mode, nz_dtype, rows, cols, (cudaStream_t)stream));
}

int dfss_meta_hw_to_logical(const uint32_t* meta_hw, uint8_t* meta_logical, int mode, int64_t bh, int rows, int cols,
                            void* stream) {
  if (!valid_mode(mode) || rows < 0 || cols < 0 || cols % mode || bh < 0)
    return fail(DFSS_ERR_INVALID, "invalid metadata geometry");
  if (!meta_hw || !meta_logical) return fail(DFSS_ERR_INVALID, "null tensor pointer");
  return cuda_status(dfss::launch_meta_hw_to_logical(meta_hw, meta_logical, mode, bh, rows, cols, (cudaStream_t)stream));
}

int dfss_meta_logical_to_hw(const uint8_t* meta_logical, uint32_t* meta_hw, int mode, int64_t bh, int rows, int cols,
                            void* stream) {
  if (!valid_mode(mode) || rows < 0 || cols < 0 || cols % mode || bh < 0)
    return fail(DFSS_ERR_INVALID, "invalid metadata geometry");
  if (!meta_hw || !meta_logical) return fail(DFSS_ERR_INVALID, "null tensor pointer");
  return cuda_status(dfss::launch_meta_logical_to_hw(meta_logical, meta_hw, mode, bh, rows, cols, (cudaStream_t)stream));
}

// ---------------------------------------------------------------- reference kernel module (float64)

int dfss_kmod_sddmm_compress(const double* q, const double* k, double scale, int group_size, int n, int m, int d,
                             int tile_rows, int tile_cols, const uint8_t* keep, double* nonzeros, uint8_t* meta,
                             void* stream) {
  if (group_size != 2 && group_size != 4) return fail(DFSS_ERR_INVALID, "group size must be 2 or 4");
  if (n < 0 || m < 0 || d < 0) return fail(DFSS_ERR_INVALID, "shape dimensions must be non-negative");
  if (m % group_size) return fail(DFSS_ERR_INVALID, "score columns not group-aligned for the mode");
  if (tile_rows < 1 || tile_cols < 1 || tile_cols % group_size)
    return fail(DFSS_ERR_INVALID, "tile columns must be a positive multiple of the group size");
  if ((n && m && (!q || !k || !keep)) || !nonzeros || !meta) return fail(DFSS_ERR_INVALID, "null tensor pointer");
  return cuda_status(dfss::launch_kmod_sddmm_compress(q, k, scale, group_size, n, m, d, tile_rows, tile_cols, keep,
                                                      nonzeros, meta, (cudaStream_t)stream));
}

int dfss_kmod_softmax_nonzeros(const double* nz, const uint8_t* present, double* out, int64_t rows, int cols,
                               void* stream) {
  if (rows < 0 || cols < 0) return fail(DFSS_ERR_INVALID, "shape dimensions must be non-negative");
  if (rows && cols && (!nz || !out)) return fail(DFSS_ERR_INVALID, "null tensor pointer");
  return cuda_status(dfss::launch_kmod_softmax(nz, present, out, rows, cols, false, (cudaStream_t)stream));
}

int dfss_kmod_spmm_gather(const double* nz, const int64_t* cols, const uint8_t* present, const double* v,
                          double* out, int64_t rows, int nz_cols, int v_rows, int d, int32_t* err, void* stream) {
  if (rows < 0 || nz_cols < 0 || v_rows < 0 || d < 0) return fail(DFSS_ERR_INVALID, "shape dimensions must be non-negative");
  if (rows && d && (!out || (nz_cols && (!nz || !cols || !v)))) return fail(DFSS_ERR_INVALID, "null tensor pointer");
  return cuda_status(dfss::launch_kmod_spmm_gather(nz, cols, present, v, out, rows, nz_cols, v_rows, d, err,
                                                   (cudaStream_t)stream));
}

int dfss_kmod_gemm_abt(const double* a, const double* b, double scale, int64_t n, int64_t m, int kdim, double* out,
                       void* stream) {
  if (n < 0 || m < 0 || kdim < 0) return fail(DFSS_ERR_INVALID, "shape dimensions must be non-negative");
  if (n && m && (!out || (kdim && (!a || !b)))) return fail(DFSS_ERR_INVALID, "null tensor pointer");
  return cuda_status(dfss::launch_kmod_gemm_abt(a, b, scale, n, m, kdim, out, (cudaStream_t)stream));
}

int dfss_prune_scores_f64(const double* scores, double* nonzeros, uint8_t* meta_logical, uint8_t* kept, int mode,
                          int64_t rows, int cols, void* stream) {
  if (!valid_mode(mode)) return fail(DFSS_ERR_INVALID, "unknown sparsity mode (expected 2 or 4)");
  if (rows < 0 || cols < 0 || cols % mode) return fail(DFSS_ERR_INVALID, "column count not divisible by group size");
  if (rows && cols && !scores) return fail(DFSS_ERR_INVALID, "null tensor pointer");
  return cuda_status(dfss::launch_kmod_prune(scores, rows, cols, mode, nonzeros, meta_logical, kept,
                                             (cudaStream_t)stream));
}

int dfss_kmod_row_softmax_dense(const double* x, double* out, int64_t rows, int cols, void* stream) {
  if (rows < 0 || cols < 0) return fail(DFSS_ERR_INVALID, "shape dimensions must be non-negative");
  if (rows && cols && (!x || !out)) return fail(DFSS_ERR_INVALID, "null tensor pointer");
  return cuda_status(dfss::launch_kmod_softmax(x, nullptr, out, rows, cols, true, (cudaStream_t)stream));
}

}  // extern "C"
