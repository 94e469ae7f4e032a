// dfss_common.cuh -- shared device helpers for the DFSS sm_100a kernels:
// dtype conversion, the N:M selection rule, and the meta_hw word layout.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/dfss.h"

namespace dfss {

// ----------------------------------------------------------------------------
// dtype helpers

template <typename T>
struct DT;
template <>
struct DT<float> {
  static constexpr int id = DFSS_F32;
  __device__ __forceinline__ static float to_f(float x) { return x; }
  __device__ __forceinline__ static float from_f(float x) { return x; }
};
template <>
struct DT<__nv_bfloat16> {
  static constexpr int id = DFSS_BF16;
  __device__ __forceinline__ static float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
  __device__ __forceinline__ static __nv_bfloat16 from_f(float x) { return __float2bfloat16_rn(x); }
};
template <>
struct DT<__half> {
  static constexpr int id = DFSS_F16;
  __device__ __forceinline__ static float to_f(__half x) { return __half2float(x); }
  __device__ __forceinline__ static __half from_f(float x) { return __float2half_rn(x); }
};

inline int dtype_bytes(int dtype) { return dtype == DFSS_F32 ? 4 : 2; }

// ----------------------------------------------------------------------------
// N:M selection (codec.py:104-123, codec.py:289-313, _kernels_numba.py:145-184).
//
// Signed-value order with ties to the lower index.  2:4 uses the rank rule
//   rank_i = #{j : v_j > v_i} + #{j < i : v_j == v_i},  keep iff rank_i < 2,
// which is exactly "first two entries of a stable descending argsort"
// (codec.py:121) and the numba first-strict-max loops (:165-176).  Never the
// paper's pair-sum rule, which differs under fp32 ties.

// Nibble (lo | hi << 2) for each 4-bit kept mask with two bits set.
// mask 0b0011 -> 0x4, 0b0101 -> 0x8, 0b1001 -> 0xC, 0b0110 -> 0x9, 0b1010 -> 0xD, 0b1100 -> 0xE.
__device__ __forceinline__ uint32_t nibble_of_mask(uint32_t mask) {
  constexpr unsigned long long kTable = (0x4ull << (4 * 3)) | (0x8ull << (4 * 5)) | (0xCull << (4 * 9)) |
                                        (0x9ull << (4 * 6)) | (0xDull << (4 * 10)) | (0xEull << (4 * 12));
  return (uint32_t)(kTable >> (4 * mask)) & 0xFu;
}

// 2:4 select: returns the nibble, writes the kept values in ascending column order.
//
// Tournament form of the rank rule under the total order "i beats j iff
// v_i > v_j, or v_i == v_j and i < j": the pair winners w01 / w23 and losers
// l01 / l23 decide everything.  {0,1} survive iff l01 beats w23, {2,3} iff l23
// beats w01, otherwise {w01, w23}.  Every comparison puts the lower index on
// the left of >= (or the higher on the left of >), so ties resolve exactly as
// the reference's stable argsort (exhaustively checked over tie-heavy inputs,
// tests/test_gpu_parity.py).
//
// Cost model (the SDDMM epilogue is ALU-pipe bound): 4 FMNMX + 2 FSETP +
// 4 FSEL + 2 SEL on the ALU pipe; the "mixed" nibble (w01 idx) | (w23 idx) << 2
// comes from the sign bits of v0 - v1 and v2 - v3 on the FMA pipe
// (FADD + IMAD.HI by `two` == 2, a runtime value so the compiler cannot turn
// it into an ALU shift).  The sign trick needs canonical zeros (no -0.0):
// callers produce the inputs with fma(x, s, +0.0f) / x + 0.0f, which maps
// -0 to +0 -- equal values, identical ordering and ties.
__device__ __forceinline__ uint32_t sign_bit(float x, uint32_t two) { return __umulhi(__float_as_uint(x), two); }

__device__ __forceinline__ uint32_t select24(float v0, float v1, float v2, float v3, float& lo, float& hi,
                                             uint32_t two) {
  const float w01 = fmaxf(v0, v1), l01 = fminf(v0, v1);
  const float w23 = fmaxf(v2, v3), l23 = fminf(v2, v3);
  const bool keep01 = l01 >= w23;  // lower-index loser vs higher-index winner
  const bool keep23 = l23 > w01;   // higher-index loser must strictly beat the winner
  lo = keep01 ? v0 : (keep23 ? v2 : w01);
  hi = keep01 ? v1 : (keep23 ? v3 : w23);
  // w01 index = [v0 < v1], w23 index = 2 + [v2 < v3]  (ties keep the lower index)
  const uint32_t mixed = 8u + sign_bit(v0 - v1, two) + 4u * sign_bit(v2 - v3, two);
  uint32_t nib = keep23 ? 0xEu : mixed;
  nib = keep01 ? 0x4u : nib;
  return nib;
}

// Same, also folding the group's largest kept value (= max(w01, w23), the row
// maximum is always kept) into a running maximum: one extra 3-input FMNMX.
__device__ __forceinline__ uint32_t select24_max(float v0, float v1, float v2, float v3, float& lo, float& hi,
                                                 float& run_max, uint32_t two) {
  const float w01 = fmaxf(v0, v1), l01 = fminf(v0, v1);
  const float w23 = fmaxf(v2, v3), l23 = fminf(v2, v3);
  run_max = fmaxf(run_max, fmaxf(w01, w23));
  const bool keep01 = l01 >= w23;
  const bool keep23 = l23 > w01;
  lo = keep01 ? v0 : (keep23 ? v2 : w01);
  hi = keep01 ? v1 : (keep23 ? v3 : w23);
  const uint32_t mixed = 8u + sign_bit(v0 - v1, two) + 4u * sign_bit(v2 - v3, two);
  uint32_t nib = keep23 ? 0xEu : mixed;
  nib = keep01 ? 0x4u : nib;
  return nib;
}

// canonical-zero scaling used before every select: x*s + (+0) turns -0 into +0
__device__ __forceinline__ float scale_canon(float x, float s) {
  float y;
  asm("fma.rn.f32 %0, %1, %2, 0f00000000;" : "=f"(y) : "f"(x), "f"(s));
  return y;
}

// Reference rank rule (codec.py:121, kept for the self-check kernel in tests).
__device__ __forceinline__ uint32_t select24_rank(float v0, float v1, float v2, float v3) {
  const int r0 = (v1 > v0) + (v2 > v0) + (v3 > v0);
  const int r1 = (v0 >= v1) + (v2 > v1) + (v3 > v1);
  const int r2 = (v0 >= v2) + (v1 >= v2) + (v3 > v2);
  const int r3 = (v0 >= v3) + (v1 >= v3) + (v2 >= v3);
  return nibble_of_mask((uint32_t)(r0 < 2) | ((uint32_t)(r1 < 2) << 1) | ((uint32_t)(r2 < 2) << 2) |
                        ((uint32_t)(r3 < 2) << 3));
}

// 1:2 select: element 1 survives iff v1 > v0 (codec.py:114-117); 0x4 / 0xE.
__device__ __forceinline__ uint32_t select12(float v0, float v1, float& kept) {
  const bool second = v1 > v0;
  kept = second ? v1 : v0;
  return second ? 0xEu : 0x4u;
}

// Kept mask bits (bit i = element i of the group kept) from a nibble.
__device__ __forceinline__ uint32_t kept_bits(uint32_t nib, int gs) {
  if (gs == 2) return nib == 0xEu ? 2u : 1u;
  return (1u << (nib & 3u)) | (1u << ((nib >> 2) & 3u));
}

// ----------------------------------------------------------------------------
// meta_hw layout (dfss.h): words [bh][ceil(rows/128)][ceil(groups/8)][128].

constexpr uint32_t kPadNibble = 0x4u;

struct MetaGeom {
  int rows, groups;   // logical
  int rblocks, chunks;  // ceil(rows/128), ceil(groups/8)
  __host__ __device__ MetaGeom(int rows_, int groups_)
      : rows(rows_), groups(groups_), rblocks((rows_ + 127) / 128), chunks((groups_ + 7) / 8) {}
  __host__ __device__ int64_t words_per_bh() const { return (int64_t)rblocks * chunks * 128; }
  // word index (within one bh) and bit shift of the nibble of (row, group)
  __device__ __forceinline__ int64_t word_of(int row, int group, int& shift) const {
    const int rb = row >> 7, rr = row & 127;
    const int m2 = rr >> 4, m1 = (rr >> 3) & 1, m0 = rr & 7;
    const int c = group >> 3, gi = group & 7, k1 = gi >> 2, slot = gi & 3;
    shift = 16 * m1 + 4 * slot;
    return ((int64_t)rb * chunks + c) * 128 + (16 * m2 + 8 * k1 + m0);
  }
  // inverse: (rb, c, lane, nibble index 0..7 in the word) -> row, group
  __device__ __forceinline__ static void coords_of(int rb, int c, int lane, int idx, int& row, int& group) {
    const int m2 = lane >> 4, k1 = (lane >> 3) & 1, m0 = lane & 7;
    const int m1 = idx >> 2, slot = idx & 3;
    row = rb * 128 + 16 * m2 + 8 * m1 + m0;
    group = c * 8 + 4 * k1 + slot;
  }
};

}  // namespace dfss

// ----------------------------------------------------------------------------
// internal launchers (implemented in the .cu files, dispatched from capi.cu)

namespace dfss {
cudaError_t launch_sddmm_simt(const void* q, const void* k, void* nz, uint32_t* meta, float scale, int gs,
                              int in_dtype, int nz_dtype, int64_t bh, int n, int m, int d, const uint8_t* keep,
                              int tile_rows, int tile_cols, float* dbg, cudaStream_t s);
cudaError_t launch_softmax(const void* in, void* out, int in_dtype, int out_dtype, int64_t bh, int rows,
                           int cols, const uint8_t* keep, int tile_rows, int tile_cols, int32_t* err,
                           cudaStream_t s);
// fp32 SpMM with the row softmax fused (exact-FP32 nm_attention path, no mask, d <= 64)
cudaError_t launch_spmm_simt_softmax_f32(const void* p, const uint32_t* meta, const void* v, void* out, int gs,
                                        int64_t bh, int rows, int n_k, int d, cudaStream_t s);
cudaError_t launch_spmm_simt(const void* p, const uint32_t* meta, const void* v, void* out, int gs, int p_dtype,
                             int v_dtype, int out_dtype, int64_t bh, int rows, int n_k, int d, const uint8_t* keep,
                             int tile_rows, int tile_cols, cudaStream_t s);
cudaError_t launch_prune_scores(const float* scores, void* nz, uint8_t* meta, uint8_t* kept, int gs, int nz_dtype,
                                int64_t rows, int cols, cudaStream_t s);
cudaError_t launch_meta_hw_to_logical(const uint32_t* hw, uint8_t* logical, int gs, int64_t bh, int rows, int cols,
                                      cudaStream_t s);
cudaError_t launch_meta_logical_to_hw(const uint8_t* logical, uint32_t* hw, int gs, int64_t bh, int rows, int cols,
                                      cudaStream_t s);
// tcgen05 paths: return cudaErrorNotSupported when the shape is not covered.
cudaError_t launch_sddmm_tc(const void* q, const void* k, void* nz, uint32_t* meta, float scale, int gs,
                            int in_dtype, int64_t bh, int n, int m, int d, float* dbg, float* rowmax, cudaStream_t s,
                            const uint8_t* keep = nullptr, int tile_rows = 0, int tile_cols = 0);
// rowmax (nullable): [bh, rows, 2] partial row maxima from the SDDMM; when given, the SpMM
// applies softmax on the fly: P = exp(s - max) in smem, out = (P.V) / sum(P).
cudaError_t launch_spmm_tc(const void* p, const uint32_t* meta, const void* v, void* out, int gs, int dtype,
                           int out_dtype, int64_t bh, int rows, int n_k, int d, const float* rowmax, cudaStream_t s,
                           const uint8_t* keep = nullptr, int tile_rows = 0, int tile_cols = 0);
bool tc_sddmm_supported(int gs, int in_dtype, int nz_dtype, int n, int m, int d);
// fully fused attention (flash_tc.cu): no n x n tensor in HBM
bool tc_flash_supported(int gs, int dtype, int n, int d);
// tile_keep (nullable): BlockMask grid [ceil(n/tile_rows)][ceil(n/tile_cols)], uint8, shared by all bh;
// needs tile_rows % 32 == 0 and tile_cols % 32 == 0 (tc_flash_mask_supported)
bool tc_flash_mask_supported(int tile_rows, int tile_cols);
cudaError_t launch_flash_tc(const void* q, const void* k, const void* v, void* out, float scale, int gs, int dtype,
                            int64_t bh, int n, int d, const uint8_t* tile_keep, int tile_rows, int tile_cols,
                            void* workspace, cudaStream_t s);
// workspace of launch_flash_tc with a tile mask (liveness bitmaps); unmasked needs none
int64_t flash_mask_workspace_bytes(int n);
// unmasked fused 16-bit path: partial results of the split last round (flash_tc.cu SplitPlan)
int64_t flash_split_workspace_bytes(int64_t bh, int n);
// block-mask step skipping in the two-set fused kernels (flash_tc.cu): n % 256 == 0, n <= 32768
bool flash_mask_two_set_ok(int n);
int flash_mask_smem_bytes(int n);
struct TileMask;
// fills m's bitmap pointers (workspace of flash_mask_workspace_bytes(n)) and launches the
// two pre-kernels that build them on stream s
void prepare_mask_bits(TileMask& m, int n, void* workspace, cudaStream_t s);
bool tc_spmm_supported(int gs, int p_dtype, int v_dtype, int out_dtype, int rows, int n_k, int d);
// fp32 1:2 fused score + prune at fp32 accuracy on tcgen05 (3xTF32, sddmm_tf32.cu); workspace: Q / K hi / lo
bool tc_sddmm_tf32x3_supported(int gs, int n, int m, int d);
int64_t sddmm_tf32x3_workspace_bytes(int64_t bh, int n, int m);
cudaError_t launch_sddmm_tf32x3(const float* q, const float* k, float* nz, uint32_t* meta, float scale, int64_t bh,
                                int n, int m, float* dbg, float* rowmax, void* workspace, cudaStream_t s);
cudaError_t launch_split_tf32x3(const float* q, const float* k, int64_t bh, int n, int m, void* workspace,
                                cudaStream_t s);
cudaError_t launch_vt_split_tf32x3(const float* v, int64_t bh, int n_k, void* workspace, cudaStream_t s);
// fp32 1:2 SpMM at fp32 accuracy on tcgen05 (3xTF32, spmm_tf32.cu); workspace: V^T hi / lo
bool tc_spmm_tf32x3_supported(int gs, int rows, int n_k, int d);
int64_t spmm_tf32x3_workspace_bytes(int64_t bh, int n_k);
cudaError_t launch_spmm_tf32x3(const float* p, const uint32_t* meta, const float* v, float* out, int64_t bh, int rows,
                               int n_k, const float* rowmax, void* workspace, cudaStream_t s);
// fused 1:2 attention on fp32 inputs with tf32 tensor cores (flash_tf32.cu), n % 256 == 0, d = 64
bool tc_flash_tf32_supported(int gs, int n, int d);
// vt_scratch: flash_tf32_workspace_bytes of device scratch -- V^T (the kind::tf32 B operand
// must be K-major), then the block-mask bitmaps when tile_keep is given (n <= 32768)
int64_t flash_tf32_workspace_bytes(int64_t bh, int n, bool masked);
// dump_scores / dump_meta (both or neither): the DUMP kernel also stores the post-scale scores
// [bh, n, n] and the 1:2 metadata words (meta_hw layout) it fed to tcgen05.mma.sp
cudaError_t launch_flash_tf32(const void* q, const void* k, const void* v, void* out, float scale, int64_t bh, int n,
                              int d, const uint8_t* tile_keep, int tile_rows, int tile_cols, void* vt_scratch,
                              cudaStream_t s, float* dump_scores = nullptr, uint32_t* dump_meta = nullptr);
// launch_flash_tc with the DUMP kernels (flash_tc_dump.cu): post-scale scores [bh, n, n] fp32 and
// the metadata words in the 2:4 meta_hw layout (1:2 is run as the 2:4 pattern 8 + a + 4b)
cudaError_t launch_flash_tc_dump(const void* q, const void* k, const void* v, void* out, float scale, int gs,
                                 int dtype, int64_t bh, int n, int d, const uint8_t* tile_keep, int tile_rows,
                                 int tile_cols, void* workspace, float* dump_scores, uint32_t* dump_meta,
                                 cudaStream_t s);
// reference kernel module in float64 (kmod_f64.cu): bitwise the numba arithmetic (exp aside)
cudaError_t launch_kmod_sddmm_compress(const double* q, const double* k, double scale, int gs, int n, int m, int d,
                                       int tile_rows, int tile_cols, const uint8_t* keep, double* nonzeros,
                                       uint8_t* meta, cudaStream_t s);
cudaError_t launch_kmod_prune(const double* scores, int64_t rows, int cols, int gs, double* nonzeros, uint8_t* meta,
                              uint8_t* kept, cudaStream_t s);
cudaError_t launch_kmod_softmax(const double* x, const uint8_t* present, double* out, int64_t rows, int cols,
                                bool dense, cudaStream_t s);
cudaError_t launch_kmod_spmm_gather(const double* nz, const int64_t* cols, const uint8_t* present, const double* v,
                                    double* out, int64_t rows, int nzc, int v_rows, int d, int32_t* err,
                                    cudaStream_t s);
cudaError_t launch_kmod_gemm_abt(const double* a, const double* b, double scale, int64_t n, int64_t m, int kdim,
                                 double* out, cudaStream_t s);
}  // namespace dfss
