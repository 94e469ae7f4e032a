// meta_prune.cu -- parity hook (prune a given fp32 score tensor with the
// epilogue's own select routine) and meta_hw <-> logical conversions.
#include "dfss_common.cuh"

namespace dfss {

// One thread per group.  Mirrors codec._select_rows (codec.py:289-313):
// nonzeros [rows, cols/2], logical nibbles [rows, cols/gs], kept mask [rows, cols].
template <typename TNz, int GS>
__global__ void prune_scores_kernel(const float* __restrict__ scores, TNz* __restrict__ nz,
                                    uint8_t* __restrict__ meta, uint8_t* __restrict__ kept, int64_t rows,
                                    int cols, uint32_t two) {
  const int groups = cols / GS;
  const int64_t total = rows * groups;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / groups;
    const int g = (int)(t % groups);
    const float* s = scores + r * cols + (int64_t)g * GS;
    uint32_t nib;
    if (GS == 4) {
      float lo, hi;
      // same routine as the SDDMM epilogue; +0 canonicalises -0 (equal values, same ties)
      nib = select24(scale_canon(s[0], 1.f), scale_canon(s[1], 1.f), scale_canon(s[2], 1.f), scale_canon(s[3], 1.f),
                     lo, hi, two);
      if (nz) {
        nz[r * (cols / 2) + 2 * g] = DT<TNz>::from_f(lo);
        nz[r * (cols / 2) + 2 * g + 1] = DT<TNz>::from_f(hi);
      }
    } else {
      float kv;
      nib = select12(s[0], s[1], kv);
      if (nz) nz[r * (cols / 2) + g] = DT<TNz>::from_f(kv);
    }
    if (meta) meta[t] = (uint8_t)nib;
    if (kept) {
      const uint32_t kb = kept_bits(nib, GS);
#pragma unroll
      for (int i = 0; i < GS; ++i) kept[r * cols + (int64_t)g * GS + i] = (uint8_t)((kb >> i) & 1u);
    }
  }
}

template <int GS>
static cudaError_t prune_dispatch(const float* scores, void* nz, uint8_t* meta, uint8_t* kept, int nz_dtype,
                                  int64_t rows, int cols, cudaStream_t s) {
  const int64_t total = rows * (cols / GS);
  const int threads = 256;
  const int blocks = (int)((total + threads - 1) / threads < 148 * 16 ? (total + threads - 1) / threads : 148 * 16);
  if (blocks == 0) return cudaSuccess;
  switch (nz_dtype) {
    case DFSS_F32:
      prune_scores_kernel<float, GS><<<blocks, threads, 0, s>>>(scores, (float*)nz, meta, kept, rows, cols, 2u);
      break;
    case DFSS_BF16:
      prune_scores_kernel<__nv_bfloat16, GS>
          <<<blocks, threads, 0, s>>>(scores, (__nv_bfloat16*)nz, meta, kept, rows, cols, 2u);
      break;
    default:
      prune_scores_kernel<__half, GS><<<blocks, threads, 0, s>>>(scores, (__half*)nz, meta, kept, rows, cols, 2u);
  }
  return cudaGetLastError();
}

cudaError_t launch_prune_scores(const float* scores, void* nz, uint8_t* meta, uint8_t* kept, int gs, int nz_dtype,
                                int64_t rows, int cols, cudaStream_t s) {
  return gs == 4 ? prune_dispatch<4>(scores, nz, meta, kept, nz_dtype, rows, cols, s)
                 : prune_dispatch<2>(scores, nz, meta, kept, nz_dtype, rows, cols, s);
}

// One thread per (row, group): logical[bh][row][group] = nibble.
__global__ void meta_hw_to_logical_kernel(const uint32_t* __restrict__ hw, uint8_t* __restrict__ logical, int64_t bh,
                                          MetaGeom geo) {
  const int64_t per = (int64_t)geo.rows * geo.groups;
  const int64_t total = bh * per;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = t / per;
    const int64_t rem = t % per;
    const int row = (int)(rem / geo.groups), group = (int)(rem % geo.groups);
    int shift;
    const int64_t w = geo.word_of(row, group, shift);
    logical[t] = (uint8_t)((hw[b * geo.words_per_bh() + w] >> shift) & 0xFu);
  }
}

// One thread per word: gathers the 8 nibbles, padding with 0x4.
__global__ void meta_logical_to_hw_kernel(const uint8_t* __restrict__ logical, uint32_t* __restrict__ hw, int64_t bh,
                                          MetaGeom geo) {
  const int64_t per = geo.words_per_bh();
  const int64_t total = bh * per;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = t / per;
    int64_t rem = t % per;
    const int lane = (int)(rem & 127);
    rem >>= 7;
    const int c = (int)(rem % geo.chunks), rb = (int)(rem / geo.chunks);
    uint32_t word = 0;
#pragma unroll
    for (int idx = 0; idx < 8; ++idx) {
      int row, group;
      MetaGeom::coords_of(rb, c, lane, idx, row, group);
      uint32_t nib = kPadNibble;
      if (row < geo.rows && group < geo.groups)
        nib = logical[(b * geo.rows + row) * (int64_t)geo.groups + group] & 0xFu;
      word |= nib << (16 * (idx >> 2) + 4 * (idx & 3));
    }
    hw[t] = word;
  }
}

static int grid_for(int64_t total, int threads) {
  int64_t b = (total + threads - 1) / threads;
  return (int)(b < 148 * 32 ? b : 148 * 32);
}

cudaError_t launch_meta_hw_to_logical(const uint32_t* hw, uint8_t* logical, int gs, int64_t bh, int rows, int cols,
                                      cudaStream_t s) {
  MetaGeom geo(rows, cols / gs);
  const int64_t total = bh * rows * (int64_t)(cols / gs);
  if (total == 0) return cudaSuccess;
  meta_hw_to_logical_kernel<<<grid_for(total, 256), 256, 0, s>>>(hw, logical, bh, geo);
  return cudaGetLastError();
}

cudaError_t launch_meta_logical_to_hw(const uint8_t* logical, uint32_t* hw, int gs, int64_t bh, int rows, int cols,
                                      cudaStream_t s) {
  MetaGeom geo(rows, cols / gs);
  const int64_t total = bh * geo.words_per_bh();
  if (total == 0) return cudaSuccess;
  meta_logical_to_hw_kernel<<<grid_for(total, 256), 256, 0, s>>>(logical, hw, bh, geo);
  return cudaGetLastError();
}

}  // namespace dfss
