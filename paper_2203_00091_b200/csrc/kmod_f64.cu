// kmod_f64.cu -- the reference's kernel-module interface on the GPU, in float64.
//
// The reference dispatches its hot loops through a duck-typed kernel module (backend.kernels(),
// backend.py:63-67) with five functions; _kernels_numba.py implements them in float64 with
// fastmath off and one running accumulator per output, ascending in the reduction index.  These
// kernels implement the same five functions with the same arithmetic: every product and every
// sum is a separately rounded __dmul_rn / __dadd_rn (no FMA contraction) in the reference's
// order, so sddmm_compress, spmm_gather and gemm_abt are bitwise equal to the numba kernels, and
// the two softmaxes differ only through exp (CUDA's double exp vs libm, <= 1 ulp) -- their sums
// are sequential in column order like the reference's.
//
// This is the exact-semantics drop-in for a maintainer who plugs a CUDA backend into the
// reference (integration/_kernels_cuda.py); the production attention path is the fused sm_100a
// kernels (flash_tc.cu, flash_tf32.cu), which never materialise what these take as arguments.
#include "dfss_common.cuh"

namespace dfss {

namespace {

// sddmm_compress (_kernels_numba.py:110-185): one thread per (row, group).  A group lies in one
// tile (tile_cols % group_size == 0, validated by fused.py:64-69), so the tile-keep test is per
// group; masked tiles are left as the caller's zeros (nonzeros 0, metadata 0), as in the
// reference, which never writes them.
template <int GS>
__global__ void __launch_bounds__(256) kmod_sddmm_compress_kernel(const double* __restrict__ q,
                                                                  const double* __restrict__ k, double scale, int n,
                                                                  int m, int d, int tile_rows, int tile_cols,
                                                                  const uint8_t* __restrict__ keep, int grid_cols,
                                                                  double* __restrict__ nonzeros,
                                                                  uint8_t* __restrict__ meta) {
  const int groups = m / GS;
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)n * groups) return;
  const int row = (int)(idx / groups), g = (int)(idx % groups), col0 = g * GS;
  if (!keep[(int64_t)(row / tile_rows) * grid_cols + col0 / tile_cols]) return;
  double v[GS];
#pragma unroll
  for (int t = 0; t < GS; ++t) {
    const double* qr = q + (int64_t)row * d;
    const double* kr = k + (int64_t)(col0 + t) * d;
    double acc = 0.0;  // tile[a, b] = 0.0; tile[a, b] += qv * kmat[j0 + b, k] for ascending k
    for (int kk = 0; kk < d; ++kk) acc = __dadd_rn(acc, __dmul_rn(qr[kk], kr[kk]));
    v[t] = __dmul_rn(acc, scale);  // tile[a, b] = tile[a, b] * scale
  }
  if (GS == 2) {  // :145-158 -- element 1 iff strictly greater
    const bool second = v[1] > v[0];
    nonzeros[(int64_t)row * (m / 2) + g] = second ? v[1] : v[0];
    meta[(int64_t)row * groups + g] = second ? 0xE : 0x4;
  } else {  // :159-184 -- first strict maximum, then the first strict maximum of the rest
    int best = 0;
    for (int t = 1; t < 4; ++t)
      if (v[t] > v[best]) best = t;
    int second = -1;
    for (int t = 0; t < 4; ++t) {
      if (t == best) continue;
      if (second < 0 || v[t] > v[second]) second = t;
    }
    const int lo = best < second ? best : second, hi = best < second ? second : best;
    nonzeros[(int64_t)row * (m / 2) + 2 * g] = v[lo];
    nonzeros[(int64_t)row * (m / 2) + 2 * g + 1] = v[hi];
    meta[(int64_t)row * groups + g] = (uint8_t)(lo | (hi << 2));
  }
}

// selection on given float64 scores (codec.py:289-313 -- the same rule as the fused epilogue
// above): one thread per (row, group); any output may be null
template <int GS>
__global__ void __launch_bounds__(256) kmod_prune_kernel(const double* __restrict__ scores, int64_t rows, int cols,
                                                         double* __restrict__ nonzeros, uint8_t* __restrict__ meta,
                                                         uint8_t* __restrict__ kept) {
  const int groups = cols / GS;
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= rows * groups) return;
  const int64_t row = idx / groups;
  const int g = (int)(idx % groups);
  const double* v = scores + row * cols + (int64_t)g * GS;
  int lo, hi;
  if (GS == 2) {
    lo = hi = v[1] > v[0] ? 1 : 0;
  } else {
    int best = 0;
    for (int t = 1; t < 4; ++t)
      if (v[t] > v[best]) best = t;
    int second = -1;
    for (int t = 0; t < 4; ++t) {
      if (t == best) continue;
      if (second < 0 || v[t] > v[second]) second = t;
    }
    lo = best < second ? best : second;
    hi = best < second ? second : best;
  }
  if (GS == 2) {
    if (nonzeros) nonzeros[row * (cols / 2) + g] = v[lo];
    if (meta) meta[row * groups + g] = lo ? 0xE : 0x4;
    if (kept) {
      kept[row * cols + 2 * g] = lo == 0;
      kept[row * cols + 2 * g + 1] = lo == 1;
    }
  } else {
    if (nonzeros) {
      nonzeros[row * (cols / 2) + 2 * g] = v[lo];
      nonzeros[row * (cols / 2) + 2 * g + 1] = v[hi];
    }
    if (meta) meta[row * groups + g] = (uint8_t)(lo | (hi << 2));
    if (kept)
      for (int t = 0; t < 4; ++t) kept[row * cols + 4 * g + t] = (t == lo || t == hi);
  }
}

// softmax_nonzeros (_kernels_numba.py:66-84) and row_softmax_dense (:43-59): one warp per row.
// The maximum is order independent (computed by the warp); the exponentials are independent
// (computed by the warp); the sum is sequential in column order (lane 0), as the reference's
// `s += e`; absent slots are 0.  DENSE: the max starts at x[0] and every entry is present.
template <bool DENSE>
__global__ void __launch_bounds__(256) kmod_softmax_kernel(const double* __restrict__ x,
                                                           const uint8_t* __restrict__ present,
                                                           double* __restrict__ out, int64_t rows, int cols) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < rows; r += nwarps) {
    const double* xr = x + r * cols;
    const uint8_t* pr = present ? present + r * cols : nullptr;
    double* orow = out + r * cols;
    double mx = DENSE ? xr[0] : -INFINITY;
    for (int j = lane; j < cols; j += 32)
      if ((DENSE || !pr || pr[j]) && xr[j] > mx) mx = xr[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    for (int j = lane; j < cols; j += 32) orow[j] = (DENSE || !pr || pr[j]) ? exp(__dsub_rn(xr[j], mx)) : 0.0;
    __syncwarp();
    double s = 0.0;
    if (lane == 0)
      for (int j = 0; j < cols; ++j)
        if (DENSE || !pr || pr[j]) s = __dadd_rn(s, orow[j]);
    s = __shfl_sync(0xffffffffu, s, 0);
    __syncwarp();
    for (int j = lane; j < cols; j += 32)
      if (DENSE || !pr || pr[j]) orow[j] = __ddiv_rn(orow[j], s);
  }
}

// spmm_gather (_kernels_numba.py:91-103): one warp per row, lanes over the d output columns;
// out[i, j] += val * v[col, j] for ascending nonzero index c, absent slots skipped.  A column
// index outside [0, v_rows) is skipped and flagged in *err (the reference indexes out of bounds).
__global__ void __launch_bounds__(256) kmod_spmm_gather_kernel(const double* __restrict__ nz,
                                                               const int64_t* __restrict__ cols,
                                                               const uint8_t* __restrict__ present,
                                                               const double* __restrict__ v, double* __restrict__ out,
                                                               int64_t rows, int nzc, int v_rows, int d,
                                                               int32_t* __restrict__ err) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < rows; r += nwarps) {
    for (int j0 = 0; j0 < d; j0 += 32) {
      const int j = j0 + lane;
      double acc = 0.0;
      for (int c = 0; c < nzc; ++c) {
        if (present && !present[r * nzc + c]) continue;
        const int64_t col = cols[r * nzc + c];
        if (col < 0 || col >= v_rows) {
          if (err && lane == 0) atomicMin(err, (int32_t)(r < INT32_MAX ? r : INT32_MAX - 1));
          continue;
        }
        if (j < d) acc = __dadd_rn(acc, __dmul_rn(nz[r * nzc + c], v[col * d + j]));
      }
      if (j < d) out[r * d + j] = acc;
    }
  }
}

// gemm_abt (_kernels_numba.py:16-36): out[i, j] = (sum_k a[i, k] b[j, k], ascending k) * scale.
// The reference's tiles and k panels only reorder the traversal: each element still has one
// running accumulator over ascending k.  16 x 16 outputs per block; a and b panels through smem.
__global__ void __launch_bounds__(256) kmod_gemm_abt_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                                            double scale, int64_t n, int64_t m, int kdim,
                                                            double* __restrict__ out) {
  __shared__ double as[16][17], bs[16][17];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t i = blockIdx.y * 16 + ty, j = blockIdx.x * 16 + tx;
  double acc = 0.0;
  for (int k0 = 0; k0 < kdim; k0 += 16) {
    const int64_t ai = blockIdx.y * 16 + ty, bj = blockIdx.x * 16 + ty;
    as[ty][tx] = (ai < n && k0 + tx < kdim) ? a[ai * kdim + k0 + tx] : 0.0;
    bs[ty][tx] = (bj < m && k0 + tx < kdim) ? b[bj * kdim + k0 + tx] : 0.0;
    __syncthreads();
    const int kk_end = kdim - k0 < 16 ? kdim - k0 : 16;
    for (int kk = 0; kk < kk_end; ++kk) acc = __dadd_rn(acc, __dmul_rn(as[ty][kk], bs[tx][kk]));
    __syncthreads();
  }
  if (i < n && j < m) out[i * m + j] = __dmul_rn(acc, scale);
}

int grid_warps(int64_t rows) {
  const int64_t blocks = (rows + 7) / 8;
  return (int)(blocks < 148 * 32 ? (blocks > 0 ? blocks : 1) : 148 * 32);
}

}  // namespace

cudaError_t launch_kmod_sddmm_compress(const double* q, const double* k, double scale, int gs, int n, int m, int d,
                                       int tile_rows, int tile_cols, const uint8_t* keep, double* nonzeros,
                                       uint8_t* meta, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(nonzeros, 0, (size_t)n * (m / 2) * sizeof(double), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(meta, 0, (size_t)n * (m / gs), s);
  if (e != cudaSuccess || n == 0 || m == 0) return e;
  const int grid_cols = (m + tile_cols - 1) / tile_cols;
  const int64_t threads = (int64_t)n * (m / gs);
  const unsigned blocks = (unsigned)((threads + 255) / 256);
  if (gs == 2)
    kmod_sddmm_compress_kernel<2><<<blocks, 256, 0, s>>>(q, k, scale, n, m, d, tile_rows, tile_cols, keep, grid_cols,
                                                         nonzeros, meta);
  else
    kmod_sddmm_compress_kernel<4><<<blocks, 256, 0, s>>>(q, k, scale, n, m, d, tile_rows, tile_cols, keep, grid_cols,
                                                         nonzeros, meta);
  return cudaGetLastError();
}

cudaError_t launch_kmod_prune(const double* scores, int64_t rows, int cols, int gs, double* nonzeros, uint8_t* meta,
                              uint8_t* kept, cudaStream_t s) {
  const int64_t threads = rows * (cols / gs);
  if (threads == 0) return cudaSuccess;
  const unsigned blocks = (unsigned)((threads + 255) / 256);
  if (gs == 2)
    kmod_prune_kernel<2><<<blocks, 256, 0, s>>>(scores, rows, cols, nonzeros, meta, kept);
  else
    kmod_prune_kernel<4><<<blocks, 256, 0, s>>>(scores, rows, cols, nonzeros, meta, kept);
  return cudaGetLastError();
}

cudaError_t launch_kmod_softmax(const double* x, const uint8_t* present, double* out, int64_t rows, int cols,
                                bool dense, cudaStream_t s) {
  if (rows == 0 || cols == 0) return cudaSuccess;
  if (dense)
    kmod_softmax_kernel<true><<<grid_warps(rows), 256, 0, s>>>(x, nullptr, out, rows, cols);
  else
    kmod_softmax_kernel<false><<<grid_warps(rows), 256, 0, s>>>(x, present, out, rows, cols);
  return cudaGetLastError();
}

cudaError_t launch_kmod_spmm_gather(const double* nz, const int64_t* cols, const uint8_t* present, const double* v,
                                    double* out, int64_t rows, int nzc, int v_rows, int d, int32_t* err,
                                    cudaStream_t s) {
  if (rows == 0 || d == 0) return cudaSuccess;
  kmod_spmm_gather_kernel<<<grid_warps(rows), 256, 0, s>>>(nz, cols, present, v, out, rows, nzc, v_rows, d, err);
  return cudaGetLastError();
}

cudaError_t launch_kmod_gemm_abt(const double* a, const double* b, double scale, int64_t n, int64_t m, int kdim,
                                 double* out, cudaStream_t s) {
  if (n == 0 || m == 0) return cudaSuccess;
  if (kdim == 0) return cudaMemsetAsync(out, 0, (size_t)(n * m) * sizeof(double), s);
  for (int64_t i0 = 0; i0 < n; i0 += 16 * 65535) {  // gridDim.y <= 65535 row tiles per launch
    const int64_t nn = n - i0 < 16 * 65535 ? n - i0 : 16 * 65535;
    const dim3 grid((unsigned)((m + 15) / 16), (unsigned)((nn + 15) / 16));
    kmod_gemm_abt_kernel<<<grid, 256, 0, s>>>(a + i0 * kdim, b, scale, nn, m, kdim, out + i0 * m);
  }
  return cudaGetLastError();
}

}  // namespace dfss
