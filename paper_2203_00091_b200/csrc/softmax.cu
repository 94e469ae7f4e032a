// softmax.cu -- stable softmax over each compressed row's present nonzeros.
//
// Replaces _softmax_nonzeros (_kernels_numba.py:66-84): pass 1 max over
// present entries, pass 2 sum of exp(x - max), pass 3 normalise; absent
// entries (block-masked tiles) are written as 0.  One warp per row, the row
// held in registers (16-byte vector loads) when it fits, so HBM sees exactly
// one read and one write of the row.  exp is computed as exp2(x*log2e - m*log2e).
// Empty rows and NaN are flagged on the device (err[0] / err[1] = 1 + first
// flattened row, atomicMin, caller initialises to INT32_MAX) so the host can
// raise the reference's ValueError (sparse_ops.py:27-32) after the fact.
#include <math_constants.h>

#include "dfss_common.cuh"

namespace dfss {

template <typename T, int VEC>
struct Vec;
template <typename T>
struct Vec<T, 1> {
  T v[1];
};
template <typename T, int VEC>
struct __align__(16) Vec {
  T v[VEC];
};

template <typename TIn, typename TOut, int VEC, int NV>
__global__ void __launch_bounds__(256) softmax_rows_kernel(const TIn* __restrict__ in, TOut* __restrict__ out,
                                                           int64_t total_rows, int rows, int cols,
                                                           const uint8_t* __restrict__ keep, int tile_rows,
                                                           int tile_cols, int32_t* __restrict__ err) {
  constexpr float kLog2e = 1.4426950408889634f;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int grid_cols = keep ? (2 * cols + tile_cols - 1) / tile_cols : 0;
  const int nvec = cols / VEC;  // cols % VEC == 0 by dispatch

  for (int64_t rg = warp; rg < total_rows; rg += nwarps) {
    const TIn* x = in + rg * cols;
    TOut* y = out + rg * cols;
    const int r = (int)(rg % rows);
    const uint8_t* keep_row = keep ? keep + (int64_t)(r / tile_rows) * grid_cols : nullptr;
    auto present = [&](int j) -> bool { return !keep_row || keep_row[(2 * j) / tile_cols]; };

    float mx = -CUDART_INF_F;
    bool nan_seen = false;
    float cache[NV > 0 ? NV * VEC : 1];
    // pass 1: max
    if (NV > 0) {
#pragma unroll
      for (int t = 0; t < NV; ++t) {
        const int vi = lane + 32 * t;
        Vec<TIn, VEC> pk;
        if (vi < nvec) pk = reinterpret_cast<const Vec<TIn, VEC>*>(x)[vi];
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          const int j = vi * VEC + e;
          float f = -CUDART_INF_F;
          if (vi < nvec && present(j)) {
            f = DT<TIn>::to_f(pk.v[e]);
            nan_seen |= isnan(f);
          }
          cache[t * VEC + e] = f;
          mx = fmaxf(mx, f);
        }
      }
    } else {
      for (int vi = lane; vi < nvec; vi += 32) {
        const Vec<TIn, VEC> pk = reinterpret_cast<const Vec<TIn, VEC>*>(x)[vi];
#pragma unroll
        for (int e = 0; e < VEC; ++e)
          if (present(vi * VEC + e)) {
            const float f = DT<TIn>::to_f(pk.v[e]);
            nan_seen |= isnan(f);
            mx = fmaxf(mx, f);
          }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    nan_seen = __any_sync(0xffffffffu, nan_seen);
    const bool empty = (mx == -CUDART_INF_F);
    if (lane == 0 && err) {
      if (empty) atomicMin(err, (int32_t)(rg + 1));
      if (nan_seen) atomicMin(err + 1, (int32_t)(rg + 1));
    }
    const float mb = empty ? 0.f : mx * kLog2e;

    // pass 2: sum of exp
    float s = 0.f;
    if (NV > 0) {
#pragma unroll
      for (int t = 0; t < NV * VEC; ++t) {
        const float e = (cache[t] == -CUDART_INF_F) ? 0.f : exp2f(fmaf(cache[t], kLog2e, -mb));
        cache[t] = e;
        s += e;
      }
    } else {
      for (int vi = lane; vi < nvec; vi += 32) {
        const Vec<TIn, VEC> pk = reinterpret_cast<const Vec<TIn, VEC>*>(x)[vi];
#pragma unroll
        for (int e = 0; e < VEC; ++e)
          if (present(vi * VEC + e)) s += exp2f(fmaf(DT<TIn>::to_f(pk.v[e]), kLog2e, -mb));
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float inv = empty ? 0.f : 1.0f / s;

    // pass 3: normalise and store (absent entries -> 0)
    if (NV > 0) {
#pragma unroll
      for (int t = 0; t < NV; ++t) {
        const int vi = lane + 32 * t;
        if (vi < nvec) {
          Vec<TOut, VEC> pk;
#pragma unroll
          for (int e = 0; e < VEC; ++e) pk.v[e] = DT<TOut>::from_f(cache[t * VEC + e] * inv);
          reinterpret_cast<Vec<TOut, VEC>*>(y)[vi] = pk;
        }
      }
    } else {
      for (int vi = lane; vi < nvec; vi += 32) {
        const Vec<TIn, VEC> pk = reinterpret_cast<const Vec<TIn, VEC>*>(x)[vi];
        Vec<TOut, VEC> po;
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          const float f = present(vi * VEC + e) ? exp2f(fmaf(DT<TIn>::to_f(pk.v[e]), kLog2e, -mb)) * inv : 0.f;
          po.v[e] = DT<TOut>::from_f(f);
        }
        reinterpret_cast<Vec<TOut, VEC>*>(y)[vi] = po;
      }
    }
  }
}

template <typename TIn, typename TOut, int VEC>
static cudaError_t softmax_vec(const void* in, void* out, int64_t bh, int rows, int cols, const uint8_t* keep,
                               int tr, int tc, int32_t* err, cudaStream_t s) {
  const int64_t total = bh * rows;
  const int threads = 256;
  int64_t blocks = (total + 7) / 8;
  if (blocks > 148 * 64) blocks = 148 * 64;
  const int per_lane = (cols + 32 * VEC - 1) / (32 * VEC);  // vectors per lane
  auto go = [&](auto kern) {
    kern<<<(int)blocks, threads, 0, s>>>((const TIn*)in, (TOut*)out, total, rows, cols, keep, tr, tc, err);
  };
  if (per_lane <= 1)
    go(softmax_rows_kernel<TIn, TOut, VEC, 1>);
  else if (per_lane <= 2)
    go(softmax_rows_kernel<TIn, TOut, VEC, 2>);
  else if (per_lane <= 4)
    go(softmax_rows_kernel<TIn, TOut, VEC, 4>);
  else if (per_lane <= 8 && VEC * 8 <= 64)
    go(softmax_rows_kernel<TIn, TOut, VEC, (VEC * 8 <= 64 ? 8 : 4)>);
  else
    go(softmax_rows_kernel<TIn, TOut, VEC, 0>);
  return cudaGetLastError();
}

template <typename TIn, typename TOut>
static cudaError_t softmax_typed(const void* in, void* out, int64_t bh, int rows, int cols, const uint8_t* keep,
                                 int tr, int tc, int32_t* err, cudaStream_t s) {
  constexpr int V = 16 / (sizeof(TIn) > sizeof(TOut) ? sizeof(TIn) : sizeof(TOut));
  const bool aligned = (cols % V == 0) && ((uintptr_t)in % 16 == 0) && ((uintptr_t)out % 16 == 0);
  if (aligned) return softmax_vec<TIn, TOut, V>(in, out, bh, rows, cols, keep, tr, tc, err, s);
  return softmax_vec<TIn, TOut, 1>(in, out, bh, rows, cols, keep, tr, tc, err, s);
}

template <typename TIn>
static cudaError_t softmax_in(const void* in, void* out, int out_dtype, int64_t bh, int rows, int cols,
                              const uint8_t* keep, int tr, int tc, int32_t* err, cudaStream_t s) {
  switch (out_dtype) {
    case DFSS_F32: return softmax_typed<TIn, float>(in, out, bh, rows, cols, keep, tr, tc, err, s);
    case DFSS_BF16: return softmax_typed<TIn, __nv_bfloat16>(in, out, bh, rows, cols, keep, tr, tc, err, s);
    default: return softmax_typed<TIn, __half>(in, out, bh, rows, cols, keep, tr, tc, err, s);
  }
}

cudaError_t launch_softmax(const void* in, void* out, int in_dtype, int out_dtype, int64_t bh, int rows, int cols,
                           const uint8_t* keep, int tile_rows, int tile_cols, int32_t* err, cudaStream_t s) {
  if (bh == 0 || rows == 0 || cols == 0) return cudaSuccess;
  switch (in_dtype) {
    case DFSS_F32: return softmax_in<float>(in, out, out_dtype, bh, rows, cols, keep, tile_rows, tile_cols, err, s);
    case DFSS_BF16:
      return softmax_in<__nv_bfloat16>(in, out, out_dtype, bh, rows, cols, keep, tile_rows, tile_cols, err, s);
    default: return softmax_in<__half>(in, out, out_dtype, bh, rows, cols, keep, tile_rows, tile_cols, err, s);
  }
}

}  // namespace dfss
