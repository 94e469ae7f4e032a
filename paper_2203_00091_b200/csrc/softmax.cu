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

#include <type_traits>

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
__global__ void __launch_bounds__(256, 2) softmax_rows_kernel(const TIn* __restrict__ in, TOut* __restrict__ out,
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

// Fast path: 16-bit in and out (same type), no tile mask, rows of NV * 256 nonzeros.  The row
// stays in registers PACKED (NV x 16 B per lane: 32 registers at 2048 nonzeros, so 3 CTAs of 8
// warps fit per SM and keep ~128 KB of loads in flight), the maximum is taken on packed pairs
// (exact in 16 bit), exp is recomputed in the normalising pass instead of cached as fp32 (MUFU has
// the headroom: 2 ex2 per element stay under the HBM time), and NaN detection costs nothing in
// the common case: a NaN input makes the row sum NaN, and only then is the row re-scanned to tell
// a NaN input (reference: ValueError) from an inf (reference: NaN output, no error).
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// the normalising pass recomputes exp: volatile, so the compiler cannot keep the first pass's
// values alive across the row-sum reduction instead (64 live floats: spills)
__device__ __forceinline__ float ex2_again(float f, float c, float nb) {  // exp2(f * c + nb)
  float y;
  asm volatile("{\n\t.reg .f32 t;\n\tfma.rn.f32 t, %1, %2, %3;\n\tex2.approx.ftz.f32 %0, t;\n\t}"
               : "=f"(y) : "f"(f), "f"(c), "f"(nb));
  return y;
}

// BlockMask on the fast path (MASK, tile_cols % 16 == 0: a lane's 8-nonzero vector = 16 dense
// columns lies in one tile): absent vectors become -inf before the maximum, so they contribute
// exp = 0 to the sum and are written as 0; a row without a present entry is flagged (err[0])
// and written as zeros, like softmax_rows_kernel.
struct SoftmaxKeep {
  const uint8_t* keep = nullptr;
  int rows = 1, tile_rows = 1, tile_cols = 16, grid_cols = 0;
};

template <typename T, int NV, int RW, bool MASK>
__global__ void __launch_bounds__(256, MASK && NV > 4 ? 2 : 3) softmax_rows16_kernel(const T* __restrict__ in, T* __restrict__ out,
                                                                int64_t total_rows, int cols,
                                                                int32_t* __restrict__ err, SoftmaxKeep mk) {
  using T2 = typename std::conditional<std::is_same<T, __half>::value, __half2, __nv_bfloat162>::type;
  constexpr float kLog2e = 1.4426950408889634f;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  auto f_lo = [](uint32_t u) -> float {
    if constexpr (std::is_same<T, __half>::value) return __half2float(__ushort_as_half((unsigned short)(u & 0xffffu)));
    else return __uint_as_float(u << 16);
  };
  auto f_hi = [](uint32_t u) -> float {
    if constexpr (std::is_same<T, __half>::value) return __half2float(__ushort_as_half((unsigned short)(u >> 16)));
    else return __uint_as_float(u & 0xffff0000u);
  };
  // RW rows per warp at a time (short rows: more loads in flight per warp)
  for (int64_t rg0 = warp * RW; rg0 < total_rows; rg0 += nwarps * RW) {
    uint4 pk[RW][NV];
#pragma unroll
    for (int q = 0; q < RW; ++q) {
      const uint4* x = reinterpret_cast<const uint4*>(in + (rg0 + q) * cols);
#pragma unroll
      for (int t = 0; t < NV; ++t) pk[q][t] = (rg0 + q < total_rows) ? __ldcs(x + lane + 32 * t) : make_uint4(0, 0, 0, 0);
    }
    bool empty[RW];
#pragma unroll
    for (int q = 0; q < RW; ++q) {
      empty[q] = false;
      if constexpr (MASK) {  // (every vector is read: predicating the loads on the tile lookups
                             // serialised them behind it, 0.80 -> 0.92 ms block-causal at c4)
        constexpr uint32_t kNegInf2 = std::is_same<T, __half>::value ? 0xFC00FC00u : 0xFF80FF80u;
        const uint8_t* krow = mk.keep + (int64_t)((int)((rg0 + q) % mk.rows) / mk.tile_rows) * mk.grid_cols;
        bool any = false;
#pragma unroll
        for (int t = 0; t < NV; ++t) {
          const bool pres = (rg0 + q < total_rows) && __ldg(krow + (16 * (lane + 32 * t)) / mk.tile_cols) != 0;
          any |= pres;
          if (!pres) pk[q][t] = make_uint4(kNegInf2, kNegInf2, kNegInf2, kNegInf2);
        }
        empty[q] = !__any_sync(0xffffffffu, any);
        if (empty[q] && lane == 0 && err && rg0 + q < total_rows) atomicMin(err, (int32_t)(rg0 + q + 1));
      }
    }
    float mb[RW], inv[RW];
#pragma unroll
    for (int q = 0; q < RW; ++q) {
      // max on packed pairs
      uint32_t m2u = pk[q][0].x;
#pragma unroll
      for (int t = 0; t < NV; ++t) {
        const uint32_t w[4] = {pk[q][t].x, pk[q][t].y, pk[q][t].z, pk[q][t].w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          T2 a = *reinterpret_cast<const T2*>(&m2u), c = *reinterpret_cast<const T2*>(&w[i]);
          a = __hmax2(a, c);
          m2u = *reinterpret_cast<uint32_t*>(&a);
        }
      }
      float mx = fmaxf(f_lo(m2u), f_hi(m2u));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      mb[q] = empty[q] ? 0.f : mx * kLog2e;
      float s0 = 0.f, s1 = 0.f;
#pragma unroll
      for (int t = 0; t < NV; ++t) {
        const uint32_t w[4] = {pk[q][t].x, pk[q][t].y, pk[q][t].z, pk[q][t].w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          s0 += ex2_approx(fmaf(f_lo(w[i]), kLog2e, -mb[q]));
          s1 += ex2_approx(fmaf(f_hi(w[i]), kLog2e, -mb[q]));
        }
      }
      float sum = s0 + s1;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      if (isnan(sum) && !empty[q]) {  // rare: a NaN input (flag it) or an inf (reference: NaN output, no error)
        bool nan_seen = false;
#pragma unroll
        for (int t = 0; t < NV; ++t) {
          const uint32_t w[4] = {pk[q][t].x, pk[q][t].y, pk[q][t].z, pk[q][t].w};
#pragma unroll
          for (int i = 0; i < 4; ++i) nan_seen |= isnan(f_lo(w[i])) || isnan(f_hi(w[i]));
        }
        if (__any_sync(0xffffffffu, nan_seen) && lane == 0 && err && rg0 + q < total_rows)
          atomicMin(err + 1, (int32_t)(rg0 + q + 1));
      }
      inv[q] = empty[q] ? 0.f : 1.0f / sum;
    }
#pragma unroll
    for (int q = 0; q < RW; ++q) {
      if (rg0 + q >= total_rows) break;
      uint4* y = reinterpret_cast<uint4*>(out + (rg0 + q) * cols);
#pragma unroll
      for (int t = 0; t < NV; ++t) {
        const uint32_t w[4] = {pk[q][t].x, pk[q][t].y, pk[q][t].z, pk[q][t].w};
        uint32_t o4[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float a = ex2_again(f_lo(w[i]), kLog2e, -mb[q]) * inv[q];
          const float c = ex2_again(f_hi(w[i]), kLog2e, -mb[q]) * inv[q];
          T2 p2;
          if constexpr (std::is_same<T, __half>::value) p2 = __floats2half2_rn(a, c);
          else p2 = __floats2bfloat162_rn(a, c);
          o4[i] = *reinterpret_cast<uint32_t*>(&p2);
        }
        __stcs(y + lane + 32 * t, make_uint4(o4[0], o4[1], o4[2], o4[3]));
      }
    }
  }
}

template <typename T, bool MASK>
static void softmax16_launch(const void* in, void* out, int64_t total, int cols, int32_t* err, const SoftmaxKeep& mk,
                             cudaStream_t s) {
  auto go = [&](auto kern, int rw) {
    int64_t blocks = (total + 8 * rw - 1) / (8 * rw);
    if (blocks > 148 * 3 * 4) blocks = 148 * 3 * 4;
    kern<<<(int)blocks, 256, 0, s>>>((const T*)in, (T*)out, total, cols, err, mk);
  };
  switch (cols / 256) {
    case 1: go(softmax_rows16_kernel<T, 1, 4, MASK>, 4); break;
    case 2: go(softmax_rows16_kernel<T, 2, 2, MASK>, 2); break;
    case 3: go(softmax_rows16_kernel<T, 3, 1, MASK>, 1); break;
    case 4: go(softmax_rows16_kernel<T, 4, 1, MASK>, 1); break;
    case 5: go(softmax_rows16_kernel<T, 5, 1, MASK>, 1); break;
    case 6: go(softmax_rows16_kernel<T, 6, 1, MASK>, 1); break;
    case 7: go(softmax_rows16_kernel<T, 7, 1, MASK>, 1); break;
    default: go(softmax_rows16_kernel<T, 8, 1, MASK>, 1); break;
  }
}

template <typename T>
static bool softmax16_fast(const void* in, void* out, int64_t bh, int rows, int cols, const uint8_t* keep, int tr,
                           int tc, int32_t* err, cudaStream_t s, cudaError_t* e) {
  if (cols % 256 || cols > 2048 || ((uintptr_t)in | (uintptr_t)out) % 16) return false;
  if (keep && (tc % 16 || tr < 1)) return false;  // a lane's 8-nonzero vector must lie in one tile
  const int64_t total = bh * rows;
  SoftmaxKeep mk;
  if (keep) {
    mk.keep = keep;
    mk.rows = rows;
    mk.tile_rows = tr;
    mk.tile_cols = tc;
    mk.grid_cols = (2 * cols + tc - 1) / tc;
    softmax16_launch<T, true>(in, out, total, cols, err, mk, s);
  } else {
    softmax16_launch<T, false>(in, out, total, cols, err, mk, s);
  }
  *e = cudaGetLastError();
  return true;
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
  if constexpr (std::is_same<TIn, TOut>::value && !std::is_same<TIn, float>::value) {
    cudaError_t e;
    if (softmax16_fast<TIn>(in, out, bh, rows, cols, keep, tr, tc, err, s, &e)) return e;
  }
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
