// spmm_simt.cu -- generic compressed SpMM on FP32 FFMA: out = decompress(P) . V.
//
// Replaces _spmm_gather (_kernels_numba.py:91-103): for every row, the
// stored nonzeros are visited in ascending order and out[i,:] += p * V[col,:],
// where the dense column comes from the nibble in meta_hw (the decode of
// codec.nonzero_columns, codec.py:346-360, done in registers).  One warp per
// output row; each lane decodes one nonzero of a 32-wide batch, the batch is
// broadcast by shuffles, lanes own output columns lane + 32*t.
// This is the exact-FP32 path (c1 at 1e-5) and the fallback for shapes the
// tcgen05.mma.sp kernel does not tile.
#include <type_traits>
#include <cstdlib>

#include "dfss_common.cuh"

namespace dfss {

// SM: the row softmax (softmax_rows, sparse_ops.py:18-37) fused in: the warp first reduces the
// row's max and sum of exp over its nonzeros, then weights each nonzero by exp(x - max) and
// scales the output row by 1 / sum (no mask; the exact-FP32 nm_attention path).
template <typename TP, typename TV, typename TO, int GS, int DPER, bool SM = false>
__global__ void __launch_bounds__(256, 4) spmm_simt_kernel(const TP* __restrict__ p, const uint32_t* __restrict__ meta,
                                                        const TV* __restrict__ v, TO* __restrict__ out,
                                                        int64_t total_rows, int rows, int n_k, int d,
                                                        const uint8_t* __restrict__ keep, int tile_rows,
                                                        int tile_cols, MetaGeom geo) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int nzc = n_k / 2;
  const int grid_cols = keep ? (n_k + tile_cols - 1) / tile_cols : 0;

  for (int64_t rg = warp; rg < total_rows; rg += nwarps) {
    const int64_t b = rg / rows;
    const int r = (int)(rg % rows);
    const TP* prow = p + rg * nzc;
    const uint32_t* mb = meta + b * geo.words_per_bh();
    const TV* vb = v + b * (int64_t)n_k * d;
    float acc[DPER];
#pragma unroll
    for (int t = 0; t < DPER; ++t) acc[t] = 0.f;
    constexpr float kLog2e = 1.4426950408889634f;
    float mlb = 0.f, inv = 1.f;
    if (SM) {
      float mx = -INFINITY;
      for (int j = lane; j < nzc; j += 32) mx = fmaxf(mx, DT<TP>::to_f(prow[j]));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      mlb = mx * kLog2e;
      float sum = 0.f;
      for (int j = lane; j < nzc; j += 32) sum += exp2f(fmaf(DT<TP>::to_f(prow[j]), kLog2e, -mlb));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      inv = 1.0f / sum;
    }

    for (int j0 = 0; j0 < nzc; j0 += 32) {
      const int j = j0 + lane;
      float pv = 0.f;
      int col = -1;  // -1: absent (masked tile) -- skipped, as the reference skips it (_kernels_numba.py:98)
      if (j < nzc) {
        const int g = (GS == 4) ? (j >> 1) : j;
        int shift;
        const uint32_t nib = (mb[geo.word_of(r, g, shift)] >> shift) & 0xFu;
        col = (GS == 4) ? 4 * g + (int)((j & 1) ? ((nib >> 2) & 3u) : (nib & 3u)) : 2 * g + (nib == 0xEu ? 1 : 0);
        pv = DT<TP>::to_f(prow[j]);
        if (SM) pv = exp2f(fmaf(pv, kLog2e, -mlb));
        if (keep && !keep[(int64_t)(r / tile_rows) * grid_cols + col / tile_cols]) col = -1;
      }
      const int cnt = min(32, nzc - j0);
      // unrolled so the V-row loads of several nonzeros are in flight together (the loop was
      // latency-bound: one dependent L2 load chain per warp)
#pragma unroll 8
      for (int l = 0; l < cnt; ++l) {
        const float pl = __shfl_sync(0xffffffffu, pv, l);
        const int cl = __shfl_sync(0xffffffffu, col, l);
        if (cl < 0) continue;  // warp-uniform
        const TV* vr = vb + (int64_t)cl * d;
#pragma unroll
        for (int t = 0; t < DPER; ++t) {
          const int c = lane + 32 * t;
          if (c < d) acc[t] = fmaf(pl, DT<TV>::to_f(vr[c]), acc[t]);
        }
      }
    }
    TO* orow = out + rg * d;
#pragma unroll
    for (int t = 0; t < DPER; ++t) {
      const int c = lane + 32 * t;
      if (c < d) orow[c] = DT<TO>::from_f(SM ? acc[t] * inv : acc[t]);
    }
  }
}

// Tiled generic variant (d == 64, n_k % 128 == 0): a CTA owns 32 rows of one (batch, head) and
// streams V through shared memory (converted to fp32) in 128-key tiles, so every V row is read
// from L2 once per CTA instead of once per nonzero -- the warp-per-row kernel above re-reads a
// 128-byte V row per nonzero and is L2-bound at long rows (c4 1:2: 48 ms).  The nonzeros of a
// row inside a 128-key tile are the contiguous range [k0 / 2, k0 / 2 + 64) for either mode.
// Absent nonzeros (BlockMask) point at an all-zero V row and weigh 0: skipped, as the reference
// skips them (_kernels_numba.py:98) -- no 0 * Inf.  Accumulation stays in ascending order.
template <typename TP, typename TV, typename TO, int GS>
__global__ void __launch_bounds__(256) spmm_tiled_kernel(const TP* __restrict__ p, const uint32_t* __restrict__ meta,
                                                         const TV* __restrict__ v, TO* __restrict__ out, int rows,
                                                         int n_k, const uint8_t* __restrict__ keep, int tile_rows,
                                                         int tile_cols, MetaGeom geo) {
  constexpr int RB = 32, KT = 128, NZT = KT / 2;
  constexpr int VE = 16 / sizeof(TV);  // V elements per 16-byte load
  __shared__ __align__(16) float Vs[KT + 1][64];
  __shared__ float Ps[RB][NZT + 1];
  __shared__ uint8_t Cs[RB][NZT];
  const int b = blockIdx.y, row0 = blockIdx.x * RB;
  const int nzc = n_k / 2;
  const int grid_cols = keep ? (n_k + tile_cols - 1) / tile_cols : 0;
  const TP* pb = p + ((int64_t)b * rows) * nzc;
  const uint32_t* mb = meta + (int64_t)b * geo.words_per_bh();
  const uint4* vb = reinterpret_cast<const uint4*>(v + (int64_t)b * n_k * 64);
  if (threadIdx.x < 64) Vs[KT][threadIdx.x] = 0.f;
  // output row; columns 4cb .. 4cb+3 and 32+4cb .. 32+4cb+3: the 8 threads of a row read two
  // contiguous 128-byte halves of the V row (one shared-memory wavefront each) -- an 8-column
  // block per thread read them at a 32-byte stride (twice the wavefronts)
  const int orow = threadIdx.x >> 3, cb = threadIdx.x & 7;
  float acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.f;
  for (int k0 = 0; k0 < n_k; k0 += KT) {
#pragma unroll
    for (int i = 0; i < (KT * 64 / VE) / 256; ++i) {
      const int idx = threadIdx.x + 256 * i;  // 16-byte unit of the [128][64] tile
      const uint4 u = vb[(int64_t)k0 * (64 / VE) + idx];
      const TV* e = reinterpret_cast<const TV*>(&u);
      float* dst = &Vs[0][0] + idx * VE;
#pragma unroll
      for (int j = 0; j < VE; ++j) dst[j] = DT<TV>::to_f(e[j]);
    }
#pragma unroll
    for (int i = 0; i < (RB * NZT) / 256; ++i) {
      const int idx = threadIdx.x + 256 * i;
      const int rr = idx / NZT, jl = idx % NZT;
      const int r = row0 + rr, j = k0 / 2 + jl;
      float w = 0.f;
      int col = KT;  // the zero row: rows past the end, absent nonzeros
      if (r < rows) {
        const int g = (GS == 4) ? (j >> 1) : j;
        int shift;
        const uint32_t nib = (mb[geo.word_of(r, g, shift)] >> shift) & 0xFu;
        const int c = (GS == 4) ? 4 * g + (int)((j & 1) ? ((nib >> 2) & 3u) : (nib & 3u)) : 2 * g + (nib == 0xEu ? 1 : 0);
        if (!keep || keep[(int64_t)(r / tile_rows) * grid_cols + c / tile_cols]) {
          w = DT<TP>::to_f(pb[(int64_t)r * nzc + j]);
          col = c - k0;
        }
      }
      Ps[rr][jl] = w;
      Cs[rr][jl] = (uint8_t)col;
    }
    __syncthreads();
#pragma unroll 4
    for (int jl = 0; jl < NZT; ++jl) {
      const float w = Ps[orow][jl];
      const float4* vr = reinterpret_cast<const float4*>(&Vs[Cs[orow][jl]][4 * cb]);
      const float4 x0 = vr[0], x1 = vr[8];
      acc[0] = fmaf(w, x0.x, acc[0]);
      acc[1] = fmaf(w, x0.y, acc[1]);
      acc[2] = fmaf(w, x0.z, acc[2]);
      acc[3] = fmaf(w, x0.w, acc[3]);
      acc[4] = fmaf(w, x1.x, acc[4]);
      acc[5] = fmaf(w, x1.y, acc[5]);
      acc[6] = fmaf(w, x1.z, acc[6]);
      acc[7] = fmaf(w, x1.w, acc[7]);
    }
    __syncthreads();
  }
  const int r = row0 + orow;
  if (r < rows) {
    TO* o = out + ((int64_t)b * rows + r) * 64 + 4 * cb;  // columns 4cb.. and 32+4cb.. (see Vs reads)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      o[i] = DT<TO>::from_f(acc[i]);
      o[32 + i] = DT<TO>::from_f(acc[4 + i]);
    }
  }
}

template <typename TP, typename TV, typename TO, int GS>
static cudaError_t spmm_simt_gs(const void* p, const uint32_t* meta, const void* v, void* out, int64_t bh, int rows,
                                int n_k, int d, const uint8_t* keep, int tr, int tc, cudaStream_t s) {
  MetaGeom geo(rows, n_k / GS);
  if (d == 64 && n_k % 128 == 0 && n_k >= 512 && ((uintptr_t)v & 15) == 0) {
    for (int64_t b0 = 0; b0 < bh; b0 += 65535) {  // bh on gridDim.y (<= 65535): slices
      const int64_t nb = bh - b0 < 65535 ? bh - b0 : 65535;
      spmm_tiled_kernel<TP, TV, TO, GS><<<dim3((unsigned)((rows + 31) / 32), (unsigned)nb), 256, 0, s>>>(
          (const TP*)p + b0 * rows * (n_k / 2), meta + b0 * geo.words_per_bh(), (const TV*)v + b0 * n_k * 64,
          (TO*)out + b0 * rows * 64, rows, n_k, keep, tr, tc, geo);
    }
    return cudaGetLastError();
  }
  const int64_t total = bh * rows;
  int64_t blocks = (total + 7) / 8;
  if (blocks > 148 * 64) blocks = 148 * 64;
  const int dper = (d + 31) / 32;
#define DFSS_SPMM_LAUNCH(DP)                                                                                    \
  spmm_simt_kernel<TP, TV, TO, GS, DP><<<(int)blocks, 256, 0, s>>>((const TP*)p, meta, (const TV*)v, (TO*)out, \
                                                                   total, rows, n_k, d, keep, tr, tc, geo)
  if (dper <= 1)
    DFSS_SPMM_LAUNCH(1);
  else if (dper <= 2)
    DFSS_SPMM_LAUNCH(2);
  else if (dper <= 4)
    DFSS_SPMM_LAUNCH(4);
  else
    DFSS_SPMM_LAUNCH(8);
#undef DFSS_SPMM_LAUNCH
  return cudaGetLastError();
}

template <typename TP, typename TV, typename TO>
static cudaError_t spmm_simt_typed(const void* p, const uint32_t* meta, const void* v, void* out, int gs, int64_t bh,
                                   int rows, int n_k, int d, const uint8_t* keep, int tr, int tc, cudaStream_t s) {
  return gs == 4 ? spmm_simt_gs<TP, TV, TO, 4>(p, meta, v, out, bh, rows, n_k, d, keep, tr, tc, s)
                 : spmm_simt_gs<TP, TV, TO, 2>(p, meta, v, out, bh, rows, n_k, d, keep, tr, tc, s);
}

template <typename TP, typename TV>
static cudaError_t spmm_simt_pv(const void* p, const uint32_t* meta, const void* v, void* out, int gs, int out_dtype,
                                int64_t bh, int rows, int n_k, int d, const uint8_t* keep, int tr, int tc,
                                cudaStream_t s) {
  switch (out_dtype) {
    case DFSS_F32: return spmm_simt_typed<TP, TV, float>(p, meta, v, out, gs, bh, rows, n_k, d, keep, tr, tc, s);
    case DFSS_BF16:
      return spmm_simt_typed<TP, TV, __nv_bfloat16>(p, meta, v, out, gs, bh, rows, n_k, d, keep, tr, tc, s);
    default: return spmm_simt_typed<TP, TV, __half>(p, meta, v, out, gs, bh, rows, n_k, d, keep, tr, tc, s);
  }
}

template <typename TP>
static cudaError_t spmm_simt_p(const void* p, const uint32_t* meta, const void* v, void* out, int gs, int v_dtype,
                               int out_dtype, int64_t bh, int rows, int n_k, int d, const uint8_t* keep, int tr, int tc,
                               cudaStream_t s) {
  switch (v_dtype) {
    case DFSS_F32: return spmm_simt_pv<TP, float>(p, meta, v, out, gs, out_dtype, bh, rows, n_k, d, keep, tr, tc, s);
    case DFSS_BF16:
      return spmm_simt_pv<TP, __nv_bfloat16>(p, meta, v, out, gs, out_dtype, bh, rows, n_k, d, keep, tr, tc, s);
    default: return spmm_simt_pv<TP, __half>(p, meta, v, out, gs, out_dtype, bh, rows, n_k, d, keep, tr, tc, s);
  }
}

// d == 64 variant of the softmax-fused fp32 SpMM: one warp per row, the two half-warps take
// alternate 16-nonzero batches of the row and add their partial rows at the end; each lane
// owns 4 output columns loaded as one float4 (half the instructions per nonzero of the generic
// kernel, and the row's dependent load chain split in two).
template <int GS>
__global__ void __launch_bounds__(256) spmm_simt_softmax_d64_kernel(const float* __restrict__ p,
                                                                    const uint32_t* __restrict__ meta,
                                                                    const float* __restrict__ v,
                                                                    float* __restrict__ out, int64_t total_rows,
                                                                    int rows, int n_k, MetaGeom geo) {
  constexpr float kLog2e = 1.4426950408889634f;
  // launched as a programmatic dependent of the SDDMM (see the launch): wait for its results
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int lane = threadIdx.x & 31, hl = lane & 15, part = lane >> 4;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int nzc = n_k / 2;
  for (int64_t rg = warp; rg < total_rows; rg += nwarps) {
    const int64_t b = rg / rows;
    const int r = (int)(rg % rows);
    const float* prow = p + rg * nzc;
    const uint32_t* mb = meta + b * geo.words_per_bh();
    const float4* vb = reinterpret_cast<const float4*>(v + b * (int64_t)n_k * 64);
    float mx = -INFINITY;
    for (int j = lane; j < nzc; j += 32) mx = fmaxf(mx, prow[j]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const float mlb = mx * kLog2e;
    float sum = 0.f;
    for (int j = lane; j < nzc; j += 32) sum += exp2f(fmaf(prow[j], kLog2e, -mlb));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    // one batch = 32 nonzeros, 16 per half-warp; same trip count in both halves (converged
    // shuffles).  Full batches run unpredicated (all 16 V-row loads in flight); only the row's
    // last partial batch predicates its slots -- slots past the row end are skipped, not
    // weighted 0 (an Inf in an unrelated V row must not leak in as 0 * Inf).
    auto batch = [&](int j0, auto tail) {
      constexpr bool TAIL = decltype(tail)::value;
      const int j = j0 + 16 * part + hl;
      float pv = 0.f;
      int col = 0;
      if (!TAIL || j < nzc) {
        const int g = (GS == 4) ? (j >> 1) : j;
        int shift;
        const uint32_t nib = (mb[geo.word_of(r, g, shift)] >> shift) & 0xFu;
        col = (GS == 4) ? 4 * g + (int)((j & 1) ? ((nib >> 2) & 3u) : (nib & 3u)) : 2 * g + (nib == 0xEu ? 1 : 0);
        pv = exp2f(fmaf(prow[j], kLog2e, -mlb));
      }
      const int cnt = nzc - (j0 + 16 * part);
#pragma unroll
      for (int l = 0; l < 16; ++l) {
        const float pl = __shfl_sync(0xffffffffu, pv, l, 16);
        const int cl = __shfl_sync(0xffffffffu, col, l, 16);
        if (!TAIL || l < cnt) {
          const float4 x = vb[(int64_t)cl * 16 + hl];
          acc.x = fmaf(pl, x.x, acc.x);
          acc.y = fmaf(pl, x.y, acc.y);
          acc.z = fmaf(pl, x.z, acc.z);
          acc.w = fmaf(pl, x.w, acc.w);
        }
      }
    };
    const int nfull = nzc & ~31;
    for (int j0 = 0; j0 < nfull; j0 += 32) batch(j0, std::false_type{});
    if (nfull < nzc) batch(nfull, std::true_type{});
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 16);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 16);
    acc.z += __shfl_xor_sync(0xffffffffu, acc.z, 16);
    acc.w += __shfl_xor_sync(0xffffffffu, acc.w, 16);
    if (part == 0) {
      const float inv = 1.0f / sum;
      reinterpret_cast<float4*>(out + rg * 64)[hl] = make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
    }
  }
}

// Tiled variant (d == 64, n_k % 128 == 0): a CTA owns 32 rows of one (batch, head) and streams
// V through shared memory in 64-key tiles, so each V row is read from L2 once per CTA instead
// of once per nonzero (the warp-per-row kernel is L2-bandwidth-bound at larger n).  For either
// mode the nonzeros of a row that fall in a 64-key tile are the contiguous range
// [k0 / 2, k0 / 2 + 32).
// The tile's weights are scattered into a dense [32 rows][128 keys] block (zeros where a key
// is not kept) and multiplied as a dense register-blocked product: a thread owns 4 rows x 2
// columns; per 4 keys, 4 broadcast loads of 4 weights and 4 8-byte V loads feed 32 FFMAs (the
// per-nonzero gather of a V row moved ~4x more shared-memory wavefronts per FMA).  Twice the
// FMAs of the sparse gather, but the added terms are fma(0, v, acc) = acc exactly (V finite,
// dense.py:34-35), and keys are accumulated in ascending order: the result is bitwise the
// sparse accumulation in ascending nonzero order.
template <int GS>
__global__ void __launch_bounds__(256) spmm_softmax_f32_tiled_kernel(const float* __restrict__ p,
                                                                     const uint32_t* __restrict__ meta,
                                                                     const float* __restrict__ v,
                                                                     float* __restrict__ out, int rows, int n_k,
                                                                     MetaGeom geo) {
  constexpr float kLog2e = 1.4426950408889634f;
  constexpr int RB = 32, KT = 64, NZT = KT / 2;  // 64-key tiles: 16 KB of V + 8.5 KB of weights
  __shared__ __align__(16) float Vs[KT][64];
  __shared__ __align__(16) float Pd[RB][KT + 4];  // dense weights, row-major (rows 16 B aligned)
  __shared__ float s_mlb[RB], s_inv[RB];
  const int b = blockIdx.y, row0 = blockIdx.x * RB;
  const int nzc = n_k / 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float* pb = p + ((int64_t)b * rows) * nzc;
  const uint32_t* mb = meta + (int64_t)b * geo.words_per_bh();
  const float4* vb = reinterpret_cast<const float4*>(v + (int64_t)b * n_k * 64);
  // row statistics: warp w handles rows 4w .. 4w + 3
  for (int rr = 4 * warp; rr < 4 * warp + 4; ++rr) {
    const int r = row0 + rr;
    float mx = -INFINITY, sum = 0.f;
    if (r < rows) {
      const float* prow = pb + (int64_t)r * nzc;
      for (int j = lane; j < nzc; j += 32) mx = fmaxf(mx, prow[j]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      for (int j = lane; j < nzc; j += 32) sum += exp2f(fmaf(prow[j], kLog2e, -mx * kLog2e));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    }
    if (lane == 0) {
      s_mlb[rr] = mx * kLog2e;
      s_inv[rr] = 1.0f / sum;
    }
  }
  __syncthreads();
  // thread: rows 4 * warp .. + 3 (one weight float4 per key, a broadcast within the warp),
  // columns 2 * lane, 2 * lane + 1 (the warp reads a whole 256-byte V row per key)
  float acc[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = 0.f;
  for (int k0 = 0; k0 < n_k; k0 += KT) {
    // V tile [128 keys][64] (float4 per thread x 8) and the zeroed weight block
#pragma unroll
    for (int i = 0; i < (KT * 16) / 256; ++i) {
      const int idx = threadIdx.x + 256 * i;
      reinterpret_cast<float4*>(&Vs[0][0])[idx] = vb[(int64_t)k0 * 16 + idx];
    }
#pragma unroll
    for (int i = 0; i < (KT * RB / 4) / 256; ++i) {
      const int idx = threadIdx.x + 256 * i;  // float4 idx % (KT / 4) of row idx / (KT / 4)
      *reinterpret_cast<float4*>(&Pd[idx / (KT / 4)][4 * (idx % (KT / 4))]) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads();
    // scatter this tile's weights of the CTA's rows to their keys
#pragma unroll
    for (int i = 0; i < (RB * NZT) / 256; ++i) {
      const int idx = threadIdx.x + 256 * i;
      const int rr = idx / NZT, jl = idx % NZT;
      const int r = row0 + rr, j = k0 / 2 + jl;
      if (r < rows) {
        const int g = (GS == 4) ? (j >> 1) : j;
        int shift;
        const uint32_t nib = (mb[geo.word_of(r, g, shift)] >> shift) & 0xFu;
        const int col = (GS == 4) ? 4 * g + (int)((j & 1) ? ((nib >> 2) & 3u) : (nib & 3u)) : 2 * g + (nib == 0xEu ? 1 : 0);
        Pd[rr][col - k0] = exp2f(fmaf(pb[(int64_t)r * nzc + j], kLog2e, -s_mlb[rr]));
      }
    }
    __syncthreads();
#pragma unroll 2
    for (int kk = 0; kk < KT; kk += 4) {
      float w[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float4 t = *reinterpret_cast<const float4*>(&Pd[4 * warp + i][kk]);
        w[i][0] = t.x, w[i][1] = t.y, w[i][2] = t.z, w[i][3] = t.w;
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {  // keys in ascending order
        const float2 x = *reinterpret_cast<const float2*>(&Vs[kk + e][2 * lane]);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          acc[i][0] = fmaf(w[i][e], x.x, acc[i][0]);
          acc[i][1] = fmaf(w[i][e], x.y, acc[i][1]);
        }
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int rr = 4 * warp + i, r = row0 + rr;
    if (r < rows) {
      const float inv = s_inv[rr];
      *reinterpret_cast<float2*>(out + ((int64_t)b * rows + r) * 64 + 2 * lane) =
          make_float2(acc[i][0] * inv, acc[i][1] * inv);
    }
  }
}

cudaError_t launch_spmm_simt_softmax_f32(const void* p, const uint32_t* meta, const void* v, void* out, int gs,
                                        int64_t bh, int rows, int n_k, int d, cudaStream_t s) {
  if (bh == 0 || rows == 0 || d == 0) return cudaSuccess;
  if (d > 64) return cudaErrorNotSupported;
  // tiled from n_k = 512 up (L2-bound warp kernel: n = 1024 1.79 -> 1.50 ms for 96 heads), and on
  // shorter rows once there are >= 4 waves of 32-row CTAs (n = 384 x 96 heads: 0.159 vs 0.179 ms per
  // step); few CTAs (c1: 12 heads x 12 row blocks) keep the warp-per-row kernel (0.030 vs 0.037 ms)
  const bool tiled_pays = n_k >= 512 || bh * ((rows + 31) / 32) >= 4 * 148;
  if (d == 64 && n_k % 128 == 0 && tiled_pays && ((uintptr_t)v & 15) == 0 && ((uintptr_t)out & 15) == 0) {
    const MetaGeom geo(rows, n_k / gs);
    for (int64_t b0 = 0; b0 < bh; b0 += 65535) {  // bh on gridDim.y (<= 65535): slices
      const int64_t nb = bh - b0 < 65535 ? bh - b0 : 65535;
      const float* pb = (const float*)p + b0 * rows * (n_k / 2);
      const uint32_t* mb = meta + b0 * geo.words_per_bh();
      const float* vb = (const float*)v + b0 * n_k * 64;
      float* ob = (float*)out + b0 * rows * 64;
      const dim3 grid((unsigned)((rows + 31) / 32), (unsigned)nb);
      if (gs == 4)
        spmm_softmax_f32_tiled_kernel<4><<<grid, 256, 0, s>>>(pb, mb, vb, ob, rows, n_k, geo);
      else
        spmm_softmax_f32_tiled_kernel<2><<<grid, 256, 0, s>>>(pb, mb, vb, ob, rows, n_k, geo);
    }
    return cudaGetLastError();
  }
  if (d == 64 && ((uintptr_t)v & 15) == 0 && ((uintptr_t)out & 15) == 0) {
    const int64_t total = bh * rows;
    int64_t blocks = (total + 7) / 8;  // one row per warp
    if (blocks > 148 * 64) blocks = 148 * 64;
    // programmatic dependent launch: the kernel's launch overlaps the SDDMM's tail (it waits
    // for the SDDMM's results with griddepcontrol.wait) -- c1 is launch-latency-bound
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)blocks);
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const float* pf = (const float*)p;
    const float* vf = (const float*)v;
    float* of = (float*)out;
    const int64_t tr = total;
    if (gs == 4)
      return cudaLaunchKernelEx(&cfg, spmm_simt_softmax_d64_kernel<4>, pf, meta, vf, of, tr, rows, n_k,
                                MetaGeom(rows, n_k / 4));
    return cudaLaunchKernelEx(&cfg, spmm_simt_softmax_d64_kernel<2>, pf, meta, vf, of, tr, rows, n_k,
                              MetaGeom(rows, n_k / 2));
  }
  const int64_t total = bh * rows;
  int64_t blocks = (total + 7) / 8;
  if (blocks > 148 * 64) blocks = 148 * 64;
  const float* pf = (const float*)p;
  const float* vf = (const float*)v;
  float* of = (float*)out;
  if (gs == 4) {
    MetaGeom geo(rows, n_k / 4);
    spmm_simt_kernel<float, float, float, 4, 2, true>
        <<<(int)blocks, 256, 0, s>>>(pf, meta, vf, of, total, rows, n_k, d, nullptr, 1, 1, geo);
  } else {
    MetaGeom geo(rows, n_k / 2);
    spmm_simt_kernel<float, float, float, 2, 2, true>
        <<<(int)blocks, 256, 0, s>>>(pf, meta, vf, of, total, rows, n_k, d, nullptr, 1, 1, geo);
  }
  return cudaGetLastError();
}

cudaError_t launch_spmm_simt(const void* p, const uint32_t* meta, const void* v, void* out, int gs, int p_dtype,
                             int v_dtype, int out_dtype, int64_t bh, int rows, int n_k, int d, const uint8_t* keep,
                             int tile_rows, int tile_cols, cudaStream_t s) {
  if (bh == 0 || rows == 0 || d == 0) return cudaSuccess;
  switch (p_dtype) {
    case DFSS_F32:
      return spmm_simt_p<float>(p, meta, v, out, gs, v_dtype, out_dtype, bh, rows, n_k, d, keep, tile_rows, tile_cols,
                                s);
    case DFSS_BF16:
      return spmm_simt_p<__nv_bfloat16>(p, meta, v, out, gs, v_dtype, out_dtype, bh, rows, n_k, d, keep, tile_rows,
                                        tile_cols, s);
    default:
      return spmm_simt_p<__half>(p, meta, v, out, gs, v_dtype, out_dtype, bh, rows, n_k, d, keep, tile_rows, tile_cols,
                                 s);
  }
}

}  // namespace dfss
