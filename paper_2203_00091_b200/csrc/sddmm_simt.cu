// sddmm_simt.cu -- generic fused score + N:M prune on FP32 FFMA.
//
// The exact-FP32 path (fp32 inputs at the 1e-5 tolerance, where TF32 tensor
// cores would round the inputs to a 10-bit mantissa) and the fallback for
// shapes the tcgen05 kernel does not tile (ragged n, odd d, block masks).
// Same epilogue semantics as the tcgen05 kernel and as the reference
// _sddmm_compress (_kernels_numba.py:110-185): scale, then select by signed
// value with ties to the lower index, then write nonzeros + nibbles only.
#include <type_traits>

#include "dfss_common.cuh"

namespace dfss {

namespace {
constexpr int BM = 64, BN = 64, BK = 32;
}

// grid: (ceil(m/64), 2*ceil(n/128), bh); 256 threads, each a 4x4 score block:
// rows 4*ty .. 4*ty+3, columns 4*tx .. 4*tx+3 (one 2:4 group, two 1:2 groups).
// (16-bit inputs: at least 2 CTAs / SM, so ptxas keeps their conversions in registers instead of
// spilling; fp32 (the c1 exact path) keeps 64 registers / 4 CTAs: 114 registers were 10 % slower)
// four consecutive elements (16 B fp32 / 8 B 16-bit, aligned) as floats, or zeros
template <typename TIn>
__device__ __forceinline__ void load4(const TIn* __restrict__ p, bool ok, float (&x)[4]) {
  if constexpr (std::is_same<TIn, float>::value) {
    const float4 v = ok ? __ldg(reinterpret_cast<const float4*>(p)) : make_float4(0.f, 0.f, 0.f, 0.f);
    x[0] = v.x, x[1] = v.y, x[2] = v.z, x[3] = v.w;
  } else {
    const uint2 u = ok ? __ldg(reinterpret_cast<const uint2*>(p)) : make_uint2(0u, 0u);
    const TIn* h = reinterpret_cast<const TIn*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) x[e] = DT<TIn>::to_f(h[e]);
  }
}

template <typename TIn, typename TNz, int GS>
__global__ void __launch_bounds__(256, std::is_same<TIn, float>::value ? 4 : 2) sddmm_simt_kernel(const TIn* __restrict__ q, const TIn* __restrict__ k,
                                                         TNz* __restrict__ nz, uint32_t* __restrict__ meta,
                                                         float scale, int n, int m, int d,
                                                         const uint8_t* __restrict__ keep, int tile_rows,
                                                         int tile_cols, float* __restrict__ dbg, MetaGeom geo,
                                                         uint32_t two, int vec4, int pdl) {
  __shared__ __align__(16) float Qs[BK][BM + 4];
  __shared__ __align__(16) float Ks[BK][BN + 4];
  __shared__ uint8_t nibs[BM][BN / GS];
  // a programmatic dependent (the exact-FP32 SpMM) may start launching now; it waits for this
  // grid's completion before reading its results (griddepcontrol.wait)
  if (pdl) asm volatile("griddepcontrol.launch_dependents;");

  const int b = blockIdx.z;
  const int row0 = blockIdx.y * BM, col0 = blockIdx.x * BN;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  q += (int64_t)b * n * d;
  k += (int64_t)b * m * d;
  nz += (int64_t)b * n * (m / 2);
  meta += (int64_t)b * geo.words_per_bh();
  if (dbg) dbg += (int64_t)b * n * m;
  const int grid_cols = keep ? (m + tile_cols - 1) / tile_cols : 0;

  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  // a CTA tile whose mask tiles are all masked skips the dot products (the reference's tile
  // loop skips masked tiles, _kernels_numba.py:110-185); its groups encode as absent below.
  // With a score dump requested (parity hook) every score is still computed.
  bool cta_live = true;
  if (keep && !dbg) {
    cta_live = false;
    const int r_hi = min(row0 + BM, n) - 1, c_hi = min(col0 + BN, m) - 1;
    for (int tr = row0 / tile_rows; tr <= r_hi / tile_rows && !cta_live; ++tr)
      for (int tcl = col0 / tile_cols; tcl <= c_hi / tile_cols; ++tcl)
        if (keep[(int64_t)tr * grid_cols + tcl]) {
          cta_live = true;
          break;
        }
  }
  if (row0 < n && cta_live) {
    for (int k0 = 0; k0 < d; k0 += BK) {
      if (vec4) {  // d % 4 == 0, aligned rows: four elements per load (the scalar loop below
                   // spent a quarter of the kernel's instructions on loads and index math)
#pragma unroll
        for (int it = 0; it < (BM * BK / 4) / 256; ++it) {
          const int i = threadIdx.x + 256 * it;
          const int r = i / (BK / 4), kq = (i % (BK / 4)) * 4;
          const int gr = row0 + r, gc = col0 + r, gk = k0 + kq;
          float a[4], c[4];
          load4<TIn>(q + (int64_t)gr * d + gk, gr < n && gk < d, a);
          load4<TIn>(k + (int64_t)gc * d + gk, gc < m && gk < d, c);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            Qs[kq + e][r] = a[e];
            Ks[kq + e][r] = c[e];
          }
        }
      } else {
        for (int i = threadIdx.x; i < BM * BK; i += 256) {
          const int r = i / BK, kk = i % BK;
          const int gr = row0 + r, gk = k0 + kk;
          Qs[kk][r] = (gr < n && gk < d) ? DT<TIn>::to_f(q[(int64_t)gr * d + gk]) : 0.f;
          const int gc = col0 + r;
          Ks[kk][r] = (gc < m && gk < d) ? DT<TIn>::to_f(k[(int64_t)gc * d + gk]) : 0.f;
        }
      }
      __syncthreads();
#pragma unroll 8
      for (int kk = 0; kk < BK; ++kk) {
        const float4 bv = *reinterpret_cast<const float4*>(&Ks[kk][4 * tx]);
        const float4 av = *reinterpret_cast<const float4*>(&Qs[kk][4 * ty]);  // rows 4 ty .. 4 ty + 3
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float a = i == 0 ? av.x : i == 1 ? av.y : i == 2 ? av.z : av.w;
          acc[i][0] = fmaf(a, bv.x, acc[i][0]);
          acc[i][1] = fmaf(a, bv.y, acc[i][1]);
          acc[i][2] = fmaf(a, bv.z, acc[i][2]);
          acc[i][3] = fmaf(a, bv.w, acc[i][3]);
        }
      }
      __syncthreads();
    }
  }

  // ---- prune/encode epilogue: nonzeros and nibbles leave, dense scores never do
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int lr = 4 * ty + i;
    const int row = row0 + lr;
    const int c0 = col0 + 4 * tx;
    float v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = scale_canon(acc[i][j], scale);
    const bool row_ok = row < n;
    if (dbg && row_ok) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (c0 + j < m) dbg[(int64_t)row * m + c0 + j] = v[j];
    }
#pragma unroll
    for (int h = 0; h < 4 / GS; ++h) {
      const int c = c0 + GS * h;  // first dense column of this group
      uint32_t nib = kPadNibble;
      if (row_ok && c < m) {
        const bool kept_tile = !keep || keep[(row / tile_rows) * grid_cols + c / tile_cols];
        const int g = c / GS;
        if (GS == 4) {
          float lo = 0.f, hi = 0.f;
          if (kept_tile) nib = select24(v[0], v[1], v[2], v[3], lo, hi, two);
          nz[(int64_t)row * (m / 2) + 2 * g] = DT<TNz>::from_f(lo);
          nz[(int64_t)row * (m / 2) + 2 * g + 1] = DT<TNz>::from_f(hi);
        } else {
          float kv = 0.f;
          if (kept_tile) nib = select12(v[2 * h], v[2 * h + 1], kv);
          nz[(int64_t)row * (m / 2) + g] = DT<TNz>::from_f(kv);
        }
      }
      nibs[lr][(4 / GS) * tx + h] = (uint8_t)nib;
    }
  }
  __syncthreads();

  // ---- assemble meta_hw words for the 64 lanes this row half covers
  constexpr int kChunks = BN / (8 * GS);  // chunks of 8 groups inside the tile
  const int rb = row0 >> 7, half = (row0 >> 6) & 1;
  const int c_base = col0 / (8 * GS);
  if (threadIdx.x < kChunks * 64) {
    const int cl = threadIdx.x >> 6;
    const int lane = 64 * half + (threadIdx.x & 63);
    const int c = c_base + cl;
    if (c < geo.chunks) {
      uint32_t word = 0;
#pragma unroll
      for (int idx = 0; idx < 8; ++idx) {
        int row, group;
        MetaGeom::coords_of(rb, c, lane, idx, row, group);
        const uint32_t nib = nibs[row - row0][group - col0 / GS];
        word |= nib << (16 * (idx >> 2) + 4 * (idx & 3));
      }
      meta[((int64_t)rb * geo.chunks + c) * 128 + lane] = word;
    }
  }
}

template <typename TIn, typename TNz>
static cudaError_t sddmm_simt_typed(const void* q, const void* k, void* nz, uint32_t* meta, float scale, int gs,
                                    int64_t bh, int n, int m, int d, const uint8_t* keep, int tile_rows,
                                    int tile_cols, float* dbg, cudaStream_t s) {
  MetaGeom geo(n, m / gs);
  // bh on gridDim.z (<= 65535): larger batches are launched in slices
  for (int64_t b0 = 0; b0 < bh; b0 += 65535) {
    const int64_t nb = bh - b0 < 65535 ? bh - b0 : 65535;
    const TIn* qb = (const TIn*)q + b0 * n * d;
    const TIn* kb = (const TIn*)k + b0 * m * d;
    TNz* nzb = (TNz*)nz + b0 * n * (m / 2);
    uint32_t* mb = meta + b0 * geo.words_per_bh();
    float* db = dbg ? dbg + b0 * n * m : nullptr;
    dim3 grid((m + BN - 1) / BN, 2 * geo.rblocks, (unsigned)nb);
    const int vec4 = d % 4 == 0 && ((uintptr_t)qb | (uintptr_t)kb) % (4 * sizeof(TIn)) == 0;
    // early dependent launch only when this grid is a single wave (4 CTAs per SM): dependents
    // would otherwise take the slots of this grid's later CTAs
    const int pdl = (int64_t)grid.x * grid.y * grid.z <= 4 * 148;
    if (gs == 4)
      sddmm_simt_kernel<TIn, TNz, 4><<<grid, 256, 0, s>>>(qb, kb, nzb, mb, scale, n, m, d, keep, tile_rows, tile_cols,
                                                          db, geo, 2u, vec4, pdl);
    else
      sddmm_simt_kernel<TIn, TNz, 2><<<grid, 256, 0, s>>>(qb, kb, nzb, mb, scale, n, m, d, keep, tile_rows, tile_cols,
                                                          db, geo, 2u, vec4, pdl);
  }
  return cudaGetLastError();
}

template <typename TIn>
static cudaError_t sddmm_simt_in(const void* q, const void* k, void* nz, uint32_t* meta, float scale, int gs,
                                 int nz_dtype, int64_t bh, int n, int m, int d, const uint8_t* keep, int tile_rows,
                                 int tile_cols, float* dbg, cudaStream_t s) {
  switch (nz_dtype) {
    case DFSS_F32:
      return sddmm_simt_typed<TIn, float>(q, k, nz, meta, scale, gs, bh, n, m, d, keep, tile_rows, tile_cols, dbg, s);
    case DFSS_BF16:
      return sddmm_simt_typed<TIn, __nv_bfloat16>(q, k, nz, meta, scale, gs, bh, n, m, d, keep, tile_rows, tile_cols,
                                                  dbg, s);
    default:
      return sddmm_simt_typed<TIn, __half>(q, k, nz, meta, scale, gs, bh, n, m, d, keep, tile_rows, tile_cols, dbg, s);
  }
}

cudaError_t launch_sddmm_simt(const void* q, const void* k, void* nz, uint32_t* meta, float scale, int gs,
                              int in_dtype, int nz_dtype, int64_t bh, int n, int m, int d, const uint8_t* keep,
                              int tile_rows, int tile_cols, float* dbg, cudaStream_t s) {
  if (bh == 0 || n == 0 || m == 0) return cudaSuccess;
  switch (in_dtype) {
    case DFSS_F32:
      return sddmm_simt_in<float>(q, k, nz, meta, scale, gs, nz_dtype, bh, n, m, d, keep, tile_rows, tile_cols, dbg, s);
    case DFSS_BF16:
      return sddmm_simt_in<__nv_bfloat16>(q, k, nz, meta, scale, gs, nz_dtype, bh, n, m, d, keep, tile_rows, tile_cols,
                                          dbg, s);
    default:
      return sddmm_simt_in<__half>(q, k, nz, meta, scale, gs, nz_dtype, bh, n, m, d, keep, tile_rows, tile_cols, dbg, s);
  }
}

}  // namespace dfss
