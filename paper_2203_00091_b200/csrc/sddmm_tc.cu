// sddmm_tc.cu -- fused Q.K^T + 2:4 prune on tcgen05 (bf16 / fp16, head dim 64).
//
// Replaces _sddmm_compress (_kernels_numba.py:110-185) for the 16-bit
// configurations.  Persistent, warp-specialised, one CTA per SM:
//   warp 0      TMA producer: Q tile (128 x 64) once per work item, K tiles
//               (256 x 64) through a KSTAGES-deep mbarrier ring;
//   warp 1      MMA issuer: 4 x tcgen05.mma.kind::f16 (M=128, N=256, K=16) per
//               K tile into one of two TMEM accumulators (2 x 256 columns);
//   warp 2      TMEM allocator;
//   warps 4-11  epilogue: warp w reads TMEM lanes 32*(w%4).. (its 32 query rows)
//               and one 128-column half of the accumulator, scales, selects
//               2-of-4 in registers (select24, the same routine as the parity
//               hook), packs the kept pair to 16-bit, stages the nonzeros in
//               128B-swizzled smem for a TMA store, and writes the metadata
//               words of its lanes straight to meta_hw (coalesced 128 B).
// No dense score ever leaves the SM unless the debug dump is requested.
// Work item = (bh, 128-row block); items are strided over the persistent CTAs.
#include <stdio.h>

#include <cmath>

#include <type_traits>

#include "dfss_common.cuh"
#include "flash_common.cuh"  // packed fp32 helpers (FMUL2 / FFMA2)
#include "tc_common.cuh"

namespace dfss {

namespace {
constexpr int BM = 128;
constexpr int BN = 256;
constexpr int HD = 64;
constexpr int KSTAGES = 3;
constexpr int NACC = 2;
constexpr int EPI_WARPS = 16;  // (lane quarter, 64-column quarter) of the 128 x 256 tile
constexpr int NUM_THREADS = (4 + EPI_WARPS) * 32;
constexpr int Q_BYTES = BM * HD * 2;
constexpr int K_BYTES = BN * HD * 2;
constexpr int STG_BYTES = 32 * 64;  // 32 rows x 32 nonzeros x 2 B (64B-swizzled rows)
constexpr int SMEM_Q = 0;
constexpr int SMEM_K = SMEM_Q + 2 * Q_BYTES;
constexpr int SMEM_STG = SMEM_K + KSTAGES * K_BYTES;
constexpr int SMEM_BAR = SMEM_STG + EPI_WARPS * 2 * STG_BYTES;
constexpr int SMEM_TOTAL = SMEM_BAR + 256 + 1024;  // + barriers + alignment slack
}  // namespace

template <typename T>
__device__ __forceinline__ uint32_t pack2(float lo, float hi);
template <>
__device__ __forceinline__ uint32_t pack2<__nv_bfloat16>(float lo, float hi) {
  __nv_bfloat162 p = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&p);
}
template <>
__device__ __forceinline__ uint32_t pack2<__half>(float lo, float hi) {
  __half2 p = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&p);
}

// BlockMask tile grid (codec.py:150-200) for the masked instantiations: a group in a masked tile
// is structurally absent -- zero nonzeros and the padding nibble 0x4, as the FFMA kernel writes
// it (_kernels_numba.py:110-185 skips masked tiles)
struct TileKeepTc {
  const uint8_t* keep = nullptr;
  int tile_rows = 1, tile_cols = 1, grid_cols = 0;
  __device__ __forceinline__ bool kept(int row, int col) const {
    return keep[(row / tile_rows) * grid_cols + col / tile_cols] != 0;
  }
};

// Prune one 32-column chunk of a row: 8 groups of 4 scores -> 16 kept 16-bit values
// (two 16B units of the 64B-swizzled staging row) + one 32-bit nibble word that is
// traded with row^8 into the meta_hw word of this TMEM lane (include/dfss.h).
template <typename T, bool DBG, bool RMAX, bool MASK, bool PRE>
__device__ __forceinline__ void epi_chunk(const uint32_t (&r)[32], float scale, int colh, int cc, int unit0,
                                          uint8_t* stg, uint32_t lane, uint32_t* meta_b, int row_blk, float* dbg,
                                          int64_t dbg_row, int m, float& mx, uint32_t two, const TileKeepTc& tk,
                                          int grow) {
  constexpr bool SK = PRE && std::is_same<T, __half>::value;  // scale the kept values
  uint32_t packed[8];
  // the select24 rule with the metadata in float arithmetic on the FMA-lite pipe (as in the
  // fused kernel, flash_tc.cu prune_exp_tile): exact 0 / 1 pair-winner flags from saturated
  // multiplies of v0 - v1, v2 - v3 (canonical zeros: a tie gives +0 -> 0), nibble - 8 accumulated
  // as integers into 2^23 + 0x8888 floats, one PRMT -- no IMAD.HI / SEL chains on the busy pipes
  float wf[2] = {8388608.f + 34952.f, 8388608.f + 34952.f};
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    // PRE (power-of-two scale): bf16 -- Q was scaled in shared memory, the accumulator holds
    // the post-scale scores; fp16 -- select on the raw scores and scale the kept values (every
    // nonzero fp16 score is >= 2^-48 in magnitude, so the scaled score is exact: same order, no
    // new ties).  tcgen05 writes zero sums as +0: already canonical.
    const float v0 = PRE ? __uint_as_float(r[4 * g + 0]) : scale_canon(__uint_as_float(r[4 * g + 0]), scale);
    const float v1 = PRE ? __uint_as_float(r[4 * g + 1]) : scale_canon(__uint_as_float(r[4 * g + 1]), scale);
    const float v2 = PRE ? __uint_as_float(r[4 * g + 2]) : scale_canon(__uint_as_float(r[4 * g + 2]), scale);
    const float v3 = PRE ? __uint_as_float(r[4 * g + 3]) : scale_canon(__uint_as_float(r[4 * g + 3]), scale);
    if (DBG) {
      const float ds = SK ? scale : 1.f;
      *reinterpret_cast<float4*>(dbg + dbg_row * m + colh + cc * 32 + 4 * g) = make_float4(v0 * ds, v1 * ds, v2 * ds, v3 * ds);
    }
    const float w01 = fmaxf(v0, v1), l01 = fminf(v0, v1);
    const float w23 = fmaxf(v2, v3), l23 = fminf(v2, v3);
    if (RMAX) mx = fmaxf(mx, fmaxf(w01, w23));
    const bool keep01 = l01 >= w23, keep23 = l23 > w01;
    float t01, t23;
    mul2s(v0 - v1, v2 - v3, -1.7014118e38f, t01, t23);  // both first multiplies in one FMUL2
    // kept pair: (v0, v1) unless another case applies -- one predicated select per value
    float lo = v0, hi = v1;
    if (!keep01) {
      lo = keep23 ? v2 : w01;
      hi = keep23 ? v3 : w23;
    }
    const float fa = __saturatef(t01 * 1.7014118e38f);
    const float fb = __saturatef(t23 * 1.7014118e38f);
    float nf = fmaf(fb, 4.f, fa);
    nf = keep23 ? 6.f : nf;
    nf = keep01 ? -4.f : nf;
    if (MASK && !tk.kept(grow, colh + cc * 32 + 4 * g)) {  // absent: zeros, padding nibble 0x4
      lo = hi = 0.f;
      nf = -4.f;
    }
    wf[g >> 2] = fmaf(nf, (float)(1 << (4 * (g & 3))), wf[g >> 2]);
    if (SK) mul2s(lo, hi, scale, lo, hi);
    packed[g] = pack2<T>(lo, hi);
  }
  const uint32_t W = __byte_perm(__float_as_uint(wf[0]), __float_as_uint(wf[1]), 0x5410);
  (void)two;
  // 64B-swizzled staging row of this lane: 16-byte unit u at (u ^ ((row >> 1) & 3)) -- the
  // 8 lanes of a store phase hit 8 distinct 16B bank groups
  const int u0 = unit0, sw = (lane >> 1) & 3;
  *reinterpret_cast<uint4*>(stg + lane * 64 + ((u0 ^ sw) << 4)) = make_uint4(packed[0], packed[1], packed[2], packed[3]);
  *reinterpret_cast<uint4*>(stg + lane * 64 + (((u0 + 1) ^ sw) << 4)) =
      make_uint4(packed[4], packed[5], packed[6], packed[7]);
  const uint32_t partner = __shfl_xor_sync(0xffffffffu, W, 8);
  const uint32_t word = (lane & 8) ? ((partner >> 16) | (W & 0xFFFF0000u)) : ((W & 0xFFFFu) | (partner << 16));
  meta_b[(int64_t)((colh + cc * 32) >> 5) * 128 + row_blk] = word;
}

// 1:2 (codec.py:114-117: element 1 of a pair survives iff v1 > v0): the chunk's 16 pairs keep 16
// values -- the same 16 per 32 columns as 2:4, so staging and the TMA store are unchanged -- and
// their 16 nibbles (0x4 / 0xE) fill two meta_hw words (meta chunks of 8 pairs = 16 columns).
template <typename T, bool DBG, bool RMAX, bool MASK, bool PRE>
__device__ __forceinline__ void epi_chunk12(const uint32_t (&r)[32], float scale, int colh, int cc, int unit0,
                                            uint8_t* stg, uint32_t lane, uint32_t* meta_b, int row_blk, float* dbg,
                                            int64_t dbg_row, int m, float& mx, const TileKeepTc& tk, int grow) {
  constexpr bool SK = PRE && std::is_same<T, __half>::value;  // scale the kept values
  uint32_t packed[8];
  uint32_t W[2] = {0u, 0u};
#pragma unroll
  for (int g = 0; g < 8; ++g) {  // g: pairs 2g, 2g + 1
    // PRE (power-of-two scale): bf16 -- Q was scaled in shared memory, the accumulator holds
    // the post-scale scores; fp16 -- select on the raw scores and scale the kept values (every
    // nonzero fp16 score is >= 2^-48 in magnitude, so the scaled score is exact: same order, no
    // new ties).  tcgen05 writes zero sums as +0: already canonical.
    const float v0 = PRE ? __uint_as_float(r[4 * g + 0]) : scale_canon(__uint_as_float(r[4 * g + 0]), scale);
    const float v1 = PRE ? __uint_as_float(r[4 * g + 1]) : scale_canon(__uint_as_float(r[4 * g + 1]), scale);
    const float v2 = PRE ? __uint_as_float(r[4 * g + 2]) : scale_canon(__uint_as_float(r[4 * g + 2]), scale);
    const float v3 = PRE ? __uint_as_float(r[4 * g + 3]) : scale_canon(__uint_as_float(r[4 * g + 3]), scale);
    if (DBG) {
      const float ds = SK ? scale : 1.f;
      *reinterpret_cast<float4*>(dbg + dbg_row * m + colh + cc * 32 + 4 * g) = make_float4(v0 * ds, v1 * ds, v2 * ds, v3 * ds);
    }
    float k0, k1;
    uint32_t n0 = select12(v0, v1, k0), n1 = select12(v2, v3, k1);
    if (MASK) {  // (tile columns are even: a pair never straddles two tiles)
      if (!tk.kept(grow, colh + cc * 32 + 4 * g)) { n0 = 0x4u; k0 = 0.f; }
      if (!tk.kept(grow, colh + cc * 32 + 4 * g + 2)) { n1 = 0x4u; k1 = 0.f; }
    }
    if (RMAX) mx = fmaxf(mx, fmaxf(k0, k1));
    if (SK) mul2s(k0, k1, scale, k0, k1);
    packed[g] = pack2<T>(k0, k1);
    W[g >> 2] += (n0 | (n1 << 4)) << (8 * (g & 3));
  }
  // 64B-swizzled staging row of this lane: 16-byte unit u at (u ^ ((row >> 1) & 3)) -- the
  // 8 lanes of a store phase hit 8 distinct 16B bank groups
  const int u0 = unit0, sw = (lane >> 1) & 3;
  *reinterpret_cast<uint4*>(stg + lane * 64 + ((u0 ^ sw) << 4)) = make_uint4(packed[0], packed[1], packed[2], packed[3]);
  *reinterpret_cast<uint4*>(stg + lane * 64 + (((u0 + 1) ^ sw) << 4)) =
      make_uint4(packed[4], packed[5], packed[6], packed[7]);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const uint32_t partner = __shfl_xor_sync(0xffffffffu, W[h], 8);
    const uint32_t word = (lane & 8) ? ((partner >> 16) | (W[h] & 0xFFFF0000u)) : ((W[h] & 0xFFFFu) | (partner << 16));
    meta_b[(int64_t)(((colh + cc * 32) >> 4) + h) * 128 + row_blk] = word;
  }
}

template <typename T, int GS, bool DBG, bool RMAX, bool MASK, bool PRE>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    sddmm24_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                      const __grid_constant__ CUtensorMap tm_nz, uint32_t* __restrict__ meta, float scale, int bh,
                      int n, int m, float* __restrict__ dbg, float* __restrict__ rowmax, uint32_t two,
                      TileKeepTc tk) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = (uint64_t*)(smem + SMEM_BAR);
  uint64_t* q_full = bars;                 // [2]
  uint64_t* q_empty = bars + 2;            // [2]
  uint64_t* k_full = bars + 4;             // [KSTAGES]
  uint64_t* k_empty = k_full + KSTAGES;    // [KSTAGES]
  uint64_t* t_full = k_empty + KSTAGES;    // [NACC]
  uint64_t* t_empty = t_full + NACC;       // [NACC]
  uint64_t* q_ready = t_empty + NACC;     // [2] PRE: Q tile scaled in shared memory
  uint32_t* tmem_slot = (uint32_t*)(q_ready + 2);

  const uint32_t warp = tc::warp_id();
  const uint32_t lane = threadIdx.x & 31;
  const int mblocks = n / BM;
  const int items = bh * mblocks;
  const int ntiles = (m + BN - 1) / BN;

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tm_q);
    tc::prefetch_tmap(&tm_k);
    tc::prefetch_tmap(&tm_nz);
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&q_full[i], 1);
      tc::mbar_init(&q_empty[i], 1);
    }
    for (int i = 0; i < KSTAGES; ++i) {
      tc::mbar_init(&k_full[i], 1);
      tc::mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < NACC; ++i) {
      tc::mbar_init(&t_full[i], 1);
      tc::mbar_init(&t_empty[i], EPI_WARPS);
    }
    for (int i = 0; i < 2; ++i) tc::mbar_init(&q_ready[i], 1);
    tc::fence_barrier_init();
  }
  if (warp == 2) tc::tmem_alloc<512>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int ks = 0;
      uint32_t kph = 0;
      int it = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
        const int b = item / mblocks, mb = item % mblocks;
        const int qs = it & 1;
        const uint32_t qph = (it >> 1) & 1;
        tc::mbar_wait_sleep(&q_empty[qs], qph ^ 1);
        tc::mbar_arrive_expect_tx(&q_full[qs], Q_BYTES);
        tc::tma_load_3d(smem + SMEM_Q + qs * Q_BYTES, &tm_q, &q_full[qs], 0, mb * BM, b);
        for (int t = 0; t < ntiles; ++t) {
          tc::mbar_wait_sleep(&k_empty[ks], kph ^ 1);
          tc::mbar_arrive_expect_tx(&k_full[ks], K_BYTES);
          tc::tma_load_3d(smem + SMEM_K + ks * K_BYTES, &tm_k, &k_full[ks], 0, t * BN, b);
          if (++ks == KSTAGES) { ks = 0; kph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t fmt = std::is_same<T, __nv_bfloat16>::value ? 1u : 0u;
      constexpr uint32_t idesc256 = tc::instr_desc(fmt, BM, 256, false, false, false);
      constexpr uint32_t idesc128 = tc::instr_desc(fmt, BM, 128, false, false, false);
      int ks = 0, acc = 0;
      uint32_t kph = 0, aph = 0;
      int it = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
        const int qs = it & 1;
        const uint32_t qph = (it >> 1) & 1;
        constexpr bool QS = PRE && std::is_same<T, __nv_bfloat16>::value;  // Q scaled in smem
        tc::mbar_wait_sleep(QS ? &q_ready[qs] : &q_full[qs], qph);
        const uint32_t q_addr = tc::smem_u32(smem + SMEM_Q + qs * Q_BYTES);
        for (int t = 0; t < ntiles; ++t) {
          const uint32_t idesc = (m - t * BN >= BN) ? idesc256 : idesc128;
          tc::mbar_wait_sleep(&t_empty[acc], aph ^ 1);
          tc::mbar_wait_sleep(&k_full[ks], kph);
          tc::tc_fence_after();
          const uint32_t k_addr = tc::smem_u32(smem + SMEM_K + ks * K_BYTES);
          const uint32_t d_tmem = tmem_base + acc * BN;
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {
            const uint64_t ad = tc::smem_desc(q_addr + kk * 32, 16, 1024, tc::kSwizzle128B);
            const uint64_t bd = tc::smem_desc(k_addr + kk * 32, 16, 1024, tc::kSwizzle128B);
            tc::mma_f16_ss(d_tmem, ad, bd, idesc, kk > 0 ? 1u : 0u);
          }
          tc::mma_commit(&k_empty[ks]);
          tc::mma_commit(&t_full[acc]);
          if (++ks == KSTAGES) { ks = 0; kph ^= 1; }
          if (++acc == NACC) { acc = 0; aph ^= 1; }
        }
        tc::mma_commit(&q_empty[qs]);
      }
    }
  } else if (warp == 3) {
    // ------------------------------------------------------------ Q scaler (PRE)
    // the attention scale is an exact power of two and the inputs bf16 (fp32's exponent range):
    // Q * scale is exact, so the MMA accumulates the post-scale scores directly and the epilogue
    // drops its per-score multiply (4 of ~29 instructions per group)
    if (PRE && std::is_same<T, __nv_bfloat16>::value) {
      const __nv_bfloat162 s2 = __float2bfloat162_rn(scale);
      int it = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
        const int qs = it & 1;
        tc::mbar_wait_sleep(&q_full[qs], (it >> 1) & 1);
        uint4* qv = reinterpret_cast<uint4*>(smem + SMEM_Q + qs * Q_BYTES);
#pragma unroll 4
        for (int i = lane; i < Q_BYTES / 16; i += 32) {
          uint4 u = qv[i];
          __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
          for (int j = 0; j < 4; ++j) h[j] = __hmul2(h[j], s2);
          qv[i] = u;
        }
        tc::fence_proxy_async();  // generic-proxy writes -> the tensor core's async-proxy reads
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&q_ready[qs]);
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    // warp (quad, cq) owns TMEM lanes 32*quad.. (its 32 query rows) and accumulator columns
    // [64*cq, 64*cq+64): 2 chunks of 32 columns, the second TMEM load in flight while the first
    // is pruned.  16 epilogue warps (4 per sub-partition) hide the epilogue's latencies.
    const int ew = warp - 4;
    const int quad = warp & 3;
    const int cq = ew >> 2;
    const int chunks = m / (8 * GS);  // meta chunks of 8 groups per row block
    uint8_t* stg_base = smem + SMEM_STG + ew * 2 * STG_BYTES;
    int acc = 0, sb = 0;
    uint32_t aph = 0;
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
      const int b = item / mblocks, mb = item % mblocks;
      const int row_blk = quad * 32 + lane;  // row within the 128-row block
      const int grow = mb * BM + row_blk;    // row within the head
      uint32_t* meta_b = meta + ((int64_t)b * mblocks + mb) * chunks * 128;
      float mx = -INFINITY;  // running max of this thread's row half (RMAX)
      for (int t = 0; t < ntiles; ++t) {
        const int width = min(BN, m - t * BN);
        const bool active = cq * 64 < width;
        tc::mbar_wait(&t_full[acc], aph);
        tc::tc_fence_after();
        uint8_t* stg = stg_base + sb * STG_BYTES;
        if (active) {
          if (lane == 0) tc::bulk_wait_read<1>();  // staging buffer from two tiles ago drained
          __syncwarp();
          const uint32_t tbase = tmem_base + ((uint32_t)(quad * 32) << 16) + acc * BN + cq * 64;
          const int colh = t * BN + cq * 64;
          const int64_t drow = (int64_t)b * n + grow;
          uint32_t ra[32], rb[32];
          // chunk cc+1 is in flight while cc is pruned
          auto chunk = [&](const uint32_t (&rr)[32], int cc) {
            if constexpr (GS == 4)
              epi_chunk<T, DBG, RMAX, MASK, PRE>(rr, scale, colh, cc, 2 * cc, stg, lane, meta_b, row_blk, dbg, drow, m, mx,
                                            two, tk, grow);
            else
              epi_chunk12<T, DBG, RMAX, MASK, PRE>(rr, scale, colh, cc, 2 * cc, stg, lane, meta_b, row_blk, dbg, drow, m,
                                              mx, tk, grow);
          };
          tc::tmem_ld_32x32b_x32(tbase, ra);
          tc::tmem_ld_wait(ra);
          tc::tmem_ld_32x32b_x32(tbase + 32, rb);
          chunk(ra, 0);
          tc::tmem_ld_wait(rb);
          chunk(rb, 1);
        }
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&t_empty[acc]);
        if (active) {
          tc::fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            tc::tma_store_3d(&tm_nz, stg, t * (BN / 2) + cq * 32, mb * BM + quad * 32, b);
            tc::bulk_commit();
          }
          sb ^= 1;
        }
        if (++acc == NACC) { acc = 0; aph ^= 1; }
      }
      // per-row partial maxima [bh, n, 4] fp32, one per column quarter (fused softmax input)
      if (RMAX) rowmax[((int64_t)b * n + grow) * 4 + cq] = (PRE && std::is_same<T, __half>::value) ? mx * scale : mx;
    }
    if (lane == 0) tc::bulk_wait<0>();
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc::tc_fence_after();
    tc::tmem_dealloc<512>(tmem_base);
  }
}

// ---------------------------------------------------------------- host side

bool tc_sddmm_supported(int gs, int in_dtype, int nz_dtype, int n, int m, int d) {
  return (gs == 4 || gs == 2) && (in_dtype == DFSS_BF16 || in_dtype == DFSS_F16) && nz_dtype == in_dtype && d == HD &&
         n % BM == 0 && m % 128 == 0 && n > 0 && m > 0;
}

static int num_sms() {
  static int cached = 0;
  if (!cached) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
    if (cached <= 0) cached = 148;
  }
  return cached;
}

template <typename T, int GS, bool PRE>
static auto pick_kernel(bool mask, bool dbg, bool rowmax) -> decltype(&sddmm24_tc_kernel<T, GS, false, false, false, PRE>) {
  if (mask) return dbg ? sddmm24_tc_kernel<T, GS, true, false, true, PRE> : sddmm24_tc_kernel<T, GS, false, false, true, PRE>;
  if (dbg) return rowmax ? sddmm24_tc_kernel<T, GS, true, true, false, PRE> : sddmm24_tc_kernel<T, GS, true, false, false, PRE>;
  return rowmax ? sddmm24_tc_kernel<T, GS, false, true, false, PRE> : sddmm24_tc_kernel<T, GS, false, false, false, PRE>;
}

// scale = 2^e, -60 <= e <= 0: bf16 Q * scale is exact (fp32's exponent range); fp16 scores
// (>= 2^-48 when nonzero) times scale stay normal fp32, so scaling them is exact
static bool exact_prescale(float scale) {
  int e = 0;
  return std::isfinite(scale) && scale > 0.f && scale <= 1.f && scale >= 0x1p-60f && std::frexp(scale, &e) == 0.5f;
}

template <typename T, int GS>
static cudaError_t launch_typed(const void* q, const void* k, void* nz, uint32_t* meta, float scale, int64_t bh, int n,
                                int m, float* dbg, float* rowmax, const TileKeepTc& tk, cudaStream_t s) {
  const CUtensorMapDataType dt =
      std::is_same<T, __nv_bfloat16>::value ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  CUtensorMap tq, tkm, tn;
  if (!encode_tmap_3d(&tq, dt, 2, (void*)q, HD, n, bh, HD, BM, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !encode_tmap_3d(&tkm, dt, 2, (void*)k, HD, m, bh, HD, BN, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !encode_tmap_3d(&tn, dt, 2, nz, m / 2, n, bh, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B))
    return cudaErrorInvalidValue;
  auto kern = exact_prescale(scale) ? pick_kernel<T, GS, true>(tk.keep != nullptr, dbg != nullptr, rowmax != nullptr)
                                    : pick_kernel<T, GS, false>(tk.keep != nullptr, dbg != nullptr, rowmax != nullptr);
  if (tk.keep && rowmax) return cudaErrorNotSupported;  // row maxima are unmasked-only
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_TOTAL);
  if (e != cudaSuccess) return e;
  const int items = (int)bh * (n / BM);
  const int grid = items < num_sms() ? items : num_sms();
  kern<<<grid, NUM_THREADS, SMEM_TOTAL, s>>>(tq, tkm, tn, meta, scale, (int)bh, n, m, dbg, rowmax, 2u, tk);
  return cudaGetLastError();
}

cudaError_t launch_sddmm_tc(const void* q, const void* k, void* nz, uint32_t* meta, float scale, int gs, int in_dtype,
                            int64_t bh, int n, int m, int d, float* dbg, float* rowmax, cudaStream_t s,
                            const uint8_t* keep, int tile_rows, int tile_cols) {
  if (!tc_sddmm_supported(gs, in_dtype, in_dtype, n, m, d)) return cudaErrorNotSupported;
  if (bh == 0) return cudaSuccess;
  TileKeepTc tk;
  if (keep) {
    tk.keep = keep;
    tk.tile_rows = tile_rows;
    tk.tile_cols = tile_cols;
    tk.grid_cols = (m + tile_cols - 1) / tile_cols;
  }
  if (gs == 2) {
    if (in_dtype == DFSS_BF16) return launch_typed<__nv_bfloat16, 2>(q, k, nz, meta, scale, bh, n, m, dbg, rowmax, tk, s);
    return launch_typed<__half, 2>(q, k, nz, meta, scale, bh, n, m, dbg, rowmax, tk, s);
  }
  if (in_dtype == DFSS_BF16) return launch_typed<__nv_bfloat16, 4>(q, k, nz, meta, scale, bh, n, m, dbg, rowmax, tk, s);
  return launch_typed<__half, 4>(q, k, nz, meta, scale, bh, n, m, dbg, rowmax, tk, s);
}

}  // namespace dfss
