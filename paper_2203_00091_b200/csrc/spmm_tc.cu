// spmm_tc.cu -- compressed SpMM O = P_sparse . V on tcgen05.mma.sp (2:4, bf16/fp16, d = 64),
// optionally with the row softmax fused in.
//
// Replaces _spmm_gather (_kernels_numba.py:91-103) for the 16-bit path.  The
// compressed P rows ARE the sparse A operand (kept values in ascending column
// order, K-major) and meta_hw words ARE the TMEM metadata columns, so nothing
// is decoded: the SDDMM output is consumed as written.  Persistent,
// warp-specialised, one CTA per SM:
//   warp 0       TMA producer: P tile (128 rows x 64 stored = 128 logical K) and
//                V tile (128 K-rows x 64, MN-major) per stage, STAGES-deep ring;
//   warp 1       MMA issuer: 4 x tcgen05.mma.sp.kind::f16 (M=128, N=64, K=32) per
//                stage, metadata column s*4+kk, accumulator double-buffered;
//   warp 2       TMEM allocator;
//   warps 4-7    metadata loaders: warp w copies the words of TMEM lanes
//                32*(w%4).. for the stage's 4 K-chunks global -> tcgen05.st;
//   warps 8-11   epilogue: TMEM -> registers (x 1/rowsum when fused) -> O rows;
//   warps 12-19  (SOFTMAX only) transform: warp (quad, half) rewrites the
//                4 16-byte chunks [4*half, 4*half+4) of rows 32*quad.. of the
//                staged P tile in smem as exp(s - m_r) (m_r = row max from the
//                SDDMM epilogue, so no rescaling pass) and accumulates partial row
//                sums -- softmax_rows (sparse_ops.py:18-37) fused between TMA and
//                MMA; two warps per SM sub-partition hide the MUFU latency.
#include <math_constants.h>

#include <type_traits>

#include "dfss_common.cuh"
#include "tc_common.cuh"

namespace dfss {

namespace {
constexpr int BM = 128;
constexpr int HD = 64;
constexpr int BKL = 128;  // logical K per stage
constexpr int STAGES = 6;
constexpr int NACC = 2;
constexpr int P_BYTES = BM * (BKL / 2) * 2;  // 16 KB
constexpr int V_BYTES = BKL * HD * 2;        // 16 KB
constexpr int SMEM_P = 0;
constexpr int SMEM_V = SMEM_P + STAGES * P_BYTES;
constexpr int SMEM_L = SMEM_V + STAGES * V_BYTES;  // [NACC][2][128] partial row sums (fused softmax)
constexpr int SMEM_BAR = SMEM_L + NACC * 2 * BM * 4;
constexpr int XF_WARPS = 8;
constexpr int SMEM_TOTAL = SMEM_BAR + 512 + 1024;
constexpr int TMEM_COLS = 256;
constexpr int E_COL0 = NACC * HD;  // metadata columns start after the accumulators
constexpr float kLog2e = 1.4426950408889634f;
}  // namespace

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <typename T>
__device__ __forceinline__ float2 unpack2(uint32_t u);
template <>
__device__ __forceinline__ float2 unpack2<__nv_bfloat16>(uint32_t u) {
  return make_float2(__uint_as_float(u << 16), __uint_as_float(u & 0xFFFF0000u));
}
template <>
__device__ __forceinline__ float2 unpack2<__half>(uint32_t u) {
  __half2 h = *reinterpret_cast<__half2*>(&u);
  return __half22float2(h);
}
template <typename T>
__device__ __forceinline__ uint32_t pack2f(float lo, float hi);
template <>
__device__ __forceinline__ uint32_t pack2f<__nv_bfloat16>(float lo, float hi) {
  __nv_bfloat162 p = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&p);
}
template <>
__device__ __forceinline__ uint32_t pack2f<__half>(float lo, float hi) {
  __half2 p = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&p);
}

// 1:2 metadata (include/dfss.h: one nibble 0x4 / 0xE per pair, meta chunks of 8 pairs) as the
// tcgen05 2:4 pattern "one survivor per pair" (nibble 8 + a + 4b: elements a and 2 + b of each
// group of 4): the 1:2 nonzeros already ARE that pattern's stored values in order, so only the
// metadata is rewritten -- the word of TMEM lane L (m2, k1, m0) for the 32-key chunk kk is built
// from the 1:2 words of chunk 2 kk + k1 at lanes 16 m2 + m0 (pairs 0-3) and 16 m2 + 8 + m0
// (pairs 4-7), bit 3 of a 1:2 nibble being "element 1 kept".
__device__ __forceinline__ uint32_t meta12_to_24(uint32_t w0, uint32_t w1) {
  const uint32_t x0 = (w0 >> 3) & 0x11111111u, x1 = (w1 >> 3) & 0x11111111u;
  // byte k of v = the 2:4 nibble of source pairs (2k, 2k + 1) of the word
  const uint32_t v0 = (x0 & 0x01010101u) | ((x0 & 0x10101010u) >> 2) | 0x08080808u;
  const uint32_t v1 = (x1 & 0x01010101u) | ((x1 & 0x10101010u) >> 2) | 0x08080808u;
  return (v0 & 0x000F000Fu) | ((v0 & 0x0F000F00u) >> 4) | ((v1 & 0x000F000Fu) << 8) | ((v1 & 0x0F000F00u) << 4);
}

// BlockMask for the tcgen05 SpMM (MASKZ): the transform warps zero the absent nonzeros of each
// staged P tile before its MMAs (the reference skips them, sparse_ops.py:57-64), so whatever a
// caller left in the absent slots never reaches the product.
struct SpmmKeep {
  const uint8_t* keep = nullptr;
  int tile_rows = 1, tile_cols = 2, grid_cols = 0;
};

template <typename T, typename TO, bool SOFTMAX, int GS, bool MASKZ = false>
__global__ void __launch_bounds__(SOFTMAX || MASKZ ? 640 : 384, 1)
    spmm24_tc_kernel(const __grid_constant__ CUtensorMap tm_p, const __grid_constant__ CUtensorMap tm_v,
                     const uint32_t* __restrict__ meta, TO* __restrict__ out, int bh, int rows, int n_k,
                     const float* __restrict__ rowmax, SpmmKeep mk) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = (uint64_t*)(smem + SMEM_BAR);
  uint64_t* full = bars;                 // [STAGES] TMA bytes landed
  uint64_t* e_full = full + STAGES;      // [STAGES] metadata columns written (4 warps)
  uint64_t* empty = e_full + STAGES;     // [STAGES] MMAs of the stage retired
  uint64_t* p_ready = empty + STAGES;    // [STAGES] (SOFTMAX) P tile rewritten as exp (4 warps)
  uint64_t* d_full = p_ready + STAGES;   // [NACC]
  uint64_t* d_empty = d_full + NACC;     // [NACC] (4 epilogue warps)
  uint64_t* l_full = d_empty + NACC;     // [NACC] (SOFTMAX) row sums in smem (4 warps)
  uint32_t* tmem_slot = (uint32_t*)(l_full + NACC);
  float* lsum = (float*)(smem + SMEM_L);

  const uint32_t warp = tc::warp_id();
  const uint32_t lane = threadIdx.x & 31;
  const int rblocks = rows / BM;
  const int items = bh * rblocks;
  const int kblocks = n_k / BKL;
  const int chunks = n_k / (8 * GS);  // meta_hw chunks per row block

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tm_p);
    tc::prefetch_tmap(&tm_v);
    for (int i = 0; i < STAGES; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&e_full[i], 4);
      tc::mbar_init(&empty[i], 1);
      tc::mbar_init(&p_ready[i], XF_WARPS);
    }
    for (int i = 0; i < NACC; ++i) {
      tc::mbar_init(&d_full[i], 1);
      tc::mbar_init(&d_empty[i], 4);
      tc::mbar_init(&l_full[i], XF_WARPS);
    }
    tc::fence_barrier_init();
  }
  if (warp == 2) tc::tmem_alloc<TMEM_COLS>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x) {
        const int b = item / rblocks, rb = item % rblocks;
        for (int kb = 0; kb < kblocks; ++kb) {
          tc::mbar_wait(&empty[s], ph ^ 1);
          tc::mbar_arrive_expect_tx(&full[s], P_BYTES + V_BYTES);
          tc::tma_load_3d(smem + SMEM_P + s * P_BYTES, &tm_p, &full[s], kb * (BKL / 2), rb * BM, b);
          tc::tma_load_3d(smem + SMEM_V + s * V_BYTES, &tm_v, &full[s], 0, kb * BKL, b);
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t fmt = std::is_same<T, __nv_bfloat16>::value ? 1u : 0u;
      constexpr uint32_t idesc = tc::instr_desc(fmt, BM, HD, /*a_mn=*/false, /*b_mn=*/true, /*sparse=*/true);
      int s = 0, acc = 0;
      uint32_t ph = 0, aph = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x) {
        tc::mbar_wait(&d_empty[acc], aph ^ 1);
        const uint32_t d_tmem = tmem_base + acc * HD;
        for (int kb = 0; kb < kblocks; ++kb) {
          tc::mbar_wait(&full[s], ph);
          if (SOFTMAX || MASKZ) tc::mbar_wait(&p_ready[s], ph);
          tc::mbar_wait(&e_full[s], ph);
          tc::tc_fence_after();
          const uint32_t p_addr = tc::smem_u32(smem + SMEM_P + s * P_BYTES);
          const uint32_t v_addr = tc::smem_u32(smem + SMEM_V + s * V_BYTES);
#pragma unroll
          for (int kk = 0; kk < BKL / 32; ++kk) {
            // A: K-major, 16 stored elements (32 B) per MMA inside the 128B swizzle row
            const uint64_t ad = tc::smem_desc(p_addr + kk * 32, 16, 1024, tc::kSwizzle128B);
            // B: MN-major, 32 K-rows of 128 B per MMA = 4 whole swizzle atoms
            const uint64_t bd = tc::smem_desc(v_addr + kk * 32 * 128, V_BYTES, 1024, tc::kSwizzle128B);
            // metadata column: even address + sparse_id2 (idesc bits [0,2)) selects the odd one
            const uint32_t e_col = tmem_base + E_COL0 + s * 4 + kk;
            tc::mma_sp_f16_ss(d_tmem, ad, bd, e_col & ~1u, idesc | (e_col & 1u), (kb | kk) ? 1u : 0u);
          }
          tc::mma_commit(&empty[s]);
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
        tc::mma_commit(&d_full[acc]);
        if (++acc == NACC) { acc = 0; aph ^= 1; }
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ------------------------------------------------------------ metadata -> TMEM
    const int quad = warp & 3;
    int s = 0;
    uint32_t ph = 0;
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
      const int b = item / rblocks, rb = item % rblocks;
      const uint32_t* mrow = meta + ((int64_t)b * rblocks + rb) * chunks * 128 + quad * 32 + lane;
      // 1:2: this lane's source words are at lanes 16 m2 + m0 and + 8 of chunk 2 kk + k1
      const int L = quad * 32 + (int)lane;
      const uint32_t* mrow12 = meta + ((int64_t)b * rblocks + rb) * chunks * 128 + 16 * (L >> 4) + (L & 7);
      const int k1 = (L >> 3) & 1;
      for (int kb = 0; kb < kblocks; ++kb) {
        uint32_t w0, w1, w2, w3;
        if constexpr (GS == 4) {
          w0 = __ldg(mrow + (int64_t)(kb * 4 + 0) * 128);
          w1 = __ldg(mrow + (int64_t)(kb * 4 + 1) * 128);
          w2 = __ldg(mrow + (int64_t)(kb * 4 + 2) * 128);
          w3 = __ldg(mrow + (int64_t)(kb * 4 + 3) * 128);
        } else {
          uint32_t src[8];
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint32_t* c = mrow12 + (int64_t)(kb * 8 + 2 * kk + k1) * 128;
            src[2 * kk] = __ldg(c);
            src[2 * kk + 1] = __ldg(c + 8);
          }
          w0 = meta12_to_24(src[0], src[1]);
          w1 = meta12_to_24(src[2], src[3]);
          w2 = meta12_to_24(src[4], src[5]);
          w3 = meta12_to_24(src[6], src[7]);
        }
        tc::mbar_wait(&empty[s], ph ^ 1);
        tc::tc_fence_after();
        tc::tmem_st_32x32b_x4(tmem_base + ((uint32_t)(quad * 32) << 16) + E_COL0 + s * 4, w0, w1, w2, w3);
        tc::tmem_st_wait();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&e_full[s]);
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp >= 8 && warp < 12) {
    // ------------------------------------------------------------ epilogue
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    int acc = 0;
    uint32_t aph = 0;
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
      const int b = item / rblocks, rb = item % rblocks;
      tc::mbar_wait(&d_full[acc], aph);
      float inv = 1.f;
      if (SOFTMAX) {
        tc::mbar_wait(&l_full[acc], aph);
        inv = 1.0f / (lsum[(acc * 2 + 0) * BM + r] + lsum[(acc * 2 + 1) * BM + r]);
      }
      tc::tc_fence_after();
      uint32_t r0[32], r1[32];
      const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + acc * HD;
      tc::tmem_ld_32x32b_x32(taddr, r0);
      tc::tmem_ld_32x32b_x32(taddr + 32, r1);
      tc::tmem_ld_wait(r0);
      tc::tmem_ld_wait(r1);
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&d_empty[acc]);
      TO* orow = out + ((int64_t)b * rows + rb * BM + r) * HD;
      if constexpr (std::is_same<TO, float>::value) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          reinterpret_cast<float4*>(orow)[j] =
              make_float4(__uint_as_float(r0[4 * j]) * inv, __uint_as_float(r0[4 * j + 1]) * inv,
                          __uint_as_float(r0[4 * j + 2]) * inv, __uint_as_float(r0[4 * j + 3]) * inv);
          reinterpret_cast<float4*>(orow)[8 + j] =
              make_float4(__uint_as_float(r1[4 * j]) * inv, __uint_as_float(r1[4 * j + 1]) * inv,
                          __uint_as_float(r1[4 * j + 2]) * inv, __uint_as_float(r1[4 * j + 3]) * inv);
        }
      } else {
        uint32_t pk[32];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          pk[j] = pack2f<TO>(__uint_as_float(r0[2 * j]) * inv, __uint_as_float(r0[2 * j + 1]) * inv);
          pk[16 + j] = pack2f<TO>(__uint_as_float(r1[2 * j]) * inv, __uint_as_float(r1[2 * j + 1]) * inv);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)
          reinterpret_cast<uint4*>(orow)[j] = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
      }
      if (++acc == NACC) { acc = 0; aph ^= 1; }
    }
  } else if (MASKZ && warp >= 12) {
    // ------------------------------------------------------------ BlockMask: zero absent nonzeros
    // warp (quad, half): row r of the block, 16-byte units 4 half .. 4 half + 3 (8 nonzeros =
    // 16 dense columns each) of the 128B-swizzled P row
    const int quad = warp & 3;
    const int half = (warp - 12) >> 2;
    const int r = quad * 32 + lane;
    const bool unit_tiles = mk.tile_cols % 16 == 0;  // a unit lies in one tile: one lookup, no read
    int s = 0;
    uint32_t ph = 0;
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
      const int rb = item % rblocks;
      const uint8_t* krow = mk.keep + (int64_t)((rb * BM + r) / mk.tile_rows) * mk.grid_cols;
      for (int kb = 0; kb < kblocks; ++kb) {
        tc::mbar_wait(&full[s], ph);
        uint8_t* prow = smem + SMEM_P + s * P_BYTES + r * 128;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int u = 4 * half + c;
          const int d0 = 2 * (kb * (BKL / 2) + 8 * u);  // first dense column of the unit
          uint4* dst = reinterpret_cast<uint4*>(prow + ((u ^ (r & 7)) << 4));
          if (unit_tiles) {
            if (!__ldg(krow + d0 / mk.tile_cols)) *dst = make_uint4(0u, 0u, 0u, 0u);
          } else {
            uint4 x = *dst;
            uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int e = 0; e < 8; ++e)
              if (!__ldg(krow + (d0 + 2 * e) / mk.tile_cols)) w[e >> 1] &= (e & 1) ? 0x0000ffffu : 0xffff0000u;
            *dst = make_uint4(w[0], w[1], w[2], w[3]);
          }
        }
        tc::fence_proxy_async();  // generic-proxy smem writes -> visible to the tensor core
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&p_ready[s]);
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
    }
  } else if (SOFTMAX && warp >= 12) {
    // ------------------------------------------------------------ softmax transform
    const int quad = warp & 3;
    const int half = (warp - 12) >> 2;
    const int r = quad * 32 + lane;  // row within the 128-row block == TMEM lane
    int s = 0, acc = 0;
    uint32_t ph = 0, aph = 0;
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
      const int b = item / rblocks, rb = item % rblocks;
      const float4 mp = *reinterpret_cast<const float4*>(rowmax + ((int64_t)b * rows + rb * BM + r) * 4);
      const float mb = fmaxf(fmaxf(mp.x, mp.y), fmaxf(mp.z, mp.w)) * kLog2e;
      float l0 = 0.f, l1 = 0.f;
      for (int kb = 0; kb < kblocks; ++kb) {
        tc::mbar_wait(&full[s], ph);
        uint8_t* prow = smem + SMEM_P + s * P_BYTES + r * 128;
        uint4 x[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) x[c] = *reinterpret_cast<const uint4*>(prow + (((4 * half + c) ^ (r & 7)) << 4));
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t w[4] = {x[c].x, x[c].y, x[c].z, x[c].w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float2 f = unpack2<T>(w[j]);
            const float e0 = ex2_approx(fmaf(f.x, kLog2e, -mb));
            const float e1 = ex2_approx(fmaf(f.y, kLog2e, -mb));
            l0 += e0;
            l1 += e1;
            w[j] = pack2f<T>(e0, e1);
          }
          *reinterpret_cast<uint4*>(prow + (((4 * half + c) ^ (r & 7)) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        tc::fence_proxy_async();  // generic-proxy smem writes -> visible to the tensor core
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&p_ready[s]);
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
      // hand the partial row sums to the epilogue (buffer acc is free once its previous O was drained)
      tc::mbar_wait(&d_empty[acc], aph ^ 1);
      lsum[(acc * 2 + half) * BM + r] = l0 + l1;
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&l_full[acc]);
      if (++acc == NACC) { acc = 0; aph ^= 1; }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc::tc_fence_after();
    tc::tmem_dealloc<TMEM_COLS>(tmem_base);
  }
}

bool tc_spmm_supported(int gs, int p_dtype, int v_dtype, int out_dtype, int rows, int n_k, int d) {
  return (gs == 4 || gs == 2) && (p_dtype == DFSS_BF16 || p_dtype == DFSS_F16) && v_dtype == p_dtype &&
         (out_dtype == p_dtype || out_dtype == DFSS_F32) && d == HD && rows % BM == 0 && n_k % BKL == 0 && rows > 0;
}

static int num_sms_spmm() {
  static int cached = 0;
  if (!cached) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
    if (cached <= 0) cached = 148;
  }
  return cached;
}

template <typename T, typename TO, int GS>
static cudaError_t spmm_launch_typed(const void* p, const uint32_t* meta, const void* v, void* out, int64_t bh, int rows,
                                     int n_k, const float* rowmax, const SpmmKeep& mk, cudaStream_t s) {
  const CUtensorMapDataType dt =
      std::is_same<T, __nv_bfloat16>::value ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  CUtensorMap tp, tv;
  if (!encode_tmap_3d(&tp, dt, 2, (void*)p, n_k / 2, rows, bh, BKL / 2, BM, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !encode_tmap_3d(&tv, dt, 2, (void*)v, HD, n_k, bh, HD, BKL, CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  const int items = (int)bh * (rows / BM);
  const int grid = items < num_sms_spmm() ? items : num_sms_spmm();
  if (rowmax && mk.keep) return cudaErrorNotSupported;  // the fused softmax is unmasked-only
  if (rowmax) {
    auto kern = spmm24_tc_kernel<T, TO, true, GS>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_TOTAL);
    if (e != cudaSuccess) return e;
    kern<<<grid, 640, SMEM_TOTAL, s>>>(tp, tv, meta, (TO*)out, (int)bh, rows, n_k, rowmax, mk);
  } else if (mk.keep) {
    auto kern = spmm24_tc_kernel<T, TO, false, GS, true>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_TOTAL);
    if (e != cudaSuccess) return e;
    kern<<<grid, 640, SMEM_TOTAL, s>>>(tp, tv, meta, (TO*)out, (int)bh, rows, n_k, nullptr, mk);
  } else {
    auto kern = spmm24_tc_kernel<T, TO, false, GS>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_TOTAL);
    if (e != cudaSuccess) return e;
    kern<<<grid, 384, SMEM_TOTAL, s>>>(tp, tv, meta, (TO*)out, (int)bh, rows, n_k, nullptr, mk);
  }
  return cudaGetLastError();
}

cudaError_t launch_spmm_tc(const void* p, const uint32_t* meta, const void* v, void* out, int gs, int dtype,
                           int out_dtype, int64_t bh, int rows, int n_k, int d, const float* rowmax, cudaStream_t s,
                           const uint8_t* keep, int tile_rows, int tile_cols) {
  if (!tc_spmm_supported(gs, dtype, dtype, out_dtype, rows, n_k, d)) return cudaErrorNotSupported;
  if (bh == 0) return cudaSuccess;
  SpmmKeep mk;
  if (keep) {
    mk.keep = keep;
    mk.tile_rows = tile_rows;
    mk.tile_cols = tile_cols;
    mk.grid_cols = (n_k + tile_cols - 1) / tile_cols;
  }
  auto go = [&](auto gs_tag) {
    constexpr int G = decltype(gs_tag)::value;
    if (dtype == DFSS_BF16)
      return out_dtype == DFSS_F32
                 ? spmm_launch_typed<__nv_bfloat16, float, G>(p, meta, v, out, bh, rows, n_k, rowmax, mk, s)
                 : spmm_launch_typed<__nv_bfloat16, __nv_bfloat16, G>(p, meta, v, out, bh, rows, n_k, rowmax, mk, s);
    return out_dtype == DFSS_F32 ? spmm_launch_typed<__half, float, G>(p, meta, v, out, bh, rows, n_k, rowmax, mk, s)
                                 : spmm_launch_typed<__half, __half, G>(p, meta, v, out, bh, rows, n_k, rowmax, mk, s);
  };
  return gs == 2 ? go(std::integral_constant<int, 2>{}) : go(std::integral_constant<int, 4>{});
}

}  // namespace dfss
