// flash_tc.cu -- fully fused DFSS attention on tcgen05 (2:4, bf16/fp16, head dim 64).
//
// pipeline.nm_attention (pipeline.py:15-32) in one kernel, with no n x n tensor of
// any kind in HBM:
//   phase A  S_t = Q K_t^T for every 128-key tile t -> TMEM; softmax warps reduce the
//            row maximum (the row maximum is always kept by 2:4, so this is the max of
//            the kept scores, the softmax shift of _softmax_nonzeros, _kernels_numba.py:66-84);
//   phase B  S_t again -> TMEM; softmax warps scale, prune 2-of-4 with select24 (the
//            reference rule, codec.py:104-123), exponentiate ONLY the kept half,
//            accumulate row sums, write the kept probabilities as the compressed sparse
//            A operand (K-major, 128B-swizzled smem) and the nibbles as tcgen05.mma.sp
//            metadata (tcgen05.st into TMEM, layout include/dfss.h); the MMA warp then
//            issues O += P_sparse . V_t with tcgen05.mma.sp (_spmm_gather, :91-103);
//   end      O / rowsum -> HBM.
// The two-phase max avoids any O rescaling.  K/V tiles stream through TMA rings;
// S is double-buffered in TMEM so the tensor core computes S_{t+1} while the softmax
// warps prune S_t.  Warp roles (one CTA per SM, persistent over (bh, 128-row block)):
//   warp 0 TMA producer (Q, K), warp 3 TMA producer (V), warp 1 MMA issuer, warp 2 TMEM allocator,
//   warps 4-19 softmax (warp (quad, quarter): TMEM lanes 32*quad.., columns [32*quarter, +32);
//   four warps per SM sub-partition hide TMEM / MUFU latency), the quarter-0 warps also
//   write the output rows.
#include <stdlib.h>

#include <type_traits>

#include "dfss_common.cuh"
#include "tc_common.cuh"

namespace dfss {

namespace {
constexpr int BM = 128;   // query rows per item (TMEM lanes)
constexpr int BN = 128;   // keys per tile
constexpr int HD = 64;    // head dim
constexpr int KST = 4;    // K ring
constexpr int VST = 3;    // V ring
constexpr int PST = 2;    // P (smem) + E (TMEM) stages
constexpr int SM_WARPS = 16;
constexpr int NUM_THREADS = (4 + SM_WARPS) * 32;
constexpr int Q_BYTES = BM * HD * 2;       // 16 KB
constexpr int K_BYTES = BN * HD * 2;       // 16 KB
constexpr int V_BYTES = BN * HD * 2;       // 16 KB
constexpr int P_BYTES = BM * (BN / 2) * 2;  // 16 KB: 128 rows x 64 kept values
constexpr int SMEM_Q = 0;
constexpr int SMEM_K = SMEM_Q + 2 * Q_BYTES;
constexpr int SMEM_V = SMEM_K + KST * K_BYTES;
constexpr int SMEM_P = SMEM_V + VST * V_BYTES;
constexpr int SMEM_RED = SMEM_P + PST * P_BYTES;  // [2][4 quarters][128] floats: row max / row sum exchange
constexpr int SMEM_BAR = SMEM_RED + 2 * 4 * BM * 4;
constexpr int SMEM_TOTAL = SMEM_BAR + 512 + 1024;
constexpr int SBUF = 3;             // S tiles in flight
constexpr int TM_S = 0;             // SBUF x 128 columns of scores
constexpr int TM_O = SBUF * BN;     // 64 columns of output accumulator
constexpr int TM_E = TM_O + HD;     // PST x 4 metadata columns
constexpr float kLog2e = 1.4426950408889634f;
}  // namespace

__device__ __forceinline__ float fex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <typename T>
__device__ __forceinline__ uint32_t fpack2(float lo, float hi) {
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    __nv_bfloat162 p = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&p);
  } else {
    __half2 p = __floats2half2_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&p);
  }
}

template <typename T>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    dfss_flash_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                      const __grid_constant__ CUtensorMap tm_v, T* __restrict__ out, float scale, int bh, int n,
                      uint32_t two, int dbg) {
  // dbg (timing experiments only, results invalid when non-zero): bit0 skip phase A,
  // bit1 skip the PV MMAs, bit2 skip the prune/exp arithmetic, bit3 skip V loads, bit4 skip K loads
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = (uint64_t*)(smem + SMEM_BAR);
  uint64_t* q_full = bars;               // [2]
  uint64_t* q_empty = q_full + 2;        // [2]
  uint64_t* k_full = q_empty + 2;        // [KST]
  uint64_t* k_empty = k_full + KST;      // [KST]
  uint64_t* v_full = k_empty + KST;      // [VST]
  uint64_t* v_empty = v_full + VST;      // [VST]
  uint64_t* s_full = v_empty + VST;      // [SBUF] S tile in TMEM
  uint64_t* s_empty = s_full + SBUF;     // [SBUF] (SM_WARPS)
  uint64_t* p_full = s_empty + SBUF;     // [PST] P smem + E TMEM written (SM_WARPS)
  uint64_t* p_empty = p_full + PST;      // [PST] PV MMAs retired
  uint64_t* o_full = p_empty + PST;      // [1] item's last PV retired
  uint64_t* o_empty = o_full + 1;        // [1] O drained (4 output warps)
  uint32_t* tmem_slot = (uint32_t*)(o_empty + 1);
  float* red = (float*)(smem + SMEM_RED);

  const uint32_t warp = tc::warp_id();
  const uint32_t lane = threadIdx.x & 31;
  const int mblocks = n / BM;
  const int items = bh * mblocks;
  const int ntiles = n / BN;

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tm_q);
    tc::prefetch_tmap(&tm_k);
    tc::prefetch_tmap(&tm_v);
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&q_full[i], 1);
      tc::mbar_init(&q_empty[i], 1);
    }
    for (int i = 0; i < SBUF; ++i) {
      tc::mbar_init(&s_full[i], 1);
      tc::mbar_init(&s_empty[i], SM_WARPS);
    }
    for (int i = 0; i < KST; ++i) {
      tc::mbar_init(&k_full[i], 1);
      tc::mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < VST; ++i) {
      tc::mbar_init(&v_full[i], 1);
      tc::mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < PST; ++i) {
      tc::mbar_init(&p_full[i], SM_WARPS);
      tc::mbar_init(&p_empty[i], 1);
    }
    tc::mbar_init(o_full, 1);
    tc::mbar_init(o_empty, 4);
    tc::fence_barrier_init();
  }
  if (warp == 2) tc::tmem_alloc<512>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer: Q and K
    if (lane == 0) {
      int ks = 0, it = 0;
      uint32_t kph = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
        const int b = item / mblocks, mb = item % mblocks;
        const int qs = it & 1;
        tc::mbar_wait(&q_empty[qs], ((it >> 1) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(&q_full[qs], Q_BYTES);
        tc::tma_load_3d(smem + SMEM_Q + qs * Q_BYTES, &tm_q, &q_full[qs], 0, mb * BM, b);
        for (int pass = (dbg & 1); pass < 2; ++pass) {
          for (int t = 0; t < ntiles; ++t) {
            tc::mbar_wait(&k_empty[ks], kph ^ 1);
            if (dbg & 16) {
              tc::mbar_arrive(&k_full[ks]);
            } else {
              tc::mbar_arrive_expect_tx(&k_full[ks], K_BYTES);
              tc::tma_load_3d(smem + SMEM_K + ks * K_BYTES, &tm_k, &k_full[ks], 0, t * BN, b);
            }
            if (++ks == KST) { ks = 0; kph ^= 1; }
          }
        }
      }
    }
  } else if (warp == 3) {
    // ------------------------------------------------------------ TMA producer: V (phase B only)
    if (lane == 0) {
      int vs = 0;
      uint32_t vph = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x) {
        const int b = item / mblocks;
        for (int t = 0; t < ntiles; ++t) {
          tc::mbar_wait(&v_empty[vs], vph ^ 1);
          if (dbg & 8) {
            tc::mbar_arrive(&v_full[vs]);
          } else {
            tc::mbar_arrive_expect_tx(&v_full[vs], V_BYTES);
            tc::tma_load_3d(smem + SMEM_V + vs * V_BYTES, &tm_v, &v_full[vs], 0, t * BN, b);
          }
          if (++vs == VST) { vs = 0; vph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ S issuer: S_t = Q K_t^T, up to SBUF ahead
    if (lane == 0) {
      constexpr uint32_t fmt = std::is_same<T, __nv_bfloat16>::value ? 1u : 0u;
      constexpr uint32_t idesc_s = tc::instr_desc(fmt, BM, BN, false, false, false);
      int ks = 0, sb = 0, it = 0;
      uint32_t kph = 0, sph = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
        const int qs = it & 1;
        tc::mbar_wait(&q_full[qs], (it >> 1) & 1);
        const uint32_t q_addr = tc::smem_u32(smem + SMEM_Q + qs * Q_BYTES);
        const int total = ((dbg & 1) ? 1 : 2) * ntiles;  // phase A (row maxima) + phase B
        for (int t = 0; t < total; ++t) {
          tc::mbar_wait(&s_empty[sb], sph ^ 1);
          tc::mbar_wait(&k_full[ks], kph);
          tc::tc_fence_after();
          const uint32_t k_addr = tc::smem_u32(smem + SMEM_K + ks * K_BYTES);
          if (dbg & 64) {
            tc::mbar_arrive(&k_empty[ks]);
            tc::mbar_arrive(&s_full[sb]);
          } else {
#pragma unroll
            for (int kk = 0; kk < HD / 16; ++kk) {
              const uint64_t ad = tc::smem_desc(q_addr + kk * 32, 16, 1024, tc::kSwizzle128B);
              const uint64_t bd = tc::smem_desc(k_addr + kk * 32, 16, 1024, tc::kSwizzle128B);
              tc::mma_f16_ss(tmem_base + TM_S + sb * BN, ad, bd, idesc_s, kk > 0 ? 1u : 0u);
            }
            tc::mma_commit(&k_empty[ks]);
            tc::mma_commit(&s_full[sb]);
          }
          if (++ks == KST) { ks = 0; kph ^= 1; }
          if (++sb == SBUF) { sb = 0; sph ^= 1; }
        }
        tc::mma_commit(&q_empty[qs]);
      }
    }
  } else if (warp == 2) {
    // ------------------------------------------------------------ PV issuer: O += P_sparse V_t
    if (lane == 0) {
      constexpr uint32_t fmt = std::is_same<T, __nv_bfloat16>::value ? 1u : 0u;
      constexpr uint32_t idesc_pv = tc::instr_desc(fmt, BM, HD, false, true, true);
      int vs = 0, pb = 0;
      uint32_t vph = 0, pph = 0, oph = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x) {
        tc::mbar_wait(o_empty, oph ^ 1);
        for (int t = 0; t < ntiles; ++t) {
          tc::mbar_wait(&p_full[pb], pph);
          tc::mbar_wait(&v_full[vs], vph);
          tc::tc_fence_after();
          if (dbg & 2) {
            tc::mbar_arrive(&p_empty[pb]);
            tc::mbar_arrive(&v_empty[vs]);
          } else {
            const uint32_t p_addr = tc::smem_u32(smem + SMEM_P + pb * P_BYTES);
            const uint32_t v_addr = tc::smem_u32(smem + SMEM_V + vs * V_BYTES);
#pragma unroll
            for (int kk = 0; kk < BN / 32; ++kk) {
              const uint64_t ad = tc::smem_desc(p_addr + kk * 32, 16, 1024, tc::kSwizzle128B);
              const uint64_t bd = tc::smem_desc(v_addr + kk * 32 * 128, V_BYTES, 1024, tc::kSwizzle128B);
              const uint32_t e_col = tmem_base + TM_E + pb * 4 + kk;
              tc::mma_sp_f16_ss(tmem_base + TM_O, ad, bd, e_col & ~1u, idesc_pv | (e_col & 1u),
                                (t == 0 && kk == 0) ? 0u : 1u);
            }
            tc::mma_commit(&p_empty[pb]);
            tc::mma_commit(&v_empty[vs]);
          }
          if (++pb == PST) { pb = 0; pph ^= 1; }
          if (++vs == VST) { vs = 0; vph ^= 1; }
        }
        if (dbg & 2)
          tc::mbar_arrive(o_full);
        else
          tc::mma_commit(o_full);
        oph ^= 1;
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax / prune warps
    const int sw = warp - 4;
    const int quad = warp & 3;
    const int quarter = sw >> 2;
    const int r = quad * 32 + lane;  // row within the item == TMEM lane
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    const uint32_t quad_bar = 1 + quad;  // the 4 warps sharing these rows
    int sb = 0, pb = 0;
    uint32_t sph = 0, pph = 0, oph = 0;
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
      const int b = item / mblocks, mb = item % mblocks;
      // ---- phase A: row maximum over this warp's 32 columns of every tile
      float mx = (dbg & 1) ? 0.f : -INFINITY;
      for (int t = 0; t < ((dbg & 1) ? 0 : ntiles); ++t) {
        tc::mbar_wait(&s_full[sb], sph);
        tc::tc_fence_after();
        uint32_t ra[32];
        tc::tmem_ld_32x32b_x32(tmem_base + lane_base + TM_S + sb * BN + quarter * 32, ra);
        tc::tmem_ld_wait(ra);
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&s_empty[sb]);
#pragma unroll
        for (int j = 0; j < 32; j += 2) mx = fmaxf(mx, fmaxf(__uint_as_float(ra[j]), __uint_as_float(ra[j + 1])));
        if (++sb == SBUF) { sb = 0; sph ^= 1; }
      }
      red[quarter * BM + r] = mx;
      tc::named_bar_sync(quad_bar, 128);
      // max of the scaled scores == scaled max (scale > 0, rounding is monotone)
      const float m =
          scale_canon(fmaxf(fmaxf(red[r], red[BM + r]), fmaxf(red[2 * BM + r], red[3 * BM + r])), scale);
      const float mlog = m * kLog2e;
      // ---- phase B: prune, exponentiate the kept half, stage P + metadata, row sums.
      // Software-pipelined over tiles: the TMEM load of S_{t+1} is in flight while S_t is pruned.
      float l = 0.f;
      uint32_t sa[32], sn[32];
      if (dbg & 32) {
        for (int t = 0; t < ntiles; ++t) {
          tc::mbar_wait(&s_full[sb], sph);
          if (lane == 0) tc::mbar_arrive(&s_empty[sb]);
          if (++sb == SBUF) { sb = 0; sph ^= 1; }
          tc::mbar_wait(&p_empty[pb], pph ^ 1);
          if (lane == 0) tc::mbar_arrive(&p_full[pb]);
          if (++pb == PST) { pb = 0; pph ^= 1; }
        }
      } else {
      tc::mbar_wait(&s_full[sb], sph);
      tc::tc_fence_after();
      tc::tmem_ld_32x32b_x32(tmem_base + lane_base + TM_S + sb * BN + quarter * 32, sn);
      for (int t = 0; t < ntiles; ++t) {
        tc::tmem_ld_wait(sn);
#pragma unroll
        for (int j = 0; j < 32; ++j) sa[j] = sn[j];
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&s_empty[sb]);  // S buffer free: MMA may compute S_{t+2}
        if (++sb == SBUF) { sb = 0; sph ^= 1; }
        if (t + 1 < ntiles) {
          tc::mbar_wait(&s_full[sb], sph);
          tc::tc_fence_after();
          tc::tmem_ld_32x32b_x32(tmem_base + lane_base + TM_S + sb * BN + quarter * 32, sn);
        }
        uint32_t packed[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        uint32_t W = (dbg & 4) ? 0x44444444u : 0u;
#pragma unroll
        for (int g = 0; g < ((dbg & 4) ? 0 : 8); ++g) {
          const float v0 = scale_canon(__uint_as_float(sa[4 * g + 0]), scale);
          const float v1 = scale_canon(__uint_as_float(sa[4 * g + 1]), scale);
          const float v2 = scale_canon(__uint_as_float(sa[4 * g + 2]), scale);
          const float v3 = scale_canon(__uint_as_float(sa[4 * g + 3]), scale);
          float lo, hi;
          const uint32_t nib = select24(v0, v1, v2, v3, lo, hi, two);
          const float p0 = fex2(fmaf(lo, kLog2e, -mlog));
          const float p1 = fex2(fmaf(hi, kLog2e, -mlog));
          l += p0 + p1;
          packed[g] = fpack2<T>(p0, p1);
          W += nib * (1u << (4 * g));
        }
        const uint32_t partner = __shfl_xor_sync(0xffffffffu, W, 8);
        const uint32_t word = (lane & 8) ? ((partner >> 16) | (W & 0xFFFF0000u)) : ((W & 0xFFFFu) | (partner << 16));
        tc::mbar_wait(&p_empty[pb], pph ^ 1);  // P stage / E columns no longer read by PV_{t-2}
        tc::tc_fence_after();
        // P row r: 16-byte units (2*quarter, +1) of the 128B-swizzled row
        uint8_t* prow = smem + SMEM_P + pb * P_BYTES + r * 128;
        const int u0 = 2 * quarter, swz = r & 7;
        *reinterpret_cast<uint4*>(prow + ((u0 ^ swz) << 4)) = make_uint4(packed[0], packed[1], packed[2], packed[3]);
        *reinterpret_cast<uint4*>(prow + (((u0 + 1) ^ swz) << 4)) = make_uint4(packed[4], packed[5], packed[6], packed[7]);
        // metadata word of TMEM lane r (rows r and r^8 traded 16-bit halves above)
        tc::tmem_st_32x32b_x1(tmem_base + lane_base + TM_E + pb * 4 + quarter, word);
        tc::tmem_st_wait();
        tc::fence_proxy_async();  // P smem writes -> tensor core
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&p_full[pb]);
        if (++pb == PST) { pb = 0; pph ^= 1; }
      }
      }
      // ---- output rows: O / rowsum (quarter-0 warps), rowsum partials exchanged through smem
      red[4 * BM + quarter * BM + r] = l;
      tc::named_bar_sync(quad_bar, 128);
      if (quarter == 0) {
        const float inv = 1.0f / ((red[4 * BM + r] + red[5 * BM + r]) + (red[6 * BM + r] + red[7 * BM + r]));
        tc::mbar_wait(o_full, oph);
        tc::tc_fence_after();
        uint32_t o0[32], o1[32];
        tc::tmem_ld_32x32b_x32(tmem_base + lane_base + TM_O, o0);
        tc::tmem_ld_32x32b_x32(tmem_base + lane_base + TM_O + 32, o1);
        tc::tmem_ld_wait(o0);
        tc::tmem_ld_wait(o1);
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(o_empty);
        T* orow = out + ((int64_t)b * n + mb * BM + r) * HD;
        uint32_t pk[32];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          pk[j] = fpack2<T>(__uint_as_float(o0[2 * j]) * inv, __uint_as_float(o0[2 * j + 1]) * inv);
          pk[16 + j] = fpack2<T>(__uint_as_float(o1[2 * j]) * inv, __uint_as_float(o1[2 * j + 1]) * inv);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)
          reinterpret_cast<uint4*>(orow)[j] = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
      }
      oph ^= 1;
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc::tc_fence_after();
    tc::tmem_dealloc<512>(tmem_base);
  }
}

bool tc_flash_supported(int gs, int dtype, int n, int d) {
  return gs == 4 && (dtype == DFSS_BF16 || dtype == DFSS_F16) && d == HD && n % BM == 0 && n > 0;
}

template <typename T>
static cudaError_t flash_launch_typed(const void* q, const void* k, const void* v, void* out, float scale, int64_t bh,
                                      int n, cudaStream_t s) {
  const CUtensorMapDataType dt =
      std::is_same<T, __nv_bfloat16>::value ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  CUtensorMap tq, tk, tv;
  if (!encode_tmap_3d(&tq, dt, 2, (void*)q, HD, n, bh, HD, BM, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !encode_tmap_3d(&tk, dt, 2, (void*)k, HD, n, bh, HD, BN, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !encode_tmap_3d(&tv, dt, 2, (void*)v, HD, n, bh, HD, BN, CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  auto kern = dfss_flash_kernel<T>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_TOTAL);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int items = (int)bh * (n / BM);
  const int grid = items < sms ? items : sms;
  static const int dbg = getenv("DFSS_FLASH_DEBUG") ? atoi(getenv("DFSS_FLASH_DEBUG")) : 0;
  kern<<<grid, NUM_THREADS, SMEM_TOTAL, s>>>(tq, tk, tv, (T*)out, scale, (int)bh, n, 2u, dbg);
  return cudaGetLastError();
}

cudaError_t launch_flash_tc(const void* q, const void* k, const void* v, void* out, float scale, int gs, int dtype,
                            int64_t bh, int n, int d, cudaStream_t s) {
  if (!tc_flash_supported(gs, dtype, n, d)) return cudaErrorNotSupported;
  if (bh == 0) return cudaSuccess;
  if (dtype == DFSS_BF16) return flash_launch_typed<__nv_bfloat16>(q, k, v, out, scale, bh, n, s);
  return flash_launch_typed<__half>(q, k, v, out, scale, bh, n, s);
}

}  // namespace dfss
