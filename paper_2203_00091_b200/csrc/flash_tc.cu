// flash_tc.cu -- fully fused DFSS attention on tcgen05 (2:4, bf16/fp16, head dim 64).
//
// pipeline.nm_attention (pipeline.py:15-32) in one kernel with no n x n tensor of any
// kind in HBM.  Per 128-query block ("item") and 128-key tile t:
//   S_t = Q K_t^T                      tcgen05.mma -> TMEM (fp32), double-buffered
//   prune 2-of-4 in registers          select24 rule of the reference (codec.py:104-123,
//                                      _kernels_numba.py:159-184): signed value, ties to
//                                      the lower index -- on the fp32 scores of S_t
//   P_t = exp(s - m) of the kept half  compressed K-major A operand in smem, nibbles as
//                                      tcgen05.mma.sp metadata in TMEM
//   O_q += P_t V_t                     tcgen05.mma.sp (_spmm_gather, :91-103)
//   O = sum_q 2^(m_q - M) O_q / L      once per item
//
// Softmax (_softmax_nonzeros, _kernels_numba.py:66-84: exp(x - max) / sum over the kept
// entries) is evaluated online with a lazily updated shift: the shift m only has to stay
// within 2^8 of the running maximum for the fp32 sums and the 16-bit P to be safe, so a
// tile whose partial sum exceeds 2^8 (or is not finite) takes a slow path that raises m to
// the true maximum and rescales the running O and sum; in steady state no max is computed
// at all.  The result is mathematically the reference's exp(x - max)/sum; only rounding
// differs.
//
// Work split inside a 128-row item: 16 softmax warps, warp (quad, quarter) owns TMEM lanes
// 32*quad.. (rows) and score columns [32*quarter, +32) of every tile.  Each quarter keeps
// its own shift m_q, row sum l_q and output accumulator O_q (TMEM columns 256 + 64*q):
// the quarter's 32 columns are exactly one K = 32 tcgen05.mma.sp, so the MMA for quarter q
// accumulates into O_q and no cross-warp agreement on the shift is ever needed inside the
// tile loop.  The four partial outputs are combined once per item.
//
// Register pairing for FADD2/FFMA2: the K tile is loaded through a 5-D tensor map whose
// strides permute the keys of every group of 4 into (k0, k2, k1, k3), so S columns arrive
// as (v0, v2, v1, v3) and the differences v0 - v1, v2 - v3 are one FADD2 of two natural
// register pairs.  The selection itself still names v0..v3 by their true key index, so
// tie-breaking is unchanged; V and the metadata stay in true key order.
//
// TMEM (512 columns): S buffers at 0 and 128 (the metadata column of quarter q for the
// tile in buffer b is column 128b + 32q, written after that quarter's scores were read);
// O_q at 256 + 64q.
//
// Warp roles (one CTA per SM, persistent over items): warp 0 TMA Q/K, warp 1 S issuer,
// warp 2 TMEM allocator + PV issuer, warp 3 TMA V, warps 4-19 softmax / prune / epilogue.
#include <type_traits>

#include "dfss_common.cuh"
#include "tc_common.cuh"

namespace dfss {

namespace {
constexpr int BM = 128;   // query rows per item (TMEM lanes)
constexpr int BN = 128;   // keys per tile
constexpr int HD = 64;    // head dim
constexpr int KST = 4;    // K ring
constexpr int VST = 4;    // V ring
constexpr int SM_WARPS = 16;
constexpr int NUM_THREADS = (4 + SM_WARPS) * 32;
constexpr int Q_BYTES = BM * HD * 2;        // 16 KB
constexpr int K_BYTES = BN * HD * 2;        // 16 KB
constexpr int V_BYTES = BN * HD * 2;        // 16 KB
constexpr int P_BYTES = BM * (BN / 2) * 2;  // 16 KB: 128 rows x 64 kept values
constexpr int SMEM_Q = 0;
constexpr int SMEM_K = SMEM_Q + 2 * Q_BYTES;
constexpr int SMEM_V = SMEM_K + KST * K_BYTES;
constexpr int SMEM_P = SMEM_V + VST * V_BYTES;
constexpr int SMEM_RED = SMEM_P + 2 * P_BYTES;  // [2 items][2 (m, l)][4 quarters][128] floats
constexpr int SMEM_BAR = SMEM_RED + 2 * 2 * 4 * BM * 4;
constexpr int SMEM_TOTAL = SMEM_BAR + 256 + 1024;
constexpr int TM_O = 2 * BN;  // O_q at TM_O + 64 q
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kSumLimit = 256.0f;  // a quarter-tile partial sum above 2^8 triggers a shift update
}  // namespace

// ---------------------------------------------------------------- packed fp32 helpers (sm_100 FADD2/FFMA2)
__device__ __forceinline__ void sub2(float a0, float a1, float b0, float b1, float& d0, float& d1) {
  asm("{\n\t.reg .b64 a, b, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
      "sub.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
__device__ __forceinline__ void add2(float a0, float a1, float b0, float b1, float& d0, float& d1) {
  asm("{\n\t.reg .b64 a, b, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
      "add.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
// (a0, a1) * c + (b, b)
__device__ __forceinline__ void fma2s(float a0, float a1, float c, float b, float& d0, float& d1) {
  asm("{\n\t.reg .b64 a, cc, bb, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 cc, {%4, %4};\n\tmov.b64 bb, {%5, %5};\n\t"
      "fma.rn.f32x2 d, a, cc, bb;\n\tmov.b64 {%0, %1}, d;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(c), "f"(b));
}

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

__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

// One quarter-tile of one row: 8 groups of 4 scores s[] in (v0, v2, v1, v3) register order.
// Prunes 2:4 (reference rule), exponentiates the kept half against the shift `mlog`
// (= m * c), packs P, builds the metadata word W (group g at bits 4g) and the partial sum.
template <typename T>
__device__ __forceinline__ void prune_exp_tile(const uint32_t (&s)[32], float c, float mlog, uint32_t two,
                                               uint32_t (&pk)[8], uint32_t& W, float& lt0, float& lt1) {
  W = 0x88888888u;
  lt0 = 0.f;
  lt1 = 0.f;
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    const float v0 = __uint_as_float(s[4 * g + 0]);
    const float v2 = __uint_as_float(s[4 * g + 1]);
    const float v1 = __uint_as_float(s[4 * g + 2]);
    const float v3 = __uint_as_float(s[4 * g + 3]);
    // winner index of each pair from the sign of the difference; +0 added so that a
    // (-0) - (+0) tie reads as +0 (ties keep the lower index)
    float d01, d23;
    sub2(v0, v2, v1, v3, d01, d23);
    add2(d01, d23, 0.f, 0.f, d01, d23);
    const uint32_t a = sign_bit(d01, two), b = sign_bit(d23, two);
    const float w01 = fmaxf(v0, v1), l01 = fminf(v0, v1);
    const float w23 = fmaxf(v2, v3), l23 = fminf(v2, v3);
    const bool keep01 = l01 >= w23;  // lower-index loser vs higher-index winner
    const bool keep23 = l23 > w01;   // higher-index loser must strictly beat the winner
    const float lo = keep01 ? v0 : (keep23 ? v2 : w01);
    const float hi = keep01 ? v1 : (keep23 ? v3 : w23);
    // nibble - 8: 0x4 -> -4, 0xE -> 6, mixed 8 + a + 4b -> a + 4b
    int nib = keep23 ? 6 : (int)(a + 4u * b);
    nib = keep01 ? -4 : nib;
    W += (uint32_t)nib * (1u << (4 * g));
    float x0, x1;
    fma2s(lo, hi, c, -mlog, x0, x1);
    const float p0 = fex2(x0), p1 = fex2(x1);
    pk[g] = fpack2<T>(p0, p1);
    add2(lt0, lt1, p0, p1, lt0, lt1);
  }
}

template <typename T>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    dfss_flash_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                      const __grid_constant__ CUtensorMap tm_v, T* __restrict__ out, float scale, int bh, int n,
                      uint32_t two) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = (uint64_t*)(smem + SMEM_BAR);
  uint64_t* q_full = bars;             // [2]
  uint64_t* q_empty = q_full + 2;      // [2]
  uint64_t* k_full = q_empty + 2;      // [KST]
  uint64_t* k_empty = k_full + KST;    // [KST]
  uint64_t* v_full = k_empty + KST;    // [VST]
  uint64_t* v_empty = v_full + VST;    // [VST]
  uint64_t* s_full = v_empty + VST;    // [2] S tile in TMEM buffer b
  uint64_t* p_full = s_full + 2;       // [2] P smem + metadata written (SM_WARPS arrivals)
  uint64_t* p_empty = p_full + 2;      // [2] PV retired: P stage and S buffer b free
  uint64_t* o_full = p_empty + 2;      // [1] item's last PV retired
  uint64_t* o_empty = o_full + 1;      // [1] O drained (SM_WARPS arrivals)
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
      tc::mbar_init(&s_full[i], 1);
      tc::mbar_init(&p_full[i], SM_WARPS);
      tc::mbar_init(&p_empty[i], 1);
    }
    for (int i = 0; i < KST; ++i) {
      tc::mbar_init(&k_full[i], 1);
      tc::mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < VST; ++i) {
      tc::mbar_init(&v_full[i], 1);
      tc::mbar_init(&v_empty[i], 1);
    }
    tc::mbar_init(o_full, 1);
    tc::mbar_init(o_empty, SM_WARPS);
    tc::fence_barrier_init();
  }
  if (warp == 2) tc::tmem_alloc<512>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer: Q and K (keys permuted)
    if (lane == 0) {
      int ks = 0, it = 0;
      uint32_t kph = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
        const int b = item / mblocks, mb = item % mblocks;
        const int qs = it & 1;
        tc::mbar_wait_sleep(&q_empty[qs], ((it >> 1) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(&q_full[qs], Q_BYTES);
        tc::tma_load_3d(smem + SMEM_Q + qs * Q_BYTES, &tm_q, &q_full[qs], 0, mb * BM, b);
        for (int t = 0; t < ntiles; ++t) {
          tc::mbar_wait_sleep(&k_empty[ks], kph ^ 1);
          tc::mbar_arrive_expect_tx(&k_full[ks], K_BYTES);
          tc::tma_load_5d(smem + SMEM_K + ks * K_BYTES, &tm_k, &k_full[ks], 0, 0, 0, t * (BN / 4), b);
          if (++ks == KST) { ks = 0; kph ^= 1; }
        }
      }
    }
  } else if (warp == 3) {
    // ------------------------------------------------------------ TMA producer: V
    if (lane == 0) {
      int vs = 0;
      uint32_t vph = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x) {
        const int b = item / mblocks;
        for (int t = 0; t < ntiles; ++t) {
          tc::mbar_wait_sleep(&v_empty[vs], vph ^ 1);
          tc::mbar_arrive_expect_tx(&v_full[vs], V_BYTES);
          tc::tma_load_3d(smem + SMEM_V + vs * V_BYTES, &tm_v, &v_full[vs], 0, t * BN, b);
          if (++vs == VST) { vs = 0; vph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ S issuer: S_T = Q K_t^T into buffer T & 1
    if (lane == 0) {
      constexpr uint32_t fmt = std::is_same<T, __nv_bfloat16>::value ? 1u : 0u;
      constexpr uint32_t idesc_s = tc::instr_desc(fmt, BM, BN, false, false, false);
      int ks = 0, it = 0;
      uint32_t kph = 0, gt = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
        const int qs = it & 1;
        tc::mbar_wait_sleep(&q_full[qs], (it >> 1) & 1);
        const uint32_t q_addr = tc::smem_u32(smem + SMEM_Q + qs * Q_BYTES);
        for (int t = 0; t < ntiles; ++t, ++gt) {
          const uint32_t sb = gt & 1;
          tc::mbar_wait_sleep(&p_empty[sb], ((gt >> 1) & 1) ^ 1);  // PV_{T-2} retired: buffer free
          tc::mbar_wait_sleep(&k_full[ks], kph);
          tc::tc_fence_after();
          const uint32_t k_addr = tc::smem_u32(smem + SMEM_K + ks * K_BYTES);
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {
            const uint64_t ad = tc::smem_desc(q_addr + kk * 32, 16, 1024, tc::kSwizzle128B);
            const uint64_t bd = tc::smem_desc(k_addr + kk * 32, 16, 1024, tc::kSwizzle128B);
            tc::mma_f16_ss(tmem_base + sb * BN, ad, bd, idesc_s, kk > 0 ? 1u : 0u);
          }
          tc::mma_commit(&k_empty[ks]);
          tc::mma_commit(&s_full[sb]);
          if (++ks == KST) { ks = 0; kph ^= 1; }
        }
        tc::mma_commit(&q_empty[qs]);
      }
    }
  } else if (warp == 2) {
    // ------------------------------------------------------------ PV issuer: O_q += P_T[:, quarter q] V_t[q rows]
    if (lane == 0) {
      constexpr uint32_t fmt = std::is_same<T, __nv_bfloat16>::value ? 1u : 0u;
      constexpr uint32_t idesc_pv = tc::instr_desc(fmt, BM, HD, false, true, true);
      int vs = 0;
      uint32_t vph = 0, oph = 0, gt = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x) {
        tc::mbar_wait_sleep(o_empty, oph ^ 1);
        for (int t = 0; t < ntiles; ++t, ++gt) {
          const uint32_t pb = gt & 1;
          tc::mbar_wait_sleep(&p_full[pb], (gt >> 1) & 1);
          tc::mbar_wait_sleep(&v_full[vs], vph);
          tc::tc_fence_after();
          const uint32_t p_addr = tc::smem_u32(smem + SMEM_P + pb * P_BYTES);
          const uint32_t v_addr = tc::smem_u32(smem + SMEM_V + vs * V_BYTES);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint64_t ad = tc::smem_desc(p_addr + q * 32, 16, 1024, tc::kSwizzle128B);
            const uint64_t bd = tc::smem_desc(v_addr + q * 32 * 128, V_BYTES, 1024, tc::kSwizzle128B);
            tc::mma_sp_f16_ss(tmem_base + TM_O + q * HD, ad, bd, tmem_base + pb * BN + 32 * q, idesc_pv,
                              t > 0 ? 1u : 0u);
          }
          tc::mma_commit(&p_empty[pb]);
          tc::mma_commit(&v_empty[vs]);
          if (++vs == VST) { vs = 0; vph ^= 1; }
        }
        tc::mma_commit(o_full);
        oph ^= 1;
      }
    }
  } else {
    // ------------------------------------------------------------ softmax / prune / epilogue warps
    const int quad = warp & 3;
    const int quarter = (warp - 4) >> 2;
    const int r = quad * 32 + lane;  // row within the item == TMEM lane
    const uint32_t lane_base = tmem_base + ((uint32_t)(quad * 32) << 16);
    const float c = scale * kLog2e;
    // P row r, 16-byte units (2*quarter, +1) of the 128B-swizzled row, for both stages
    const uint32_t p_row = tc::smem_u32(smem + SMEM_P) + r * 128;
    const uint32_t u0 = (uint32_t)(((2 * quarter) ^ (r & 7)) << 4), u1 = (uint32_t)(((2 * quarter + 1) ^ (r & 7)) << 4);
    uint32_t gt = 0, oph = 0;
    int it = 0;
    for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
      const int b = item / mblocks, mb = item % mblocks;
      float mlog = 0.f;        // shift in log2 units (m * c)
      float l0 = 0.f, l1 = 0.f;  // running row sum (pair)
      for (int t = 0; t < ntiles; ++t, ++gt) {
        const uint32_t sb = gt & 1;
        tc::mbar_wait(&s_full[sb], (gt >> 1) & 1);
        tc::tc_fence_after();
        uint32_t s[32];
        tc::tmem_ld_32x32b_x32(lane_base + sb * BN + quarter * 32, s);
        tc::tmem_ld_wait(s);
        uint32_t pk[8], W;
        float lt0, lt1;
        if (t == 0) {
          // first tile of the item: the shift starts at this quarter's maximum
          float mt = -INFINITY;
#pragma unroll
          for (int j = 0; j < 32; j += 2) mt = fmaxf(mt, fmaxf(__uint_as_float(s[j]), __uint_as_float(s[j + 1])));
          mlog = mt * c;
          prune_exp_tile<T>(s, c, mlog, two, pk, W, lt0, lt1);
        } else {
          prune_exp_tile<T>(s, c, mlog, two, pk, W, lt0, lt1);
          const bool need = !(lt0 + lt1 <= kSumLimit);
          if (__any_sync(0xffffffffu, need)) {
            // ---- slow path: raise the shift to the true maximum, rescale O_q and the sum
            float mt = -INFINITY;
#pragma unroll
            for (int j = 0; j < 32; j += 2) mt = fmaxf(mt, fmaxf(__uint_as_float(s[j]), __uint_as_float(s[j + 1])));
            const float mnew = need ? fmaxf(mlog, mt * c) : mlog;
            const float f = fex2(mlog - mnew);
            l0 *= f;
            l1 *= f;
            // every PV issued so far (up to T-1) must have retired before O_q is rescaled
            tc::mbar_wait(&p_empty[(gt - 1) & 1], ((gt - 1) >> 1) & 1);
            tc::tc_fence_after();
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              uint32_t o[32];
              const uint32_t oaddr = lane_base + TM_O + quarter * HD + h * 32;
              tc::tmem_ld_32x32b_x32(oaddr, o);
              tc::tmem_ld_wait(o);
#pragma unroll
              for (int j = 0; j < 32; ++j) o[j] = __float_as_uint(__uint_as_float(o[j]) * f);
              tc::tmem_st_32x32b_x32(oaddr, o);
            }
            tc::tmem_st_wait();
            mlog = mnew;
            prune_exp_tile<T>(s, c, mlog, two, pk, W, lt0, lt1);
          }
        }
        add2(l0, l1, lt0, lt1, l0, l1);
        // metadata word of TMEM lane r: rows r and r^8 trade 16-bit halves (include/dfss.h)
        const uint32_t partner = __shfl_xor_sync(0xffffffffu, W, 8);
        const uint32_t word = (lane & 8) ? ((partner >> 16) | (W & 0xFFFF0000u)) : ((W & 0xFFFFu) | (partner << 16));
        // P stage sb / the metadata column are free: S_T was computed after PV_{T-2} retired
        const uint32_t prow = p_row + sb * P_BYTES;
        sts128(prow + u0, pk[0], pk[1], pk[2], pk[3]);
        sts128(prow + u1, pk[4], pk[5], pk[6], pk[7]);
        tc::tmem_st_32x32b_x1(lane_base + sb * BN + 32 * quarter, word);
        tc::tmem_st_wait();
        tc::fence_proxy_async();  // P smem writes -> tensor core
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&p_full[sb]);
      }
      // ---- epilogue: combine the four quarter accumulators of row r
      float* red_m = red + (it & 1) * (2 * 4 * BM);
      float* red_l = red_m + 4 * BM;
      red_m[quarter * BM + r] = mlog;
      red_l[quarter * BM + r] = l0 + l1;
      tc::named_bar_sync(1 + quad, 128);
      float mq[4], lq[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        mq[q] = red_m[q * BM + r];
        lq[q] = red_l[q * BM + r];
      }
      const float M = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3]));
      float coef[4], L = 0.f;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        coef[q] = fex2(mq[q] - M);
        L += coef[q] * lq[q];
      }
      const float inv = 1.0f / L;
      tc::mbar_wait(o_full, oph);
      oph ^= 1;
      tc::tc_fence_after();
      uint32_t o[4][16];
#pragma unroll
      for (int q = 0; q < 4; ++q) tc::tmem_ld_32x32b_x16(lane_base + TM_O + q * HD + 16 * quarter, o[q]);
#pragma unroll
      for (int q = 0; q < 4; ++q) tc::tmem_ld_wait(o[q]);
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(o_empty);
      uint32_t pko[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float a0 = 0.f, a1 = 0.f;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float w = coef[q] * inv;
          a0 = fmaf(__uint_as_float(o[q][2 * j]), w, a0);
          a1 = fmaf(__uint_as_float(o[q][2 * j + 1]), w, a1);
        }
        pko[j] = fpack2<T>(a0, a1);
      }
      uint4* orow = reinterpret_cast<uint4*>(out + ((int64_t)b * n + mb * BM + r) * HD + 16 * quarter);
      orow[0] = make_uint4(pko[0], pko[1], pko[2], pko[3]);
      orow[1] = make_uint4(pko[4], pko[5], pko[6], pko[7]);
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
  // K as [bh][n/4 groups][j2][j1][d] with key = 4g + 2 j1 + j2 and j1 iterated before j2:
  // the smem rows of a tile come out in key order (k0, k2, k1, k3) per group of 4.
  const uint64_t row = HD * 2;
  const uint64_t kdims[5] = {(uint64_t)HD, 2, 2, (uint64_t)n / 4, (uint64_t)bh};
  const uint64_t kstr[4] = {2 * row, row, 4 * row, (uint64_t)n * row};
  const uint32_t kbox[5] = {(uint32_t)HD, 2, 2, BN / 4, 1};
  if (!encode_tmap_3d(&tq, dt, 2, (void*)q, HD, n, bh, HD, BM, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !encode_tmap(&tk, dt, 5, (void*)k, kdims, kstr, kbox, CU_TENSOR_MAP_SWIZZLE_128B) ||
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
  kern<<<grid, NUM_THREADS, SMEM_TOTAL, s>>>(tq, tk, tv, (T*)out, scale, (int)bh, n, 2u);
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
