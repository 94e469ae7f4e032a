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
//   O += P_t V_t                       tcgen05.mma.sp (_spmm_gather, :91-103)
//   O / L                              once per item
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
// 32*quad.. (rows) and score columns [32*quarter, +32) of every tile (= one K = 32
// tcgen05.mma.sp).  The four warps of a quad share the rows, hence the shift: each tile they
// OR-reduce their "partial sum too large" flags with one bar.red.or over the quad (the four
// warps sit on the same SM sub-partition, so this costs a barrier, not a round trip), and
// on the rare update exchange their maxima through shared memory.
//
// Register pairing for FADD2/FFMA2: the K tile is loaded through a 5-D tensor map whose
// strides permute the keys of every group of 4 into (k0, k2, k1, k3), so S columns arrive
// as (v0, v2, v1, v3) and the differences v0 - v1, v2 - v3 are one FADD2 of two natural
// register pairs.  The selection itself still names v0..v3 by their true key index, so
// tie-breaking is unchanged; V and the metadata stay in true key order.
//
// TMEM (512 columns): three S buffers at 0/128/256 (released as soon as every warp has
// read its scores, so S runs up to three tiles ahead of the softmax), O at 384, the
// metadata of P stage p at columns 448 + 4p + quarter.
//
// Warp roles (one CTA per SM, persistent over items): warp 0 TMA Q/K, warp 1 S issuer,
// warp 2 TMEM allocator + PV issuer, warp 3 TMA V, warps 4-19 softmax / prune / epilogue.
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
constexpr int PST = 2;    // P stages (smem) / metadata stages (TMEM)
constexpr int SBUF = 3;   // S buffers (TMEM)
constexpr int SMEM_RED = SMEM_P + PST * P_BYTES;  // [2 (max, sum)][4 quarters][128] floats
constexpr int SMEM_BAR = SMEM_RED + 2 * 4 * BM * 4;
constexpr int SMEM_TOTAL = SMEM_BAR + 256 + 1024;
constexpr int TM_O = SBUF * BN;  // 64 columns of output accumulator
constexpr int TM_E = TM_O + HD;  // PST x 4 metadata columns
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

// bar.red.or over `count` threads of named barrier `id`: true iff any thread passed true
__device__ __forceinline__ bool bar_any(uint32_t id, uint32_t count, bool pred) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\tsetp.ne.u32 p, %1, 0;\n\tbar.red.or.pred q, %2, %3, p;\n\tselp.u32 %0, 1, 0, q;\n\t}"
      : "=r"(r)
      : "r"((uint32_t)pred), "r"(id), "r"(count)
      : "memory");
  return r != 0;
}

// role-warp wait: sleeping try_wait (default) or spinning (variant bit 10, experiment)
__device__ __forceinline__ void wait_role(int variant, uint64_t* bar, uint32_t parity) {
  if (variant & 1024)
    tc::mbar_wait(bar, parity);
  else
    tc::mbar_wait_sleep(bar, parity);
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
                      uint32_t two, int variant) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = (uint64_t*)(smem + SMEM_BAR);
  uint64_t* q_full = bars;              // [2]
  uint64_t* q_empty = q_full + 2;       // [2]
  uint64_t* k_full = q_empty + 2;       // [KST]
  uint64_t* k_empty = k_full + KST;     // [KST]
  uint64_t* v_full = k_empty + KST;     // [VST]
  uint64_t* v_empty = v_full + VST;     // [VST]
  uint64_t* s_full = v_empty + VST;     // [SBUF] S tile computed
  uint64_t* s_empty = s_full + SBUF;    // [SBUF] every softmax warp read its scores (SM_WARPS)
  uint64_t* p_full = s_empty + SBUF;    // [PST] P smem + metadata written (SM_WARPS)
  uint64_t* p_empty = p_full + PST;     // [PST] PV retired
  uint64_t* o_full = p_empty + PST;     // [1] item's last PV retired
  uint64_t* o_empty = o_full + 1;       // [1] O drained (SM_WARPS)
  uint32_t* tmem_slot = (uint32_t*)(o_empty + 1);
  float* red_max = (float*)(smem + SMEM_RED);
  float* red_sum = red_max + 4 * BM;

  const uint32_t warp = tc::warp_id();
  const uint32_t lane = threadIdx.x & 31;
  const int mblocks = n / BM;
  const int ntiles = n / BN;
  // clusters of cs CTAs work on cs consecutive 128-row blocks of one head and share every
  // K / V tile: each CTA loads 1/cs of it and multicasts to the cluster (L2 traffic / cs)
  const int cs = (int)tc::cluster_nctarank();
  const int crank = (int)tc::cluster_ctarank();
  const uint16_t cmask = (uint16_t)((1u << cs) - 1u);
  const int gpb = mblocks / cs;  // groups per (batch, head)
  const int items = bh * gpb;    // one item = this CTA's block of a group
  const int cid = blockIdx.x / cs, ncl = gridDim.x / cs;

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
    for (int i = 0; i < PST; ++i) {
      tc::mbar_init(&p_full[i], SM_WARPS);
      tc::mbar_init(&p_empty[i], 1);
    }
    for (int i = 0; i < KST; ++i) {
      tc::mbar_init(&k_full[i], 1);
      tc::mbar_init(&k_empty[i], cs);  // released by every CTA of the cluster
    }
    for (int i = 0; i < VST; ++i) {
      tc::mbar_init(&v_full[i], 1);
      tc::mbar_init(&v_empty[i], cs);
    }
    tc::mbar_init(o_full, 1);
    tc::mbar_init(o_empty, SM_WARPS);
    tc::fence_barrier_init();
  }
  if (warp == 2) tc::tmem_alloc<512>(tmem_slot);
  tc::tc_fence_before();
  tc::cluster_sync();  // remote CTAs multicast into our smem / barriers only after init
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer: Q and K (keys permuted)
    if (lane == 0) {
      int ks = 0, it = 0;
      uint32_t kph = 0;
      for (int item = cid; item < items; item += ncl, ++it) {
        const int b = item / gpb, mb = (item % gpb) * cs + crank;
        const int qs = it & 1;
        wait_role(variant, &q_empty[qs], ((it >> 1) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(&q_full[qs], Q_BYTES);
        tc::tma_load_3d(smem + SMEM_Q + qs * Q_BYTES, &tm_q, &q_full[qs], 0, mb * BM, b);
        for (int t = 0; t < ntiles; ++t) {
          wait_role(variant, &k_empty[ks], kph ^ 1);
          tc::mbar_arrive_expect_tx(&k_full[ks], K_BYTES);
          tc::tma_load_5d_mc(smem + SMEM_K + ks * K_BYTES + crank * (K_BYTES / cs), &tm_k, &k_full[ks], 0, 0, 0,
                             t * (BN / 4) + crank * (BN / 4 / cs), b, cmask);
          if (++ks == KST) { ks = 0; kph ^= 1; }
        }
      }
    }
  } else if (warp == 3) {
    // ------------------------------------------------------------ TMA producer: V
    if (lane == 0) {
      int vs = 0;
      uint32_t vph = 0;
      for (int item = cid; item < items; item += ncl) {
        const int b = item / gpb;
        for (int t = 0; t < ntiles; ++t) {
          wait_role(variant, &v_empty[vs], vph ^ 1);
          tc::mbar_arrive_expect_tx(&v_full[vs], V_BYTES);
          tc::tma_load_3d_mc(smem + SMEM_V + vs * V_BYTES + crank * (V_BYTES / cs), &tm_v, &v_full[vs], 0,
                             t * BN + crank * (BN / cs), b, cmask);
          if (++vs == VST) { vs = 0; vph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ S issuer: S_T = Q K_t^T into buffer T % SBUF
    if (lane == 0) {
      constexpr uint32_t fmt = std::is_same<T, __nv_bfloat16>::value ? 1u : 0u;
      constexpr uint32_t idesc_s = tc::instr_desc(fmt, BM, BN, false, false, false);
      int ks = 0, it = 0, sb = 0;
      uint32_t kph = 0, sph = 0;
      for (int item = cid; item < items; item += ncl, ++it) {
        const int qs = it & 1;
        wait_role(variant, &q_full[qs], (it >> 1) & 1);
        const uint32_t q_addr = tc::smem_u32(smem + SMEM_Q + qs * Q_BYTES);
        for (int t = 0; t < ntiles; ++t) {
          wait_role(variant, &s_empty[sb], sph ^ 1);  // S_{T-SBUF} read by every softmax warp
          wait_role(variant, &k_full[ks], kph);
          tc::tc_fence_after();
          const uint32_t k_addr = tc::smem_u32(smem + SMEM_K + ks * K_BYTES);
          if (!(variant & 32)) {
#pragma unroll
            for (int kk = 0; kk < HD / 16; ++kk) {
              const uint64_t ad = tc::smem_desc(q_addr + kk * 32, 16, 1024, tc::kSwizzle128B);
              const uint64_t bd = tc::smem_desc(k_addr + kk * 32, 16, 1024, tc::kSwizzle128B);
              tc::mma_f16_ss(tmem_base + sb * BN, ad, bd, idesc_s, kk > 0 ? 1u : 0u);
            }
          }
          tc::mma_commit_mc(&k_empty[ks], cmask);
          tc::mma_commit(&s_full[sb]);
          if (++ks == KST) { ks = 0; kph ^= 1; }
          if (++sb == SBUF) { sb = 0; sph ^= 1; }
        }
        tc::mma_commit(&q_empty[qs]);
      }
    }
  } else if (warp == 2) {
    // ------------------------------------------------------------ PV issuer: O += P_T V_t (4 sparse K=32 MMAs)
    if (lane == 0) {
      constexpr uint32_t fmt = std::is_same<T, __nv_bfloat16>::value ? 1u : 0u;
      constexpr uint32_t idesc_pv = tc::instr_desc(fmt, BM, HD, false, true, true);
      int vs = 0, pb = 0;
      uint32_t vph = 0, pph = 0, oph = 0;
      for (int item = cid; item < items; item += ncl) {
        wait_role(variant, o_empty, oph ^ 1);
        for (int t = 0; t < ntiles; ++t) {
          wait_role(variant, &p_full[pb], pph);
          wait_role(variant, &v_full[vs], vph);
          tc::tc_fence_after();
          const uint32_t p_addr = tc::smem_u32(smem + SMEM_P + pb * P_BYTES);
          const uint32_t v_addr = tc::smem_u32(smem + SMEM_V + vs * V_BYTES);
#pragma unroll
          for (int q = 0; q < ((variant & 16) ? 0 : 4); ++q) {
            const uint64_t ad = tc::smem_desc(p_addr + q * 32, 16, 1024, tc::kSwizzle128B);
            const uint64_t bd = tc::smem_desc(v_addr + q * 32 * 128, V_BYTES, 1024, tc::kSwizzle128B);
            // metadata column: even address + sparse_id2 (idesc bits [0,2)) selects the odd one
            const uint32_t e_col = tmem_base + TM_E + pb * 4 + q;
            tc::mma_sp_f16_ss(tmem_base + TM_O, ad, bd, e_col & ~1u, idesc_pv | (e_col & 1u),
                              (t > 0 || q > 0) ? 1u : 0u);
          }
          tc::mma_commit(&p_empty[pb]);
          tc::mma_commit_mc(&v_empty[vs], cmask);
          if (++vs == VST) { vs = 0; vph ^= 1; }
          if (++pb == PST) { pb = 0; pph ^= 1; }
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
    const uint32_t qbar = 1 + quad;  // named barrier of the four warps sharing these rows
    const float c = scale * kLog2e;
    // P row r, 16-byte units (2*quarter, +1) of the 128B-swizzled row
    const uint32_t p_row = tc::smem_u32(smem + SMEM_P) + r * 128;
    const uint32_t u0 = (uint32_t)(((2 * quarter) ^ (r & 7)) << 4), u1 = (uint32_t)(((2 * quarter + 1) ^ (r & 7)) << 4);
    int sb = 0, pb = 0;
    uint32_t sph = 0, pph = 0, oph = 0;
    // row maximum of the current tile over the quad's four quarters (scaled to log2 units)
    auto row_max = [&](const uint32_t (&s)[32]) {
      float mt = -INFINITY;
#pragma unroll
      for (int j = 0; j < 32; j += 2) mt = fmaxf(mt, fmaxf(__uint_as_float(s[j]), __uint_as_float(s[j + 1])));
      red_max[quarter * BM + r] = mt;
      tc::named_bar_sync(qbar, 128);
      const float m = fmaxf(fmaxf(red_max[r], red_max[BM + r]), fmaxf(red_max[2 * BM + r], red_max[3 * BM + r]));
      return m * c;
    };
    for (int item = cid; item < items; item += ncl) {
      const int b = item / gpb, mb = (item % gpb) * cs + crank;
      float mlog = 0.f;          // shift in log2 units (m * c), shared by the quad's four warps
      float l0 = 0.f, l1 = 0.f;  // this quarter's running row sum (pair)
      for (int t = 0; t < ntiles; ++t) {
        tc::mbar_wait(&s_full[sb], sph);
        tc::tc_fence_after();
        uint32_t s[32];
        tc::tmem_ld_32x32b_x32(lane_base + sb * BN + quarter * 32, s);
        tc::tmem_ld_wait(s);
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&s_empty[sb]);
        if (++sb == SBUF) { sb = 0; sph ^= 1; }
        uint32_t pk[8], W;
        float lt0, lt1;
        if (t == 0) {
          // first tile of the item: the shift starts at the row maximum of this tile
          mlog = row_max(s);
          prune_exp_tile<T>(s, c, mlog, two, pk, W, lt0, lt1);
        } else {
          if (variant & 8) {  // timing experiment: no prune / exp arithmetic
#pragma unroll
            for (int j = 0; j < 8; ++j) pk[j] = s[j] ^ s[j + 8];
            W = 0x44444444u;
            lt0 = lt1 = 0.f;
          } else {
            prune_exp_tile<T>(s, c, mlog, two, pk, W, lt0, lt1);
          }
          if (!(variant & 128) && bar_any(qbar, 128, !(lt0 + lt1 <= kSumLimit))) {
            // ---- slow path (whole quad): raise the shift to the row maximum, rescale O and the sums
            const float mnew = fmaxf(mlog, row_max(s));
            const float f = fex2(mlog - mnew);
            l0 *= f;
            l1 *= f;
            // every PV issued so far (up to T-1) must have retired before O is rescaled
            const int prev = pb == 0 ? PST - 1 : pb - 1;
            tc::mbar_wait(&p_empty[prev], prev == PST - 1 ? pph ^ 1 : pph);
            tc::tc_fence_after();
            uint32_t o[16];
            const uint32_t oaddr = lane_base + TM_O + 16 * quarter;
            tc::tmem_ld_32x32b_x16(oaddr, o);
            tc::tmem_ld_wait(o);
#pragma unroll
            for (int j = 0; j < 16; ++j) o[j] = __float_as_uint(__uint_as_float(o[j]) * f);
            tc::tmem_st_32x32b_x16(oaddr, o);
            tc::tmem_st_wait();
            mlog = mnew;
            prune_exp_tile<T>(s, c, mlog, two, pk, W, lt0, lt1);
          }
        }
        add2(l0, l1, lt0, lt1, l0, l1);
        // metadata word of TMEM lane r: rows r and r^8 trade 16-bit halves (include/dfss.h)
        const uint32_t partner = __shfl_xor_sync(0xffffffffu, W, 8);
        const uint32_t word = (lane & 8) ? ((partner >> 16) | (W & 0xFFFF0000u)) : ((W & 0xFFFFu) | (partner << 16));
        tc::mbar_wait(&p_empty[pb], pph ^ 1);  // PV_{T-PST} retired: P stage and metadata columns free
        tc::tc_fence_after();
        const uint32_t prow = p_row + pb * P_BYTES;
        if (!(variant & 256)) {
          sts128(prow + u0, pk[0], pk[1], pk[2], pk[3]);
          sts128(prow + u1, pk[4], pk[5], pk[6], pk[7]);
        }
        if (!(variant & 512)) {
          tc::tmem_st_32x32b_x1(lane_base + TM_E + pb * 4 + quarter, word);
          tc::tmem_st_wait();
        }
        if (!(variant & 64)) tc::fence_proxy_async();  // P smem writes -> tensor core
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&p_full[pb]);
        if (++pb == PST) { pb = 0; pph ^= 1; }
      }
      // ---- epilogue: O / (sum over the four quarters' row sums); warp writes columns [16q, +16)
      red_sum[quarter * BM + r] = l0 + l1;
      tc::named_bar_sync(qbar, 128);
      const float inv =
          1.0f / ((red_sum[r] + red_sum[BM + r]) + (red_sum[2 * BM + r] + red_sum[3 * BM + r]));
      tc::mbar_wait(o_full, oph);
      oph ^= 1;
      tc::tc_fence_after();
      uint32_t o[16];
      tc::tmem_ld_32x32b_x16(lane_base + TM_O + 16 * quarter, o);
      tc::tmem_ld_wait(o);
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(o_empty);
      uint32_t pko[8];
#pragma unroll
      for (int j = 0; j < 8; ++j)
        pko[j] = fpack2<T>(__uint_as_float(o[2 * j]) * inv, __uint_as_float(o[2 * j + 1]) * inv);
      uint4* orow = reinterpret_cast<uint4*>(out + ((int64_t)b * n + mb * BM + r) * HD + 16 * quarter);
      orow[0] = make_uint4(pko[0], pko[1], pko[2], pko[3]);
      orow[1] = make_uint4(pko[4], pko[5], pko[6], pko[7]);
    }
  }
  tc::tc_fence_before();
  tc::cluster_sync();  // no CTA leaves while cluster peers may still signal its barriers
  if (warp == 2) {
    tc::tc_fence_after();
    tc::tmem_dealloc<512>(tmem_base);
  }
}

bool tc_flash_supported(int gs, int dtype, int n, int d) {
  return gs == 4 && (dtype == DFSS_BF16 || dtype == DFSS_F16) && d == HD && n % BM == 0 && n > 0;
}

// cluster size: 4 when the 128-row blocks of a head split evenly, else 2, else 1
// (DFSS_FLASH_CLUSTER overrides, for experiments)
static int pick_cluster(int mblocks) {
  static const int forced = getenv("DFSS_FLASH_CLUSTER") ? atoi(getenv("DFSS_FLASH_CLUSTER")) : 0;
  if (forced == 1 || forced == 2 || forced == 4) return mblocks % forced == 0 ? forced : 1;
  return mblocks % 4 == 0 ? 4 : (mblocks % 2 == 0 ? 2 : 1);
}

template <typename T>
static cudaError_t flash_launch_typed(const void* q, const void* k, const void* v, void* out, float scale, int64_t bh,
                                      int n, cudaStream_t s) {
  const CUtensorMapDataType dt =
      std::is_same<T, __nv_bfloat16>::value ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  const int mblocks = n / BM;
  const int cs = pick_cluster(mblocks);
  CUtensorMap tq, tk, tv;
  // K as [bh][n/4 groups][j2][j1][d] with key = 4g + 2 j1 + j2 and j1 iterated before j2:
  // the smem rows of a tile come out in key order (k0, k2, k1, k3) per group of 4.  Each CTA
  // of a cluster loads 1/cs of the tile (boxes of BN/cs keys) and multicasts it.
  const uint64_t row = HD * 2;
  const uint64_t kdims[5] = {(uint64_t)HD, 2, 2, (uint64_t)n / 4, (uint64_t)bh};
  const uint64_t kstr[4] = {2 * row, row, 4 * row, (uint64_t)n * row};
  const uint32_t kbox[5] = {(uint32_t)HD, 2, 2, (uint32_t)(BN / 4 / cs), 1};
  if (!encode_tmap_3d(&tq, dt, 2, (void*)q, HD, n, bh, HD, BM, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !encode_tmap(&tk, dt, 5, (void*)k, kdims, kstr, kbox, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !encode_tmap_3d(&tv, dt, 2, (void*)v, HD, n, bh, HD, BN / cs, CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  auto kern = dfss_flash_kernel<T>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_TOTAL);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = SMEM_TOTAL;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // persistent: as many clusters as fit at once (not every GPC holds a multiple of cs SMs)
  cfg.gridDim = dim3(sms / cs * cs);
  int max_clusters = 0;
  if (cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg) != cudaSuccess || max_clusters < 1)
    max_clusters = sms / cs;
  const int64_t groups = bh * (mblocks / cs);
  const int ncl = (int)(groups < max_clusters ? groups : max_clusters);
  cfg.gridDim = dim3(ncl * cs);
  // DFSS_FLASH_VARIANT (timing experiments only; results invalid when bits 3-9 are set):
  // bit3 skip prune/exp arithmetic, bit4 skip PV MMAs, bit5 skip S MMAs, bit6 skip the proxy fence,
  // bit7 skip the per-tile quad barrier, bit8 skip the P stores, bit9 skip the metadata store,
  // bit10 role warps spin instead of sleeping
  static const int variant = getenv("DFSS_FLASH_VARIANT") ? atoi(getenv("DFSS_FLASH_VARIANT")) : 0;
  return cudaLaunchKernelEx(&cfg, kern, tq, tk, tv, (T*)out, scale, (int)bh, n, 2u, variant);
}

cudaError_t launch_flash_tc(const void* q, const void* k, const void* v, void* out, float scale, int gs, int dtype,
                            int64_t bh, int n, int d, cudaStream_t s) {
  if (!tc_flash_supported(gs, dtype, n, d)) return cudaErrorNotSupported;
  if (bh == 0) return cudaSuccess;
  if (dtype == DFSS_BF16) return flash_launch_typed<__nv_bfloat16>(q, k, v, out, scale, bh, n, s);
  return flash_launch_typed<__half>(q, k, v, out, scale, bh, n, s);
}

}  // namespace dfss
