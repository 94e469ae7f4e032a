// flash_tf32.cu -- fully fused DFSS attention, 1:2 on fp32 inputs with tf32 tensor cores
// (BASELINE configs[4] "1:2 tf32"), head dim 64, n % 256 == 0.
//
// Same structure as the 16-bit two-set kernel (flash_tc.cu): an item is 256 query rows of
// one head, two independent softmax sets of 8 warps (one per 128-row half), a ring of three
// 128-column TMEM S buffers shared by the steps g = 2t + h, lazily updated softmax shift,
// P and metadata written back into the step's S buffer, sparse PV with A from TMEM.
// What changes for 32-bit elements:
//   S = Q K^T           tcgen05.mma kind::tf32, K = 8 per MMA (8 MMAs for d = 64); Q, K, V
//                       tiles are fp32 in two 128-byte swizzle atoms along the 64 dims
//   prune 1:2           keep element 1 of each pair iff v1 > v0 (codec.py:114-117), i.e.
//                       the pair maximum; nibble 0x4 / 0xE (codec.py:60-76) -- the tf32
//                       sparse-MMA metadata, one 4-bit field per pair
//   O += P V            tcgen05.mma.sp kind::tf32, K = 16 dense (8 kept) per MMA: per 32-key
//                       chunk two MMAs, metadata words in chunk columns 0 and 4, the kept
//                       fp32 P in columns 16..23 and 24..31.  kind::tf32 reads B only
//                       K-major (an MN-major tf32 B contributes zeros, tools/tf32_probe.cu),
//                       so V is transposed once per call into the workspace (V^T [bh][64][n])
//                       and streamed as four 32-key swizzle atoms per tile
// The tf32 metadata lane layout equals the f16 one with "group" read as "pair" (CUTLASS
// tmem_e_frg TF32 atom, mma_traits_sm100.hpp:612-621): lane 16 m2 + 8 k1 + m0 holds pairs
// 4 k1 .. 4 k1 + 3 of rows 16 m2 + m0 (bits 0-15) and 16 m2 + 8 + m0 (bits 16-31).
// Q is single-buffered (2 x 32 KB) to fit two-stage K and V rings in shared memory.
#include <type_traits>

#include "flash_common.cuh"

namespace dfss {

namespace {
constexpr int BM = 128, BN = 128, HD = 64;
constexpr int SM_WARPS = 16;
constexpr int NUM_THREADS = (4 + SM_WARPS) * 32;
constexpr uint32_t W_QK = SM_WARPS, W_S = SM_WARPS + 1, W_PV = SM_WARPS + 2, W_PV1 = SM_WARPS + 3;
constexpr int ATOM = BM * 128;               // 16 KB: 128 rows x 32 fp32 (one 128B swizzle column)
constexpr int Q_BYTES = 2 * ATOM;            // 32 KB per half
constexpr int KV_BYTES = 2 * ATOM;           // 32 KB per tile (K: 2 atoms of 32 dims; V^T: 4 atoms of 32 keys)
constexpr int VT_ATOM = HD * 128;            // 8 KB: 64 dims x 32 keys
constexpr int KST = 2, VST = 2;
constexpr int F_Q = 0;                        // [2 halves]
constexpr int F_K = F_Q + 2 * Q_BYTES;
constexpr int F_V = F_K + KST * KV_BYTES;
constexpr int F_RED = F_V + VST * KV_BYTES;   // red_max / red_sum [2 halves][2 pairs][128]
constexpr int F_BAR = F_RED + 2 * 2 * 2 * BM * 4;
constexpr int F_LIVE = F_BAR + 512;           // BlockMask step bitmap + row-block order (sized at launch)
constexpr int F_TOTAL = F_LIVE + 1024;
constexpr int RING = 3;
constexpr int T_O = RING * BN;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kSumLimit = 256.0f;
static_assert(F_TOTAL <= 227 * 1024, "shared memory budget");
static_assert(T_O + 2 * HD <= 512, "TMEM budget");
}  // namespace

// One 32-key chunk of one row, 1:2: 16 pairs (register order (v0, v2, v1, v3) per 4 keys).
// Writes the 16 kept probabilities (fp32), the two metadata words (pairs 0-7, 8-15 at
// bits 4p, nibble 0x4 / 0xE) and the partial row sum.
__device__ __forceinline__ void prune12_chunk(const uint32_t (&s)[32], float c, float mlog, uint32_t (&p)[16],
                                              uint32_t& W0, uint32_t& W1, float& lt0, float& lt1) {
  W0 = W1 = 0x44444444u;
  lt0 = lt1 = 0.f;
#pragma unroll
  for (int g = 0; g < 8; ++g) {  // 4 keys = pairs 2g, 2g + 1
    const float v0 = __uint_as_float(s[4 * g + 0]);
    const float v2 = __uint_as_float(s[4 * g + 1]);
    const float v1 = __uint_as_float(s[4 * g + 2]);
    const float v3 = __uint_as_float(s[4 * g + 3]);
    float d01, d23;
    sub2(v0, v2, v1, v3, d01, d23);  // ties -> +0 (tcgen05 zero sums are +0) -> element 0
    const uint32_t a = __float_as_uint(d01) >> 31, b = __float_as_uint(d23) >> 31;
    // nibble 0x4 + 0xA * [v1 > v0]; W accumulates on top of 0x4 per field
    const uint32_t fields = a * 0xAu + (b * 0xAu << 4);
    if (g < 4)
      W0 += fields << (8 * g);
    else
      W1 += fields << (8 * (g - 4));
    float x0, x1;
    fma2s(fmaxf(v0, v1), fmaxf(v2, v3), c, -mlog, x0, x1);
    const float p0 = fex2(x0), p1 = fex2(x1);
    p[2 * g] = __float_as_uint(p0);
    p[2 * g + 1] = __float_as_uint(p1);
    add2(lt0, lt1, p0, p1, lt0, lt1);
  }
}

__device__ __forceinline__ void tmem_st_x16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

__device__ __forceinline__ void mma_tf32_w(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_sp_tf32_ts_w(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t e_tmem,
                                                 uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %5, 0;\n\t"
      "@e tcgen05.mma.sp.cta_group::1.kind::tf32 [%0], [%1], %2, [%3], %4, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(e_tmem), "r"(idesc), "r"(accumulate)
      : "memory");
}

template <bool MASKED, bool DUMP>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    dfss_flash_tf32_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                           const __grid_constant__ CUtensorMap tm_v, float* __restrict__ out, float scale, int bh,
                           int n, FlashDump dump, TileMask tmask) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = (uint64_t*)(smem + F_BAR);
  uint64_t* q_full = bars;               // [1]
  uint64_t* q_empty = q_full + 1;        // [1]
  uint64_t* k_full = q_empty + 1;        // [KST]
  uint64_t* k_empty = k_full + KST;      // [KST]
  uint64_t* v_full = k_empty + KST;      // [VST]
  uint64_t* v_empty = v_full + VST;      // [VST]
  uint64_t* s_full = v_empty + VST;      // [2 halves][RING] (per half: see dfss_flash2_kernel)
  uint64_t* s_free = s_full + 2 * RING;  // [RING]
  uint64_t* p_full = s_free + RING;      // [2 halves][RING] (8 warps)
  uint64_t* o_full = p_full + 2 * RING;  // [2 halves]
  uint64_t* o_empty = o_full + 2;        // [2 halves] (8 warps)
  uint64_t* pv_done = o_empty + 2;       // [2 halves]
  uint32_t* tmem_slot = (uint32_t*)(pv_done + 2);
  float* red_max = (float*)(smem + F_RED);
  float* red_sum = red_max + 2 * 2 * BM;

  const uint32_t warp = tc::warp_id();
  const uint32_t lane = threadIdx.x & 31;
  // 256-row items; n % 256 == 128 leaves the second half of the last row block empty: that
  // half is treated like a fully masked one (no S / softmax / PV, output not stored)
  const int iblocks = (n + 2 * BM - 1) / (2 * BM);
  const int items = bh * iblocks;
  auto half_ok = [&](int ib, int hh) { return (ib * 2 + hh) * BM < n; };
  const int ntiles = n / BN;
  // BlockMask step skipping and the cost-ranked snake schedule: exactly as dfss_flash2_kernel
  // (flash_tc.cu), which documents the scheme
  uint32_t* s_live = (uint32_t*)(smem + F_LIVE);
  int* s_order = (int*)(s_live + (n / BM) * tmask.sbw);
  if (MASKED) {
    for (int i = threadIdx.x; i < (n / BM) * tmask.sbw; i += blockDim.x) s_live[i] = __ldg(tmask.sbits + i);
    for (int i = threadIdx.x; i < iblocks; i += blockDim.x) s_order[i] = __ldg(tmask.order + i);
  }
  auto pos_at = [&](int k) -> int {
    const int g = gridDim.x;
    return k * g + (MASKED && (k & 1) ? g - 1 - (int)blockIdx.x : (int)blockIdx.x);
  };
  auto item_of = [&](int p) -> int {
    if (!MASKED) return p;
    const int info = s_order[p / bh], r0 = (info >> 8) & 255, m = info >> 16, o = p - r0 * bh;
    return (o / m) * iblocks + (s_order[r0 + o % m] & 255);
  };
  auto live_words = [&](int ib, int t, uint32_t& w0, uint32_t& w1) {
    if (MASKED && (t & 31) == 0) {
      w0 = s_live[(ib * 2) * tmask.sbw + (t >> 5)];
      w1 = half_ok(ib, 1) ? s_live[(ib * 2 + 1) * tmask.sbw + (t >> 5)] : 0u;
    }
  };
  auto bit_u = [&](uint32_t w, int t) { return !MASKED || __any_sync(0xffffffffu, (w >> (t & 31)) & 1u); };
  // liveness of half 1 also needs the half inside the sequence (uniform)
  auto bit1_u = [&](uint32_t w, int t, int ib) { return half_ok(ib, 1) && bit_u(w, t); };

  if (warp == W_QK && lane == 0) {
    tc::prefetch_tmap(&tm_q);
    tc::prefetch_tmap(&tm_k);
    tc::prefetch_tmap(&tm_v);
    tc::mbar_init(q_full, 1);
    tc::mbar_init(q_empty, 1);
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&o_full[i], 1);
      tc::mbar_init(&o_empty[i], 8);
      tc::mbar_init(&pv_done[i], 1);
    }
    for (int i = 0; i < RING; ++i) tc::mbar_init(&s_free[i], 1);
    for (int i = 0; i < 2 * RING; ++i) tc::mbar_init(&s_full[i], 1);
    for (int i = 0; i < 2 * RING; ++i) tc::mbar_init(&p_full[i], 8);
    for (int i = 0; i < KST; ++i) {
      tc::mbar_init(&k_full[i], 1);
      tc::mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < VST; ++i) {
      tc::mbar_init(&v_full[i], 1);
      tc::mbar_init(&v_empty[i], 2);
    }
    tc::fence_barrier_init();
  }
  if (warp == W_PV) tc::tmem_alloc<512>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == W_QK) {
    // ------------------------------------------------------------ TMA: Q (both halves), K (keys permuted), V
    if (lane == 0) {
      int ks = 0, vs = 0, it = 0;
      uint32_t kph = 0, vph = 0;
      for (int kk_ = 0, pos = pos_at(0); pos < items; pos = pos_at(++kk_), ++it) {
        const int item = item_of(pos);
        uint32_t lw0 = 0, lw1 = 0;
        const int b = item / iblocks, ib = item % iblocks;
        tc::mbar_wait_sleep(q_empty, (it & 1) ^ 1);
        tc::mbar_arrive_expect_tx(q_full, 2 * Q_BYTES);
        for (int h = 0; h < 2; ++h)
          for (int a = 0; a < 2; ++a)
            tc::tma_load_3d(smem + F_Q + h * Q_BYTES + a * ATOM, &tm_q, q_full, 32 * a, (ib * 2 + h) * BM, b);
        for (int t = 0; t < ntiles; ++t) {
          live_words(ib, t, lw0, lw1);
          if (MASKED && !(((lw0 | lw1) >> (t & 31)) & 1u)) continue;  // (half 0 is always inside)
          tc::mbar_wait_sleep(&k_empty[ks], kph ^ 1);
          tc::mbar_arrive_expect_tx(&k_full[ks], KV_BYTES);
          for (int a = 0; a < 2; ++a)
            tc::tma_load_5d(smem + F_K + ks * KV_BYTES + a * ATOM, &tm_k, &k_full[ks], 32 * a, 0, 0, t * (BN / 4), b);
          if (++ks == KST) { ks = 0; kph ^= 1; }
          tc::mbar_wait_sleep(&v_empty[vs], vph ^ 1);
          tc::mbar_arrive_expect_tx(&v_full[vs], KV_BYTES);
          for (int a = 0; a < 4; ++a)
            tc::tma_load_3d(smem + F_V + vs * KV_BYTES + a * VT_ATOM, &tm_v, &v_full[vs], t * BN + 32 * a, 0, b);
          if (++vs == VST) { vs = 0; vph ^= 1; }
        }
      }
    }
  } else if (warp == W_S) {
    // ------------------------------------------------------------ S issuer (tf32, 8 MMAs of K = 8)
    {
      constexpr uint32_t idesc_s = tc::instr_desc(2, BM, BN, false, false, false);
      int ks = 0, it = 0, sb = 0;
      uint32_t kph = 0, sph = 0;
      for (int kk_ = 0, pos = pos_at(0); pos < items; pos = pos_at(++kk_), ++it) {
        const int item = item_of(pos);
        uint32_t lw0 = 0, lw1 = 0;
        const int ib = item % iblocks;
        tc::mbar_wait_sleep(q_full, it & 1);
        for (int t = 0; t < ntiles; ++t) {
          live_words(ib, t, lw0, lw1);
          const bool lv[2] = {bit_u(lw0, t), bit1_u(lw1, t, ib)};
          if (!lv[0] && !lv[1]) continue;
          tc::mbar_wait_sleep(&k_full[ks], kph);
          const uint32_t k_addr = tc::smem_u32(smem + F_K + ks * KV_BYTES);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (!lv[h]) continue;
            tc::mbar_wait_sleep(&s_free[sb], sph ^ 1);
            tc::tc_fence_after();
            const uint32_t q_addr = tc::smem_u32(smem + F_Q + h * Q_BYTES);
#pragma unroll
            for (int kk = 0; kk < HD / 8; ++kk) {
              const uint32_t off = (kk >> 2) * ATOM + (kk & 3) * 32;
              const uint64_t ad = tc::smem_desc(q_addr + off, 16, 1024, tc::kSwizzle128B);
              const uint64_t bd = tc::smem_desc(k_addr + off, 16, 1024, tc::kSwizzle128B);
              mma_tf32_w(tmem_base + sb * BN, ad, bd, idesc_s, kk > 0 ? 1u : 0u);
            }
            tc::mma_commit_w(&s_full[h * RING + sb]);
            if (++sb == RING) { sb = 0; sph ^= 1; }
          }
          tc::mma_commit_w(&k_empty[ks]);
          if (++ks == KST) { ks = 0; kph ^= 1; }
        }
        tc::mma_commit_w(q_empty);  // all S MMAs of the item read Q
      }
    }
  } else if (warp == W_PV || warp == W_PV1) {
    // ------------------------------------------------------------ PV issuer of half h (sparse tf32, A in TMEM)
    {
      const int h = warp == W_PV ? 0 : 1;
      constexpr uint32_t idesc_pv = tc::instr_desc(2, BM, HD, false, false, true);  // B = V^T, K-major
      int vs = 0, it = 0;
      uint32_t vph = 0, gcount = 0, pbits = 0;  // live steps so far (both halves); p_full phase per slot
      for (int kk_ = 0, pos = pos_at(0); pos < items; pos = pos_at(++kk_), ++it) {
        const int item = item_of(pos);
        uint32_t lw0 = 0, lw1 = 0;
        const int ib = item % iblocks;
        bool o_free = false;  // O_h drained: awaited lazily, as in dfss_flash2_kernel
        auto await_o_free = [&]() {
          if (!o_free) tc::mbar_wait_sleep(&o_empty[h], (it & 1) ^ 1);
          o_free = true;
        };
        bool first = true;
        for (int t = 0; t < ntiles; ++t) {
          live_words(ib, t, lw0, lw1);
          const bool l0 = bit_u(lw0, t), l1 = bit1_u(lw1, t, ib);
          if (MASKED && !l0 && !l1) continue;  // tile not loaded
          const uint32_t g = gcount + (h ? (uint32_t)l0 : 0u), slot = g % RING;
          gcount += (uint32_t)l0 + (uint32_t)l1;
          if (!(h ? l1 : l0)) {  // this half masked / empty here: release the V stage unused (after its load)
            tc::mbar_wait_sleep(&v_full[vs], vph);
            if (lane == 0) tc::mbar_arrive(&v_empty[vs]);
            if (++vs == VST) { vs = 0; vph ^= 1; }
            continue;
          }
          await_o_free();
          tc::mbar_wait_sleep(&v_full[vs], vph);
          tc::mbar_wait_sleep(&p_full[h * RING + slot], (pbits >> slot) & 1);
          pbits ^= 1u << slot;
          tc::tc_fence_after();
          const uint32_t v_addr = tc::smem_u32(smem + F_V + vs * KV_BYTES);
          const uint32_t s_col = tmem_base + slot * BN;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              // B: keys 32q + 16j .. +16 of V^T (K-major): atom q, 64-byte offset j inside its 128B rows
              const uint64_t bd = tc::smem_desc(v_addr + q * VT_ATOM + 64 * j, 16, 1024, tc::kSwizzle128B);
              mma_sp_tf32_ts_w(tmem_base + T_O + h * HD, s_col + 32 * q + 16 + 8 * j, bd, s_col + 32 * q + 4 * j,
                               idesc_pv, (!first || q > 0 || j > 0) ? 1u : 0u);
            }
          }
          first = false;
          tc::mma_commit_w(&s_free[slot]);
          tc::mma_commit_w(&v_empty[vs]);
          tc::mma_commit_w(&pv_done[h]);
          if (++vs == VST) { vs = 0; vph ^= 1; }
        }
        await_o_free();
        tc::mma_commit_w(&o_full[h]);
      }
    }
  } else if (warp < SM_WARPS) {
    // ------------------------------------------------------------ softmax / prune / epilogue sets
    const int h = warp >> 3;
    const int pr = (warp >> 2) & 1;
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const uint32_t lane_base = tmem_base + ((uint32_t)(quad * 32) << 16);
    const uint32_t pbar = 1 + h * 4 + quad;
    const float c = scale * kLog2e;
    float* rmax = red_max + h * 2 * BM;
    float* rsum = red_sum + h * 2 * BM;
    uint32_t gcount = 0, hcount = 0, scol = 0, sfbits = 0;
    int it = 0;
    bool cm[2] = {false, false};
    auto row_max = [&]() {
      float mt = -INFINITY;
#pragma unroll
      for (int ch = 0; ch < 2; ++ch) {
        uint32_t s[32];
        tc::tmem_ld_32x32b_x32(scol + 32 * ch, s);
        tc::tmem_ld_wait(s);
        float mc = -INFINITY;
#pragma unroll
        for (int j = 0; j < 32; j += 2) mc = fmaxf(mc, fmaxf(__uint_as_float(s[j]), __uint_as_float(s[j + 1])));
        if (!cm[ch]) mt = fmaxf(mt, mc);
      }
      rmax[pr * BM + r] = mt;
      tc::named_bar_sync(pbar, 64);
      const float m = fmaxf(rmax[r], rmax[BM + r]);
      tc::named_bar_sync(pbar, 64);
      return m * c;
    };
    bool pend = false;
    int pend_b = 0, pend_ib = 0, pend_it = 0;
    float pend_l = 0.f;
    auto cword = [&](int pos_) -> uint32_t {  // chunk-keep word `lane` of this warp's strip
      if (!MASKED || pos_ >= items || (int)lane >= tmask.cbw) return 0u;
      if (!half_ok(item_of(pos_) % iblocks, h)) return 0u;
      const int strip = ((item_of(pos_) % iblocks) * 2 + h) * (BM / 32) + quad;
      return __ldg(tmask.cbits + (int64_t)strip * tmask.cbw + lane);
    };
    uint32_t cw = cword(pos_at(0));
    auto epilogue = [&]() {
      rsum[pr * BM + r] = pend_l;
      tc::named_bar_sync(pbar, 64);
      const float inv = 1.0f / (rsum[r] + rsum[BM + r]);
      tc::named_bar_sync(pbar, 64);
      tc::mbar_wait(&o_full[h], pend_it & 1);
      tc::tc_fence_after();
      uint32_t o[32];
      tc::tmem_ld_32x32b_x32(lane_base + T_O + h * HD + 32 * pr, o);
      tc::tmem_ld_wait(o);
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&o_empty[h]);
      pend = false;
      if (!half_ok(pend_ib, h)) return;  // empty half of the last row block
      const int64_t row = (int64_t)pend_b * n + (pend_ib * 2 + h) * BM + r;
      float4* orow = reinterpret_cast<float4*>(out + row * HD + 32 * pr);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        orow[j] = make_float4(__uint_as_float(o[4 * j]) * inv, __uint_as_float(o[4 * j + 1]) * inv,
                              __uint_as_float(o[4 * j + 2]) * inv, __uint_as_float(o[4 * j + 3]) * inv);
    };
    for (int kk_ = 0, pos = pos_at(0); pos < items; pos = pos_at(++kk_), ++it) {
        const int item = item_of(pos);
        uint32_t lw0 = 0, lw1 = 0;
      const int b = item / iblocks, ib = item % iblocks;
      const uint32_t cwn = cword(pos_at(kk_ + 1));
      float mlog = 0.f, l0 = 0.f, l1 = 0.f;
      bool first = true;
      for (int t = 0; t < ntiles; ++t) {
        live_words(ib, t, lw0, lw1);
        const bool lv0 = bit_u(lw0, t), lv1 = bit1_u(lw1, t, ib);
        const uint32_t g = gcount + (h ? (uint32_t)lv0 : 0u);  // global live step
        gcount += (uint32_t)lv0 + (uint32_t)lv1;
        if (!(h ? lv1 : lv0)) continue;
        ++hcount;
        const uint32_t slot = g % RING;
        scol = lane_base + slot * BN + 64 * pr;
        tc::mbar_wait(&s_full[h * RING + slot], (sfbits >> slot) & 1);  // k-th use of (h, slot): parity k & 1
        sfbits ^= 1u << slot;
        tc::tc_fence_after();
        bool anym = false;
        if (MASKED) {
          const int c32 = 4 * t + 2 * pr;
          const uint32_t w = __shfl_sync(0xffffffffu, cw, c32 >> 5) >> (c32 & 31);
          cm[0] = !(w & 1u);
          cm[1] = !(w & 2u);
          anym = __any_sync(0xffffffffu, (~w & 3u) != 0);
        }
        if (first) mlog = row_max();
        uint32_t p[2][16], W[2][2];
        float lt0 = 0.f, lt1 = 0.f;
        auto compute = [&](auto masked_variant) {
          constexpr bool MV = decltype(masked_variant)::value;
          lt0 = lt1 = 0.f;
#pragma unroll
          for (int ch = 0; ch < 2; ++ch) {
            float a0, a1;
            uint32_t s[32];
            tc::tmem_ld_32x32b_x32(scol + 32 * ch, s);
            tc::tmem_ld_wait(s);
            if constexpr (DUMP)
              dump_chunk_scores<true>(dump.s + ((int64_t)b * n + (ib * 2 + h) * BM + r) * n + t * BN + 64 * pr + 32 * ch, s,
                                scale);
            prune12_chunk(s, c, mlog, p[ch], W[ch][0], W[ch][1], a0, a1);
            if (MV && cm[ch]) {  // masked chunk: structurally absent
#pragma unroll
              for (int j = 0; j < 16; ++j) p[ch][j] = 0u;
              W[ch][0] = W[ch][1] = 0x44444444u;
              a0 = a1 = 0.f;
            }
            add2(lt0, lt1, a0, a1, lt0, lt1);
          }
        };
#pragma unroll 1
        for (int pass = 0;; ++pass) {
          if (MASKED && anym) compute(std::true_type{});
          else compute(std::false_type{});
          if (pass > 0 || first || !bar_any(pbar, 64, !(lt0 + lt1 <= kSumLimit))) break;
          tc::mbar_wait(&pv_done[h], (hcount - 2) & 1);
          tc::tc_fence_after();
          const float mnew = fmaxf(mlog, row_max());
          const float f = fex2(mlog - mnew);
          l0 *= f;
          l1 *= f;
#pragma unroll 1
          for (int hh = 0; hh < 2; ++hh) {
            uint32_t o[16];
            const uint32_t oaddr = lane_base + T_O + h * HD + 32 * pr + 16 * hh;
            tc::tmem_ld_32x32b_x16(oaddr, o);
            tc::tmem_ld_wait(o);
#pragma unroll
            for (int j = 0; j < 16; ++j) o[j] = __float_as_uint(__uint_as_float(o[j]) * f);
            tc::tmem_st_32x32b_x16(oaddr, o);
          }
          tc::tmem_st_wait();
          mlog = mnew;
        }
        add2(l0, l1, lt0, lt1, l0, l1);
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const uint32_t Wj = W[ch][j];
            const uint32_t partner = __shfl_xor_sync(0xffffffffu, Wj, 8);
            const uint32_t word =
                (lane & 8) ? ((partner >> 16) | (Wj & 0xFFFF0000u)) : ((Wj & 0xFFFFu) | (partner << 16));
            tc::tmem_st_32x32b_x1(scol + 32 * ch + 4 * j, word);
            if constexpr (DUMP)  // 1:2 meta_hw: 8 pairs (16 columns) per word
              dump.meta[(((int64_t)b * (n / BM) + ib * 2 + h) * (n / 16) + 2 * (4 * t + 2 * pr + ch) + j) * BM + r] =
                  word;
          }
          tmem_st_x16(scol + 32 * ch + 16, p[ch]);
        }
        tc::tmem_st_wait();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&p_full[h * RING + slot]);
        first = false;
        if (pend) epilogue();
      }
      if (pend) epilogue();  // the previous item's, if this item had no live step for this set
      pend = true;
      pend_b = b;
      pend_ib = ib;
      pend_it = it;
      pend_l = l0 + l1;
      cw = cwn;
    }
    if (pend) epilogue();
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == W_PV) {
    tc::tc_fence_after();
    tc::tmem_dealloc<512>(tmem_base);
  }
}

// V [bh][n][64] -> V^T [bh][64][n] (fp32), 32 keys x 64 dims per block through shared memory;
// blockIdx.y strides over bh (gridDim.y is capped at 65535)
__global__ void __launch_bounds__(256) transpose_v_kernel(const float* __restrict__ v, float* __restrict__ vt, int n,
                                                          int64_t bh) {
  __shared__ float tile[32][HD + 1];
  const int k0 = blockIdx.x * 32;
  for (int64_t b = blockIdx.y; b < bh; b += gridDim.y) {
    const float* src = v + ((int64_t)b * n + k0) * HD;
    for (int i = threadIdx.x; i < 32 * HD; i += blockDim.x) tile[i / HD][i % HD] = src[i];
    __syncthreads();
    float* dst = vt + (int64_t)b * HD * n + k0;
    for (int i = threadIdx.x; i < 32 * HD; i += blockDim.x) {
      const int dim = i / 32, key = i % 32;
      dst[(int64_t)dim * n + key] = tile[key][dim];
    }
    __syncthreads();
  }
}

bool tc_flash_tf32_supported(int gs, int n, int d) { return gs == 2 && d == HD && n > 0 && n % BM == 0; }

static int64_t vt_bytes(int64_t bh, int n) { return (bh * (int64_t)n * HD * 4 + 255) / 256 * 256; }

int64_t flash_tf32_workspace_bytes(int64_t bh, int n, bool masked) {
  return vt_bytes(bh, n) + (masked ? flash_mask_workspace_bytes(n) : 0);
}

cudaError_t launch_flash_tf32(const void* q, const void* k, const void* v, void* out, float scale, int64_t bh, int n,
                              int d, const uint8_t* tile_keep, int tile_rows, int tile_cols, void* vt_scratch,
                              cudaStream_t s, float* dump_scores, uint32_t* dump_meta) {
  if (!tc_flash_tf32_supported(2, n, d)) return cudaErrorNotSupported;
  if (tile_keep && (!tc_flash_mask_supported(tile_rows, tile_cols) || !flash_mask_two_set_ok(n)))
    return cudaErrorNotSupported;
  if (bh == 0) return cudaSuccess;
  const CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  CUtensorMap tq, tk, tv;
  const uint64_t row = HD * 4;
  const uint64_t qdims[3] = {(uint64_t)HD, (uint64_t)n, (uint64_t)bh};
  const uint64_t qstr[2] = {row, (uint64_t)n * row};
  const uint32_t qbox[3] = {32, BM, 1};
  // K: keys of every group of 4 permuted to (k0, k2, k1, k3) (see flash_tc.cu)
  const uint64_t kdims[5] = {(uint64_t)HD, 2, 2, (uint64_t)n / 4, (uint64_t)bh};
  const uint64_t kstr[4] = {2 * row, row, 4 * row, (uint64_t)n * row};
  const uint32_t kbox[5] = {32, 2, 2, BN / 4, 1};
  // V^T [bh][64][n]: boxes of 32 keys x 64 dims (one 128B-swizzle atom each)
  const uint64_t vdims[3] = {(uint64_t)n, (uint64_t)HD, (uint64_t)bh};
  const uint64_t vstr[2] = {(uint64_t)n * 4, (uint64_t)n * HD * 4};
  const uint32_t vbox[3] = {32, HD, 1};
  if (!vt_scratch) return cudaErrorInvalidValue;
  if (!encode_tmap(&tq, dt, 3, (void*)q, qdims, qstr, qbox, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !encode_tmap(&tk, dt, 5, (void*)k, kdims, kstr, kbox, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !encode_tmap(&tv, dt, 3, vt_scratch, vdims, vstr, vbox, CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  transpose_v_kernel<<<dim3(n / 32, (unsigned)(bh < 65535 ? bh : 65535)), 256, 0, s>>>((const float*)v, (float*)vt_scratch,
                                                                                n, bh);
  TileMask m{tile_keep, tile_keep ? tile_rows : 1, tile_keep ? tile_cols : 1,
             tile_keep ? (n + tile_cols - 1) / tile_cols : 1};
  // workspace: V^T, then the block-mask bitmaps (flash_tf32_workspace_bytes)
  if (tile_keep) prepare_mask_bits(m, n, (char*)vt_scratch + vt_bytes(bh, n), s);
  const bool dumping = dump_scores != nullptr || dump_meta != nullptr;
  if (dumping && (!dump_scores || !dump_meta)) return cudaErrorInvalidValue;
  FlashDump dump;
  dump.s = dump_scores;
  dump.meta = dump_meta;
  auto kern = tile_keep ? (dumping ? dfss_flash_tf32_kernel<true, true> : dfss_flash_tf32_kernel<true, false>)
                        : (dumping ? dfss_flash_tf32_kernel<false, true> : dfss_flash_tf32_kernel<false, false>);
  const int smem_total = F_TOTAL + (tile_keep ? flash_mask_smem_bytes(n) : 0);
  if (smem_total > 227 * 1024) return cudaErrorNotSupported;
  const int dev = current_device();
  static std::atomic<uint64_t> attr[4];
  cudaError_t e = set_max_smem_once((const void*)kern, attr[(tile_keep ? 2 : 0) + (dumping ? 1 : 0)], dev);
  if (e != cudaSuccess) return e;
  const int sms = device_sms(dev);
  const int64_t items = bh * ((n + 2 * BM - 1) / (2 * BM));
  const int grid = (int)(items < sms ? items : sms);
  kern<<<grid, NUM_THREADS, smem_total, s>>>(tq, tk, tv, (float*)out, scale, (int)bh, n, dump, m);
  return cudaGetLastError();
}

}  // namespace dfss
