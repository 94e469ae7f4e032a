// flash_tc.cu -- fully fused DFSS attention on tcgen05 (2:4 and 1:2, bf16/fp16, head dim 64).
//
// pipeline.nm_attention (pipeline.py:15-32) in one kernel with no n x n tensor of any
// kind in HBM.  Per 128-query half-block h and 128-key tile t:
//   S = Q_h K_t^T                      tcgen05.mma -> TMEM (fp32)
//   prune 2-of-4 in registers          select24 rule of the reference (codec.py:104-123,
//                                      _kernels_numba.py:159-184): signed value, ties to
//                                      the lower index -- on the fp32 scores of S
//   P = exp(s - m) of the kept half    compressed K-major A operand in smem, nibbles as
//                                      tcgen05.mma.sp metadata in TMEM
//   O_h += P V_t                       tcgen05.mma.sp (_spmm_gather, :91-103)
//   O_h / L                            once per item
//
// An item is HALVES x 128 query rows of one head; every K / V tile that streams through
// shared memory serves all halves.  Each SM must ingest 32 KB of K and V per 128 keys, and
// L2 -> SM delivery (~55 B/clk/SM measured) makes that ~600 clocks -- as long as the whole
// prune / exp epilogue of a 128 x 128 tile -- so two halves per K / V tile (HALVES = 2,
// n % 256 == 0) halve the ingress per score.
//
// Softmax (_softmax_nonzeros, _kernels_numba.py:66-84: exp(x - max) / sum over the kept
// entries) is evaluated online with a lazily updated shift: the shift m only has to stay
// within 2^8 of the running maximum for the fp32 sums and the 16-bit P to be safe, so a
// step whose partial sum exceeds 2^8 (or is not finite) takes a slow path that raises m to
// the true maximum and rescales the running O and sum; in steady state no max is computed
// at all.  The result is mathematically the reference's exp(x - max)/sum; only rounding
// differs.
//
// Work split: 16 softmax warps, warp (quad, quarter) owns TMEM lanes 32*quad.. (rows) and
// score columns [32*quarter, +32) of every tile (= one K = 32 tcgen05.mma.sp).  The four
// warps of a quad share the rows, hence the shift: every step they OR-reduce their "partial
// sum too large" flags with one bar.red.or over the quad, and on the rare update exchange
// their maxima through shared memory.  Steps run (t, h) = (0,0), (0,1), (1,0), ...
//
// Register pairing for FADD2/FFMA2: the K tile is loaded through a 5-D tensor map whose
// strides permute the keys of every group of 4 into (k0, k2, k1, k3), so S columns arrive
// as (v0, v2, v1, v3) and the differences v0 - v1, v2 - v3 are one FADD2 of two natural
// register pairs.  The selection itself still names v0..v3 by their true key index, so
// tie-breaking is unchanged; V and the metadata stay in true key order.
//
// TMEM (512 columns): S buffers at 0 / 128 (step parity), O_h at 256 + 64h, metadata of
// P stage p at 384 + 4p + quarter.
//
// Warp roles (one CTA per SM, persistent over items): warps 0-15 softmax / prune / epilogue,
// warp 16 TMA Q/K, warp 17 S issuer, warp 18 TMEM allocator + PV issuer, warp 19 TMA V.
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <type_traits>

#include "flash_common.cuh"


namespace dfss {

namespace {
constexpr int BM = 128;   // query rows per half (TMEM lanes)
constexpr int BN = 128;   // keys per tile
constexpr int HD = 64;    // head dim
constexpr int KST = 3;    // K ring
constexpr int VST = 3;    // V ring
constexpr int PST = 2;    // P stages (smem) / metadata stages (TMEM)
constexpr int SM_WARPS = 16;
constexpr int NUM_THREADS = (4 + SM_WARPS) * 32;
// Role warps sit at the highest warp ids (16..19): the sub-partition scheduler prefers high
// warp ids, so a single-thread TMA producer / MMA issuer is served as soon as it is ready
// instead of waiting for a stall of the four arithmetic warps sharing its sub-partition.
constexpr uint32_t W_QK = SM_WARPS, W_S = SM_WARPS + 1, W_PV = SM_WARPS + 2, W_V = SM_WARPS + 3;
constexpr uint32_t W_PV1 = W_V;  // two-set kernel: PV issuer of half 1 (V is loaded by W_QK there)
constexpr int Q_BYTES = BM * HD * 2;        // 16 KB per half
constexpr int K_BYTES = BN * HD * 2;        // 16 KB
constexpr int V_BYTES = BN * HD * 2;        // 16 KB
constexpr int P_BYTES = BM * (BN / 2) * 2;  // 16 KB: 128 rows x 64 kept values
constexpr int SMEM_Q = 0;                   // [2 stages][2 halves]
constexpr int SMEM_K = SMEM_Q + 4 * Q_BYTES;
constexpr int SMEM_V = SMEM_K + KST * K_BYTES;
constexpr int SMEM_P = SMEM_V + VST * V_BYTES;
constexpr int SMEM_RED = SMEM_P + PST * P_BYTES;  // [2 (max, sum)][4 quarters][128] floats
constexpr int SMEM_BAR = SMEM_RED + 2 * 4 * BM * 4;
constexpr int SMEM_TOTAL = SMEM_BAR + 256 + 1024;
constexpr int TM_O = 2 * BN;     // O_h at TM_O + 64 h
constexpr int TM_E = TM_O + 2 * HD;  // PST x 4 metadata columns
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kSumLimit = 256.0f;  // a quarter-tile partial sum above 2^8 triggers a shift update
// an item's first step summing below the floor: its start shift (carried from the previous item)
// is too high -- recompute with the exact maximum.  fp16 P must stay out of the denormal range
// (< 2^-14): 2^-6 keeps the significant terms normal; bf16 shares fp32's exponent range.
template <typename T>
__host__ __device__ constexpr float sum_floor() {
  return std::is_same<T, __half>::value ? 1.0f / 64.0f : 1.0f / 65536.0f;
}
}  // namespace

// Split of the last round (two-set kernel, unmasked): `items` equal items on G persistent CTAs
// leave items % G of them for a last round in which the other CTAs idle (c2: 768 items on 148
// SMs = 5.19 rounds, 14 % of the kernel).  Those `rem` items are cut along the keys into
// `parts` contiguous tile ranges, one per CTA; parts 1.. leave their unnormalised O, shift and
// row sum in the workspace behind a flag holding the launch's token (so no memset is needed:
// a reused workspace holds older tokens) and part 0 merges them:
// O = sum_p 2^(m_p - M) O_p / sum_p 2^(m_p - M) l_p, M = max_p m_p.
struct SplitPlan {
  int rounds = 0;   // whole rounds: unit k < rounds of CTA b is item k * G + b
  int rem = 0;      // items of the last round
  int parts = 1;    // key ranges per last-round item (1: no split)
  unsigned long long token = 0;   // per launch: a part's flag holds it once its data is written
  float* part_ws = nullptr;       // [rem][2 halves][8 warps][parts][34][32 lanes]
  unsigned long long* counters = nullptr;  // flags [rem][2 halves][8 warps][parts]
};

// One quarter-tile of one row: 8 groups of 4 scores s[] in key order.  Prunes 2:4 (reference
// rule), exponentiates the kept half against the shift `mlog` (= m * c), packs P, builds the
// metadata word W (group g at bits 4g) and the partial sum.
//
// Instruction budget per group (the kernel is bound by instruction issue: 23 warp instructions
// per group, tools/sass_region.py): ALU -- 4 FMNMX, 2 FSETP, 4 FSEL (lo, hi, two nibble
// overrides), F2FP; FMA pipe -- 2 FADD (pair differences), FMUL2 + 2 FMUL.SAT (pair-winner
// flags), 2 FFMA (nibble), FFMA2 (exponent arguments), FADD2 (row sums); XU -- 2 MUFU.EX2.
// Key-order registers make the kept pair land in the
// registers of (v0, v1) -- an aligned pair for FFMA2 -- and each of lo / hi is one FSEL
// predicated on "that register's own value is not the kept one" (keep01 keeps v0 / v1).
//
// PAIRS (mode 1:2 on 16-bit data): keep the larger of each pair, element 1 iff v1 > v0
// (codec.py:114-117) -- on the tensor core this is the 2:4 pattern with one survivor per
// pair, nibble 8 + a + 4b, so the same sparse MMA consumes it.
template <typename T, bool PAIRS>
__device__ __forceinline__ void prune_exp_tile(const uint32_t (&s)[32], float c, float mlog, uint32_t two,
                                               uint32_t (&pk)[8], uint32_t& W, float& lt0, float& lt1) {
#ifdef DFSS_EXP_NO_PRUNE  // timing experiment: no selection, no exp (results invalid)
  W = 0x44444444u ^ (s[0] & 0x11111111u);
  lt0 = __uint_as_float(s[1]) * 0.f;
  lt1 = 0.f;
#pragma unroll
  for (int g = 0; g < 8; ++g) pk[g] = s[4 * g] ^ s[4 * g + 2];
  return;
#endif
  W = 0x88888888u;
  lt0 = 0.f;
  lt1 = 0.f;
  // 2:4 metadata in float arithmetic on the otherwise idle FMA-lite pipe: nibble - 8 of groups
  // 0-3 / 4-7 accumulated exactly as integers into 2^23 + 0x8888 (ulp 1), low halves merged by
  // one PRMT at the end (tools/epi_probe.cu: -12 % against sign bits by IMAD.HI + SEL chains)
  float wf[2] = {8388608.f + 34952.f, 8388608.f + 34952.f};
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    const float v0 = __uint_as_float(s[4 * g + 0]);
    const float v1 = __uint_as_float(s[4 * g + 1]);
    const float v2 = __uint_as_float(s[4 * g + 2]);
    const float v3 = __uint_as_float(s[4 * g + 3]);
    // winner index of each pair from the sign of the difference (ties -> +0 -> lower index).
    // tcgen05.mma writes every zero score as +0 (tools/negzero_probe.cu; covered by
    // test_flash_tie_lattice_and_zero_queries), so (-0) - (+0) cannot occur and the
    // differences need no canonicalisation.
    const float d01 = v0 - v1, d23 = v2 - v3;
    const float w01 = fmaxf(v0, v1), w23 = fmaxf(v2, v3);
    float lo = w01, hi = w23;
    if (PAIRS) {
      // sign bits on the otherwise idle ALU pipe (1:2 is FMA / MUFU-bound); nibble 8 + a + 4b
      const uint32_t a = __float_as_uint(d01) >> 31, b = __float_as_uint(d23) >> 31;
      W += (a + 4u * b) * (1u << (4 * g));
    } else {
      const float l01 = fminf(v0, v1), l23 = fminf(v2, v3);
      const bool keep01 = l01 >= w23;  // lower-index loser vs higher-index winner
      const bool keep23 = l23 > w01;   // higher-index loser must strictly beat the winner
      lo = keep01 ? v0 : (keep23 ? v2 : w01);
      hi = keep01 ? v1 : (keep23 ? v3 : w23);
      // a = [v1 > v0], b = [v3 > v2] as exact 0 / 1 floats: sat(d * -2^127 * 2^127) is 1 for
      // every d < 0 down to the smallest subnormal and 0 for d >= 0 (ties: d = +0 -> lower index)
      // (the first multiplies of both pairs are one FMUL2: c4 -2 %, c2 -2 %; pairing groups g and
      // g + 4 for the nibble FFMAs as well saved another instruction per group statically but ran
      // 1-2 % slower)
      float t01, t23;
      mul2s(d01, d23, -1.7014118e38f, t01, t23);
      const float fa = __saturatef(t01 * 1.7014118e38f);
      const float fb = __saturatef(t23 * 1.7014118e38f);
      // nibble - 8: 0x4 -> -4, 0xE -> 6, mixed 8 + a + 4b -> a + 4b
      float n = fmaf(fb, 4.f, fa);
      n = keep23 ? 6.f : n;
      n = keep01 ? -4.f : n;
      wf[g >> 2] = fmaf(n, (float)(1 << (4 * (g & 3))), wf[g >> 2]);
      if (g == 7) W = __byte_perm(__float_as_uint(wf[0]), __float_as_uint(wf[1]), 0x5410);
    }
    float x0, x1;
    fma2s(lo, hi, c, -mlog, x0, x1);
    const float p0 = fex2(x0), p1 = fex2(x1);
    pk[g] = fpack2<T>(p0, p1);
    add2(lt0, lt1, p0, p1, lt0, lt1);
  }
}

template <typename T, int HALVES, bool PAIRS, bool MASKED, bool DUMP>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    dfss_flash_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                      const __grid_constant__ CUtensorMap tm_v, T* __restrict__ out, float scale, int bh, int n,
                      uint32_t two, FlashDump dump, TileMask tmask, SplitPlan /*two-set kernel only*/) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = (uint64_t*)(smem + SMEM_BAR);
  uint64_t* q_full = bars;              // [2]
  uint64_t* q_empty = q_full + 2;       // [2]
  uint64_t* k_full = q_empty + 2;       // [KST]
  uint64_t* k_empty = k_full + KST;     // [KST]
  uint64_t* v_full = k_empty + KST;     // [VST]
  uint64_t* v_empty = v_full + VST;     // [VST]
  uint64_t* s_full = v_empty + VST;     // [2] S of a step computed
  uint64_t* s_empty = s_full + 2;       // [2] every softmax warp read its scores (SM_WARPS)
  uint64_t* p_full = s_empty + 2;       // [PST] P smem + metadata written (SM_WARPS)
  uint64_t* p_empty = p_full + PST;     // [PST] PV retired
  uint64_t* o_full = p_empty + PST;     // [1] item's last PV retired
  uint64_t* o_empty = o_full + 1;       // [1] O drained (SM_WARPS)
  uint32_t* tmem_slot = (uint32_t*)(o_empty + 1);
  float* red_max = (float*)(smem + SMEM_RED);
  float* red_sum = red_max + 4 * BM;

  const uint32_t warp = tc::warp_id();
  const uint32_t lane = threadIdx.x & 31;
  const int iblocks = n / (BM * HALVES);  // items per (batch, head)
  const int items = bh * iblocks;
  const int ntiles = n / BN;

  if (warp == W_QK && lane == 0) {
    tc::prefetch_tmap(&tm_q);
    tc::prefetch_tmap(&tm_k);
    tc::prefetch_tmap(&tm_v);
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&q_full[i], 1);
      tc::mbar_init(&q_empty[i], 1);
      tc::mbar_init(&s_full[i], 1);
      tc::mbar_init(&s_empty[i], SM_WARPS);
    }
    for (int i = 0; i < PST; ++i) {
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
  if (warp == W_PV) tc::tmem_alloc<512>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == W_QK) {
    // ------------------------------------------------------------ TMA producer: Q (all halves) and K (keys permuted)
    if (lane == 0) {
      int ks = 0, it = 0;
      uint32_t kph = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
        const int b = item / iblocks, ib = item % iblocks;
        const int qs = it & 1;
        tc::mbar_wait_sleep(&q_empty[qs], ((it >> 1) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(&q_full[qs], HALVES * Q_BYTES);
#pragma unroll
        for (int h = 0; h < HALVES; ++h)
          tc::tma_load_3d(smem + SMEM_Q + (2 * qs + h) * Q_BYTES, &tm_q, &q_full[qs], 0, (ib * HALVES + h) * BM, b);
        for (int t = 0; t < ntiles; ++t) {
          tc::mbar_wait_sleep(&k_empty[ks], kph ^ 1);
          tc::mbar_arrive_expect_tx(&k_full[ks], K_BYTES);
          tc::tma_load_3d(smem + SMEM_K + ks * K_BYTES, &tm_k, &k_full[ks], 0, t * BN, b);
          if (++ks == KST) { ks = 0; kph ^= 1; }
        }
      }
    }
  } else if (warp == W_V) {
    // ------------------------------------------------------------ TMA producer: V
    if (lane == 0) {
      int vs = 0;
      uint32_t vph = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x) {
        const int b = item / iblocks;
        for (int t = 0; t < ntiles; ++t) {
          tc::mbar_wait_sleep(&v_empty[vs], vph ^ 1);
          tc::mbar_arrive_expect_tx(&v_full[vs], V_BYTES);
          tc::tma_load_3d(smem + SMEM_V + vs * V_BYTES, &tm_v, &v_full[vs], 0, t * BN, b);
          if (++vs == VST) { vs = 0; vph ^= 1; }
        }
      }
    }
  } else if (warp == W_S) {
    // ------------------------------------------------------------ S issuer: step g = (t, h) -> S buffer g & 1
    if (lane == 0) {
      constexpr uint32_t fmt = std::is_same<T, __nv_bfloat16>::value ? 1u : 0u;
      constexpr uint32_t idesc_s = tc::instr_desc(fmt, BM, BN, false, false, false);
      int ks = 0, it = 0;
      uint32_t kph = 0, g = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
        const int qs = it & 1;
        tc::mbar_wait_sleep(&q_full[qs], (it >> 1) & 1);
        for (int t = 0; t < ntiles; ++t) {
          tc::mbar_wait_sleep(&k_full[ks], kph);
          const uint32_t k_addr = tc::smem_u32(smem + SMEM_K + ks * K_BYTES);
#pragma unroll
          for (int h = 0; h < HALVES; ++h, ++g) {
            const uint32_t sb = g & 1;
            tc::mbar_wait_sleep(&s_empty[sb], ((g >> 1) & 1) ^ 1);  // step g-2 read by every softmax warp
            tc::tc_fence_after();
            const uint32_t q_addr = tc::smem_u32(smem + SMEM_Q + (2 * qs + h) * Q_BYTES);
#pragma unroll
            for (int kk = 0; kk < HD / 16; ++kk) {
              const uint64_t ad = tc::smem_desc(q_addr + kk * 32, 16, 1024, tc::kSwizzle128B);
              const uint64_t bd = tc::smem_desc(k_addr + kk * 32, 16, 1024, tc::kSwizzle128B);
              tc::mma_f16_ss(tmem_base + sb * BN, ad, bd, idesc_s, kk > 0 ? 1u : 0u);
            }
            tc::mma_commit(&s_full[sb]);
          }
          tc::mma_commit(&k_empty[ks]);
          if (++ks == KST) { ks = 0; kph ^= 1; }
        }
        tc::mma_commit(&q_empty[qs]);
      }
    }
  } else if (warp == W_PV) {
    // ------------------------------------------------------------ PV issuer: O_h += P V_t (4 sparse K=32 MMAs)
    if (lane == 0) {
      constexpr uint32_t fmt = std::is_same<T, __nv_bfloat16>::value ? 1u : 0u;
      constexpr uint32_t idesc_pv = tc::instr_desc(fmt, BM, HD, false, true, true);
      int vs = 0, pb = 0;
      uint32_t vph = 0, pph = 0, oph = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x) {
        tc::mbar_wait_sleep(o_empty, oph ^ 1);
        for (int t = 0; t < ntiles; ++t) {
          tc::mbar_wait_sleep(&v_full[vs], vph);
          const uint32_t v_addr = tc::smem_u32(smem + SMEM_V + vs * V_BYTES);
#pragma unroll
          for (int h = 0; h < HALVES; ++h) {
            tc::mbar_wait_sleep(&p_full[pb], pph);
            tc::tc_fence_after();
            const uint32_t p_addr = tc::smem_u32(smem + SMEM_P + pb * P_BYTES);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint64_t ad = tc::smem_desc(p_addr + q * 32, 16, 1024, tc::kSwizzle128B);
              const uint64_t bd = tc::smem_desc(v_addr + q * 32 * 128, V_BYTES, 1024, tc::kSwizzle128B);
              // metadata column: even address + sparse_id2 (idesc bits [0,2)) selects the odd one
              const uint32_t e_col = tmem_base + TM_E + pb * 4 + q;
              tc::mma_sp_f16_ss(tmem_base + TM_O + h * HD, ad, bd, e_col & ~1u, idesc_pv | (e_col & 1u),
                                (t > 0 || q > 0) ? 1u : 0u);
            }
            tc::mma_commit(&p_empty[pb]);
            if (++pb == PST) { pb = 0; pph ^= 1; }
          }
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
    const int quarter = warp >> 2;
    const int r = quad * 32 + lane;  // row within the half == TMEM lane
    const uint32_t lane_base = tmem_base + ((uint32_t)(quad * 32) << 16);
    const uint32_t qbar = 1 + quad;  // named barrier of the four warps sharing these rows
    const float c = scale * kLog2e;
    // P row r, 16-byte units (2*quarter, +1) of the 128B-swizzled row
    const uint32_t p_row = tc::smem_u32(smem + SMEM_P) + r * 128;
    const uint32_t u0 = (uint32_t)(((2 * quarter) ^ (r & 7)) << 4), u1 = (uint32_t)(((2 * quarter + 1) ^ (r & 7)) << 4);
    int pb = 0;
    uint32_t pph = 0, oph = 0, g = 0;
    // row maximum of the current step over the quad's four quarters (scaled to log2 units)
    bool cmask = false;  // this warp's chunk of the current tile is masked (BlockMask)
    auto row_max = [&](const uint32_t (&s)[32]) {
      float mt = -INFINITY;
      if (!cmask) {
#pragma unroll
        for (int j = 0; j < 32; j += 2) mt = fmaxf(mt, fmaxf(__uint_as_float(s[j]), __uint_as_float(s[j + 1])));
      }
      red_max[quarter * BM + r] = mt;
      tc::named_bar_sync(qbar, 128);
      const float m = fmaxf(fmaxf(red_max[r], red_max[BM + r]), fmaxf(red_max[2 * BM + r], red_max[3 * BM + r]));
      tc::named_bar_sync(qbar, 128);  // red_max is reused by the next exchange
      return m * c;
    };
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
      const int b = item / iblocks, ib = item % iblocks;
      float mlog[HALVES];          // shift in log2 units (m * c), shared by the quad's four warps
      float l0[HALVES], l1[HALVES];  // this quarter's running row sums (pairs)
      for (int t = 0; t < ntiles; ++t) {
#pragma unroll
        for (int h = 0; h < HALVES; ++h, ++g) {
          const uint32_t sb = g & 1;
          tc::mbar_wait(&s_full[sb], (g >> 1) & 1);
          tc::tc_fence_after();
          uint32_t s[32];
          tc::tmem_ld_32x32b_x32(lane_base + sb * BN + quarter * 32, s);
          tc::tmem_ld_wait(s);
          tc::tc_fence_before();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&s_empty[sb]);
          if constexpr (DUMP)
            dump_chunk_scores<false>(dump.s + ((int64_t)b * n + (ib * HALVES + h) * BM + r) * n + t * BN + quarter * 32, s,
                              scale);
          uint32_t pk[8], W;
          float lt0, lt1;
          cmask = MASKED && tmask.masked((ib * HALVES + h) * BM + quad * 32, t * BN + quarter * 32);
          // P stage pb: PV of step g - PST (for PST = 2 and two halves: this half's previous tile) retired
          tc::mbar_wait(&p_empty[pb], pph ^ 1);
          tc::tc_fence_after();
          if (t == 0) {
            // first tile of the item: the shift starts at the row maximum of this tile
            mlog[h] = row_max(s);
            l0[h] = l1[h] = 0.f;
            if (cmask) masked_chunk(pk, W, lt0, lt1); else prune_exp_tile<T, PAIRS>(s, c, mlog[h], two, pk, W, lt0, lt1);
          } else {
            if (cmask) masked_chunk(pk, W, lt0, lt1); else prune_exp_tile<T, PAIRS>(s, c, mlog[h], two, pk, W, lt0, lt1);
            if (bar_any(qbar, 128, !(lt0 + lt1 <= kSumLimit) || W == ~0u)) {  // W: see the two-set kernel
              // ---- slow path (whole quad): raise the shift to the row maximum, rescale O_h and the sums.
              // Every PV into O_h issued so far has retired: with PST == HALVES the P-stage wait
              // above was for this half's previous tile; otherwise wait for the step before.
              if (PST != HALVES) tc::mbar_wait(&p_empty[pb ^ 1], pb == 0 ? pph ^ 1 : pph);
              tc::tc_fence_after();
              const float mnew = fmaxf(mlog[h], row_max(s));
              const float f = fex2(mlog[h] - mnew);
              l0[h] *= f;
              l1[h] *= f;
              uint32_t o[16];
              const uint32_t oaddr = lane_base + TM_O + h * HD + 16 * quarter;
              tc::tmem_ld_32x32b_x16(oaddr, o);
              tc::tmem_ld_wait(o);
#pragma unroll
              for (int j = 0; j < 16; ++j) o[j] = __float_as_uint(__uint_as_float(o[j]) * f);
              tc::tmem_st_32x32b_x16(oaddr, o);
              tc::tmem_st_wait();
              mlog[h] = mnew;
              if (cmask) masked_chunk(pk, W, lt0, lt1); else prune_exp_tile<T, PAIRS>(s, c, mlog[h], two, pk, W, lt0, lt1);
            }
          }
          add2(l0[h], l1[h], lt0, lt1, l0[h], l1[h]);
          const uint32_t prow = p_row + pb * P_BYTES;
          sts128(prow + u0, pk[0], pk[1], pk[2], pk[3]);
          sts128(prow + u1, pk[4], pk[5], pk[6], pk[7]);
          // metadata word of TMEM lane r: rows r and r^8 trade 16-bit halves (include/dfss.h)
          const uint32_t partner = __shfl_xor_sync(0xffffffffu, W, 8);
          const uint32_t word = (lane & 8) ? ((partner >> 16) | (W & 0xFFFF0000u)) : ((W & 0xFFFFu) | (partner << 16));
          tc::tmem_st_32x32b_x1(lane_base + TM_E + pb * 4 + quarter, word);
          if constexpr (DUMP)
            dump.meta[(((int64_t)b * (n / BM) + ib * HALVES + h) * (n / 32) + 4 * t + quarter) * BM + r] = word;
          tc::tmem_st_wait();
          tc::fence_proxy_async();  // P smem writes -> tensor core
          tc::tc_fence_before();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&p_full[pb]);
          if (++pb == PST) { pb = 0; pph ^= 1; }
        }
      }
      // ---- epilogue: O_h / (sum over the four quarters' row sums); warp writes columns [16q, +16)
      tc::mbar_wait(o_full, oph);
      oph ^= 1;
      tc::tc_fence_after();
      uint32_t o[HALVES][16];
#pragma unroll
      for (int h = 0; h < HALVES; ++h) tc::tmem_ld_32x32b_x16(lane_base + TM_O + h * HD + 16 * quarter, o[h]);
#pragma unroll
      for (int h = 0; h < HALVES; ++h) tc::tmem_ld_wait(o[h]);
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(o_empty);
#pragma unroll
      for (int h = 0; h < HALVES; ++h) {
        red_sum[quarter * BM + r] = l0[h] + l1[h];
        tc::named_bar_sync(qbar, 128);
        const float inv =
            1.0f / ((red_sum[r] + red_sum[BM + r]) + (red_sum[2 * BM + r] + red_sum[3 * BM + r]));
        tc::named_bar_sync(qbar, 128);
        uint32_t pko[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
          pko[j] = fpack2<T>(__uint_as_float(o[h][2 * j]) * inv, __uint_as_float(o[h][2 * j + 1]) * inv);
        const int64_t row = (int64_t)b * n + (ib * HALVES + h) * BM + r;
        uint4* orow = reinterpret_cast<uint4*>(out + row * HD + 16 * quarter);
        orow[0] = make_uint4(pko[0], pko[1], pko[2], pko[3]);
        orow[1] = make_uint4(pko[4], pko[5], pko[6], pko[7]);
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == W_PV) {
    tc::tc_fence_after();
    tc::tmem_dealloc<512>(tmem_base);
  }
}

// ============================================================================ two-set kernel
// n % 256 == 0: an item is 256 query rows (halves h = 0, 1) of one head.  The 16 softmax
// warps split into two independent sets of 8, set h owning half h: warp (quad, pair) of a
// set holds rows 32*quad.. and score columns [64*pair, +64) of every 128-key tile as two
// 32-column chunks (= two K = 32 tcgen05.mma.sp).  The sets share the K / V stream but
// not their latency chains, so one set's TMEM / barrier latencies overlap the other set's
// arithmetic on every SM sub-partition (2 + 2 warps each).
//
// Steps g = 2t + h use a ring of three 128-column TMEM S buffers.  The compressed P of a
// step (16 kept values per row and quarter = 8 columns of 16-bit pairs) and its metadata
// are written with tcgen05.st back into the step's own S buffer (quarter q: metadata at
// column 32q, P at 32q + 16, both already read) and the sparse PV reads A straight from
// TMEM: no shared-memory staging and no generic -> async proxy fence per tile.  A buffer
// is free again once its PV retired; a set's next S (step g + 2) lands in the buffer of
// step g - 1 and is computed while the set is still pruning step g.
//
// Tensor cost per 128 x 128 step (measured, tools/mma_probe.cu): 4 x 64 clk for S (SS,
// N = 128) + 4 x 46 clk for the sparse PV (A in TMEM) -- an M = 128 MMA costs >= ~46 clk
// whatever its N, so 128-key tiles, not 64, keep the tensor pipe under the epilogue.
namespace {
constexpr int K2ST = 4, V2ST = 4;             // K ring, V ring (128-key tiles, 16 KB each)
constexpr int S2_Q = 0;                        // [2 stages][2 halves] x 16 KB
constexpr int S2_K = S2_Q + 4 * Q_BYTES;
constexpr int S2_V = S2_K + K2ST * K_BYTES;
constexpr int S2_RED = S2_V + V2ST * V_BYTES;  // red_max / red_sum: [2 halves][2 pairs][128] floats each
constexpr int S2_BAR = S2_RED + 2 * 2 * 2 * BM * 4;
constexpr int S2_LIVE = S2_BAR + 512;             // BlockMask step bitmap (masked kernels; sized at launch)
constexpr int S2_TOTAL = S2_LIVE + 1024;
constexpr int S2RING = 3;                      // S buffers (TMEM), 128 columns each
constexpr int T2_O = S2RING * BN;              // O_h at T2_O + 64 h
static_assert(T2_O + 2 * HD <= 512, "TMEM budget");
static_assert(S2_TOTAL <= 227 * 1024, "shared memory budget");
}  // namespace

// bring-up timeline (DFSS_FLASH_TRACE=<file>): clock64 at pipeline events of CTA 0, first 2
// items.  Compiled in only with -DDFSS_FLASH_TRACE_BUILD (DFSS_NVCC_EXTRA, tools/trace_flash.py):
// the per-lane trace predicates cost ~5 % issue slots in the epilogue-bound kernel.
#ifdef DFSS_FLASH_TRACE_BUILD
__device__ unsigned long long* g_flash_trace = nullptr;
#define FTRACE(slot, it_, t_, h_)                                                                  \
  do {                                                                                             \
    if (trace && (it_) < 2 && (t_) < 64)                                                           \
      trace[((((slot) * 2 + (it_)) * 64 + (t_)) * 2 + (h_))] = clock64();                          \
  } while (0)
// per-CTA unit timeline: [CTA < 148][unit < 16][event < 8] after the CTA-0 trace
#define UTRACE(k_, ev_)                                                                                  \
  do {                                                                                                   \
    if (g_flash_trace && blockIdx.x < 148 && (k_) < 16)                                                  \
      g_flash_trace[16 * 2 * 64 * 2 + ((blockIdx.x * 16 + (k_)) * 8 + (ev_))] = clock64();               \
  } while (0)
#else
#define FTRACE(slot, it_, t_, h_) \
  do {                            \
  } while (0)
#define UTRACE(k_, ev_) \
  do {                  \
  } while (0)
#endif

// One warp's part of a split last-round item (SplitPlan): parts 1.. leave their 32 rows x 32
// columns of unnormalised O, the rows' shift (log2 units) and sum in the workspace and publish
// them with a release store of the launch token; part 0 keeps its own in registers, waits for
// the other parts' tokens (one lane per part, acquire loads) and merges.  Part 0 of an item
// is the CTA with the lowest id; all parts hold (nearly) the same number of tiles.
template <typename T>
__device__ __forceinline__ void split_part_epilogue(const SplitPlan& sp, int ui, int h, int w, int part, uint32_t lane,
                                                    const uint32_t (&o)[32], float mlog, float lsum, T* dst) {
  const int64_t slot = ((int64_t)(ui * 2 + h) * 8 + w) * sp.parts;
  unsigned long long* flags = sp.counters + slot;
  if (part > 0) {
    float* mine = sp.part_ws + (slot + part) * 34 * 32 + lane;
#pragma unroll
    for (int j = 0; j < 32; ++j) __stcg(mine + j * 32, __uint_as_float(o[j]));
    __stcg(mine + 32 * 32, mlog);
    __stcg(mine + 33 * 32, lsum);
    __syncwarp();
    if (lane == 0) {
      __threadfence();
      asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(flags + part), "l"(sp.token) : "memory");
    }
    return;
  }
  // part 0: wait for parts 1 .. parts-1 (lane p polls part p)
  for (;;) {
    bool ok = true;
    if (lane > 0 && (int)lane < sp.parts) {
      unsigned long long f;
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(f) : "l"(flags + lane) : "memory");
      ok = f == sp.token;
    }
    if (__all_sync(0xffffffffu, ok)) break;
    __nanosleep(64);
  }
  __threadfence();
  float m = mlog;
  for (int p = 1; p < sp.parts; ++p) m = fmaxf(m, __ldcg(sp.part_ws + ((slot + p) * 34 + 32) * 32 + lane));
  const float f0 = exp2f(mlog - m);
  float acc[32], l = f0 * lsum;
#pragma unroll
  for (int j = 0; j < 32; ++j) acc[j] = f0 * __uint_as_float(o[j]);
  for (int p = 1; p < sp.parts; ++p) {
    const float* q = sp.part_ws + (slot + p) * 34 * 32 + lane;
    float x[34];
#pragma unroll
    for (int j = 0; j < 34; ++j) x[j] = __ldcg(q + j * 32);
    const float f = exp2f(x[32] - m);
    l = fmaf(f, x[33], l);
#pragma unroll
    for (int j = 0; j < 32; ++j) acc[j] = fmaf(f, x[j], acc[j]);
  }
  const float inv = 1.0f / l;
  uint32_t pko[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) pko[j] = fpack2<T>(acc[2 * j] * inv, acc[2 * j + 1] * inv);
  uint4* orow = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int j = 0; j < 4; ++j) orow[j] = make_uint4(pko[4 * j], pko[4 * j + 1], pko[4 * j + 2], pko[4 * j + 3]);
}

template <typename T, bool PAIRS, bool MASKED, bool DUMP>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    dfss_flash2_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                       const __grid_constant__ CUtensorMap tm_v, T* __restrict__ out, float scale, int bh, int n,
                       uint32_t two, FlashDump dump, TileMask tmask, SplitPlan sp) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = (uint64_t*)(smem + S2_BAR);
  uint64_t* q_full = bars;                // [2]
  uint64_t* q_empty = q_full + 2;         // [2]
  uint64_t* k_full = q_empty + 2;         // [K2ST]
  uint64_t* k_empty = k_full + K2ST;      // [K2ST]
  uint64_t* v_full = k_empty + K2ST;      // [V2ST]
  uint64_t* v_empty = v_full + V2ST;      // [V2ST]
  // [2 halves][S2RING] S of a step computed.  Per half: when one set runs several live steps in
  // a row (masks, an empty half) a shared slot barrier could complete two phases past a waiting
  // set, whose parity wait would then succeed on the wrong step.  (P + metadata of a step
  // written is signalled on named barriers 9.. 14, per half, see the PV issuer.)
  uint64_t* s_full = v_empty + V2ST;
  uint64_t* s_free = s_full + 2 * S2RING; // [S2RING] PV of that step retired (buffer free)
  uint64_t* o_full = s_free + S2RING;     // [2 halves]
  uint64_t* o_empty = o_full + 2;         // [2 halves] (8 warps)
  uint64_t* pv_done = o_empty + 2;        // [2 halves] every PV of this half so far retired
  uint32_t* tmem_slot = (uint32_t*)(pv_done + 2);
  float* red_max = (float*)(smem + S2_RED);  // [h][pair][128]
  float* red_sum = red_max + 2 * 2 * BM;

  const uint32_t warp = tc::warp_id();
  const uint32_t lane = threadIdx.x & 31;
#ifdef DFSS_FLASH_TRACE_BUILD
  unsigned long long* trace = blockIdx.x == 0 ? g_flash_trace : nullptr;
#endif
  const int iblocks = n / (2 * BM);
  const int items = bh * iblocks;
  const int ntiles = n / BN;
  // BlockMask tile skipping: a 128 x 128 step whose mask tiles are all
  // masked is not computed at all -- no K / V load when both halves are dead, no S MMA, no
  // softmax work, no PV.  Every role evaluates the same predicate and counts only live steps,
  // so the S ring / barrier phases stay in lock-step (identical to the dense sequence when
  // nothing is masked).
  // Liveness comes from the step bitmap (copied to shared memory below) and, for the softmax
  // warps, from per-strip chunk words held one per lane: no mask load on any critical path.
  uint32_t* s_live = (uint32_t*)(smem + S2_LIVE);
  int* s_order = (int*)(s_live + (n / BM) * tmask.sbw);
  if (MASKED) {
    for (int i = threadIdx.x; i < (n / BM) * tmask.sbw; i += blockDim.x) s_live[i] = __ldg(tmask.sbits + i);
    for (int i = threadIdx.x; i < iblocks; i += blockDim.x) s_order[i] = __ldg(tmask.order + i);
  }
  // k-th item of this CTA.  Dense: round robin (item = b * iblocks + ib).  Masked: items cost
  // their live steps, which depend on the row block only; row blocks are ranked by cost
  // (mask_order_kernel) and the ranked items dealt out in snake order -- heaviest first,
  // alternating direction per round -- so CTAs finish together (an all-kept mask reproduces the
  // dense order).  Every role walks the same sequence.
  // The position sequence is a pure function of (k, blockIdx) so loop control stays warp-uniform
  // for the MMA issuers (a trip count read from shared memory would make every loop divergent
  // in the compiler's eyes: no uniform datapath, R2UR / ELECT around each MMA).
  auto pos_at = [&](int k) -> int {
    const int g = gridDim.x;
    return k * g + (MASKED && (k & 1) ? g - 1 - (int)blockIdx.x : (int)blockIdx.x);
  };
  auto item_of = [&](int p) -> int {
    if (!MASKED) return p;
    // within a group of equal-cost row blocks keep the dense head-major order (K / V reuse in L2)
    const int info = s_order[p / bh], r0 = (info >> 8) & 255, m = info >> 16, o = p - r0 * bh;
    return (o / m) * iblocks + (s_order[r0 + o % m] & 255);
  };
  // k-th unit of this CTA: an item, its tile range [t0, t1) and its part of a split last-round
  // item (-1: the whole item); false past the CTA's last unit
  auto unit_at = [&](int k, int& item, int& t0, int& t1, int& part) -> bool {
    t0 = 0;
    t1 = ntiles;
    part = -1;
    if (MASKED || sp.parts <= 1 || k < sp.rounds) {
      const int pos = pos_at(k);
      item = pos < items ? item_of(pos) : 0;
      return pos < items;
    }
    if (k > sp.rounds || (int)blockIdx.x >= sp.rem * sp.parts) return false;
    item = sp.rounds * (int)gridDim.x + (int)blockIdx.x / sp.parts;
    part = (int)blockIdx.x % sp.parts;
    t0 = part * ntiles / sp.parts;
    t1 = (part + 1) * ntiles / sp.parts;
    return true;
  };
  // step-liveness words of an item's two halves for tiles [32 (t / 32), +32), refreshed every
  // 32 tiles; bit_u reads one as a warp vote so branches on it stay uniform in the converged
  // role warps
  auto live_words = [&](int ib, int t, uint32_t& w0, uint32_t& w1) {
    if (MASKED && (t & 31) == 0) {
      w0 = s_live[(ib * 2) * tmask.sbw + (t >> 5)];
      w1 = s_live[(ib * 2 + 1) * tmask.sbw + (t >> 5)];
    }
  };
  auto bit_u = [&](uint32_t w, int t) {
    return !MASKED || __any_sync(0xffffffffu, (w >> (t & 31)) & 1u);
  };

  if (threadIdx.x == 0) FTRACE(15, 0, 0, 0);  // CTA start
  if (warp == W_QK && lane == 0) {
    tc::prefetch_tmap(&tm_q);
    tc::prefetch_tmap(&tm_k);
    tc::prefetch_tmap(&tm_v);
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&q_full[i], 1);
      tc::mbar_init(&q_empty[i], 1);
      tc::mbar_init(&o_full[i], 1);
      tc::mbar_init(&o_empty[i], 8);
      tc::mbar_init(&pv_done[i], 1);
    }
    for (int i = 0; i < S2RING; ++i) tc::mbar_init(&s_free[i], 1);
    for (int i = 0; i < 2 * S2RING; ++i) tc::mbar_init(&s_full[i], 1);
    for (int i = 0; i < K2ST; ++i) {
      tc::mbar_init(&k_full[i], 1);
      tc::mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < V2ST; ++i) {
      tc::mbar_init(&v_full[i], 1);
      tc::mbar_init(&v_empty[i], 2);  // released by both PV issuers
    }
    tc::fence_barrier_init();
  }
  if (warp == W_PV) tc::tmem_alloc<512>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) FTRACE(15, 0, 1, 0);  // setup done

  if (warp >= SM_WARPS) {
  regs_role();
  if (warp == W_QK) {
    // ------------------------------------------------------------ TMA producer: Q (both halves), K (keys permuted), V
    if (lane == 0) {
      int ks = 0, vs = 0, it = 0;
      uint32_t kph = 0, vph = 0;
      int item, t0, t1, part;
      for (int kk_ = 0; unit_at(kk_, item, t0, t1, part); ++kk_, ++it) {
        uint32_t lw0 = 0, lw1 = 0;
        const int b = item / iblocks, ib = item % iblocks;
        const int qs = it & 1;
        UTRACE(kk_, 0);
        wait_role(&q_empty[qs], ((it >> 1) & 1) ^ 1);
        UTRACE(kk_, 1);
        tc::mbar_arrive_expect_tx(&q_full[qs], 2 * Q_BYTES);
        tc::tma_load_3d(smem + S2_Q + (2 * qs) * Q_BYTES, &tm_q, &q_full[qs], 0, ib * 2 * BM, b);
        tc::tma_load_3d(smem + S2_Q + (2 * qs + 1) * Q_BYTES, &tm_q, &q_full[qs], 0, ib * 2 * BM + BM, b);
        for (int t = t0; t < t1; ++t) {
          live_words(ib, t, lw0, lw1);
          if (MASKED && !(((lw0 | lw1) >> (t & 31)) & 1u)) continue;
          wait_role(&k_empty[ks], kph ^ 1);
          tc::mbar_arrive_expect_tx(&k_full[ks], K_BYTES);
          tc::tma_load_3d(smem + S2_K + ks * K_BYTES, &tm_k, &k_full[ks], 0, t * BN, b);
          FTRACE(8, it, t, 0);
          if (++ks == K2ST) { ks = 0; kph ^= 1; }
          wait_role(&v_empty[vs], vph ^ 1);
          tc::mbar_arrive_expect_tx(&v_full[vs], V_BYTES);
          tc::tma_load_3d(smem + S2_V + vs * V_BYTES, &tm_v, &v_full[vs], 0, t * BN, b);
          FTRACE(9, it, t, 0);
          if (++vs == V2ST) { vs = 0; vph ^= 1; }
        }
      }
    }
  } else if (warp == W_S) {
    // ------------------------------------------------------------ S issuer: step g = 2t + h -> buffer g % 3
    {  // whole warp, converged; elected lanes issue
      constexpr uint32_t fmt = std::is_same<T, __nv_bfloat16>::value ? 1u : 0u;
      constexpr uint32_t idesc_s = tc::instr_desc(fmt, BM, BN, false, false, false);
      int ks = 0, it = 0, sb = 0;
      uint32_t kph = 0, sph = 0;
      int item, t0, t1, part;
      for (int kk_ = 0; unit_at(kk_, item, t0, t1, part); ++kk_, ++it) {
        uint32_t lw0 = 0, lw1 = 0;
        const int qs = it & 1;
        const int ib = item % iblocks;
        wait_role(&q_full[qs], (it >> 1) & 1);
        for (int t = t0; t < t1; ++t) {
          live_words(ib, t, lw0, lw1);
          const bool lv[2] = {bit_u(lw0, t), bit_u(lw1, t)};
          if (MASKED && !lv[0] && !lv[1]) continue;
          wait_role(&k_full[ks], kph);
          if (lane == 0) FTRACE(10, it, t, 0);
          const uint32_t k_addr = tc::smem_u32(smem + S2_K + ks * K_BYTES);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (MASKED && !lv[h]) continue;
            if (lane == 0) FTRACE(3, it, t, h);
            wait_role(&s_free[sb], sph ^ 1);  // PV of step g - 3 retired
            if (lane == 0) FTRACE(4, it, t, h);
            tc::tc_fence_after();
            const uint32_t q_addr = tc::smem_u32(smem + S2_Q + (2 * qs + h) * Q_BYTES);
#pragma unroll
            for (int kk = 0; kk < HD / 16; ++kk) {
              const uint64_t ad = tc::smem_desc(q_addr + kk * 32, 16, 1024, tc::kSwizzle128B);
              const uint64_t bd = tc::smem_desc(k_addr + kk * 32, 16, 1024, tc::kSwizzle128B);
#ifndef DFSS_EXP_NO_MMA
              tc::mma_f16_ss_w(tmem_base + sb * BN, ad, bd, idesc_s, kk > 0 ? 1u : 0u);
#endif
            }
            tc::mma_commit_w(&s_full[h * S2RING + sb]);
            if (lane == 0) FTRACE(5, it, t, h);
            if (++sb == S2RING) { sb = 0; sph ^= 1; }
          }
          tc::mma_commit_w(&k_empty[ks]);
          if (++ks == K2ST) { ks = 0; kph ^= 1; }
        }
        tc::mma_commit_w(&q_empty[qs]);
      }
    }
  } else if (warp == W_PV || warp == W_PV1) {
    // ------------------------------------------------------------ PV issuer of half h: O_h += P V_t (4 sparse K=32
    // MMAs, A in TMEM); one issuer per half, so a lagging set never blocks the other's PV
    {  // whole warp, converged; elected lanes issue
      const int h = warp == W_PV ? 0 : 1;
      constexpr uint32_t fmt = std::is_same<T, __nv_bfloat16>::value ? 1u : 0u;
      constexpr uint32_t idesc_pv = tc::instr_desc(fmt, BM, HD, false, true, true);
      int vs = 0, it = 0;
      uint32_t vph = 0, gcount = 0, hc = 0;  // live steps so far (both halves / this half)
      int item, t0, t1, part;
      for (int kk_ = 0; unit_at(kk_, item, t0, t1, part); ++kk_, ++it) {
        uint32_t lw0 = 0, lw1 = 0;
        const int ib = item % iblocks;
        // O_h free (previous item drained) is awaited only before the first PV MMA of the item --
        // or before o_full when the half has no live step: a set whose first live step comes late
        // drains the previous item only then, and the V stages of the steps before it must be
        // released meanwhile or the producer stalls (deadlock on one-sided masks).
        bool o_free = false;
        auto await_o_free = [&]() {
          if (!o_free) wait_role(&o_empty[h], (it & 1) ^ 1);
          o_free = true;
        };
        bool first = true;  // first live step of this half-item initialises O_h
        for (int t = t0; t < t1; ++t) {
          live_words(ib, t, lw0, lw1);
          const bool l0 = bit_u(lw0, t), l1 = bit_u(lw1, t);
          if (MASKED && !l0 && !l1) continue;  // tile not loaded
          const uint32_t g = gcount + (h ? (uint32_t)l0 : 0u), slot = g % S2RING;
          gcount += (uint32_t)l0 + (uint32_t)l1;
          if (MASKED && !(h ? l1 : l0)) {  // this half is masked here: release the V stage unused
            // wait for the load first: arriving early could complete the stage's PREVIOUS phase
            // while the other half's PV still reads it
            wait_role(&v_full[vs], vph);
            if (lane == 0) tc::mbar_arrive(&v_empty[vs]);
            if (++vs == V2ST) { vs = 0; vph ^= 1; }
            continue;
          }
          await_o_free();
          wait_role(&v_full[vs], vph);
          // P of this half's hc-th live step published: named barrier 9 + 3h + hc % 3 over the
          // set's 8 warps (bar.arrive) and this warp -- a hardware wait that issues nothing while
          // it blocks (an mbarrier wait re-polled at each of the 8 arrivals: c4 -1.4 %, c2 -1 %).
          // Three ids per half rotate; the set cannot run more than one live step ahead of this
          // wait (its next S needs K(t+1), which the producer loads only after V(t), whose
          // load this issuer awaits before it), so an id is never re-armed early.
          ++hc;
          tc::named_bar_sync(9 + 3 * h + hc % 3, 288);
          if (lane == 0) FTRACE(6, it, t, h);
          tc::tc_fence_after();
          const uint32_t v_addr = tc::smem_u32(smem + S2_V + vs * V_BYTES);
          const uint32_t s_col = tmem_base + slot * BN;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint64_t bd = tc::smem_desc(v_addr + q * 32 * 128, V_BYTES, 1024, tc::kSwizzle128B);
#ifndef DFSS_EXP_NO_MMA
            tc::mma_sp_f16_ts_w(tmem_base + T2_O + h * HD, s_col + 32 * q + 16, bd, s_col + 32 * q, idesc_pv,
                                (!first || q > 0) ? 1u : 0u);
#endif
          }
          first = false;
          tc::mma_commit_w(&s_free[slot]);
          tc::mma_commit_w(&v_empty[vs]);
          tc::mma_commit_w(&pv_done[h]);
          if (lane == 0) FTRACE(7, it, t, h);
          if (++vs == V2ST) { vs = 0; vph ^= 1; }
        }
        await_o_free();
        tc::mma_commit_w(&o_full[h]);
      }
    }
  }
  // end of the role warpgroup (no code after the branches: ptxas needs one register budget
  // per region, so each branch finishes the CTA itself)
  tc::tc_fence_before();
  __syncthreads();
  if (warp == W_PV) {
    tc::tc_fence_after();
    tc::tmem_dealloc<512>(tmem_base);
  }
  } else {
    regs_softmax();
    // the per-step barriers as 32-bit shared addresses (see tc::mbar_wait_u32)
    // (materialised through asm so the compiler keeps them instead of re-deriving them from the
    // generic smem pointer -- window base + alignment -- at every use)
    uint32_t s_full32;
    asm volatile("mov.b32 %0, %1;" : "=r"(s_full32) : "r"(tc::smem_u32(s_full)));
    // ------------------------------------------------------------ softmax / prune / epilogue sets
    const int h = warp >> 3;              // half owned by this set
    const int pr = (warp >> 2) & 1;       // column pair: quarters 2pr, 2pr + 1
    const int quad = warp & 3;
    const int r = quad * 32 + lane;       // row within the half == TMEM lane
    const uint32_t lane_base = tmem_base + ((uint32_t)(quad * 32) << 16);
    const uint32_t pbar = 1 + h * 4 + quad;  // named barrier of the two warps sharing these rows
    const float c = scale * kLog2e;
    float* rmax = red_max + h * 2 * BM;
    float* rsum = red_sum + h * 2 * BM;
    [[maybe_unused]] const bool tw = quad == 0 && pr == 0 && lane == 0;
    uint32_t gcount = 0, hcount = 0, scol = 0, sfbits = 0;  // live steps (both halves / this half); this warp's S column
    int it = 0;
    // maximum of this row over the set's 128 columns of the current S (both warps of the pair)
    bool cm[2] = {false, false};  // this warp's two chunks of the current tile masked (BlockMask)
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
    auto chunk0_max = [&]() {
      uint32_t s0[32];
      tc::tmem_ld_32x32b_x32(scol - 64 * pr, s0);
      tc::tmem_ld_wait(s0);
      float mc = -INFINITY;
#pragma unroll
      for (int j = 0; j < 32; j += 2) mc = fmaxf(mc, fmaxf(__uint_as_float(s0[j]), __uint_as_float(s0[j + 1])));
      return mc * c;
    };
    // ---- epilogue of a finished item: O_h / row sum; this warp writes columns [32 pr, +32) of its rows.
    // The row sums of the two warps of a pair are combined when the item ends (lsum, below);
    // O_h is drained, normalised and stored during the next item's first live step, after its
    // compute but BEFORE its P is published: that item's first PV overwrites O_h, so it (and with
    // it the S ring) is never held up waiting for this epilogue (it was when the epilogue ran after
    // the publication: ~2500 clk per item boundary, tools/trace_items.py).
    bool pend = false;
    int pend_b = 0, pend_ib = 0, pend_it = 0, pend_item = 0, pend_part = -1;
    float pend_lsum = 0.f, pend_m = 0.f;
    // drain_o: O_h of the pending item into registers, O_h released (o_empty); finish_o: normalise
    // and store.  Split so that the next item's first P can be published in between.
    auto drain_o = [&](uint32_t (&o)[32]) {
      tc::mbar_wait(&o_full[h], pend_it & 1);
      tc::tc_fence_after();
      tc::tmem_ld_32x32b_x32(lane_base + T2_O + h * HD + 32 * pr, o);
      tc::tmem_ld_wait(o);
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&o_empty[h]);
    };
    auto finish_o = [&](const uint32_t (&o)[32]) {
      const int64_t row = (int64_t)pend_b * n + (pend_ib * 2 + h) * BM + r;
      pend = false;
      if (!MASKED && pend_part >= 0) {
        split_part_epilogue<T>(sp, pend_item - sp.rounds * (int)gridDim.x, h, (int)(warp & 7), pend_part, lane, o,
                               pend_m, pend_lsum, out + row * HD + 32 * pr);
        return;
      }
      const float inv = 1.0f / pend_lsum;
      uint32_t pko[16];
#pragma unroll
      for (int j = 0; j < 16; ++j)
        pko[j] = fpack2<T>(__uint_as_float(o[2 * j]) * inv, __uint_as_float(o[2 * j + 1]) * inv);
      uint4* orow = reinterpret_cast<uint4*>(out + row * HD + 32 * pr);
#pragma unroll
      for (int j = 0; j < 4; ++j) orow[j] = make_uint4(pko[4 * j], pko[4 * j + 1], pko[4 * j + 2], pko[4 * j + 3]);
    };
    auto epilogue = [&]() {
      uint32_t o[32];
      drain_o(o);
      finish_o(o);
    };
    // chunk-keep word `lane` of this warp's 32-row strip (cbits), next item's prefetched
    auto cword = [&](int pos_) -> uint32_t {
      if (!MASKED || pos_ >= items || (int)lane >= tmask.cbw) return 0u;
      const int strip = ((item_of(pos_) % iblocks) * 2 + h) * (BM / 32) + quad;
      return __ldg(tmask.cbits + (int64_t)strip * tmask.cbw + lane);
    };
    uint32_t cw = cword(pos_at(0));
    float carry_mlog = -INFINITY;  // the shift this row ended the set's previous item with
    const uint32_t word_sel = (lane & 8) ? 0x3276u : 0x5410u;
    int item, t0, t1, part;
    for (int kk_ = 0; unit_at(kk_, item, t0, t1, part); ++kk_, ++it) {
      uint32_t lw0 = 0, lw1 = 0;
      const int b = item / iblocks, ib = item % iblocks;
      const uint32_t cwn = cword(pos_at(kk_ + 1));
      float mlog = carry_mlog, l0 = 0.f, l1 = 0.f;
      bool first = true;  // first live step of this half-item: establishes the shift
      for (int t = t0; t < t1; ++t) {
        live_words(ib, t, lw0, lw1);
        const bool lv0 = bit_u(lw0, t), lv1 = bit_u(lw1, t);
        const uint32_t g = gcount + (h ? (uint32_t)lv0 : 0u);  // global live step
        gcount += (uint32_t)lv0 + (uint32_t)lv1;
        if (MASKED && !(h ? lv1 : lv0)) continue;  // whole 128 x 128 step masked for this half
        ++hcount;
        const uint32_t slot = g % S2RING;
        scol = lane_base + slot * BN + 64 * pr;
#ifndef DFSS_EXP_NO_SWAIT
        tc::mbar_wait_u32(s_full32 + 8 * (h * S2RING + slot), (sfbits >> slot) & 1);  // k-th use of (h, slot): parity k & 1
#endif
        sfbits ^= 1u << slot;
        if (tw) FTRACE(0, it, t, h);
        if (tw && h == 0 && t == t0) UTRACE(kk_, 2);
        tc::tc_fence_after();
        bool anym = false;  // a chunk of this warp masked (uniform): the masked compute variant
        if (MASKED) {
          const int c32 = 4 * t + 2 * pr;  // this warp's first 32-column chunk
          const uint32_t w = __shfl_sync(0xffffffffu, cw, c32 >> 5) >> (c32 & 31);
          cm[0] = !(w & 1u);
          cm[1] = !(w & 2u);
          anym = __any_sync(0xffffffffu, (~w & 3u) != 0);
        }
        // the shift starts at the row maximum of the item's first live tile -- unmasked: the
        // shift the row of this set's previous item ended with (attention rows of one launch
        // share their scale; no TMEM pass, no barrier), or the max of the first 32 columns for
        // the first item, read by both warps of the pair alike; a first step whose sums leave
        // [2^-16, 2^8] recomputes with the exact maximum (below)
        if (first) mlog = MASKED ? row_max() : (carry_mlog == -INFINITY ? chunk0_max() : carry_mlog);
        uint32_t pk[2][8], W[2];
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
            if (tw) FTRACE(11 + 2 * ch, it, t, h);
            if constexpr (DUMP)
              dump_chunk_scores<false>(dump.s + ((int64_t)b * n + (ib * 2 + h) * BM + r) * n + t * BN + 64 * pr + 32 * ch, s,
                                scale);
            prune_exp_tile<T, PAIRS>(s, c, mlog, two, pk[ch], W[ch], a0, a1);
            // masked chunk (structurally absent): computed like the others -- straight-line code
            // keeps the two chunks interleaved -- then overwritten (predicated moves)
            if (MV && cm[ch]) masked_chunk(pk[ch], W[ch], a0, a1);
            add2(lt0, lt1, a0, a1, lt0, lt1);
            if (tw) FTRACE(12 + 2 * ch, it, t, h);
          }
        };
        // one copy of the compute code (instruction-cache footprint): the slow path loops back
#pragma unroll 1
        for (int pass = 0;; ++pass) {
          if (MASKED && anym) compute(std::true_type{});
          else compute(std::false_type{});
          // (W[0] & W[1]) == ~0 never holds (no nibble is 0xF); it makes the vote consume the
          // metadata so ptxas builds W before the branch instead of keeping every group's
          // keep predicates / operands alive across it (which spilled to local memory)
#ifdef DFSS_EXP_NO_VOTE
          if (pass > 0 || first || !((W[0] & W[1]) == ~0u && lt0 + lt1 > 1e30f)) break;
#else
          if (pass > 0 || (MASKED && first) ||
              !bar_any(pbar, 64, !(lt0 + lt1 <= kSumLimit) || (first && !(lt0 + lt1 >= sum_floor<T>())) ||
                                     (W[0] & W[1]) == ~0u))
            break;
#endif
          if (!MASKED && first) {  // estimated shift off: exact row maximum, nothing accumulated yet
            mlog = row_max();
            continue;
          }
          // ---- slow path (both warps of the pair): raise the shift to the row maximum,
          // rescale O_h and the sums once every PV into O_h so far (this half's tile t-1) retired.
          // (pv_done[h] completes once per tile of this half and cannot run ahead of this set,
          // unlike the ring barriers, which the other set may advance twice meanwhile.)
          tc::mbar_wait(&pv_done[h], (hcount - 2) & 1);  // completion of this half's previous live step
          tc::tc_fence_after();
          const float mnew = fmaxf(mlog, row_max());
          const float f = fex2(mlog - mnew);
          l0 *= f;
          l1 *= f;
#pragma unroll 1
          for (int hh = 0; hh < 2; ++hh) {
            uint32_t o[16];
            const uint32_t oaddr = lane_base + T2_O + h * HD + 32 * pr + 16 * hh;
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
        if (tw) FTRACE(1, it, t, h);
        // P (8 columns of 16-bit pairs at 32q + 16) and the metadata word (column 32q) of each
        // chunk into this warp's own, already read S columns; rows r and r^8 trade metadata
        // halves (include/dfss.h): one PRMT with a lane-dependent selector
        auto publish = [&]() {
#pragma unroll
          for (int ch = 0; ch < 2; ++ch) {
            const uint32_t partner = __shfl_xor_sync(0xffffffffu, W[ch], 8);
            const uint32_t word = __byte_perm(W[ch], partner, word_sel);
            tc::tmem_st_32x32b_x8(scol + 32 * ch + 16, pk[ch]);
            tc::tmem_st_32x32b_x1(scol + 32 * ch, word);
            if constexpr (DUMP)
              dump.meta[(((int64_t)b * (n / BM) + ib * 2 + h) * (n / 32) + 4 * t + 2 * pr + ch) * BM + r] = word;
          }
          tc::tmem_st_wait();
          tc::tc_fence_before();
          __syncwarp();
          tc::named_bar_arrive(9 + 3 * h + hcount % 3, 288);  // P published (PV issuer of this half)
        };
        if (!MASKED && pend) {
          // the previous item's O_h leaves TMEM before this item's first P goes out (that P's PV
          // overwrites O_h); normalising and storing it follows the publication (masked kernels:
          // the whole epilogue after it -- their extra live state would spill around it here)
          uint32_t o[32];
          drain_o(o);
          publish();
          finish_o(o);
        } else {
          publish();
          if (MASKED && pend) epilogue();
        }
        if (tw) FTRACE(2, it, t, h);
        first = false;
      }
      if (tw && h == 0) UTRACE(kk_, 3);
      // the epilogue of this item runs in step 0 of the next one (above), so the wait for the
      // item's last PV overlaps that step's compute instead of idling the set at the boundary
      if (pend) epilogue();  // the previous item's, if this item had no live step for this set
      rsum[pr * BM + r] = l0 + l1;  // row sum over both warps of the pair
      tc::named_bar_sync(pbar, 64);
      pend_lsum = rsum[r] + rsum[BM + r];
      tc::named_bar_sync(pbar, 64);
      carry_mlog = mlog;
      pend = true;
      pend_b = b;
      pend_ib = ib;
      pend_it = it;
      pend_m = mlog;
      pend_item = item;
      pend_part = part;
      cw = cwn;
    }
    if (tw && h == 0) UTRACE(15, 4);
    if (pend) epilogue();
    if (tw && h == 0) UTRACE(15, 5);
    if (threadIdx.x == 0) FTRACE(15, 1, 0, 0);  // CTA end
    tc::tc_fence_before();
    __syncthreads();
  }
}

#ifndef DFSS_FLASH_DUMP_TU  // defined once, in flash_tc.cu
// BlockMask tile grid -> step / chunk bitmaps (TileMask::sbits / cbits) for the two-set
// kernel; one thread per bit, a warp writes one word.
__global__ void mask_bits_kernel(TileMask m, int n, uint32_t* __restrict__ sbits, uint32_t* __restrict__ cbits) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t ns = (int64_t)(n / BM) * m.sbw * 32, nc = (int64_t)(n / 32) * m.cbw * 32;
  bool bit = false;
  if (i < ns) {
    const int row = (int)(i / (m.sbw * 32)), t = (int)(i % (m.sbw * 32));
    bit = t < n / BN && m.region_live(row * BM, BM, t * BN, BN);
  } else if (i < ns + nc) {
    const int64_t j = i - ns;
    const int strip = (int)(j / (m.cbw * 32)), c = (int)(j % (m.cbw * 32));
    bit = c < n / 32 && !m.masked(strip * 32, c * 32);
  }
  const uint32_t w = __ballot_sync(0xffffffffu, bit);
  if ((threadIdx.x & 31) == 0) {
    if (i < ns) sbits[i >> 5] = w;
    else if (i < ns + nc) cbits[(i - ns) >> 5] = w;
  }
}

// row blocks (256 rows, one two-set item) ranked by live steps, heaviest first (ties: lower
// block first); one thread per row block, n <= 32768
__global__ void mask_order_kernel(const uint32_t* __restrict__ sbits, int sbw, int nrows, int iblocks,
                                  int* __restrict__ order) {
  __shared__ int cost[128];
  const int i = threadIdx.x;
  if (i < iblocks) {  // (the last block's second half may lie beyond n: rows n / 128 of sbits)
    int c = 0;
    for (int w = 0; w < 2 * sbw && (2 * i * sbw + w) < nrows * sbw; ++w) c += __popc(sbits[2 * i * sbw + w]);
    cost[i] = c;
  }
  __syncthreads();
  if (i < iblocks) {  // order[rank] = block | first rank of its equal-cost group << 8 | group size << 16
    int r = 0, r0 = 0, m = 0;
    for (int j = 0; j < iblocks; ++j) {
      r += cost[j] > cost[i] || (cost[j] == cost[i] && j < i);
      r0 += cost[j] > cost[i];
      m += cost[j] == cost[i];
    }
    order[r] = i | r0 << 8 | m << 16;
  }
}

static int mask_sbw(int n) { return (n / BN + 31) / 32; }
static int mask_cbw(int n) { return (n / 32 + 31) / 32; }
static int64_t mask_words(int n) { return (int64_t)(n / BM) * mask_sbw(n) + (int64_t)(n / 32) * mask_cbw(n); }

int64_t flash_mask_workspace_bytes(int n) {
  return ((mask_words(n) + (n + 2 * BM - 1) / (2 * BM)) * 4 + 255) / 256 * 256;  // bitmaps + row-block order
}

bool flash_mask_two_set_ok(int n) { return n % BM == 0 && mask_cbw(n) <= 32; }

int flash_mask_smem_bytes(int n) { return ((n / BM) * mask_sbw(n) + (n + 2 * BM - 1) / (2 * BM)) * 4; }

void prepare_mask_bits(TileMask& m, int n, void* workspace, cudaStream_t s) {
  m.sbw = mask_sbw(n);
  m.cbw = mask_cbw(n);
  m.sbits = (const uint32_t*)workspace;
  m.cbits = m.sbits + (int64_t)(n / BM) * m.sbw;
  m.order = (const int*)(m.sbits + mask_words(n));
  const int64_t bits = mask_words(n) * 32;
  mask_bits_kernel<<<(unsigned)((bits + 255) / 256), 256, 0, s>>>(m, n, (uint32_t*)m.sbits, (uint32_t*)m.cbits);
  mask_order_kernel<<<1, 128, 0, s>>>(m.sbits, m.sbw, n / BM, (n + 2 * BM - 1) / (2 * BM), (int*)m.order);
}

bool tc_flash_supported(int gs, int dtype, int n, int d) {
  return (gs == 4 || gs == 2) && (dtype == DFSS_BF16 || dtype == DFSS_F16) && d == HD && n % BM == 0 && n > 0;
}

#endif  // DFSS_FLASH_DUMP_TU

unsigned long long next_split_token();

// Last-round split of the two-set kernel for bh heads of n keys on `sms` persistent CTAs
// (SplitPlan); workspace bytes in *bytes (0: no split).
static SplitPlan split_plan(int64_t bh, int n, int sms, int64_t* bytes) {
  SplitPlan sp;
  *bytes = 0;
  if (n % (2 * BM) != 0 || bh <= 0) return sp;
  const int64_t items = bh * (n / (2 * BM));
  const int64_t g = items < sms ? items : sms;
  const int64_t rem = items % g;
  const int ntiles = n / BN;
  // >= 4 tiles per part: a part's epilogue (publish / merge through L2) costs about one tile
  // of work, so 1-tile parts (c2: 28 items x 4 parts) measured slower than no split
  const int64_t parts = rem ? std::min<int64_t>(ntiles / 4, g / rem) : 1;
  if (parts < 2 || items / g > (1 << 20)) return sp;
  sp.rounds = (int)(items / g);
  sp.rem = (int)rem;
  sp.parts = (int)parts;
  const int64_t part_bytes = (rem * 2 * 8 * parts * 34 * 32 * 4 + 255) / 256 * 256;
  *bytes = part_bytes + (rem * 2 * 8 * parts * 8 + 255) / 256 * 256;
  return sp;
}

#ifndef DFSS_FLASH_DUMP_TU
// one token per launch of any instantiation (the counters of a reused workspace may hold the
// previous launch's token; a per-instantiation count would repeat across instantiations)
unsigned long long next_split_token() {
  static std::atomic<unsigned long long> launches{0};
  return (++launches) & ((1ull << 56) - 1);
}

// workspace of the unmasked fused 16-bit path: the last-round split's partial results (SplitPlan)
int64_t flash_split_workspace_bytes(int64_t bh, int n) {
  int64_t bytes = 0;
  split_plan(bh, n, device_sms(current_device()), &bytes);
  return bytes;
}
#endif

template <typename T, bool PAIRS, bool MASKED, bool DUMP>
static cudaError_t flash_launch_typed(const void* q, const void* k, const void* v, void* out, float scale, int64_t bh,
                                      int n, TileMask tmask, void* workspace, FlashDump dump, cudaStream_t s) {
  const CUtensorMapDataType dt =
      std::is_same<T, __nv_bfloat16>::value ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  CUtensorMap tq, tk, tv;
  // n % 256 == 0: the two-set kernel (256-row items, independent softmax sets per half);
  // otherwise 128-row items with all 16 softmax warps on one half
  const bool two_set = n % (2 * BM) == 0 && (!MASKED || flash_mask_two_set_ok(n));
  if (!encode_tmap_3d(&tq, dt, 2, (void*)q, HD, n, bh, HD, BM, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !encode_tmap_3d(&tk, dt, 2, (void*)k, HD, n, bh, HD, BN, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !encode_tmap_3d(&tv, dt, 2, (void*)v, HD, n, bh, HD, BN, CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  const int halves = two_set ? 2 : 1;
  auto kern = two_set ? dfss_flash2_kernel<T, PAIRS, MASKED, DUMP> : dfss_flash_kernel<T, 1, PAIRS, MASKED, DUMP>;
  const int smem_total = two_set ? S2_TOTAL + (MASKED ? flash_mask_smem_bytes(n) : 0) : SMEM_TOTAL;
  if (smem_total > 227 * 1024) return cudaErrorNotSupported;
  if (MASKED && two_set) prepare_mask_bits(tmask, n, workspace, s);
  const int dev = current_device();
  SplitPlan sp;
  if (two_set && !MASKED && workspace) {
    int64_t split_bytes = 0;
    sp = split_plan(bh, n, device_sms(dev), &split_bytes);
    if (split_bytes) {
      sp.token = next_split_token();
      sp.part_ws = (float*)workspace;
      sp.counters = (unsigned long long*)((char*)workspace + split_bytes -
                                          ((int64_t)sp.rem * 2 * 8 * sp.parts * 8 + 255) / 256 * 256);
    }
  }
  static std::atomic<uint64_t> attr1{0}, attr2{0};
  cudaError_t e = set_max_smem_once((const void*)kern, two_set ? attr2 : attr1, dev);
  if (e != cudaSuccess) return e;
  const int sms = device_sms(dev);
  const int64_t items = bh * (n / (BM * halves));
  const int grid = (int)(items < sms ? items : sms);
#ifdef DFSS_FLASH_TRACE_BUILD
  // bring-up timeline (tools/trace_flash.py): DFSS_FLASH_TRACE=<file> in trace builds only
  static const char* trace_file = getenv("DFSS_FLASH_TRACE");
  unsigned long long* trace = nullptr;
  const size_t trace_n = 16 * 2 * 64 * 2 + 148 * 16 * 8;
  if (trace_file && two_set) {
    cudaMalloc(&trace, trace_n * 8);
    cudaMemset(trace, 0, trace_n * 8);
    cudaMemcpyToSymbol(g_flash_trace, &trace, sizeof(trace));
  }
#endif
  kern<<<grid, NUM_THREADS, smem_total, s>>>(tq, tk, tv, (T*)out, scale, (int)bh, n, 2u, dump, tmask, sp);
#ifdef DFSS_FLASH_TRACE_BUILD
  if (trace) {
    cudaStreamSynchronize(s);
    unsigned long long* host = (unsigned long long*)malloc(trace_n * 8);
    cudaMemcpy(host, trace, trace_n * 8, cudaMemcpyDeviceToHost);
    FILE* f = fopen(trace_file, "wb");
    if (f) {
      fwrite(host, 8, trace_n, f);
      fclose(f);
    }
    free(host);
    unsigned long long* null = nullptr;
    cudaMemcpyToSymbol(g_flash_trace, &null, sizeof(null));
    cudaFree(trace);
  }
#endif
  return cudaGetLastError();
}

#ifndef DFSS_FLASH_DUMP_TU
bool tc_flash_mask_supported(int tile_rows, int tile_cols) {
  return tile_rows > 0 && tile_cols > 0 && tile_rows % 32 == 0 && tile_cols % 32 == 0;
}
#endif

template <bool DUMP>
static cudaError_t launch_flash_tc_impl(const void* q, const void* k, const void* v, void* out, float scale, int gs,
                                        int dtype, int64_t bh, int n, int d, const uint8_t* tile_keep, int tile_rows,
                                        int tile_cols, void* workspace, FlashDump dump, cudaStream_t s) {
  if (!tc_flash_supported(gs, dtype, n, d)) return cudaErrorNotSupported;
  if (tile_keep && !tc_flash_mask_supported(tile_rows, tile_cols)) return cudaErrorNotSupported;
  if (tile_keep && !workspace) return cudaErrorInvalidValue;  // flash_mask_workspace_bytes(n)
  if (bh == 0) return cudaSuccess;
  TileMask m{tile_keep, tile_keep ? tile_rows : 1, tile_keep ? tile_cols : 1,
             tile_keep ? (n + tile_cols - 1) / tile_cols : 1};
  const bool bf = dtype == DFSS_BF16, masked = tile_keep != nullptr;
#define DFSS_FLASH_CALL(T, P, M) flash_launch_typed<T, P, M, DUMP>(q, k, v, out, scale, bh, n, m, workspace, dump, s)
  if (gs == 2) {
    if (masked) return bf ? DFSS_FLASH_CALL(__nv_bfloat16, true, true) : DFSS_FLASH_CALL(__half, true, true);
    return bf ? DFSS_FLASH_CALL(__nv_bfloat16, true, false) : DFSS_FLASH_CALL(__half, true, false);
  }
  if (masked) return bf ? DFSS_FLASH_CALL(__nv_bfloat16, false, true) : DFSS_FLASH_CALL(__half, false, true);
  return bf ? DFSS_FLASH_CALL(__nv_bfloat16, false, false) : DFSS_FLASH_CALL(__half, false, false);
#undef DFSS_FLASH_CALL
}

#ifndef DFSS_FLASH_DUMP_TU
cudaError_t launch_flash_tc(const void* q, const void* k, const void* v, void* out, float scale, int gs, int dtype,
                            int64_t bh, int n, int d, const uint8_t* tile_keep, int tile_rows, int tile_cols,
                            void* workspace, cudaStream_t s) {
  return launch_flash_tc_impl<false>(q, k, v, out, scale, gs, dtype, bh, n, d, tile_keep, tile_rows, tile_cols,
                                     workspace, FlashDump{}, s);
}
#else
cudaError_t launch_flash_tc_dump(const void* q, const void* k, const void* v, void* out, float scale, int gs,
                                 int dtype, int64_t bh, int n, int d, const uint8_t* tile_keep, int tile_rows,
                                 int tile_cols, void* workspace, float* dump_scores, uint32_t* dump_meta,
                                 cudaStream_t s) {
  FlashDump dump;
  dump.s = dump_scores;
  dump.meta = dump_meta;
  return launch_flash_tc_impl<true>(q, k, v, out, scale, gs, dtype, bh, n, d, tile_keep, tile_rows, tile_cols,
                                    workspace, dump, s);
}
#endif

}  // namespace dfss
