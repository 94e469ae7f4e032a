// sddmm_tf32.cu -- fused score + 1:2 prune for fp32 inputs on the tensor cores at fp32 accuracy
// (3xTF32: Q = Qh + Ql, K = Kh + Kl with Xh = tf32(X), Xl = tf32(X - Xh), both rounded to
// nearest; S = Qh Kh^T + Qh Kl^T + Ql Kh^T accumulated in fp32 by tcgen05.mma.kind::tf32).
//
// The exact-FP32 attention path (nm_attention on fp32 inputs, math "auto", 1e-5 bar).  The
// dropped Ql Kl^T term and the rounding of the split parts leave the scores within a few fp32
// ulps of the FFMA scores (tools/x3_accuracy.py, profiles/x3_accuracy.txt: same maximum error against float64
// as FFMA on the c1 inputs); the selection is bit-exact on the scores this kernel computes
// (the dump hook writes them), as for every other SDDMM here (codec.py:104-123: element 1 of a
// pair survives iff v1 > v0, ties to the lower index).  The explicit "ffma" math mode keeps
// the pure-FFMA SIMT kernel.
//
// Persistent, warp-specialised, one CTA per SM; items are 128-row blocks of one head:
//   warp 0       TMA: Q hi / lo of the item (single-buffered, two 128B-swizzle atoms of 32
//                dims each) and K hi / lo tiles of 128 keys (two-stage ring);
//   warp 1       MMA issuer: per tile 8 k-steps of K = 8, three MMAs each, into one of two
//                128-column TMEM accumulators;
//   warp 2       TMEM allocator;
//   warps 4-11   epilogue: warp (quad, half) prunes rows 32 quad.. x columns 64 half.. of the
//                tile: scale, 1:2 selection, fp32 kept values and the meta_hw words (1:2: two
//                per 32 columns, rows r / r^8 traded, include/dfss.h) straight to global.
#include <math_constants.h>

#include <algorithm>
#include <type_traits>

#include "dfss_common.cuh"
#include "tc_common.cuh"

namespace dfss {

namespace {
constexpr int BM = 128, BN = 128, HD = 64;
constexpr int ATOM = BM * 128;           // 16 KB: 128 rows x 32 fp32
constexpr int TILE = 2 * ATOM;           // 32 KB: 128 rows x 64 dims
constexpr int KST = 2;
constexpr int S_QH = 0, S_QL = TILE, S_K = 2 * TILE;  // K ring: [stage][hi, lo]
constexpr int STG_BYTES = 32 * 128;  // per epilogue warp: 32 rows x 32 kept fp32 (128B-swizzled rows)
constexpr int S_STG = S_K + KST * 2 * TILE;
constexpr int SMEM_BAR = S_STG + 8 * STG_BYTES;
constexpr int SMEM_TOTAL = SMEM_BAR + 256 + 1024;
constexpr int NACC = 2;
constexpr int NTHREADS = 12 * 32;
}  // namespace

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ float tf32_round(float x) {
  uint32_t y;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(y) : "f"(x));
  return __uint_as_float(y);
}

// x -> hi = tf32(x), lo = tf32(x - hi) (both with zero low mantissa bits), for Q and K in one launch
__global__ void __launch_bounds__(256) split_tf32_kernel(const float4* __restrict__ xa, float4* __restrict__ ha,
                                                         float4* __restrict__ la, int64_t na,
                                                         const float4* __restrict__ xb, float4* __restrict__ hb,
                                                         float4* __restrict__ lb, int64_t nb) {
  asm volatile("griddepcontrol.launch_dependents;");  // the V^T split (independent) may start now
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < na + nb; j += (int64_t)gridDim.x * blockDim.x) {
    const bool first = j < na;
    const int64_t i = first ? j : j - na;
    const float4* x = first ? xa : xb;
    float4* hi = first ? ha : hb;
    float4* lo = first ? la : lb;
    const float4 v = x[i];
    float4 h, l;
    h.x = tf32_round(v.x), l.x = tf32_round(v.x - h.x);
    h.y = tf32_round(v.y), l.y = tf32_round(v.y - h.y);
    h.z = tf32_round(v.z), l.z = tf32_round(v.z - h.z);
    h.w = tf32_round(v.w), l.w = tf32_round(v.w - h.w);
    hi[i] = h;
    lo[i] = l;
  }
}

template <bool DBG>
__global__ void __launch_bounds__(NTHREADS, 1)
    sddmm12_tf32x3_kernel(const __grid_constant__ CUtensorMap tm_qh, const __grid_constant__ CUtensorMap tm_ql,
                          const __grid_constant__ CUtensorMap tm_kh, const __grid_constant__ CUtensorMap tm_kl,
                          const __grid_constant__ CUtensorMap tm_nz, float* __restrict__ nz, uint32_t* __restrict__ meta, float scale, int bh, int n, int m,
                          float* __restrict__ dbg, float* __restrict__ rowmax) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = (uint64_t*)(smem + SMEM_BAR);
  uint64_t* q_full = bars;             // [1]
  uint64_t* q_empty = q_full + 1;      // [1]
  uint64_t* k_full = q_empty + 1;      // [KST]
  uint64_t* k_empty = k_full + KST;    // [KST]
  uint64_t* t_full = k_empty + KST;    // [NACC]
  uint64_t* t_empty = t_full + NACC;   // [NACC] (8 epilogue warps)
  uint32_t* tmem_slot = (uint32_t*)(t_empty + NACC);

  const uint32_t warp = tc::warp_id();
  const uint32_t lane = threadIdx.x & 31;
  const int mblocks = n / BM;
  const int items = bh * mblocks;
  const int ntiles = m / BN;

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tm_qh);
    tc::prefetch_tmap(&tm_ql);
    tc::prefetch_tmap(&tm_kh);
    tc::prefetch_tmap(&tm_kl);
    tc::prefetch_tmap(&tm_nz);
    tc::mbar_init(q_full, 1);
    tc::mbar_init(q_empty, 1);
    for (int i = 0; i < KST; ++i) {
      tc::mbar_init(&k_full[i], 1);
      tc::mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < NACC; ++i) {
      tc::mbar_init(&t_full[i], 1);
      tc::mbar_init(&t_empty[i], 8);
    }
    tc::fence_barrier_init();
  }
  if (warp == 2) tc::tmem_alloc<256>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // launched as a programmatic dependent of the operand splits: the prologue above overlapped
  // them; their results are read from here on
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int ks = 0, it = 0;
      uint32_t kph = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
        const int b = item / mblocks, mb = item % mblocks;
        tc::mbar_wait_sleep(q_empty, (it & 1) ^ 1);
        tc::mbar_arrive_expect_tx(q_full, 2 * TILE);
#pragma unroll
        for (int a = 0; a < 2; ++a) {
          tc::tma_load_3d(smem + S_QH + a * ATOM, &tm_qh, q_full, 32 * a, mb * BM, b);
          tc::tma_load_3d(smem + S_QL + a * ATOM, &tm_ql, q_full, 32 * a, mb * BM, b);
        }
        for (int t = 0; t < ntiles; ++t) {
          tc::mbar_wait_sleep(&k_empty[ks], kph ^ 1);
          tc::mbar_arrive_expect_tx(&k_full[ks], 2 * TILE);
          uint8_t* kt = smem + S_K + ks * 2 * TILE;
#pragma unroll
          for (int a = 0; a < 2; ++a) {
            tc::tma_load_3d(kt + a * ATOM, &tm_kh, &k_full[ks], 32 * a, t * BN, b);
            tc::tma_load_3d(kt + TILE + a * ATOM, &tm_kl, &k_full[ks], 32 * a, t * BN, b);
          }
          if (++ks == KST) { ks = 0; kph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = tc::instr_desc(2, BM, BN, false, false, false);  // tf32, K-major A / B
      int ks = 0, acc = 0, it = 0;
      uint32_t kph = 0, aph = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
        tc::mbar_wait_sleep(q_full, it & 1);
        const uint32_t qh = tc::smem_u32(smem + S_QH), ql = tc::smem_u32(smem + S_QL);
        for (int t = 0; t < ntiles; ++t) {
          tc::mbar_wait_sleep(&t_empty[acc], aph ^ 1);
          tc::mbar_wait_sleep(&k_full[ks], kph);
          tc::tc_fence_after();
          const uint32_t kh = tc::smem_u32(smem + S_K + ks * 2 * TILE), kl = kh + TILE;
          const uint32_t d = tmem_base + acc * BN;
#pragma unroll
          for (int kk = 0; kk < HD / 8; ++kk) {
            const uint32_t off = (kk >> 2) * ATOM + (kk & 3) * 32;
            const uint64_t a_h = tc::smem_desc(qh + off, 16, 1024, tc::kSwizzle128B);
            const uint64_t a_l = tc::smem_desc(ql + off, 16, 1024, tc::kSwizzle128B);
            const uint64_t b_h = tc::smem_desc(kh + off, 16, 1024, tc::kSwizzle128B);
            const uint64_t b_l = tc::smem_desc(kl + off, 16, 1024, tc::kSwizzle128B);
            // small terms first: the large hi.hi product is added to the already summed corrections
            mma_tf32(d, a_h, b_l, idesc, kk > 0 ? 1u : 0u);
            mma_tf32(d, a_l, b_h, idesc, 1u);
            mma_tf32(d, a_h, b_h, idesc, 1u);
          }
          tc::mma_commit(&k_empty[ks]);
          tc::mma_commit(&t_full[acc]);
          if (++ks == KST) { ks = 0; kph ^= 1; }
          if (++acc == NACC) { acc = 0; aph ^= 1; }
        }
        tc::mma_commit(q_empty);
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const int ew = warp - 4;
    const int quad = warp & 3;
    const int half = ew >> 2;
    const int row_blk = quad * 32 + lane;
    const int words = m / 16;  // 1:2 meta_hw words per row-block lane
    // kept values leave through a shared-memory staging tile and one TMA store per tile (direct
    // 16-byte stores, one row per lane, kept L1 68 % busy for 113 us at n = 1024)
    uint8_t* stg = smem + S_STG + ew * STG_BYTES;
    int acc = 0;
    uint32_t aph = 0;
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
      const int b = item / mblocks, mb = item % mblocks;
      const int grow = mb * BM + row_blk;
      uint32_t* meta_b = meta + ((int64_t)b * mblocks + mb) * words * 128;
      float mx = -INFINITY;  // this row's maximum kept score over the warp's column half
      for (int t = 0; t < ntiles; ++t) {
        tc::mbar_wait_sleep(&t_full[acc], aph);
        tc::tc_fence_after();
        const uint32_t tbase = tmem_base + ((uint32_t)(quad * 32) << 16) + acc * BN + half * 64;
        uint32_t ra[32], rb[32];
        tc::tmem_ld_32x32b_x32(tbase, ra);
        tc::tmem_ld_32x32b_x32(tbase + 32, rb);
        tc::tmem_ld_wait(ra);
        tc::tmem_ld_wait(rb);
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&t_empty[acc]);
        if (lane == 0) tc::bulk_wait_read<0>();  // the previous tile's store has read the staging tile
        __syncwarp();
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          const uint32_t(&r)[32] = cc ? rb : ra;
          const int col = t * BN + half * 64 + cc * 32;  // first dense column of the chunk
          float kept[16];
          uint32_t W[2] = {0u, 0u};
#pragma unroll
          for (int pr = 0; pr < 16; ++pr) {
            const float v0 = scale_canon(__uint_as_float(r[2 * pr]), scale);
            const float v1 = scale_canon(__uint_as_float(r[2 * pr + 1]), scale);
            if (DBG) *reinterpret_cast<float2*>(dbg + ((int64_t)b * n + grow) * m + col + 2 * pr) = make_float2(v0, v1);
            W[pr >> 3] |= select12(v0, v1, kept[pr]) << (4 * (pr & 7));
            mx = fmaxf(mx, kept[pr]);
          }
#pragma unroll
          for (int j = 0; j < 4; ++j)  // 16-byte unit 4 cc + j of this lane's 128-byte row, swizzled
            *reinterpret_cast<float4*>(stg + lane * 128 + (((4 * cc + j) ^ (lane & 7)) << 4)) =
                make_float4(kept[4 * j], kept[4 * j + 1], kept[4 * j + 2], kept[4 * j + 3]);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t partner = __shfl_xor_sync(0xffffffffu, W[h], 8);
            const uint32_t word =
                (lane & 8) ? ((partner >> 16) | (W[h] & 0xFFFF0000u)) : ((W[h] & 0xFFFFu) | (partner << 16));
            meta_b[(int64_t)((col >> 4) + h) * 128 + row_blk] = word;
          }
        }
        tc::fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          tc::tma_store_3d(&tm_nz, stg, (t * BN + half * 64) / 2, mb * BM + quad * 32, b);
          tc::bulk_commit();
        }
        if (++acc == NACC) { acc = 0; aph ^= 1; }
      }
      // per-row partial maxima [bh, n, 4] (halves 0, 1; 2, 3 unused): the SpMM's fused softmax
      rowmax[((int64_t)b * n + grow) * 4 + half] = mx;
      rowmax[((int64_t)b * n + grow) * 4 + 2 + half] = -INFINITY;
    }
    if (lane == 0) tc::bulk_wait<0>();
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc::tc_fence_after();
    tc::tmem_dealloc<256>(tmem_base);
  }
}

bool tc_sddmm_tf32x3_supported(int gs, int n, int m, int d) {
  return gs == 2 && d == HD && n > 0 && m > 0 && n % BM == 0 && m % BN == 0;
}

int64_t sddmm_tf32x3_workspace_bytes(int64_t bh, int n, int m) {
  const auto al = [](int64_t x) { return (x + 255) / 256 * 256; };
  return 2 * al(bh * (int64_t)n * HD * 4) + 2 * al(bh * (int64_t)m * HD * 4);
}

cudaError_t launch_sddmm_tf32x3(const float* q, const float* k, float* nz, uint32_t* meta, float scale, int64_t bh,
                                int n, int m, float* dbg, float* rowmax, void* workspace, cudaStream_t s) {
  if (!tc_sddmm_tf32x3_supported(2, n, m, HD)) return cudaErrorNotSupported;
  if (bh == 0) return cudaSuccess;
  if (!workspace || !rowmax || ((uintptr_t)q | (uintptr_t)k) % 16) return cudaErrorInvalidValue;
  const auto al = [](int64_t x) { return (x + 255) / 256 * 256; };
  char* ws = (char*)workspace;
  float* qh = (float*)ws;
  float* ql = (float*)(ws + al(bh * (int64_t)n * HD * 4));
  float* kh = (float*)(ws + 2 * al(bh * (int64_t)n * HD * 4));
  float* kl = (float*)(ws + 2 * al(bh * (int64_t)n * HD * 4) + al(bh * (int64_t)m * HD * 4));
  const int sms = device_sms(current_device());
  const CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  CUtensorMap tqh, tql, tkh, tkl, tnz;
  const uint64_t row = HD * 4;
  const uint64_t qdims[3] = {(uint64_t)HD, (uint64_t)n, (uint64_t)bh}, qstr[2] = {row, (uint64_t)n * row};
  const uint64_t kdims[3] = {(uint64_t)HD, (uint64_t)m, (uint64_t)bh}, kstr[2] = {row, (uint64_t)m * row};
  const uint32_t box[3] = {32, BM, 1};
  if (!encode_tmap(&tqh, dt, 3, qh, qdims, qstr, box, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !encode_tmap(&tql, dt, 3, ql, qdims, qstr, box, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !encode_tmap(&tkh, dt, 3, kh, kdims, kstr, box, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !encode_tmap(&tkl, dt, 3, kl, kdims, kstr, box, CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  const uint64_t ndims[3] = {(uint64_t)m / 2, (uint64_t)n, (uint64_t)bh};
  const uint64_t nstr[2] = {(uint64_t)m / 2 * 4, (uint64_t)n * (m / 2) * 4};
  const uint32_t nbox[3] = {32, 32, 1};
  if (!encode_tmap(&tnz, dt, 3, nz, ndims, nstr, nbox, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorInvalidValue;
  auto kern = dbg ? sddmm12_tf32x3_kernel<true> : sddmm12_tf32x3_kernel<false>;
  static std::atomic<uint64_t> attr[2];
  cudaError_t e = set_max_smem_once((const void*)kern, attr[dbg ? 1 : 0], current_device());
  if (e != cudaSuccess) return e;
  const int64_t items = bh * (n / BM);
  const int grid = (int)(items < sms ? items : sms);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(NTHREADS);
  cfg.dynamicSmemBytes = SMEM_TOTAL;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, tqh, tql, tkh, tkl, tnz, nz, meta, scale, (int)bh, n, m, dbg, rowmax);
}

// Q, K -> tf32 hi / lo in the workspace (one launch; the first of the 3xTF32 chain: split, V^T
// split, SDDMM, SpMM, each later one a programmatic dependent of the one before)
cudaError_t launch_split_tf32x3(const float* q, const float* k, int64_t bh, int n, int m, void* workspace,
                                cudaStream_t s) {
  if (bh == 0) return cudaSuccess;
  if (!workspace || ((uintptr_t)q | (uintptr_t)k) % 16) return cudaErrorInvalidValue;
  const auto al = [](int64_t x) { return (x + 255) / 256 * 256; };
  char* ws = (char*)workspace;
  float* qh = (float*)ws;
  float* ql = (float*)(ws + al(bh * (int64_t)n * HD * 4));
  float* kh = (float*)(ws + 2 * al(bh * (int64_t)n * HD * 4));
  float* kl = (float*)(ws + 2 * al(bh * (int64_t)n * HD * 4) + al(bh * (int64_t)m * HD * 4));
  const int64_t nq4 = bh * (int64_t)n * HD / 4, nk4 = bh * (int64_t)m * HD / 4;
  const int sms = device_sms(current_device());
  split_tf32_kernel<<<(unsigned)std::min<int64_t>((nq4 + nk4 + 255) / 256, sms * 8), 256, 0, s>>>(
      (const float4*)q, (float4*)qh, (float4*)ql, nq4, (const float4*)k, (float4*)kh, (float4*)kl, nk4);
  return cudaGetLastError();
}

}  // namespace dfss
