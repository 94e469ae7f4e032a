// spmm_tf32.cu -- O = softmax_rows(P_sparse) . V for fp32 1:2 operands on the tensor cores at fp32
// accuracy (3xTF32: E = Eh + El, V = Vh + Vl with Xh = tf32(X), Xl = X - Xh; O += Eh Vh + Eh Vl +
// El Vh, E = exp(P - row max), O divided by the row sums at the end).
//
// The exact-FP32 attention path (nm_attention on fp32 inputs, math "auto", 1e-5 bar): the
// selection is already made on the SDDMM's fp32-accurate scores (sddmm_tf32.cu, which also
// records the row maxima), so the tensor cores only see fixed weights; the dropped El Vl term
// and the tf32 truncation of the low parts leave a relative error of ~2^-21 per product, far
// inside 1e-5 (sparse_ops.py:18-68 / _kernels_numba.py:66-103 compute in float64).
//
// tcgen05.mma.sp.kind::tf32 (M = 128, N = 64, K = 16 dense / 8 kept) with A and the metadata in
// TMEM and B = V^T (kind::tf32 reads B only K-major, tools/tf32_probe.cu), as in the fused
// tf32 kernel (flash_tf32.cu).  The staged 1:2 meta_hw words (8 pairs per word, rows r / r^8
// traded) are exactly the tf32 sparse metadata words, so they go to TMEM unchanged.
// Persistent, warp-specialised, one CTA per SM, 64-key stages:
//   warp 0       TMA producer: P tile (128 rows x 32 stored fp32, one 128B-swizzle atom) and
//                V^T hi / lo tiles (64 dims x 64 keys, two atoms each) per stage;
//   warp 1       MMA issuer: per 16-key step three sparse MMAs (hi.hi, hi.lo, lo.hi);
//   warp 2       TMEM allocator;
//   warps 4-7    softmax + split: a lane's P row from shared memory -> exp2(p log2e - row max)
//                (row sum accumulated) -> tf32 hi / lo -> TMEM A columns, its meta_hw words ->
//                TMEM metadata columns (two TMEM A stages); the row sum to the epilogue;
//   warps 8-11   epilogue: TMEM -> fp32 O rows / row sum.
// V^T hi / lo are produced once per call by vt_split_kernel into the workspace.
#include <type_traits>

#include "dfss_common.cuh"
#include "tc_common.cuh"

namespace dfss {

namespace {
constexpr int BM = 128, HD = 64;
constexpr int BKL = 64;                     // logical keys per stage (32 stored nonzeros)
constexpr int STAGES = 4;
constexpr int NACC = 2;
constexpr int ASTAGES = 2;                  // TMEM A stages
constexpr int P_BYTES = BM * (BKL / 2) * 4;  // 16 KB: one 128B-swizzle atom
constexpr int VT_ATOM = HD * 128;            // 8 KB: 64 dims x 32 keys
constexpr int VT_BYTES = 2 * VT_ATOM;        // 16 KB per part (hi / lo)
constexpr int STAGE_BYTES = P_BYTES + 2 * VT_BYTES;
constexpr int SMEM_L = STAGES * STAGE_BYTES;  // [NACC][128] row sums of the fused softmax
constexpr int SMEM_BAR = SMEM_L + NACC * BM * 4;
constexpr int SMEM_TOTAL = SMEM_BAR + 256 + 1024;
constexpr int T_A = NACC * HD;  // A stages start after the accumulators: [stage][part][chunk] x 32 cols
constexpr int NTHREADS = 12 * 32;
constexpr float kLog2e = 1.4426950408889634f;
}  // namespace

__device__ __forceinline__ void mma_sp_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t e_tmem,
                                               uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %5, 0;\n\t"
      "tcgen05.mma.sp.cta_group::1.kind::tf32 [%0], [%1], %2, [%3], %4, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(e_tmem), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ uint32_t tf32_rna(float x) {
  uint32_t y;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(y) : "f"(x));
  return y;
}

__global__ void __launch_bounds__(NTHREADS, 1)
    spmm12_tf32x3_kernel(const __grid_constant__ CUtensorMap tm_p, const __grid_constant__ CUtensorMap tm_vh,
                         const __grid_constant__ CUtensorMap tm_vl, const uint32_t* __restrict__ meta,
                         float* __restrict__ out, int bh, int rows, int n_k, const float* __restrict__ rowmax) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = (uint64_t*)(smem + SMEM_BAR);
  uint64_t* full = bars;                   // [STAGES] TMA bytes landed
  uint64_t* empty = full + STAGES;         // [STAGES] the stage's MMAs retired (P already split)
  uint64_t* a_full = empty + STAGES;       // [ASTAGES] A hi / lo + metadata in TMEM (4 warps)
  uint64_t* a_empty = a_full + ASTAGES;    // [ASTAGES] MMAs reading that A stage retired
  uint64_t* d_full = a_empty + ASTAGES;    // [NACC]
  uint64_t* d_empty = d_full + NACC;       // [NACC] (4 epilogue warps)
  uint64_t* l_full = d_empty + NACC;       // [NACC] row sums in smem (4 split warps)
  uint32_t* tmem_slot = (uint32_t*)(l_full + NACC);
  float* lsum = (float*)(smem + SMEM_L);

  const uint32_t warp = tc::warp_id();
  const uint32_t lane = threadIdx.x & 31;
  const int rblocks = rows / BM;
  const int items = bh * rblocks;
  const int kblocks = n_k / BKL;
  const int words = n_k / 16;  // meta_hw words per row block lane (8 pairs each)

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tm_p);
    tc::prefetch_tmap(&tm_vh);
    tc::prefetch_tmap(&tm_vl);
    for (int i = 0; i < STAGES; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < ASTAGES; ++i) {
      tc::mbar_init(&a_full[i], 4);
      tc::mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < NACC; ++i) {
      tc::mbar_init(&d_full[i], 1);
      tc::mbar_init(&d_empty[i], 4);
      tc::mbar_init(&l_full[i], 4);
    }
    tc::fence_barrier_init();
  }
  if (warp == 2) tc::tmem_alloc<512>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic dependent of the SDDMM

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x) {
        const int b = item / rblocks, rb = item % rblocks;
        for (int kb = 0; kb < kblocks; ++kb) {
          tc::mbar_wait_sleep(&empty[s], ph ^ 1);
          uint8_t* st = smem + s * STAGE_BYTES;
          tc::mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
          tc::tma_load_3d(st, &tm_p, &full[s], kb * (BKL / 2), rb * BM, b);
#pragma unroll
          for (int a = 0; a < 2; ++a) {
            tc::tma_load_3d(st + P_BYTES + a * VT_ATOM, &tm_vh, &full[s], kb * BKL + 32 * a, 0, b);
            tc::tma_load_3d(st + P_BYTES + VT_BYTES + a * VT_ATOM, &tm_vl, &full[s], kb * BKL + 32 * a, 0, b);
          }
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = tc::instr_desc(2, BM, HD, false, false, true);  // tf32, B = V^T K-major, sparse
      int s = 0, as = 0, acc = 0;
      uint32_t ph = 0, aph = 0, dph = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x) {
        tc::mbar_wait_sleep(&d_empty[acc], dph ^ 1);
        const uint32_t d_tmem = tmem_base + acc * HD;
        for (int kb = 0; kb < kblocks; ++kb) {
          tc::mbar_wait_sleep(&full[s], ph);
          tc::mbar_wait_sleep(&a_full[as], aph);
          tc::tc_fence_after();
          const uint32_t vh = tc::smem_u32(smem + s * STAGE_BYTES + P_BYTES);
          const uint32_t vl = vh + VT_BYTES;
          const uint32_t abase = tmem_base + T_A + as * 128;
#pragma unroll
          for (int c = 0; c < 2; ++c) {  // 32-key chunk = V^T atom c
#pragma unroll
            for (int j = 0; j < 2; ++j) {  // 16 keys: 64-byte offset j inside the atom's rows
              const uint64_t bh_ = tc::smem_desc(vh + c * VT_ATOM + 64 * j, 16, 1024, tc::kSwizzle128B);
              const uint64_t bl_ = tc::smem_desc(vl + c * VT_ATOM + 64 * j, 16, 1024, tc::kSwizzle128B);
              const uint32_t a_hi = abase + c * 32 + 16 + 8 * j, a_lo = abase + 64 + c * 32 + 16 + 8 * j;
              const uint32_t e = abase + c * 32 + 4 * j;
              mma_sp_tf32_ts(d_tmem, a_hi, bh_, e, idesc, (kb | c | j) ? 1u : 0u);
              mma_sp_tf32_ts(d_tmem, a_hi, bl_, e, idesc, 1u);
              mma_sp_tf32_ts(d_tmem, a_lo, bh_, e, idesc, 1u);
            }
          }
          tc::mma_commit(&empty[s]);
          tc::mma_commit(&a_empty[as]);
          if (++s == STAGES) { s = 0; ph ^= 1; }
          if (++as == ASTAGES) { as = 0; aph ^= 1; }
        }
        tc::mma_commit(&d_full[acc]);
        if (++acc == NACC) { acc = 0; dph ^= 1; }
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ------------------------------------------------------------ split P into tf32 hi / lo (TMEM)
    const int quad = warp & 3;
    const int r = quad * 32 + lane;  // row within the 128-row block == TMEM lane
    const uint32_t lane_base = tmem_base + ((uint32_t)(quad * 32) << 16);
    int s = 0, as = 0, acc = 0;
    uint32_t ph = 0, aph = 0, dph = 0;
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
      const int b = item / rblocks, rb = item % rblocks;
      const uint32_t* mrow = meta + ((int64_t)b * rblocks + rb) * words * 128 + r;
      // fused row softmax (sparse_ops.py:18-37): the SDDMM's row maximum, exp2 of the scaled
      // difference per kept value, the row sum handed to the epilogue
      const float4 mp = *reinterpret_cast<const float4*>(rowmax + ((int64_t)b * rows + rb * BM + r) * 4);
      const float mb = fmaxf(fmaxf(mp.x, mp.y), fmaxf(mp.z, mp.w)) * kLog2e;
      float l = 0.f;
      for (int kb = 0; kb < kblocks; ++kb) {
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) w[i] = __ldg(mrow + (int64_t)(kb * 4 + i) * 128);
        tc::mbar_wait_sleep(&full[s], ph);
        tc::mbar_wait_sleep(&a_empty[as], aph ^ 1);
        tc::tc_fence_after();
        const uint8_t* prow = smem + s * STAGE_BYTES + r * 128;
        const uint32_t abase = lane_base + T_A + as * 128;
#pragma unroll
        for (int c = 0; c < 2; ++c) {  // 16 stored values = 32 keys
          uint32_t hi[16], lo[16];
#pragma unroll
          for (int u = 0; u < 4; ++u) {  // 16-byte unit 4c + u of the 128B-swizzled row
            const float4 x = *reinterpret_cast<const float4*>(prow + (((4 * c + u) ^ (r & 7)) << 4));
            const float xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float p = exp2f(fmaf(xv[e], kLog2e, -mb));
              l += p;
              hi[4 * u + e] = tf32_rna(p);
              lo[4 * u + e] = __float_as_uint(p - __uint_as_float(hi[4 * u + e]));
            }
          }
          tc::tmem_st_32x32b_x16(abase + c * 32 + 16, hi);
          tc::tmem_st_32x32b_x16(abase + 64 + c * 32 + 16, lo);
          tc::tmem_st_32x32b_x1(abase + c * 32, w[2 * c]);
          tc::tmem_st_32x32b_x1(abase + c * 32 + 4, w[2 * c + 1]);
        }
        tc::tmem_st_wait();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&a_full[as]);
        if (++s == STAGES) { s = 0; ph ^= 1; }
        if (++as == ASTAGES) { as = 0; aph ^= 1; }
      }
      // the row sum to the epilogue (buffer acc is free once its previous O was drained)
      tc::mbar_wait_sleep(&d_empty[acc], dph ^ 1);
      lsum[acc * BM + r] = l;
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&l_full[acc]);
      if (++acc == NACC) { acc = 0; dph ^= 1; }
    }
  } else if (warp >= 8) {
    // ------------------------------------------------------------ epilogue
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    int acc = 0;
    uint32_t dph = 0;
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
      const int b = item / rblocks, rb = item % rblocks;
      tc::mbar_wait_sleep(&d_full[acc], dph);
      tc::mbar_wait_sleep(&l_full[acc], dph);
      const float inv = 1.0f / lsum[acc * BM + r];
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
      float4* orow = reinterpret_cast<float4*>(out + ((int64_t)b * rows + rb * BM + r) * HD);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        orow[j] = make_float4(__uint_as_float(r0[4 * j]) * inv, __uint_as_float(r0[4 * j + 1]) * inv,
                              __uint_as_float(r0[4 * j + 2]) * inv, __uint_as_float(r0[4 * j + 3]) * inv);
        orow[8 + j] = make_float4(__uint_as_float(r1[4 * j]) * inv, __uint_as_float(r1[4 * j + 1]) * inv,
                                  __uint_as_float(r1[4 * j + 2]) * inv, __uint_as_float(r1[4 * j + 3]) * inv);
      }
      if (++acc == NACC) { acc = 0; dph ^= 1; }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc::tc_fence_after();
    tc::tmem_dealloc<512>(tmem_base);
  }
}

// V [bh][n][64] fp32 -> V^T hi / lo [bh][64][n] (hi = tf32(v) round-to-nearest, lo = v - hi)
__global__ void __launch_bounds__(256) vt_split_kernel(const float* __restrict__ v, float* __restrict__ vth,
                                                       float* __restrict__ vtl, int n, int64_t bh) {
  asm volatile("griddepcontrol.launch_dependents;");  // the SDDMM may launch (it waits on this grid)
  __shared__ float tile[32][HD + 1];
  const int k0 = blockIdx.x * 32;
  for (int64_t b = blockIdx.y; b < bh; b += gridDim.y) {
    const float* src = v + ((int64_t)b * n + k0) * HD;
    for (int i = threadIdx.x; i < 32 * HD; i += blockDim.x) tile[i / HD][i % HD] = src[i];
    __syncthreads();
    for (int i = threadIdx.x; i < 32 * HD; i += blockDim.x) {
      const int dim = i / 32, key = i % 32;
      const float x = tile[key][dim];
      const uint32_t h = tf32_rna(x);
      const int64_t o = (int64_t)b * HD * n + (int64_t)dim * n + k0 + key;
      vth[o] = __uint_as_float(h);
      vtl[o] = x - __uint_as_float(h);
    }
    __syncthreads();
  }
  // a programmatic dependent of the Q / K split: run alongside it (independent work), but finish
  // only after it, so the SDDMM that waits on this grid sees both
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

bool tc_spmm_tf32x3_supported(int gs, int rows, int n_k, int d) {
  return gs == 2 && d == HD && rows > 0 && rows % BM == 0 && n_k > 0 && n_k % BKL == 0;
}

int64_t spmm_tf32x3_workspace_bytes(int64_t bh, int n_k) { return 2 * ((bh * (int64_t)n_k * HD * 4 + 255) / 256 * 256); }

cudaError_t launch_spmm_tf32x3(const float* p, const uint32_t* meta, const float* v, float* out, int64_t bh, int rows,
                               int n_k, const float* rowmax, void* workspace, cudaStream_t s) {
  if (!tc_spmm_tf32x3_supported(2, rows, n_k, HD)) return cudaErrorNotSupported;
  if (bh == 0) return cudaSuccess;
  if (!workspace || !rowmax) return cudaErrorInvalidValue;
  float* vth = (float*)workspace;
  float* vtl = (float*)((char*)workspace + spmm_tf32x3_workspace_bytes(bh, n_k) / 2);
  const CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  CUtensorMap tp, th, tl;
  const uint64_t pdims[3] = {(uint64_t)n_k / 2, (uint64_t)rows, (uint64_t)bh};
  const uint64_t pstr[2] = {(uint64_t)n_k / 2 * 4, (uint64_t)rows * (n_k / 2) * 4};
  const uint32_t pbox[3] = {BKL / 2, BM, 1};
  const uint64_t vdims[3] = {(uint64_t)n_k, (uint64_t)HD, (uint64_t)bh};
  const uint64_t vstr[2] = {(uint64_t)n_k * 4, (uint64_t)n_k * HD * 4};
  const uint32_t vbox[3] = {32, HD, 1};
  if (!encode_tmap(&tp, dt, 3, (void*)p, pdims, pstr, pbox, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !encode_tmap(&th, dt, 3, vth, vdims, vstr, vbox, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !encode_tmap(&tl, dt, 3, vtl, vdims, vstr, vbox, CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  const int dev = current_device();
  static std::atomic<uint64_t> attr{0};
  cudaError_t e = set_max_smem_once((const void*)spmm12_tf32x3_kernel, attr, dev);
  if (e != cudaSuccess) return e;
  const int sms = device_sms(dev);
  const int64_t items = bh * (rows / BM);
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
  return cudaLaunchKernelEx(&cfg, spmm12_tf32x3_kernel, tp, th, tl, meta, out, (int)bh, rows, n_k, rowmax);
}

// V -> V^T hi / lo in the workspace, as a programmatic dependent of the Q / K split (see the kernel)
cudaError_t launch_vt_split_tf32x3(const float* v, int64_t bh, int n_k, void* workspace, cudaStream_t s) {
  if (bh == 0) return cudaSuccess;
  if (!workspace) return cudaErrorInvalidValue;
  float* vth = (float*)workspace;
  float* vtl = (float*)((char*)workspace + spmm_tf32x3_workspace_bytes(bh, n_k) / 2);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n_k / 32, (unsigned)(bh < 65535 ? bh : 65535));
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, vt_split_kernel, v, vth, vtl, n_k, bh);
}

}  // namespace dfss
