// sp_probe.cu -- hardware probe for the tcgen05.mma.sp metadata layout (bring-up tool,
// not part of the product library).  One CTA, 128 threads: A = all ones (128 x 16 stored
// bf16, K-major SW128), B[k][n] = (n == k) for k < 32 (MN-major SW128), E = 128 given
// 32-bit words in one TMEM column.  Then D[r][n] = 1 iff logical column n of row r is
// kept by the metadata, which exposes the (lane, bit) -> (row, group) map directly.
#include <cuda_bf16.h>

#include "../paper_2203_00091_b200/csrc/tc_common.cuh"

using namespace dfss;

__global__ void probe_kernel(const uint32_t* e_words, float* d_out, int dense, int ecol, int id2mode) {
  __shared__ __align__(1024) uint8_t a_s[128 * 128];
  __shared__ __align__(1024) uint8_t b_s[32 * 128];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  __nv_bfloat16 one = __float2bfloat16(1.0f), zero = __float2bfloat16(0.0f);
  for (int i = tid; i < 128 * 64; i += blockDim.x) reinterpret_cast<__nv_bfloat16*>(a_s)[i] = one;
  for (int i = tid; i < 32 * 64; i += blockDim.x) {
    const int k = i / 64, n = i % 64;
    const int byte = k * 128 + ((((n * 2) >> 4) ^ (k & 7)) << 4) + ((n * 2) & 15);
    *reinterpret_cast<__nv_bfloat16*>(b_s + byte) = (n == k) ? one : zero;
  }
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_barrier_init();
  }
  if (warp == 0) tc::tmem_alloc<128>(&tslot);
  tc::fence_proxy_async();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = tslot;
  tc::tmem_st_32x32b_x1(tbase + ((uint32_t)(warp * 32) << 16) + ecol, e_words[warp * 32 + lane]);
  tc::tmem_st_wait();
  tc::tc_fence_before();
  __syncthreads();
  if (tid == 0) {
    tc::tc_fence_after();
    const uint64_t ad = tc::smem_desc(tc::smem_u32(a_s), 16, 1024, tc::kSwizzle128B);
    const uint64_t bd = tc::smem_desc(tc::smem_u32(b_s), 32 * 128, 1024, tc::kSwizzle128B);
    if (dense) {
      tc::mma_f16_ss(tbase, ad, bd, tc::instr_desc(1, 128, 64, false, true, false), 0);
    } else {
      const uint32_t e = tbase + ecol;
      if (id2mode)
        tc::mma_sp_f16_ss(tbase, ad, bd, e & ~1u, tc::instr_desc(1, 128, 64, false, true, true) | (e & 1u), 0);
      else
        tc::mma_sp_f16_ss(tbase, ad, bd, e, tc::instr_desc(1, 128, 64, false, true, true), 0);
    }
    tc::mma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::tc_fence_after();
  uint32_t r0[32], r1[32];
  tc::tmem_ld_32x32b_x32(tbase + ((uint32_t)(warp * 32) << 16), r0);
  tc::tmem_ld_32x32b_x32(tbase + ((uint32_t)(warp * 32) << 16) + 32, r1);
  tc::tmem_ld_wait();
  for (int j = 0; j < 32; ++j) {
    d_out[tid * 64 + j] = __uint_as_float(r0[j]);
    d_out[tid * 64 + 32 + j] = __uint_as_float(r1[j]);
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<128>(tbase);
}

extern "C" int probe_sp(const uint32_t* e_words, float* d_out, int dense, int ecol, int id2mode) {
  probe_kernel<<<1, 128>>>(e_words, d_out, dense, ecol, id2mode);
  cudaError_t e = cudaDeviceSynchronize();
  return (int)e;
}
