// sp_order_probe.cu -- does tcgen05.mma.sp accept metadata nibbles whose two indices are not in
// ascending order (idx0 > idx1) or equal (bring-up tool).  A stores 1 in slot 0 and 2 in slot 1
// of every group, B = identity, so D[r][4g + i] shows which slot each column received.
#include <cstdio>
#include <cuda_bf16.h>

#include "../paper_2203_00091_b200/csrc/tc_common.cuh"

using namespace dfss;

__global__ void probe_kernel(uint32_t nib, float* d_out) {
  __shared__ __align__(1024) uint8_t a_s[128 * 128];
  __shared__ __align__(1024) uint8_t b_s[32 * 128];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  __nv_bfloat16 one = __float2bfloat16(1.0f), two = __float2bfloat16(2.0f), zero = __float2bfloat16(0.0f);
  for (int i = tid; i < 128 * 64; i += blockDim.x) {
    const int r = i / 64, k = i % 64;
    const int byte = r * 128 + ((((k * 2) >> 4) ^ (r & 7)) << 4) + ((k * 2) & 15);
    *reinterpret_cast<__nv_bfloat16*>(a_s + byte) = k < 16 ? ((k & 1) ? two : one) : zero;
  }
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
  const uint32_t ecol = 64;
  tc::tmem_st_32x32b_x1(tbase + ((uint32_t)(warp * 32) << 16) + ecol, nib * 0x11111111u);
  tc::tmem_st_wait();
  tc::tc_fence_before();
  __syncthreads();
  if (tid == 0) {
    tc::tc_fence_after();
    const uint64_t ad = tc::smem_desc(tc::smem_u32(a_s), 16, 1024, tc::kSwizzle128B);
    const uint64_t bd = tc::smem_desc(tc::smem_u32(b_s), 32 * 128, 1024, tc::kSwizzle128B);
    tc::mma_sp_f16_ss(tbase, ad, bd, tbase + ecol, tc::instr_desc(1, 128, 64, false, true, true), 0);
    tc::mma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::tc_fence_after();
  uint32_t r0[32];
  tc::tmem_ld_32x32b_x32(tbase + ((uint32_t)(warp * 32) << 16), r0);
  tc::tmem_ld_wait();
  if (tid == 0)
    for (int j = 0; j < 8; ++j) d_out[j] = __uint_as_float(r0[j]);
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<128>(tbase);
}

int main() {
  float* d;
  float h[8];
  cudaMalloc(&d, 8 * 4);
  const uint32_t nibs[] = {0x4, 0x8, 0xC, 0x9, 0xD, 0xE, 0x1, 0x2, 0x3, 0x6, 0x7, 0xB, 0x0, 0x5, 0xA, 0xF};
  for (uint32_t nb : nibs) {
    cudaMemset(d, 0xff, 32);
    probe_kernel<<<1, 128>>>(nb, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    printf("nibble 0x%X (idx0 %u, idx1 %u): %s  D[0][0..7] = %g %g %g %g | %g %g %g %g\n", nb, nb & 3, nb >> 2,
           cudaGetErrorString(e), h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
