// negzero_probe.cu -- does tcgen05.mma (kind::f16, fp32 accumulate) ever write -0.0?  A = +/-0 rows,
// B = +/- values; dumps the sign of zero results (bring-up check for dropping score canonicalization).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "tc_common.cuh"
using namespace dfss;

__global__ void k(uint16_t a_val, uint16_t b_val, int accumulate_twice, int alt, uint32_t* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  uint16_t* a = (uint16_t*)smem;              // 128 x 64 bf16, 128B-swizzled layout irrelevant: all equal
  uint16_t* b = (uint16_t*)(smem + 16384);    // 128 x 64
  for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) { a[i] = a_val; b[i] = (alt && (i & 1)) ? (uint16_t)(b_val ^ 0x8000) : b_val; }
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_barrier_init(); }
  if (warp == 0) tc::tmem_alloc<128>(&slot);
  tc::fence_proxy_async();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = tc::instr_desc(1, 128, 128, false, false, false);
    for (int rep = 0; rep < 1 + accumulate_twice; ++rep)
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t ad = tc::smem_desc(tc::smem_u32(a) + kk * 32, 16, 1024, tc::kSwizzle128B);
        const uint64_t bd = tc::smem_desc(tc::smem_u32(b) + kk * 32, 16, 1024, tc::kSwizzle128B);
        tc::mma_f16_ss(tm, ad, bd, idesc, (kk > 0 || rep > 0) ? 1u : 0u);
      }
    tc::mma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::tc_fence_after();
  if (warp < 4) {
    uint32_t r[32];
    tc::tmem_ld_32x32b_x32(tm + ((warp * 32) << 16), r);
    tc::tmem_ld_wait(r);
    uint32_t negz = 0, posz = 0, other = 0;
    for (int j = 0; j < 32; ++j) {
      negz += r[j] == 0x80000000u;
      posz += r[j] == 0u;
      other += (r[j] & 0x7fffffffu) != 0;
    }
    atomicAdd(&out[0], negz);
    atomicAdd(&out[1], posz);
    atomicAdd(&out[2], other);
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<128>(tm);
}

int main() {
  uint32_t* d;
  cudaMalloc(&d, 12);
  struct { const char* name; uint16_t a, b; int twice, alt; } cs[] = {
      {"A=+0, B=+-1", 0x0000, 0x3f80, 0, 1}, {"A=-0, B=+1 (all products -0)", 0x8000, 0x3f80, 0, 0},
      {"A=+0, B=-1 (all products -0)", 0x0000, 0xbf80, 0, 0},
      {"A=-0, B=+1, accumulate twice", 0x8000, 0x3f80, 1, 0}, {"A=-0, B=-0 (products +0)", 0x8000, 0x8000, 0, 0},
      {"A=-0, B=+0 (products -0)", 0x8000, 0x0000, 0, 0}};
  for (auto& c : cs) {
    cudaMemset(d, 0, 12);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
    k<<<1, 128, 40 * 1024>>>(c.a, c.b, c.twice, c.alt, d);
    cudaError_t e = cudaDeviceSynchronize();
    uint32_t h[3];
    cudaMemcpy(h, d, 12, cudaMemcpyDeviceToHost);
    printf("%-34s err=%d  -0: %u  +0: %u  nonzero: %u\n", c.name, (int)e, h[0], h[1], h[2]);
  }
  return 0;
}
