// mixed_mma_probe.cu -- does tcgen05.mma kind::f16 accept A in f16 and B in bf16 (a_format != b_format)?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "tc_common.cuh"
using namespace dfss;

__global__ void k(uint32_t afmt, uint32_t bfmt, uint16_t aval, uint16_t bval, float* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  uint16_t* a = (uint16_t*)smem;
  uint16_t* b = (uint16_t*)(smem + 16384);
  for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) { a[i] = aval; b[i] = bval; }
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_barrier_init(); }
  if (warp == 0) tc::tmem_alloc<128>(&slot);
  tc::fence_proxy_async();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (afmt << 7) | (bfmt << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
    const uint64_t ad = tc::smem_desc(tc::smem_u32(a), 16, 1024, tc::kSwizzle128B);
    const uint64_t bd = tc::smem_desc(tc::smem_u32(b), 16, 1024, tc::kSwizzle128B);
    tc::mma_f16_ss(tm, ad, bd, idesc, 0u);
    tc::mma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::tc_fence_after();
  if (warp == 0) {
    uint32_t r[32];
    tc::tmem_ld_32x32b_x32(tm, r);
    tc::tmem_ld_wait(r);
    if (threadIdx.x == 0) out[0] = __uint_as_float(r[0]);
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<128>(tm);
}

int main() {
  float* d; float h;
  cudaMalloc(&d, 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  // f16 1.5 = 0x3E00, bf16 2.0 = 0x4000, f16 2.0 = 0x4000, bf16 1.5 = 0x3FC0; K = 16 -> expect 16 * 3 = 48
  struct { const char* n; uint32_t af, bf; uint16_t av, bv; } cs[] = {
      {"f16 x f16   (1.5 x 2.0)", 0, 0, 0x3E00, 0x4000}, {"bf16 x bf16 (1.5 x 2.0)", 1, 1, 0x3FC0, 0x4000},
      {"f16 A x bf16 B (1.5 x 2.0)", 0, 1, 0x3E00, 0x4000}, {"bf16 A x f16 B (1.5 x 2.0)", 1, 0, 0x3FC0, 0x4000}};
  for (auto& c : cs) {
    cudaMemset(d, 0, 4);
    k<<<1, 128, 40 * 1024>>>(c.af, c.bf, c.av, c.bv, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
    printf("%-30s err=%s D=%g (expect 48)\n", c.n, cudaGetErrorString(e), h);
    if (e) cudaGetLastError();
  }
  return 0;
}
