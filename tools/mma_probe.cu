// mma_probe.cu -- microbenchmark: tcgen05.mma throughput for the flash kernel's tile shapes (bring-up tool).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2203_00091_b200/csrc -o mma_probe tools/mma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "tc_common.cuh"
using namespace dfss;

// MODE 0: dense SS (A, B from smem, rotating over 4 A tiles and 4 B tiles)
// MODE 1: dense TS (A from TMEM)
// MODE 2: sparse SS (K = 32)
// MODE 3: sparse TS (K = 32)
// MODE 4: mixed: per iteration 4 dense SS N (S) + 2 sparse TS N=64 (PV), like one flash step
template <int MODE, int N>
__global__ void probe(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_barrier_init(); }
  if (warp == 0) tc::tmem_alloc<512>(&slot);
  tc::fence_proxy_async();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tm = slot;
  // TMEM: D at 0 (N cols), A at 256, E at 300, D2 at 320
  if (warp == 1) {  // fill A / E columns
    uint32_t r[8];
    for (int j = 0; j < 8; ++j) r[j] = 0x3c003c00u;
    const uint32_t lb = tm + (((threadIdx.x >> 5) & 3) * 32 << 16);
    tc::tmem_st_32x32b_x8(lb + 256, r);
    tc::tmem_st_32x32b_x8(lb + 264, r);
    tc::tmem_st_32x32b_x8(lb + 272, r);
    tc::tmem_st_32x32b_x8(lb + 280, r);
    tc::tmem_st_32x32b_x1(lb + 300, 0x44444444u);
    tc::tmem_st_wait();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (threadIdx.x == 0) {
    constexpr bool sparse = MODE == 2 || MODE == 3;
    constexpr uint32_t idesc = tc::instr_desc(1, 128, N, false, false, sparse);
    constexpr uint32_t idesc_pv = tc::instr_desc(1, 128, 64, false, true, true);
    const uint32_t a = tc::smem_u32(smem), b = tc::smem_u32(smem + 65536);
    long long t0 = clock64();
    int cnt = 0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t ad = tc::smem_desc(a + (i & 3) * 16384 + kk * 32, 16, 1024, tc::kSwizzle128B);
        const uint64_t bd = tc::smem_desc(b + (i & 3) * 16384 + kk * 32, 16, 1024, tc::kSwizzle128B);
        if (MODE == 0 || MODE == 4) tc::mma_f16_ss(tm, ad, bd, idesc, kk > 0 ? 1u : 0u);
        if (MODE == 1) {
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %4, p;\n\t}\n" ::"r"(tm),
                       "r"(tm + 256 + kk * 8), "l"(bd), "r"((uint32_t)(kk > 0)), "r"(idesc));
        }
        if (MODE == 2) tc::mma_sp_f16_ss(tm, ad, bd, tm + 300, idesc, kk > 0 ? 1u : 0u);
        if (MODE == 3) tc::mma_sp_f16_ts(tm, tm + 256 + kk * 8, bd, tm + 300, idesc, kk > 0 ? 1u : 0u);
        ++cnt;
      }
      if (MODE == 4) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const uint64_t vd = tc::smem_desc(b + 32768 + q * 4096, 8192, 1024, tc::kSwizzle128B);
          tc::mma_sp_f16_ts(tm + 320, tm + 256 + q * 8, vd, tm + 300, idesc_pv, 1u);
        }
      }
    }
    long long t1 = clock64();
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t0;
    out[2] = cnt;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tm);
}

template <int MODE, int N>
void run(long long* d, const char* name) {
  long long h[3];
  const int iters = 256;
  cudaFuncSetAttribute(probe<MODE, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  probe<MODE, N><<<1, 128, 160 * 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e) { printf("%s err %s\n", name, cudaGetErrorString(e)); return; }
  cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
  const double per_iter = (double)h[1] / iters;
  printf("%-24s N=%3d: %.1f cyc per 4-MMA group (%.1f per MMA)\n", name, N, per_iter, per_iter / 4);
}

int main() {
  long long* d;
  cudaMalloc(&d, 24);
  run<0, 64>(d, "dense SS");
  run<0, 128>(d, "dense SS");
  run<1, 64>(d, "dense TS (A tmem)");
  run<1, 128>(d, "dense TS (A tmem)");
  run<2, 64>(d, "sparse SS K32");
  run<3, 64>(d, "sparse TS K32");
  run<4, 64>(d, "S N64 x4 + 2 PV sp TS");
  run<4, 128>(d, "S N128 x4 + 2 PV sp TS");
  return 0;
}
