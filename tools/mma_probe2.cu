// mma_probe2.cu -- tcgen05.mma throughput under the flash kernel's concurrency (bring-up tool):
// one vs two issuing threads, with / without 16 warps streaming tcgen05.ld from TMEM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "tc_common.cuh"
using namespace dfss;

template <int MODE>
__global__ void probe(int iters, long long* out, int ld_warps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[2];
  __shared__ uint32_t slot;
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 128 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { tc::mbar_init(&bar[0], 1); tc::mbar_init(&bar[1], 1); tc::fence_barrier_init(); done = 0; }
  if (warp == 0) tc::tmem_alloc<512>(&slot);
  tc::fence_proxy_async();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tm = slot;
  {  // P / E columns of both slots (TMEM 256.. for A, 300 for E) -- any 16-bit data
    uint32_t r[8];
    for (int j = 0; j < 8; ++j) r[j] = 0x3c003c00u;
    const uint32_t lb = tm + (((warp & 3) * 32) << 16);
    if (warp < 4) {
      for (int c = 0; c < 4; ++c) tc::tmem_st_32x32b_x8(lb + 256 + 8 * c, r);
      tc::tmem_st_32x32b_x1(lb + 300, 0x44444444u);
      tc::tmem_st_wait();
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  constexpr uint32_t idesc_s = tc::instr_desc(1, 128, 128, false, false, false);
  constexpr uint32_t idesc_pv = tc::instr_desc(1, 128, 64, false, true, true);
  const uint32_t a = tc::smem_u32(smem), b = tc::smem_u32(smem + 65536);
  auto issue_s = [&](int i) {
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const uint64_t ad = tc::smem_desc(a + (i & 1) * 16384 + kk * 32, 16, 1024, tc::kSwizzle128B);
      const uint64_t bd = tc::smem_desc(b + (i & 1) * 16384 + kk * 32, 16, 1024, tc::kSwizzle128B);
      tc::mma_f16_ss(tm, ad, bd, idesc_s, kk > 0 ? 1u : 0u);
    }
  };
  auto issue_pv = [&](int i) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint64_t vd = tc::smem_desc(b + 32768 + q * 4096, 16384, 1024, tc::kSwizzle128B);
      tc::mma_sp_f16_ts(tm + 384, tm + 256 + q * 8, vd, tm + 300, idesc_pv, 1u);
    }
  };
  long long t0 = clock64();
  if (MODE == 0) {  // one thread: S then PV
    if (threadIdx.x == 32) {
      for (int i = 0; i < iters; ++i) { issue_s(i); issue_pv(i); }
      tc::mma_commit(&bar[0]);
      tc::mbar_wait(&bar[0], 0);
      out[0] = clock64() - t0;
      done = 1;
    }
  } else {  // two threads
    if (threadIdx.x == 32) {
      for (int i = 0; i < iters; ++i) issue_s(i);
      tc::mma_commit(&bar[0]);
      tc::mbar_wait(&bar[0], 0);
      out[0] = clock64() - t0;
    }
    if (threadIdx.x == 64) {
      for (int i = 0; i < iters; ++i) issue_pv(i);
      tc::mma_commit(&bar[1]);
      tc::mbar_wait(&bar[1], 0);
      out[1] = clock64() - t0;
      done = 1;
    }
  }
  if (warp >= 4 && warp < 4 + ld_warps) {  // TMEM readers, columns 128..255
    uint32_t acc = 0, r[32];
    const uint32_t lb = tm + (((warp & 3) * 32) << 16) + 128 + ((warp >> 2) & 3) * 32;
    while (!done) {
      tc::tmem_ld_32x32b_x32(lb, r);
      tc::tmem_ld_wait(r);
      for (int j = 0; j < 32; ++j) acc += r[j];
    }
    if (acc == 12345) out[2] = acc;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tm);
}

int main() {
  long long* d;
  long long h[3];
  cudaMalloc(&d, 24);
  const int iters = 256;
  for (int mode = 0; mode < 2; ++mode) {
    for (int ldw : {0, 8, 16}) {
      auto k = mode == 0 ? probe<0> : probe<1>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
      cudaMemset(d, 0, 24);
      k<<<1, 640, 128 * 1024>>>(iters, d, ldw);
      cudaError_t e = cudaDeviceSynchronize();
      if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
      printf("%s issuer(s), %2d TMEM-ld warps: %.1f cyc per (4 S N128 + 4 PV sparse TS)  [S-only thread %.1f]\n",
             mode == 0 ? "one" : "two", ldw, (double)(mode == 0 ? h[0] : (h[0] > h[1] ? h[0] : h[1])) / iters,
             (double)h[0] / iters);
    }
  }
  return 0;
}
