// tmem_probe.cu -- microbenchmark: tcgen05.ld throughput per SM (bytes/cycle) vs warps and load width,
// and FADD2/FFMA2/FMNMX/FSEL issue rates.  Bring-up tool, not product code.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_probe tools/tmem_probe.cu && ./tmem_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int X>
__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t* r);
template <>
__device__ __forceinline__ void ld32<32>(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
template <>
__device__ __forceinline__ void ld32<16>(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

template <int X>
__global__ void tmem_ld_kernel(int iters, uint32_t* out, long long* cycles) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16);
  uint32_t acc = 0, r[32];
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const uint32_t col = ((i * 4 + (warp >> 2)) * X) & 511;
    ld32<X>(base + col, r);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < X; ++j) acc ^= r[j];
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

// ALU / FMA issue probe: 8 independent chains of op per thread
template <int OP>
__global__ void op_kernel(int iters, float* out, long long* cycles) {
  float a[8], b[8];
  for (int j = 0; j < 8; ++j) { a[j] = threadIdx.x * 0.001f + j; b[j] = 1.0f + j * 1e-3f; }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; j += 2) {
      if (OP == 0) {  // FMNMX
        a[j] = fmaxf(a[j], b[j]); a[j + 1] = fminf(a[j + 1], b[j + 1]);
      } else if (OP == 1) {  // FFMA 3-reg
        a[j] = fmaf(a[j], b[j], b[j + 1]); a[j + 1] = fmaf(a[j + 1], b[j + 1], b[j]);
      } else if (OP == 2) {  // FFMA2
        uint64_t A = ((uint64_t)__float_as_uint(a[j + 1]) << 32) | __float_as_uint(a[j]);
        uint64_t B = ((uint64_t)__float_as_uint(b[j + 1]) << 32) | __float_as_uint(b[j]);
        uint64_t D;
        asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(D) : "l"(A), "l"(B), "l"(B));
        a[j] = __uint_as_float((uint32_t)D); a[j + 1] = __uint_as_float((uint32_t)(D >> 32));
      } else if (OP == 3) {  // FSEL via predicate
        bool p = a[j] > b[j + 1];
        a[j] = p ? b[j] : a[j + 1]; a[j + 1] = p ? a[j + 1] : b[j];
      } else if (OP == 4) {  // MUFU ex2
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[j])); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[j + 1]));
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
  for (int j = 0; j < 8; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

int main() {
  uint32_t* out; long long* cyc; float* fo;
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8); cudaMalloc(&fo, 148 * 1024 * 4);
  long long h[148];
  const int iters = 4096;
  for (int warps : {4, 8, 16}) {
    for (int x : {16, 32}) {
      if (x == 32) tmem_ld_kernel<32><<<148, warps * 32>>>(iters, out, cyc);
      else tmem_ld_kernel<16><<<148, warps * 32>>>(iters, out, cyc);
      cudaError_t e = cudaDeviceSynchronize();
      if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      double bytes = (double)iters * warps * 32 * x * 4;
      printf("tcgen05.ld x%d warps=%d: %lld cycles, %.1f B/cycle/SM\n", x, warps, h[0], bytes / h[0]);
    }
  }
  const char* names[] = {"FMNMX", "FFMA", "FFMA2", "FSETP+FSEL", "MUFU.EX2"};
  for (int op = 0; op < 5; ++op) {
    for (int warps : {4, 8, 16}) {
      switch (op) {
        case 0: op_kernel<0><<<148, warps * 32>>>(iters, fo, cyc); break;
        case 1: op_kernel<1><<<148, warps * 32>>>(iters, fo, cyc); break;
        case 2: op_kernel<2><<<148, warps * 32>>>(iters, fo, cyc); break;
        case 3: op_kernel<3><<<148, warps * 32>>>(iters, fo, cyc); break;
        case 4: op_kernel<4><<<148, warps * 32>>>(iters, fo, cyc); break;
      }
      cudaDeviceSynchronize();
      cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      double ops = (double)iters * 8 * warps;  // warp-level "op slots" (FFMA2 = 2 lanes-ops per slot pair)
      printf("%-10s warps=%2d: %lld cycles, %.3f warp-ops/cycle/SMSP\n", names[op], warps, h[0], ops / h[0] / 4);
    }
  }
  return 0;
}
