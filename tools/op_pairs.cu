// op_pairs.cu -- issue cost of each epilogue instruction alone and paired with every other one
// (8 independent chains per thread, 16 warps per SM): which instructions share a pipe (bring-up tool).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define NOPS 14
const char* names[NOPS] = {"FMNMX", "FSEL", "SEL", "FSETP", "LOP3", "SHF", "PRMT", "IADD3", "IMAD", "IMAD.HI",
                           "FADD", "FFMA", "FADD2", "F2FP"};
template <int OP>
__device__ __forceinline__ void op(float& f, uint32_t& u, float g, uint32_t v) {
  if (OP == 0) asm volatile("max.f32 %0, %0, %1;" : "+f"(f) : "f"(g));
  if (OP == 1) asm volatile("{.reg .pred p; setp.ne.b32 p, %2, 0; selp.f32 %0, %0, %1, p;}" : "+f"(f) : "f"(g), "r"(v & 1));
  if (OP == 2) asm volatile("{.reg .pred p; setp.ne.b32 p, %2, 0; selp.b32 %0, %0, %1, p;}" : "+r"(u) : "r"(v), "r"(v & 2));
  if (OP == 3) asm volatile("{.reg .pred p; setp.gt.f32 p, %1, %2; selp.b32 %0, 1, 0, p; }" : "=r"(u) : "f"(f), "f"(g));
  if (OP == 4) asm volatile("xor.b32 %0, %0, %1;" : "+r"(u) : "r"(v));
  if (OP == 5) asm volatile("shf.l.clamp.b32 %0, %1, %0, 1;" : "+r"(u) : "r"(v));
  if (OP == 6) asm volatile("prmt.b32 %0, %0, %1, 0x5140;" : "+r"(u) : "r"(v));
  if (OP == 7) asm volatile("add.u32 %0, %0, %1;" : "+r"(u) : "r"(v));
  if (OP == 8) asm volatile("mad.lo.u32 %0, %0, %1, %1;" : "+r"(u) : "r"(v));
  if (OP == 9) asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(u) : "r"(v));
  if (OP == 10) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(f) : "f"(g));
  if (OP == 11) asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(f) : "f"(g));
  if (OP == 12) asm volatile("{.reg .b64 x; mov.b64 x, {%0, %1}; add.rn.f32x2 x, x, x; mov.b64 {%0, %1}, x;}" : "+f"(f), "+f"(g));
  if (OP == 13) asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u) : "f"(f), "f"(g));
}
template <int A, int B>
__global__ void __launch_bounds__(512, 1) k(int iters, long long* cyc, float* o) {
  float f[8], g[8], f2[8], g2[8];
  uint32_t u[8], v[8], u2[8];
  for (int j = 0; j < 8; ++j) {
    f[j] = threadIdx.x * 1e-4f + j; g[j] = 0.5f + j; f2[j] = f[j] + 1; g2[j] = g[j] + 2;
    u[j] = threadIdx.x * 0x9E3779B9u + j; v[j] = u[j] * 3 + 1; u2[j] = u[j] ^ 5;
  }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      op<A>(f[j], u[j], g[j], v[j]);
      if (B >= 0) op<B < 0 ? 0 : B>(f2[j], u2[j], g2[j], v[j]);
    }
  }
  long long t1 = clock64();
  float acc = 0;
  for (int j = 0; j < 8; ++j) acc += f[j] + f2[j] + g[j] + g2[j] + (float)(u[j] ^ u2[j]);
  o[blockIdx.x * 512 + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
long long* cyc; float* o;
template <int A, int B>
double run() {
  const int iters = 2048;
  k<A, B><<<148, 512>>>(iters, cyc, o);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  return (double)h / (iters * 8.0 * 4);  // cycles per (A [+ B]) per warp per SMSP (4 warps / SMSP)
}
template <int A, int B>
void row_b(double* r) {
  r[B] = run<A, B>();
  if constexpr (B + 1 < NOPS) row_b<A, B + 1>(r);
}
template <int A>
void rows() {
  double r[NOPS];
  const double alone = run<A, -1>();
  row_b<A, 0>(r);
  printf("%-8s %5.2f |", names[A], alone);
  for (int b = 0; b < NOPS; ++b) printf(" %5.2f", r[b]);
  printf("\n");
  if constexpr (A + 1 < NOPS) rows<A + 1>();
}
int main() {
  cudaMalloc(&cyc, 148 * 8);
  cudaMalloc(&o, 148 * 512 * 4);
  printf("cycles per instruction (or pair) per warp per SMSP, 4 warps / SMSP\n%-8s %5s |", "op", "alone");
  for (int b = 0; b < NOPS; ++b) printf(" %5.5s", names[b]);
  printf("\n");
  rows<0>();
  return 0;
}
