// op_probe3.cu -- dispatch cost model: ops alone and mixed with full-rate FFMA (bring-up tool).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define REP8(X) X(0) X(1) X(2) X(3) X(4) X(5) X(6) X(7)

template <int OP>
__global__ void __launch_bounds__(512, 1) k(int iters, uint32_t* out, long long* cyc) {
  float f[8], g[8];
  uint32_t u[8];
  for (int j = 0; j < 8; ++j) { f[j] = threadIdx.x * 1e-4f + j * 0.01f; g[j] = 0.999f + j * 1e-4f; u[j] = threadIdx.x * 0x9E3779B9u + j; }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#define FF(j) asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(g[j]) : "f"(f[j]));
#define OPX(j)                                                                                                  \
  if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[j]));                                          \
  if (OP == 1) { asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[j])); FF(j) FF((j+1)&7) FF((j+2)&7) FF((j+3)&7) } \
  if (OP == 2) asm volatile("max.f32 %0, %0, %1;" : "+f"(f[j]) : "f"(g[j]));                                     \
  if (OP == 3) { asm volatile("max.f32 %0, %0, %1;" : "+f"(f[j]) : "f"(g[j])); FF(j) }                           \
  if (OP == 4) asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(u[j]) : "r"(u[(j + 3) & 7]));                        \
  if (OP == 5) { asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(u[j]) : "r"(u[(j + 3) & 7])); FF(j) FF((j+1)&7) }  \
  if (OP == 6) asm volatile("xor.b32 %0, %0, %1;" : "+r"(u[j]) : "r"(u[(j + 3) & 7]));                           \
  if (OP == 7) { asm volatile("xor.b32 %0, %0, %1;" : "+r"(u[j]) : "r"(u[(j + 3) & 7])); FF(j) }                 \
  if (OP == 8) asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(g[j]) : "f"(f[j]));                              \
  if (OP == 9) asm volatile("{.reg .b64 x; mov.b64 x, {%0, %1}; add.rn.f32x2 x, x, x; mov.b64 {%0, %1}, x;}" : "+f"(f[j]), "+f"(g[j])); \
  if (OP == 10) { asm volatile("{.reg .b64 x; mov.b64 x, {%0, %1}; add.rn.f32x2 x, x, x; mov.b64 {%0, %1}, x;}" : "+f"(f[j]), "+f"(g[(j+4)&7])); asm volatile("xor.b32 %0, %0, %1;" : "+r"(u[j]) : "r"(u[(j + 3) & 7])); } \
  if (OP == 11) { asm volatile("max.f32 %0, %0, %1;" : "+f"(f[j]) : "f"(g[j])); asm volatile("xor.b32 %0, %0, %1;" : "+r"(u[j]) : "r"(u[(j + 3) & 7])); }
    REP8(OPX)
  }
  long long t1 = clock64();
  uint32_t s = 0;
  for (int j = 0; j < 8; ++j) s += u[j] + __float_as_uint(f[j] + g[j]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, uint32_t* o, long long* c) {
  long long h;
  const int warps = 16, iters = 2048;
  k<OP><<<148, warps * 32>>>(iters, o, c);
  cudaDeviceSynchronize();
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("%-40s %.2f cycles per unit (per warp, per SMSP)\n", name, (double)h / ((double)iters * 8 * warps / 4));
}

int main() {
  uint32_t* o; long long* c;
  cudaMalloc(&o, 148 * 512 * 4); cudaMalloc(&c, 148 * 8);
  run<8>("FFMA", o, c);
  run<0>("MUFU.EX2", o, c);
  run<1>("MUFU.EX2 + 4 FFMA", o, c);
  run<2>("FMNMX", o, c);
  run<3>("FMNMX + FFMA", o, c);
  run<4>("IMAD.HI", o, c);
  run<5>("IMAD.HI + 2 FFMA", o, c);
  run<6>("LOP3", o, c);
  run<7>("LOP3 + FFMA", o, c);
  run<9>("FADD2", o, c);
  run<10>("FADD2 + LOP3", o, c);
  run<11>("FMNMX + LOP3", o, c);
  return 0;
}
