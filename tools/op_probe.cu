// op_probe.cu -- per-SMSP issue rate of the instructions in the prune/exp epilogue (bring-up tool).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define REP8(X) X(0) X(1) X(2) X(3) X(4) X(5) X(6) X(7)

template <int OP>
__global__ void __launch_bounds__(512, 1) k(int iters, float* out, long long* cyc) {
  float a[8], b[8];
  uint32_t u[8];
  for (int j = 0; j < 8; ++j) { a[j] = threadIdx.x * 1e-3f + j; b[j] = 1.0f + j * 1e-3f; u[j] = threadIdx.x * 3 + j; }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#define OPX(j)                                                                                              \
  if (OP == 0) asm volatile("max.f32 %0, %0, %1;" : "+f"(a[j]) : "f"(b[j]));                              \
  if (OP == 1) asm volatile("{.reg .pred p; setp.gt.f32 p, %0, %1; selp.f32 %0, %1, %0, p;}" : "+f"(a[j]) : "f"(b[j])); \
  if (OP == 2) asm volatile("{.reg .pred p; setp.gt.f32 p, %0, %1; selp.b32 %2, 5, %2, p;}" : "+f"(a[j]), "+r"(u[j]) : "f"(b[j])); \
  if (OP == 3) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[j]) : "f"(b[j]));                          \
  if (OP == 4) asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(a[j]) : "f"(b[j]));                       \
  if (OP == 5) asm volatile("{.reg .b64 x; mov.b64 x, {%0, %1}; add.rn.f32x2 x, x, x; mov.b64 {%0, %1}, x;}" : "+f"(a[j]), "+f"(b[j])); \
  if (OP == 6) asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(u[j]) : "r"(u[(j + 1) & 7]));                 \
  if (OP == 7) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[j]));                                   \
  if (OP == 8) asm volatile("{.reg .b32 t; cvt.rn.bf16x2.f32 t, %0, %1; mov.b32 %2, t;}" : "+f"(a[j]), "+f"(b[j]), "+r"(u[j])); \
  if (OP == 9) asm volatile("add.u32 %0, %0, %1;" : "+r"(u[j]) : "r"(u[(j + 3) & 7]));                    \
  if (OP == 10) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(u[j]) : "r"(u[(j + 3) & 7]), "r"(u[(j + 5) & 7])); \
  if (OP == 11) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(u[j]) : "r"(u[(j + 3) & 7]), "r"(u[(j + 5) & 7])); \
  if (OP == 12) asm volatile("{.reg .pred p; setp.ge.f32 p, %0, %1; @p add.f32 %0, %0, 1.0;}" : "+f"(a[j]) : "f"(b[j])); \
  if (OP == 13) asm volatile("min.f32 %0, %0, %1;" : "+f"(a[j]) : "f"(b[j]));
    REP8(OPX)
  }
  long long t1 = clock64();
  float s = 0;
  for (int j = 0; j < 8; ++j) s += a[j] + b[j] + u[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, float* o, long long* c) {
  long long h;
  const int warps = 16, iters = 2048;
  k<OP><<<148, warps * 32>>>(iters, o, c);
  cudaDeviceSynchronize();
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("%-28s %.3f warp-instr / clk / SMSP\n", name, (double)iters * 8 * warps / 4 / h);
}

int main() {
  float* o; long long* c;
  cudaMalloc(&o, 148 * 512 * 4); cudaMalloc(&c, 148 * 8);
  run<0>("FMNMX (max.f32)", o, c);
  run<13>("FMNMX (min.f32)", o, c);
  run<1>("FSETP + FSEL (2 instr)", o, c);
  run<2>("FSETP + SEL (2 instr)", o, c);
  run<3>("FADD", o, c);
  run<4>("FFMA", o, c);
  run<5>("FADD2", o, c);
  run<6>("IMAD.HI", o, c);
  run<7>("MUFU.EX2", o, c);
  run<8>("F2FP bf16x2", o, c);
  run<9>("IADD3", o, c);
  run<10>("LOP3", o, c);
  run<11>("IMAD", o, c);
  run<12>("FSETP + @p FADD (2 instr)", o, c);
  return 0;
}
