// op_probe2.cu -- issue rates of select / compare / convert / shift instructions (bring-up tool).
// Each op is emitted through inline PTX whose SASS is checked with cuobjdump; loop-carried
// operands keep the compiler from hoisting anything.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define REP8(X) X(0) X(1) X(2) X(3) X(4) X(5) X(6) X(7)

template <int OP>
__global__ void __launch_bounds__(512, 1) k(int iters, uint32_t* out, long long* cyc) {
  uint32_t u[8], w[8];
  for (int j = 0; j < 8; ++j) { u[j] = threadIdx.x * 0x9E3779B9u + j * 0x85EBCA6Bu; w[j] = u[j] ^ 0x3c003c00u; }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#define OPX(j)                                                                                              \
  if (OP == 0) asm volatile("{.reg .pred p; setp.lt.s32 p, %0, 0; selp.f32 %1, %1, %0, p;}" : "+r"(u[j]), "+r"(w[j])); \
  if (OP == 1) asm volatile("{.reg .pred p; setp.lt.s32 p, %1, 0; selp.b32 %0, %0, %1, p;}" : "+r"(u[j]), "+r"(w[j])); \
  if (OP == 2) asm volatile("{.reg .pred p; setp.gt.f32 p, %0, %1; selp.b32 %1, 1, %0, p;}" : "+f"(*(float*)&u[j]), "+r"(w[j])); \
  if (OP == 3) asm volatile("cvt.rn.bf16x2.f32 %0, %0, %1;" : "+r"(u[j]) : "f"(*(float*)&w[j]));                    \
  if (OP == 4) asm volatile("shr.u32 %0, %0, 31; xor.b32 %0, %0, %1;" : "+r"(u[j]) : "r"(w[j]));                      \
  if (OP == 5) asm volatile("prmt.b32 %0, %0, %1, 0x3254;" : "+r"(u[j]) : "r"(w[j]));                               \
  if (OP == 6) asm volatile("mul.hi.u32 %0, %0, 2; xor.b32 %0, %0, %1;" : "+r"(u[j]) : "r"(w[j]));                   \
  if (OP == 7) asm volatile("xor.b32 %0, %0, %1;" : "+r"(u[j]) : "r"(w[j]));
    REP8(OPX)
  }
  long long t1 = clock64();
  uint32_t s = 0;
  for (int j = 0; j < 8; ++j) s += u[j] ^ w[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, uint32_t* o, long long* c, int per) {
  long long h;
  const int warps = 16, iters = 2048;
  k<OP><<<148, warps * 32>>>(iters, o, c);
  cudaDeviceSynchronize();
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("%-34s %.1f cycles per %d-instr unit per warp-SMSP\n", name, (double)h / ((double)iters * 8 * warps / 4), per);
}

int main() {
  uint32_t* o; long long* c;
  cudaMalloc(&o, 148 * 512 * 4); cudaMalloc(&c, 148 * 8);
  run<7>("LOP3 (xor)", o, c, 1);
  run<0>("ISETP + FSEL", o, c, 2);
  run<1>("ISETP + SEL", o, c, 2);
  run<2>("FSETP + SEL", o, c, 2);
  run<3>("F2FP bf16x2", o, c, 1);
  run<4>("SHF + LOP3", o, c, 2);
  run<5>("PRMT", o, c, 1);
  run<6>("IMAD.HI + LOP3", o, c, 2);
  return 0;
}
