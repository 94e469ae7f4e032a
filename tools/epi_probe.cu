// epi_probe.cu -- the fused kernel's prune + exp + pack epilogue alone, 16 warps / SM as in the
// kernel, S fed from shared memory (stands in for tcgen05.ld) and P / metadata stored back to
// shared memory (stands in for tcgen05.st): cycles per warp-step (16 groups per warp, 4 warps
// per SMSP) for alternative formulations of the 2:4 selection (bring-up tool).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_2203_00091_b200/csrc/flash_common.cuh"

using namespace dfss;

__device__ __forceinline__ uint32_t shl_in(uint32_t w, float src) {  // (w << 1) | sign(src)
  uint32_t r;
  asm("shf.l.clamp.b32 %0, %1, %2, 1;" : "=r"(r) : "r"(__float_as_uint(src)), "r"(w));
  return r;
}
__device__ __forceinline__ uint32_t lop_and_andn(float a, float b, float c) {  // a & b & ~c
  return __float_as_uint(a) & __float_as_uint(b) & ~__float_as_uint(c);
}
__device__ __forceinline__ uint32_t lop_or_orn(float a, float b, float c) {  // a | ~b | c
  return __float_as_uint(a) | ~__float_as_uint(b) | __float_as_uint(c);
}

__device__ __forceinline__ void mul2(float a0, float a1, float b0, float b1, float& d0, float& d1) {
  asm("{\n\t.reg .b64 a, b, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
      "mul.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
__device__ __forceinline__ float fset_gt(float a, float b) {  // 1.0f if a > b else 0.0f
  float r;
  asm("set.gt.f32.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float fset_ge(float a, float b) {
  float r;
  asm("set.ge.f32.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

template <int MODE>
__device__ __forceinline__ void prune(const uint32_t (&s)[32], float c, float mlog, uint32_t two, uint32_t (&pk)[8],
                                      uint32_t& W, float& lt0, float& lt1) {
  using T = __nv_bfloat16;
  W = (MODE == 2) ? 0u : 0x88888888u;
  lt0 = 0.f;
  lt1 = 0.f;
  float wf[2] = {8388608.f + 34952.f, 8388608.f + 34952.f};  // 2^23 + 0x8888: nibble - 8 accumulated
#pragma unroll
  for (int gg = 0; gg < 8; ++gg) {
    const int g = (MODE == 2) ? 7 - gg : gg;  // funnel shifts build W from the top nibble down
    if (MODE == 15) {
      // registers hold (v0, v2, v1, v3): differences are one FADD2, the flag multiply one FMUL2
      const float v0 = __uint_as_float(s[4 * g + 0]), v2 = __uint_as_float(s[4 * g + 1]);
      const float v1 = __uint_as_float(s[4 * g + 2]), v3 = __uint_as_float(s[4 * g + 3]);
      float d01, d23, m01, m23;
      sub2(v0, v2, v1, v3, d01, d23);
      mul2(d01, d23, -1.7014118e38f, -1.7014118e38f, m01, m23);
      const float fa = __saturatef(m01 * 1.7014118e38f), fb = __saturatef(m23 * 1.7014118e38f);
      const float w01 = fmaxf(v0, v1), w23 = fmaxf(v2, v3), l01 = fminf(v0, v1), l23 = fminf(v2, v3);
      const bool keep01 = l01 >= w23, keep23 = l23 > w01;
      const float lo = keep01 ? v0 : (keep23 ? v2 : w01);
      const float hi = keep01 ? v1 : (keep23 ? v3 : w23);
      float n = fmaf(fb, 4.f, fa);
      n = keep23 ? 6.f : n;
      n = keep01 ? -4.f : n;
      wf[g >> 2] = fmaf(n, (float)(1 << (4 * (g & 3))), wf[g >> 2]);
      if (g == 7) W = __byte_perm(__float_as_uint(wf[0]), __float_as_uint(wf[1]), 0x5410);
      const float x0 = fmaf(lo, c, -mlog), x1 = fmaf(hi, c, -mlog);
      const float p0 = fex2(x0), p1 = fex2(x1);
      pk[g] = fpack2<T>(p0, p1);
      add2(lt0, lt1, p0, p1, lt0, lt1);
      continue;
    }
    const float v0 = __uint_as_float(s[4 * g + 0]);
    const float v1 = __uint_as_float(s[4 * g + 1]);
    const float v2 = __uint_as_float(s[4 * g + 2]);
    const float v3 = __uint_as_float(s[4 * g + 3]);
    const float d01 = v0 - v1, d23 = v2 - v3;
    const float w01 = fmaxf(v0, v1), w23 = fmaxf(v2, v3);
    const float l01 = fminf(v0, v1), l23 = fminf(v2, v3);
    float lo = w01, hi = w23;
    const bool keep01 = l01 >= w23;
    const bool keep23 = l23 > w01;
    if (MODE != 5) {
      lo = keep01 ? v0 : (keep23 ? v2 : w01);
      hi = keep01 ? v1 : (keep23 ? v3 : w23);
    } else {
      lo = v0;
      hi = v1;
    }
    if (MODE == 0 || MODE == 1) {
      const uint32_t a = MODE == 0 ? sign_bit(d01, two) : __float_as_uint(d01) >> 31;
      const uint32_t b = MODE == 0 ? sign_bit(d23, two) : __float_as_uint(d23) >> 31;
      int nib = (int)(a + 4u * b);
      nib = keep23 ? 6 : nib;
      nib = keep01 ? -4 : nib;
      W += (uint32_t)nib * (1u << (4 * g));
    } else if (MODE == 2) {
      // nibble bits from sign bits: e1 < 0 <=> !keep01, e2 < 0 <=> keep23 (S holds no -0)
      const float e1 = l01 - w23, e2 = w01 - l23;
      const uint32_t t0 = lop_and_andn(d01, e1, e2);  // bit 0: a & !keep01 & !keep23
      const uint32_t t2 = lop_or_orn(d23, e1, e2);    // bit 2: b | keep01 | keep23
      W = shl_in(W, e1);                               // bit 3: !keep01
      W = shl_in(W, __uint_as_float(t2));
      W = shl_in(W, e2);                               // bit 1: keep23
      W = shl_in(W, __uint_as_float(t0));
    } else if (MODE >= 6 && MODE <= 9) {
      const uint32_t a = MODE == 7 ? __float_as_uint(d01) >> 31 : sign_bit(d01, two);
      const uint32_t b = MODE == 7 ? __float_as_uint(d23) >> 31 : sign_bit(d23, two);
      if (MODE == 6 || MODE == 7) {  // mixed nibble only (no keep SELs)
        W += (a + 4u * b) * (1u << (4 * g));
      } else if (MODE == 8) {  // keep SELs only
        int nib = keep23 ? 6 : 0;
        nib = keep01 ? -4 : nib;
        W += (uint32_t)nib * (1u << (4 * g));
        W ^= __float_as_uint(d01) ^ __float_as_uint(d23);
      } else {  // sign bits only
        W ^= a ^ b;
      }
    } else if (MODE == 10) {  // float flags (FMUL.SAT) + FSEL keep + FFMA accumulate
      const float fa = __saturatef(__fmul_rn(d01, -1.7014118e38f) * 1.7014118e38f);
      const float fb = __saturatef(__fmul_rn(d23, -1.7014118e38f) * 1.7014118e38f);
      float nf = fmaf(fb, 4.f, fa);
      nf = keep23 ? 6.f : nf;
      nf = keep01 ? -4.f : nf;
      W += __float_as_uint(nf);  // (placement not modelled: cost of the flags only)
    } else if (MODE == 13 || MODE == 14) {
      // a, b as exact 0 / 1 floats on the FMA-lite pipe: sat(d * -2^127 * 2^127) is 1 for every
      // d < 0 down to the smallest subnormal, 0 for d >= 0 (MODE 14: one multiply, subnormal-unsafe)
      const float fa = MODE == 13 ? __saturatef(__fmul_rn(d01, -1.7014118e38f) * 1.7014118e38f)
                                  : __saturatef(d01 * -1.7014118e38f);
      const float fb = MODE == 13 ? __saturatef(__fmul_rn(d23, -1.7014118e38f) * 1.7014118e38f)
                                  : __saturatef(d23 * -1.7014118e38f);
      float n = fmaf(fb, 4.f, fa);
      n = keep23 ? 6.f : n;
      n = keep01 ? -4.f : n;
      wf[g >> 2] = fmaf(n, (float)(1 << (4 * (g & 3))), wf[g >> 2]);
      if (g == 7) W = __byte_perm(__float_as_uint(wf[0]), __float_as_uint(wf[1]), 0x5410);
    } else if (MODE == 11 || MODE == 12) {  // float flags (FSET) and float nibble on the FMA-lite pipe
      const float fa = fset_gt(v1, v0), fb = fset_gt(v3, v2);
      const float m = fmaf(fb, 4.f, fa);
      float n;
      if (MODE == 11) {
        const float k01 = fset_ge(l01, w23), k23 = fset_gt(l23, w01);
        const float t = fmaf(-m, k01 + k23, m);
        n = fmaf(k01, -4.f, fmaf(k23, 6.f, t));
      } else {
        n = keep23 ? 6.f : m;
        n = keep01 ? -4.f : n;
      }
      wf[g >> 2] = fmaf(n, (float)(1 << (4 * (g & 3))), wf[g >> 2]);
      if (g == 7) W = __byte_perm(__float_as_uint(wf[0]), __float_as_uint(wf[1]), 0x5410);
    } else if (MODE == 3 || MODE == 5) {
      W ^= __float_as_uint(d01) ^ __float_as_uint(d23);  // nibble cost removed (keeps the FADDs alive)
    }
    float x0, x1;
    fma2s(lo, hi, c, -mlog, x0, x1);
    const float p0 = fex2(x0), p1 = fex2(x1);
    pk[g] = fpack2<T>(p0, p1);
    add2(lt0, lt1, p0, p1, lt0, lt1);
  }
}

template <int MODE, int NCH = 2>
__global__ void __launch_bounds__(512, 1) k(int iters, long long* cyc, float c, float mlog, uint32_t two) {
  extern __shared__ float4 sm[];  // [8 NCH float4][threads] S, then [2 NCH + 1 uint4][threads] outputs
  const int t = threadIdx.x, nt = blockDim.x;
  uint4* outs = reinterpret_cast<uint4*>(sm + 8 * NCH * nt);
  float l0 = 0.f, l1 = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    uint32_t pk[NCH][8], W[NCH];
    float lt0 = 0.f, lt1 = 0.f;
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
      uint32_t s[32];
      const int base = ((ch ^ (i & 1)) * 8) * nt + t;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float4 f = sm[base + j * nt];
        s[4 * j] = __float_as_uint(f.x); s[4 * j + 1] = __float_as_uint(f.y);
        s[4 * j + 2] = __float_as_uint(f.z); s[4 * j + 3] = __float_as_uint(f.w);
      }
      float a0, a1;
      prune<MODE>(s, c, mlog, two, pk[ch], W[ch], a0, a1);
      add2(lt0, lt1, a0, a1, lt0, lt1);
    }
    add2(l0, l1, lt0, lt1, l0, l1);
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
      outs[(ch * 2) * nt + t] = make_uint4(pk[ch][0], pk[ch][1], pk[ch][2], pk[ch][3]);
      outs[(ch * 2 + 1) * nt + t] = make_uint4(pk[ch][4], pk[ch][5], pk[ch][6], pk[ch][7]);
    }
    outs[2 * NCH * nt + t] = make_uint4(W[0], W[NCH - 1], __float_as_uint(l0), __float_as_uint(l1));
    __syncwarp();
  }
  long long t1 = clock64();
  if (t == 0) cyc[blockIdx.x] = t1 - t0;
}

// host check of MODE 2's metadata against MODE 0 on the same scores (ties included)
template <int MODE>
__global__ void meta_k(const float* s_in, uint32_t* w_out) {
  uint32_t s[32];
  for (int j = 0; j < 32; ++j) {
    const int jj = MODE == 15 ? (j & ~3) | ((j & 3) == 1 ? 2 : (j & 3) == 2 ? 1 : (j & 3)) : j;
    s[j] = __float_as_uint(s_in[threadIdx.x * 32 + jj]);
  }
  uint32_t pk[8], W;
  float a, b;
  prune<MODE>(s, 1.f, 0.f, 2u, pk, W, a, b);
  w_out[threadIdx.x] = W;
}

int main() {
  long long* cyc;
  long long h;
  cudaMalloc(&cyc, 148 * 8);
  const int smem = (16 + 5) * 512 * 16;
  float* hs = (float*)malloc(16 * 512 * 16);
  for (int i = 0; i < 16 * 512 * 4; ++i) hs[i] = (float)((i * 2654435761u >> 7) % 9) - 4.f;  // many ties
  const char* names[] = {"production (IMAD.HI sign bits, SEL nibble)", "SHF sign bits, SEL nibble",
                         "LOP3 + funnel-shift nibble", "no nibble", "-", "exp only (no select)",
                         "mixed nibble only (IMAD.HI)", "mixed nibble only (SHF)", "keep SELs only",
                         "sign bits only (IMAD.HI)", "float flags (FMUL.SAT) + FSEL", "FSET flags, float nibble (lite)",
                         "FSET a/b, FSEL keeps, float nibble", "FMUL.SAT a/b, FSEL keeps, float nibble",
                         "1-FMUL.SAT a/b (unsafe), FSEL keeps, fl. nib", "permuted regs: FADD2 + FMUL2 flags"};
  auto run = [&](auto kern, int mode) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 4096;
    kern<<<148, 512, smem>>>(iters, cyc, 0.18f, 0.5f, 2u);
    (void)mode;
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-46s %s %.0f cycles per warp-step (4 warps / SMSP)\n", names[mode], cudaGetErrorString(e), (double)h / iters);
  };
  {
    auto k4 = k<0, 4>;
    cudaFuncSetAttribute(k4, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k4<<<148, 256, smem>>>(4096, cyc, 0.18f, 0.5f, 2u);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-46s %s %.0f cycles per (2 warps x 4 chunks) / SMSP\n", "production, 8 warps x 4 chunks", cudaGetErrorString(e), (double)h / 4096);
    auto k8 = k<0, 8>;
    cudaFuncSetAttribute(k8, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k8<<<148, 128, smem>>>(4096, cyc, 0.18f, 0.5f, 2u);
    e = cudaDeviceSynchronize();
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-46s %s %.0f cycles per (1 warp x 8 chunks) / SMSP\n", "production, 4 warps x 8 chunks", cudaGetErrorString(e), (double)h / 4096);
  }
  run(k<0>, 0); run(k<1>, 1); run(k<2>, 2); run(k<3>, 3); run(k<5>, 5); run(k<6>, 6); run(k<7>, 7); run(k<8>, 8); run(k<9>, 9); run(k<10>, 10); run(k<11>, 11); run(k<12>, 12); run(k<13>, 13); run(k<14>, 14); run(k<15>, 15);
  // metadata equality of the funnel-shift form
  float* ds; uint32_t *w0, *w2;
  cudaMalloc(&ds, 512 * 32 * 4); cudaMalloc(&w0, 512 * 4); cudaMalloc(&w2, 512 * 4);
  cudaMemcpy(ds, hs, 512 * 32 * 4, cudaMemcpyHostToDevice);
  static uint32_t h0[512], h2[512];
  meta_k<0><<<1, 512>>>(ds, w0);
  cudaMemcpy(h0, w0, 2048, cudaMemcpyDeviceToHost);
  auto check = [&](auto kern, const char* what) {
    kern<<<1, 512>>>(ds, w2);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h2, w2, 2048, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < 512; ++i) bad += h0[i] != h2[i];
    printf("%s metadata == production on 512 tie-heavy rows: %s (%s, %d differ; e.g. %08x vs %08x)\n", what,
           bad ? "NO" : "yes", cudaGetErrorString(e), bad, h0[0], h2[0]);
  };
  check(meta_k<2>, "funnel-shift");
  check(meta_k<11>, "FSET float nibble");
  check(meta_k<12>, "FSET + FSEL float nibble");
  check(meta_k<13>, "FMUL.SAT float nibble");
  check(meta_k<15>, "permuted FADD2/FMUL2 float nibble");
  return 0;
}
