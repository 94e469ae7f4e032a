// tf32_probe.cu -- bring-up check of the tf32 operand layouts used by flash_tf32.cu:
// (a) dense kind::tf32 D[128x128] = A[128x64] B[128x64]^T with K split in two 128B-swizzle atoms;
// (b) sparse kind::tf32 D[128x64] = P_sparse[128x16 (8 kept/row)] V[16x64], A and metadata in TMEM,
//     V MN-major in two 32-column atoms.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>
#include "tc_common.cuh"
using namespace dfss;

// 128B swizzle: within each 1024-byte block (8 rows of 128 B), 16-byte unit u of row r goes to u ^ (r & 7)
__device__ __forceinline__ int swz(int row, int byte_in_row) {
  return row * 128 + ((((byte_in_row >> 4) ^ (row & 7)) << 4) | (byte_in_row & 15));
}

__global__ void probe(const float* A, const float* B, const float* P, const uint8_t* nib, const float* V, float* D1,
                      float* D2, int mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* sa = smem;            // A: 2 atoms x 16 KB
  uint8_t* sb = smem + 32768;    // B: 2 atoms
  uint8_t* sv = smem + 65536;    // V: 16 keys x 64 dims, 2 atoms along dims, 16 rows each (2 KB each, 1024-aligned)
  for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) {
    const int r = i / 64, c = i % 64, atom = c / 32, cc = c % 32;
    *(float*)(sa + atom * 16384 + swz(r, cc * 4)) = A[i];
    *(float*)(sb + atom * 16384 + swz(r, cc * 4)) = B[i];
  }
  for (int i = threadIdx.x; i < 16 * 64; i += blockDim.x) {
    const int r = i / 64, c = i % 64, atom = c / 32, cc = c % 32;
    *(float*)(sv + atom * 2048 + swz(r, cc * 4)) = V[i];
  }
  for (int i = threadIdx.x; i < 16 * 64; i += blockDim.x) {  // V^T K-major (rows = dims, 128 B = 32 keys), modes 3/4
    const int key = i / 64, dim = i % 64;
    *(float*)(smem + 92160 + swz(dim, key * 4)) = V[i];
  }
  for (int i = threadIdx.x; i < 128 * 8; i += blockDim.x) {  // compressed A in smem (mode 1)
    const int r = i / 8, c = i % 8;
    *(float*)(smem + 73728 + swz(r, c * 4)) = P[i];
  }
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_barrier_init(); }
  if (warp == 0) tc::tmem_alloc<512>(&slot);
  tc::fence_proxy_async();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tm = slot;
  // A_sparse (8 fp32 / row) at columns 256..263, metadata word at column 272
  if (warp < 4) {
    const int r = warp * 32 + lane;
    uint32_t pv[8];
    for (int j = 0; j < 8; ++j) pv[j] = __float_as_uint(P[r * 8 + j]);
    const uint32_t lb = tm + ((uint32_t)(warp * 32) << 16);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(lb + 256), "r"(pv[0]),
                 "r"(pv[1]), "r"(pv[2]), "r"(pv[3]), "r"(pv[4]), "r"(pv[5]), "r"(pv[6]), "r"(pv[7]));
    // word of lane L: pairs 4k1..4k1+3 of rows r0 = 16 m2 + m0 (bits 0-15) and r0 + 8 (bits 16-31)
    const int L = r, m2 = L >> 4, k1 = (L >> 3) & 1, m0 = L & 7;
    const int r0 = 16 * m2 + m0, r1 = r0 + 8;
    uint32_t w = 0;
    for (int i = 0; i < 4; ++i) {
      w |= (uint32_t)nib[r0 * 8 + 4 * k1 + i] << (4 * i);
      w |= (uint32_t)nib[r1 * 8 + 4 * k1 + i] << (16 + 4 * i);
    }
    tc::tmem_st_32x32b_x1(lb + 272, w);
    tc::tmem_st_wait();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc_s = tc::instr_desc(2, 128, 128, false, false, false);
    for (int kk = 0; kk < 8; ++kk) {
      const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
      const uint64_t ad = tc::smem_desc(tc::smem_u32(sa) + off, 16, 1024, tc::kSwizzle128B);
      const uint64_t bd = tc::smem_desc(tc::smem_u32(sb) + off, 16, 1024, tc::kSwizzle128B);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
                   "l"(ad), "l"(bd), "r"(idesc_s), "r"((uint32_t)(kk > 0)));
    }
    constexpr uint32_t idesc_pv = tc::instr_desc(2, 128, 64, false, true, true);
    const uint64_t vd = tc::smem_desc(tc::smem_u32(sv), 2048, 1024, tc::kSwizzle128B);
    if (mode == 0) {
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 1;\n\ttcgen05.mma.sp.cta_group::1.kind::tf32 [%0], [%1], %2, [%3], %4, p;\n\t}" ::"r"(tm + 384),
                   "r"(tm + 256), "l"(vd), "r"(tm + 272), "r"(idesc_pv));
    } else if (mode == 1) {  // A compressed in smem: rows of 128 B (first 8 fp32 used), 128B swizzle
      const uint64_t ad = tc::smem_desc(tc::smem_u32(smem + 73728), 16, 1024, tc::kSwizzle128B);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 1;\n\ttcgen05.mma.sp.cta_group::1.kind::tf32 [%0], %1, %2, [%3], %4, p;\n\t}" ::"r"(tm + 384),
                   "l"(ad), "l"(vd), "r"(tm + 272), "r"(idesc_pv));
    } else if (mode >= 3) {  // B = V^T K-major (64 dims x keys, 128B rows, swizzled)
      const uint64_t vkd = tc::smem_desc(tc::smem_u32(smem + 92160), 16, 1024, tc::kSwizzle128B);
      if (mode == 3) {
        constexpr uint32_t idesc_d = tc::instr_desc(2, 128, 64, false, false, false);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 1;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm + 384),
                     "r"(tm + 256), "l"(vkd), "r"(idesc_d));
      } else if (mode == 4) {
        constexpr uint32_t idesc_k = tc::instr_desc(2, 128, 64, false, false, true);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 1;\n\ttcgen05.mma.sp.cta_group::1.kind::tf32 [%0], [%1], %2, [%3], %4, p;\n\t}" ::"r"(tm + 384),
                     "r"(tm + 256), "l"(vkd), "r"(tm + 272), "r"(idesc_k));
      } else {  // mode 5: sparse SS, compressed A in smem, B K-major
        constexpr uint32_t idesc_k = tc::instr_desc(2, 128, 64, false, false, true);
        const uint64_t ad = tc::smem_desc(tc::smem_u32(smem + 73728), 16, 1024, tc::kSwizzle128B);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 1;\n\ttcgen05.mma.sp.cta_group::1.kind::tf32 [%0], %1, %2, [%3], %4, p;\n\t}" ::"r"(tm + 384),
                     "l"(ad), "l"(vkd), "r"(tm + 272), "r"(idesc_k));
      }
    } else {  // dense TS, K = 8: D = A8 (TMEM cols 256..263) x V[0:8]
      constexpr uint32_t idesc_d = tc::instr_desc(2, 128, 64, false, true, false);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 1;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm + 384),
                   "r"(tm + 256), "l"(vd), "r"(idesc_d));
    }
    tc::mma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::tc_fence_after();
  if (warp < 4) {
    const int r = warp * 32 + lane;
    const uint32_t lb = tm + ((uint32_t)(warp * 32) << 16);
    for (int c0 = 0; c0 < 128; c0 += 32) {
      uint32_t v[32];
      tc::tmem_ld_32x32b_x32(lb + c0, v);
      tc::tmem_ld_wait(v);
      for (int j = 0; j < 32; ++j) D1[r * 128 + c0 + j] = __uint_as_float(v[j]);
    }
    for (int c0 = 0; c0 < 64; c0 += 32) {
      uint32_t v[32];
      tc::tmem_ld_32x32b_x32(lb + 384 + c0, v);
      tc::tmem_ld_wait(v);
      for (int j = 0; j < 32; ++j) D2[r * 64 + c0 + j] = __uint_as_float(v[j]);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tm);
}

static float tf32r(float x) {  // round to a 10-bit mantissa (what the MMA sees; truncation vs rne both fine for the check)
  uint32_t u; memcpy(&u, &x, 4); u &= 0xFFFFE000u; float y; memcpy(&y, &u, 4); return y;
}

int main(int argc, char** argv) {
  const int pat = argc > 1 ? atoi(argv[1]) : 0;
  const int M = 128, N = 128, K = 64;
  float *A, *B, *P, *V, *D1, *D2; uint8_t* nib;
  cudaMallocManaged(&A, M * K * 4); cudaMallocManaged(&B, N * K * 4); cudaMallocManaged(&P, M * 8 * 4);
  cudaMallocManaged(&V, 16 * 64 * 4); cudaMallocManaged(&D1, M * N * 4); cudaMallocManaged(&D2, M * 64 * 4);
  cudaMallocManaged(&nib, M * 8);
  srand(1);
  for (int i = 0; i < M * K; ++i) A[i] = (rand() % 17 - 8) / 8.0f;
  for (int i = 0; i < N * K; ++i) B[i] = (rand() % 17 - 8) / 8.0f;
  for (int i = 0; i < M * 8; ++i) {
    P[i] = (pat >= 4) ? ((i % 8) == ((i / 8) % 8) ? 1.0f : 0.0f) : (rand() % 9) / 4.0f;
    const int rb = rand() & 1;
    nib[i] = (pat == 1 || pat == 4) ? 0x4 : (pat == 2 || pat == 5) ? 0xE : pat == 3 ? ((i & 1) ? 0xE : 0x4) : (rb ? 0xE : 0x4);
  }
  for (int i = 0; i < 16 * 64; ++i) V[i] = (rand() % 1023 - 511) / 64.0f;
  for (int mode = 0; mode < 6; ++mode) {
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024);
    probe<<<1, 128, 112 * 1024>>>(A, B, P, nib, V, D1, D2, mode);
    cudaError_t e = cudaDeviceSynchronize();
    if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    double e1 = 0, e2 = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double s = 0;
        for (int k = 0; k < K; ++k) s += (double)A[m * K + k] * B[n * K + k];
        e1 = fmax(e1, fabs(s - D1[m * N + n]));
      }
    for (int m = 0; m < M; ++m)
      for (int d = 0; d < 64; ++d) {
        double s = 0;
        for (int j = 0; j < 8; ++j) {  // pair j = keys 2j, 2j+1; kept key by nibble
          const int key = (mode == 2 || mode == 3) ? j : 2 * j + (nib[m * 8 + j] == 0xE ? 1 : 0);
          s += (double)P[m * 8 + j] * V[key * 64 + d];
        }
        e2 = fmax(e2, fabs(s - D2[m * 64 + d]));
      }
    if (pat >= 4 && mode >= 4) {
      char fn[64];
      snprintf(fn, sizeof fn, "gpurun_out/tf32probe_p%d_m%d.bin", pat, mode);
      FILE* f = fopen(fn, "wb");
      fwrite(D2, 4, M * 64, f); fwrite(V, 4, 16 * 64, f); fwrite(P, 4, M * 8, f); fwrite(nib, 1, M * 8, f);
      fclose(f);
    }
    if (pat >= 4 && (mode == 4 || mode == 5)) {
      // one-hot P: row m keeps stored element j = m % 8 -> D2 row = V[key] for the key the MMA used
      for (int m = 0; m < 16; ++m) {
        int found = -1;
        for (int key = 0; key < 16 && found < 0; ++key) {
          bool eq = true;
          for (int d = 0; d < 64; ++d) eq &= fabs(D2[m * 64 + d] - V[key * 64 + d]) < 1e-6;
          if (eq) found = key;
        }
        printf("  mode %d row %2d stored elem %d nib 0x%x -> key %d (D2[m][0]=%g)\n", mode, m, m % 8, nib[m * 8 + m % 8], found,
               D2[m * 64]);
      }
    }
    const char* names[] = {"sparse TS (A tmem)", "sparse SS (A smem)", "dense TS K=8", "dense TS K=8 B K-maj",
                           "sparse TS B K-major", "sparse SS B K-major"};
    printf("%-20s: dense tf32 S max err %g | PV max err %g  (D2[0]=%g)\n", names[mode], e1, e2, D2[0]);
  }
  return 0;
}
