// flash_common.cuh -- device helpers shared by the fused DFSS kernels (flash_tc.cu: 16-bit,
// flash_tf32.cu: tf32): packed fp32 math (FADD2/FFMA2), exp2, 16-bit packing, the quad/pair
// barrier reduction, role-warp waits, and the BlockMask tile test.
#pragma once

#include <type_traits>

#include "dfss_common.cuh"
#include "tc_common.cuh"

namespace dfss {

// ---------------------------------------------------------------- packed fp32 helpers (sm_100 FADD2/FFMA2)
__device__ __forceinline__ void sub2(float a0, float a1, float b0, float b1, float& d0, float& d1) {
  asm("{\n\t.reg .b64 a, b, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
      "sub.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
__device__ __forceinline__ void add2(float a0, float a1, float b0, float b1, float& d0, float& d1) {
  asm("{\n\t.reg .b64 a, b, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
      "add.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
// (a0, a1) * c + (b, b)
__device__ __forceinline__ void fma2s(float a0, float a1, float c, float b, float& d0, float& d1) {
  asm("{\n\t.reg .b64 a, cc, bb, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 cc, {%4, %4};\n\tmov.b64 bb, {%5, %5};\n\t"
      "fma.rn.f32x2 d, a, cc, bb;\n\tmov.b64 {%0, %1}, d;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(c), "f"(b));
}

// (a0, a1) * c + (b0, b1)
__device__ __forceinline__ void fma2v(float a0, float a1, float c, float b0, float b1, float& d0, float& d1) {
  asm("{\n\t.reg .b64 a, cc, bb, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 cc, {%4, %4};\n\tmov.b64 bb, {%5, %6};\n\t"
      "fma.rn.f32x2 d, a, cc, bb;\n\tmov.b64 {%0, %1}, d;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(c), "f"(b0), "f"(b1));
}
// (a0, a1) * c
__device__ __forceinline__ void mul2s(float a0, float a1, float c, float& d0, float& d1) {
  asm("{\n\t.reg .b64 a, cc, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 cc, {%4, %4};\n\t"
      "mul.rn.f32x2 d, a, cc;\n\tmov.b64 {%0, %1}, d;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(c));
}

__device__ __forceinline__ float fex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <typename T>
__device__ __forceinline__ uint32_t fpack2(float lo, float hi) {
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    __nv_bfloat162 p = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&p);
  } else {
    __half2 p = __floats2half2_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&p);
  }
}

// bar.red.or over `count` threads of named barrier `id`: true iff any thread passed true
__device__ __forceinline__ bool bar_any(uint32_t id, uint32_t count, bool pred) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\tsetp.ne.u32 p, %1, 0;\n\tbar.red.or.pred q, %2, %3, p;\n\tselp.u32 %0, 1, 0, q;\n\t}"
      : "=r"(r)
      : "r"((uint32_t)pred), "r"(id), "r"(count)
      : "memory");
  return r != 0;
}

// role-warp wait: try_wait with a suspend-time hint (the waiting warp yields its issue slots)
#ifdef DFSS_EXP_ROLE_SPIN  // timing experiment: role warps spin on try_wait without a suspend hint
__device__ __forceinline__ void wait_role(uint64_t* bar, uint32_t parity) { tc::mbar_wait(bar, parity); }
#elif defined(DFSS_EXP_ROLE_BACKOFF)  // timing experiment: test_wait + fixed nanosleep
__device__ __forceinline__ void wait_role(uint64_t* bar, uint32_t parity) {
  if (tc::mbar_test(bar, parity)) return;
  tc::mbar_wait_backoff(bar, parity, DFSS_EXP_ROLE_BACKOFF);
}
#else
__device__ __forceinline__ void wait_role(uint64_t* bar, uint32_t parity) { tc::mbar_wait_sleep(bar, parity); }
#endif

// Parity dump of the fused kernels (DUMP instantiations only, dfss_nm_attention_dump): the
// post-scale fp32 scores every prune compared, [bh, n, n] in true key order, and the metadata
// words handed to tcgen05.mma.sp, in the meta_hw layout of include/dfss.h.
struct FlashDump {
  float* s = nullptr;
  uint32_t* meta = nullptr;
};

// one 32-column chunk of one row, times the exact power-of-two scale 1/sqrt(64), in key order.
// PERMUTED: registers hold each group of 4 in (k0, k2, k1, k3) order (the tf32 kernel's
// permuted K tensor map); otherwise in key order (the 16-bit kernels).
template <bool PERMUTED>
__device__ __forceinline__ void dump_chunk_scores(float* dst, const uint32_t (&s)[32], float scale) {
  float4* d4 = reinterpret_cast<float4*>(dst);
  constexpr int i1 = PERMUTED ? 2 : 1, i2 = PERMUTED ? 1 : 2;
#pragma unroll
  for (int g = 0; g < 8; ++g)
    d4[g] = make_float4(__uint_as_float(s[4 * g]) * scale, __uint_as_float(s[4 * g + i1]) * scale,
                        __uint_as_float(s[4 * g + i2]) * scale, __uint_as_float(s[4 * g + 3]) * scale);
}

// Register budget of the warp-specialised fused kernels (640 threads = 96 registers each at
// launch): the role warpgroup (warps 16-19: TMA, MMA issuers) drops to 32 registers and the
// four softmax warpgroups take the freed 8192 -- 112 each -- so the prune / exp epilogue
// keeps two 32-column chunks in flight without spilling.  Warpgroup-uniform, and the two
// branches must not re-join (ptxas needs one register budget per code region): each one
// finishes the CTA itself.
__device__ __forceinline__ void regs_role() { asm volatile("setmaxnreg.dec.sync.aligned.u32 32;\n" ::: "memory"); }
__device__ __forceinline__ void regs_softmax() { asm volatile("setmaxnreg.inc.sync.aligned.u32 112;\n" ::: "memory"); }

__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

// Optional tile-grid keep mask (BlockMask, codec.py:150-200): keep[i * grid_cols + j] covers
// rows [i*tile_rows, +tile_rows) and key columns [j*tile_cols, +tile_cols), shared by every
// (batch, head).  The fused kernels need tile_rows and tile_cols to be multiples of 32, so a
// warp's 32 rows x 32 columns chunk lies in one tile: masked chunks are skipped warp-uniformly
// (no prune / exp work, zero P), i.e. masked tiles are structurally absent as in the reference.
struct TileMask {
  const uint8_t* keep;
  int tile_rows, tile_cols, grid_cols;
  // bitmaps derived from keep by mask_bits_kernel (flash_tc.cu), in the fused kernels' workspace:
  // sbits [n/128 row blocks][sbw words], bit t = any kept tile in the 128 x 128 step (rows, t);
  // cbits [n/32 row strips][cbw words], bit c = 32 x 32 chunk (strip, c) kept
  const uint32_t* sbits = nullptr;
  const uint32_t* cbits = nullptr;
  const int* order = nullptr;  // [n/256] row blocks by live steps, heaviest first (two-set schedule)
  int sbw = 0, cbw = 0;
  __device__ __forceinline__ bool masked(int row, int col) const {
    return keep != nullptr && __ldg(keep + (row / tile_rows) * grid_cols + col / tile_cols) == 0;
  }
  // any kept tile in rows [row0, row0 + rows) x columns [col0, col0 + cols)?
  __device__ __forceinline__ bool region_live(int row0, int rows, int col0, int cols) const {
    if (keep == nullptr) return true;
    for (int i = row0 / tile_rows; i <= (row0 + rows - 1) / tile_rows; ++i)
      for (int j = col0 / tile_cols; j <= (col0 + cols - 1) / tile_cols; ++j)
        if (__ldg(keep + i * grid_cols + j)) return true;
    return false;
  }
};

// masked chunk: no kept values, P = 0, nibble 0x4 in every group (W = 0x44444444)
__device__ __forceinline__ void masked_chunk(uint32_t (&pk)[8], uint32_t& W, float& lt0, float& lt1) {
#pragma unroll
  for (int j = 0; j < 8; ++j) pk[j] = 0u;
  W = 0x44444444u;
  lt0 = lt1 = 0.f;
}

}  // namespace dfss
