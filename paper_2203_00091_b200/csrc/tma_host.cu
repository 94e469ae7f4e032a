// tma_host.cu -- host-side TMA descriptor encoding via the runtime's driver entry point.
#include <cudaTypedefs.h>

#include <atomic>

#include "tc_common.cuh"

namespace dfss {

// ---------------------------------------------------------------- per-device attribute cache
// The C entry points run on microsecond configs (c1: ~30 us), so the per-call host work is
// kept to a cudaGetDevice: SM count and compute capability are queried once per device.
namespace {
constexpr int kMaxDev = 64;
std::atomic<int> g_sms[kMaxDev];   // 0 = not queried yet
std::atomic<int> g_cc[kMaxDev];    // major * 10 + minor + 1 (0 = not queried)
}  // namespace

int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}

int device_sms(int dev) {
  if (dev < 0 || dev >= kMaxDev) return 148;
  int v = g_sms[dev].load(std::memory_order_relaxed);
  if (!v) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    g_sms[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}

int device_cc(int dev) {
  if (dev < 0 || dev >= kMaxDev) return 0;
  int v = g_cc[dev].load(std::memory_order_relaxed);
  if (!v) {
    int major = 0, minor = 0;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess)
      return 0;  // not cached: the caller reports "no device"
    v = major * 10 + minor + 1;
    g_cc[dev].store(v, std::memory_order_relaxed);
  }
  return v - 1;
}

cudaError_t set_max_smem_once(const void* kernel, std::atomic<uint64_t>& done, int dev) {
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  // the largest opt-in size once: the persistent kernels run one CTA per SM whatever they use
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

// 3-D tiled map over a dense row-major [d2][d1][d0] tensor; box {box0, box1, 1}.
bool encode_tmap_3d(CUtensorMap* map, CUtensorMapDataType dtype, int elem_bytes, void* base, uint64_t d0, uint64_t d1,
                    uint64_t d2, uint32_t box0, uint32_t box1, CUtensorMapSwizzle swz) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {d0 * (uint64_t)elem_bytes, d0 * d1 * (uint64_t)elem_bytes};
  cuuint32_t box[3] = {box0, box1, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, dtype, 3, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// General tiled map: rank <= 5, dims innermost first, strides_bytes[i] = stride of dim i+1
// (any order: a permuted row order inside a box is expressed by non-monotonic strides).
bool encode_tmap(CUtensorMap* map, CUtensorMapDataType dtype, int rank, void* base, const uint64_t* dims,
                 const uint64_t* strides_bytes, const uint32_t* box, CUtensorMapSwizzle swz) {
  auto fn = encode_fn();
  if (!fn || rank < 1 || rank > 5) return false;
  cuuint64_t d[5], st[4];
  cuuint32_t b[5], e[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    e[i] = 1;
    if (i + 1 < rank) st[i] = strides_bytes[i];
  }
  CUresult r = fn(map, dtype, rank, base, d, st, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace dfss
