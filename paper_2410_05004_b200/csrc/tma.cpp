// tma.cpp -- TMA tensor-map encoding through the runtime's driver entry point
// (no link-time dependency on libcuda, so the library loads on GPU-less hosts).
#include <cuda.h>
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <tuple>

#include "kernels.h"

namespace hc {

namespace {
using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                 const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                 const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                 CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled get_encode() {
  static EncodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiled>(p);
  });
  return fn;
}
}  // namespace

bool make_tmap_kmajor(CUtensorMap* map, const void* base, uint64_t k, uint64_t rows,
                      uint64_t row_stride_bytes, uint32_t box_rows) {
  EncodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {k, rows};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_tmap_kmajor_cached(CUtensorMap* map, const void* base, uint64_t k, uint64_t rows,
                             uint64_t row_stride_bytes, uint32_t box_rows) {
  // a tensor map is a pure function of (address, shape, stride, box): maps of
  // reused buffers (staging-ring slots, pool allocations) are encoded once
  struct Key {
    const void* base;
    uint64_t k, rows, stride;
    uint32_t box;
    bool operator<(const Key& o) const {
      return std::tie(base, k, rows, stride, box) <
             std::tie(o.base, o.k, o.rows, o.stride, o.box);
    }
  };
  static std::mutex mu;
  static std::map<Key, CUtensorMap> cache;
  const Key key{base, k, rows, row_stride_bytes, box_rows};
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      *map = it->second;
      return true;
    }
  }
  if (!make_tmap_kmajor(map, base, k, rows, row_stride_bytes, box_rows)) return false;
  std::lock_guard<std::mutex> lk(mu);
  if (cache.size() >= 8192) cache.clear();  // bounded
  cache.emplace(key, *map);
  return true;
}

}  // namespace hc
