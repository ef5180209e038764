// common.h -- internal error plumbing and device helpers for the C ABI.
#pragma once

#include <exception>
#include <initializer_list>

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3 (no-op unless a profiler injects)

#include <atomic>
#include <cstdint>

#include <stdexcept>
#include <string>

#include "../../include/hcache_b200.h"

namespace hc {

// Internal exception carrying an hc_status; converted at the C boundary.
struct Error : std::runtime_error {
  hc_status status;
  Error(hc_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] inline void fail(hc_status s, const std::string& m) { throw Error(s, m); }

inline void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(HC_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define HC_CUDA(call) ::hc::check_cuda((call), #call)

void set_last_error(const std::string& m);
void clear_last_error();

// NVTX range over a public entry point (host enqueue span in nsys / ncu
// timelines; the device-side lanes are in the CUDA-event Timeline).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// Runs fn, mapping exceptions to hc_status + hc_last_error().
template <typename F>
hc_status guard(F&& fn) {
  try {
    clear_last_error();
    fn();
    return HC_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.status;
  } catch (const std::invalid_argument& e) {
    set_last_error(e.what());
    return HC_EINVAL;
  } catch (const std::bad_alloc&) {
    set_last_error("out of memory");
    return HC_ENOMEM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return HC_ERUNTIME;
  } catch (...) {
    set_last_error("unknown error");
    return HC_ERUNTIME;
  }
}

// Scoped cudaSetDevice.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    HC_CUDA(cudaGetDevice(&prev));
    if (prev != dev) HC_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != prev && prev >= 0) cudaSetDevice(prev);
  }
};

// Per-device properties cached once (SM count for persistent grids).
int device_sm_count(int dev);
// Fails loudly unless `dev` is an sm_100-class GPU (no CPU fallback).
void require_sm100(int dev);

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// Stream-ordered scratch (cudaMallocAsync pool), released on the same stream.
// The current device's stream-ordered pool keeps freed memory (release
// threshold = max) so per-call scratch -- e.g. a 32 MB mean-shift buffer per
// projection -- is recycled instead of being unmapped and remapped at every
// synchronisation (that doubled a back-to-back K1 loop). Once per device.
inline void retain_pool_once() {
  static std::atomic<uint64_t> done{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
  if (done.load(std::memory_order_relaxed) & (1ull << dev)) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thresh = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thresh);
  }
  done.fetch_or(1ull << dev);
}

struct StreamScratch {
  void* ptr = nullptr;
  cudaStream_t stream = nullptr;
  StreamScratch(size_t bytes, cudaStream_t s) : stream(s) {
    if (bytes) {
      retain_pool_once();
      HC_CUDA(cudaMallocAsync(&ptr, bytes, s));
    }
  }
  ~StreamScratch() {
    if (ptr) cudaFreeAsync(ptr, stream);
  }
  StreamScratch(const StreamScratch&) = delete;
  StreamScratch& operator=(const StreamScratch&) = delete;
};

// Error-path guard: when the scope unwinds by an exception, makes `stream`
// wait for everything already queued on the side lanes, so stream-ordered
// frees of scratch buffers on `stream` cannot overtake copies or kernels
// still using them. A no-op on normal exit (the code joins explicitly).
struct LaneJoin {
  cudaStream_t stream;
  cudaStream_t lanes[4] = {nullptr, nullptr, nullptr, nullptr};
  int entered;
  LaneJoin(cudaStream_t s, std::initializer_list<cudaStream_t> ls)
      : stream(s), entered(std::uncaught_exceptions()) {
    int i = 0;
    for (cudaStream_t l : ls)
      if (i < 4) lanes[i++] = l;
  }
  ~LaneJoin() {
    if (std::uncaught_exceptions() <= entered) return;
    for (cudaStream_t l : lanes) {
      if (!l || l == stream) continue;
      cudaEvent_t e;
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) continue;
      if (cudaEventRecord(e, l) == cudaSuccess) cudaStreamWaitEvent(stream, e, 0);
      cudaEventDestroy(e);
    }
  }
  LaneJoin(const LaneJoin&) = delete;
  LaneJoin& operator=(const LaneJoin&) = delete;
};

}  // namespace hc
