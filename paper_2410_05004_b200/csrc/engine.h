// engine.h -- the restore engine's per-device streams, event and timeline
// helpers (internal; defined in restore.cpp, shared with sharded.cpp).
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "common.h"
#include "store.h"

namespace hc {

// Per-device engine state: the IO lane's copy streams (a layer's gather is
// split over kCopyStreams so several copy engines share the PCIe link) and a
// memory pool that keeps the staging ring cached across restores.
constexpr int kCopyStreams = 4;
struct Engine {
  cudaStream_t copy = nullptr;  // IO lane head: orders fetches, joins the helpers
  cudaStream_t helper[kCopyStreams - 1] = {};
  cudaStream_t aux = nullptr;   // row statistics running ahead of the compute lane
  cudaStream_t aux2 = nullptr;  // second K1 lane of a resident restore
  bool init = false;
};
Engine& engine(int dev);

struct TimedOp {
  int lane, layer, kind;
  cudaEvent_t start, end;
};

// Lazily created CUDA events, destroyed with the object.
struct EventPool {
  std::vector<cudaEvent_t> all;
  bool timing;
  explicit EventPool(bool t) : timing(t) {}
  cudaEvent_t get() {
    cudaEvent_t e;
    HC_CUDA(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming));
    all.push_back(e);
    return e;
  }
  ~EventPool() {
    for (auto e : all) cudaEventDestroy(e);
  }
  EventPool(const EventPool&) = delete;
  EventPool& operator=(const EventPool&) = delete;
  static cudaEvent_t make(void* self) {
    EventPool* p = static_cast<EventPool*>(self);
    cudaEvent_t e;
    HC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    p->all.push_back(e);
    return e;
  }
};

// Gather on the IO lane: the head stream forks to the helper streams and
// joins them again, so the lane stays one ordered sequence of layer fetches.
void issue_gather(const std::vector<CopySeg>& segs, uint8_t* dst, Engine& eng,
                  std::vector<cudaEvent_t>& scratch_events, cudaEvent_t (*make)(void*), void* ctx);
void fill_timeline(hc_timeline* tl, cudaEvent_t t0, const std::vector<TimedOp>& ops);

struct LayerJob {
  int layer;
  int method;
};
// restore.cpp:50-63: recompute prefix, hidden, KV suffix
std::vector<LayerJob> compute_order(const hc_plan& p);
// staged hidden layers beyond the one in use (prefetch_depth 0 = auto)
int auto_depth(int n_staged, size_t buf_bytes, int requested);
// K1 launches alternating two streams (2) or one (1) for `rows` rows
int k1_lanes(int64_t rows);

}  // namespace hc
