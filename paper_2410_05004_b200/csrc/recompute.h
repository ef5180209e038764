// recompute.h -- K6, the RECOMPUTE complement (internal).
#pragma once

#include <functional>

#include "common.h"
#include "weights.h"

namespace hc {

// prefill_layers (proj/src/model.cpp:349-356): embed d_tokens, run layers
// [lb, le) from position 0, writing each layer's K/V into the pages.
// hook(layer, start) is called on the host around each layer's enqueue (for
// CUDA-event timelines). d_layer_inputs (optional, L x n x d bf16) receives
// each layer's input hidden state (prefill's layer_inputs, model.cpp:316).
void prefill_layers_impl(const hc_weights* w, const int32_t* d_tokens, int64_t n, int lb, int le,
                         const hc_kv_pages* pages, const int32_t* d_page_table,
                         cudaStream_t stream, const std::function<void(int, bool)>& hook,
                         void* d_layer_inputs = nullptr, int32_t* next_token = nullptr);

// Measured seconds of one recompute layer over n tokens (0 when the full
// block weights are not set).
double recompute_layer_seconds(const hc_weights* w, int n);

}  // namespace hc
