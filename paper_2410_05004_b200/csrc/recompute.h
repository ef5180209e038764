// recompute.h -- K6, the RECOMPUTE complement (internal).
#pragma once

#include <functional>

#include "common.h"
#include "weights.h"

namespace hc {

// prefill_layers (proj/src/model.cpp:349-356): embed d_tokens, run layers
// [lb, le) from position 0, writing each layer's K/V into the pages. With
// n_last in (0, n) the last layer runs only for the first n_last tokens.
// kv_only_last: the caller needs only the K/V of the last layer (a restore's
// RECOMPUTE prefix, whose next layer is restored from its stored input;
// prefill_layers), so that layer stops after its K/V projection.
// hook(layer, start) is called on the host around each layer's enqueue (for
// CUDA-event timelines). d_layer_inputs (optional, L x n x d bf16) receives
// each layer's input hidden state (prefill's layer_inputs, model.cpp:316).
void prefill_layers_impl(const hc_weights* w, const int32_t* d_tokens, int64_t n, int lb, int le,
                         const hc_kv_pages* pages, const int32_t* d_page_table,
                         cudaStream_t stream, const std::function<void(int, bool)>& hook,
                         void* d_layer_inputs = nullptr, int32_t* next_token = nullptr,
                         int64_t n_last = 0, bool kv_only_last = false);

// Sequences of a batched forward: nullptr cu = one sequence from position 0.
struct SeqBatch {
  int n_seqs = 1;
  const int32_t* cu = nullptr;         // device [n_seqs + 1] row offsets
  const int32_t* seq_start = nullptr;  // device [n_seqs] first positions
  int max_new = 0;
  int table_stride = 0;
  bool from_zero = false;  // every sequence starts at position 0 (a ragged prefill)
};

// forward_tokens / decode_step (model.cpp:305-347) for a batch of sequences
// continuing their paged caches: sequence s appends new_lens[s] tokens at
// positions start_pos[s].. (host arrays). d_next_tokens[s] = greedy token
// after the sequence's last row.
void forward_batch(const hc_weights* w, const int32_t* d_tokens, int n_seqs,
                   const int32_t* new_lens, const int32_t* start_pos, const hc_kv_pages* pages,
                   const int32_t* d_page_tables, int table_stride, void* d_layer_inputs,
                   int32_t* d_next_tokens, cudaStream_t stream);

// The same with the sequence metadata already on the device (d_cu [n_seqs+1]
// row offsets, d_starts [n_seqs] first positions; positions validated by the
// caller): no host->device traffic, so a decode step can be captured into a
// CUDA graph.
void forward_batch_dev(const hc_weights* w, const int32_t* d_tokens, int n_seqs, int64_t total,
                       int max_new, const int32_t* d_cu, const int32_t* d_starts,
                       const hc_kv_pages* pages, const int32_t* d_page_tables, int table_stride,
                       void* d_layer_inputs, int32_t* d_next_tokens, cudaStream_t stream);

// Layers [lb, le) of forward_batch_dev (the RECOMPUTE prefix of a batched
// restore: every sequence from position 0); hook as in prefill_layers_impl.
void forward_batch_layers(const hc_weights* w, const int32_t* d_tokens, int n_seqs, int64_t total,
                          int max_new, const int32_t* d_cu, const int32_t* d_starts,
                          const hc_kv_pages* pages, const int32_t* d_page_tables,
                          int table_stride, int lb, int le, cudaStream_t stream,
                          const std::function<void(int, bool)>& hook, bool kv_only_last = false);

// Measured seconds of one recompute layer over n tokens at the steady-state
// clock (after warm_s seconds of back-to-back layers); 0 when the full block
// weights are not set.
double recompute_layer_seconds(const hc_weights* w, int n, double warm_s = 0.2);

}  // namespace hc
