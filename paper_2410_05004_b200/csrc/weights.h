// weights.h -- the device-resident weight set behind hc_weights (internal).
#pragma once

#include <cuda.h>

#include <vector>

#include "common.h"
#include "kernels.h"

struct hc_weights {
  hc_model_config cfg{};
  int device = 0;
  int head_begin = 0;
  int head_count = 0;
  int d_head = 0;
  int d_kv = 0;     // local KV row width = head_count * d_head
  int d_kv_all = 0; // n_kv_heads * d_head

  struct Layer {
    const void* wkv = nullptr;   // [2*d_kv x d] bf16, K rows then V rows (local heads)
    float* colsum = nullptr;     // owned, [2*d_kv]
    CUtensorMap tm256{}, tm128{};
    bool ready = false;
    // full block (RECOMPUTE path), all heads
    const void* wq = nullptr;
    const void* wkv_all = nullptr;
    const void* wo = nullptr;
    const void* fc1 = nullptr;
    const void* fc2 = nullptr;
    float* colsum_all = nullptr;  // owned, colsum of wkv_all (2*d_kv_all)
    float* colsum_q = nullptr;    // owned, colsum of wq (d)
    float* colsum_fc1 = nullptr;  // owned, colsum of fc1 (d_ffn)
    // W_q immediately followed by [W_k;W_v] in the caller's memory: the Q, K
    // and V projections of a recompute layer run as one GEMM over this
    // [(d + 2*d_kv_all) x d] operand (nullptr: two GEMMs)
    const void* wqkv = nullptr;
    float* colsum_qkv = nullptr;  // owned, [colsum_q ; colsum_all] when wqkv is set
    bool full = false;
  };
  std::vector<Layer> layers;
  const void* embedding = nullptr;
  float2* rope = nullptr;  // owned, [rope_rows][d_head/2]
  int rope_rows = 0;
};

namespace hc {

// The epilogue arguments for a layer (LN fold + RoPE), given row stats.
EpiArgs epi_for(const hc_weights* w, const float* colsum, const float* mean, const float* rstd);

// Runs K1 for rows [0, n_rows) of a K-major bf16 hidden matrix (row stride
// d_hidden) of `layer` into `out`. Computes the row statistics itself.
// With `stats` (mean[n_rows] then rstd[n_rows], from launch_row_stats) the
// row-statistics launch is skipped; `flag` (from launch_row_stats_flagged)
// then enables the mean-shifted operand (the means may be adjusted in place).
// Without them the statistics and the flag are computed here.
// With `centered` as well, the caller has already run launch_center_rows into
// it (n_rows x d_hidden bf16) and K1 only reads it when the flag is set.
void project_rows(const hc_weights* w, int layer, const void* d_hidden, int64_t n_rows,
                  const KvOut& out, cudaStream_t stream, const float* stats = nullptr,
                  const int32_t* flag = nullptr, const void* centered = nullptr);

// KvOut for a layer of a paged cache.
KvOut kv_out_pages(const hc_kv_pages* pages, int layer, const int32_t* page_table,
                   int table_stride, const int32_t* cu_seqlens, int n_seqs);

void validate_pages(const hc_weights* w, const hc_kv_pages* pages, int d_kv_expected);

// Fails with HC_EINVAL when a sequence of a ragged batch (device offsets
// d_cu_seqlens) is longer than the RoPE table (may read the offsets back).
void check_seq_positions(const hc_weights* w, const int32_t* d_cu_seqlens, int n_seqs,
                         int64_t n_rows, cudaStream_t stream);

}  // namespace hc
