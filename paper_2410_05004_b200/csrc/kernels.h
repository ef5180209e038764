// kernels.h -- host-side launch interface of the sm_100a kernels (internal).
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace hc {

// HC_PDL=0 turns programmatic dependent launch off (A/B measurements).
bool pdl_enabled();
// Launch with programmatic stream serialization (see pdl_wait in sm100.cuh):
// the kernel must call pdl_wait() before its first global memory access.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t stream, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// Where K1 writes K and V. Dense mode (page_table == nullptr): row r of the
// projection lands at row r of k_base / v_base ([M x d_kv] row-major). Paged
// mode: row r of sequence s (rows cu_seqlens[s]..cu_seqlens[s+1]) at position
// p = start_pos + (r - cu_seqlens[s]) lands in page page_table[s*table_stride
// + p/page_size], slot p%page_size; a page holds page_size rows of d_kv.
struct KvOut {
  void* k_base = nullptr;
  void* v_base = nullptr;
  int d_kv = 0;
  int page_size = 0;
  const int32_t* page_table = nullptr;
  int table_stride = 0;
  const int32_t* cu_seqlens = nullptr;  // nullptr: one sequence of M rows
  int n_seqs = 1;
  int start_pos = 0;
  const int32_t* seq_start = nullptr;  // per-sequence first position (overrides start_pos)
  int out_f32 = 0;  // 0: bf16 KV, 1: fp32 (parity/debug)
  // Fused Q/K/V projection (recompute layers): the GEMM's first q_cols
  // columns are Q (RoPE, bf16) stored densely at q_base + row * q_cols, the
  // next 2*d_kv are K then V as above. q_cols = 0: K/V only.
  void* q_base = nullptr;
  int q_cols = 0;
};

// Epilogue inputs: LayerNorm fold (row stats + column sums of W) and RoPE.
struct EpiArgs {
  const float* row_mean = nullptr;  // nullptr: norm disabled
  const float* row_rstd = nullptr;
  const float* colsum = nullptr;    // [N] sum_k W[n,k]
  const float2* rope = nullptr;     // [rope_rows][d_head/2] (cos, sin); nullptr: off
  int d_head = 0;
  int rope_rows = 0;
};

// Epilogue modes of the shared tcgen05 GEMM (K1 and the K6 projections).
constexpr int kEpiKv = 0;     // LN fold + RoPE(K half) -> K/V rows (dense or paged)
constexpr int kEpiResid = 1;  // x += acc (fp32 residual), xb = bf16(x)
constexpr int kEpiGelu = 2;   // xb = bf16(gelu(LN fold(acc)))

// Dense outputs of the RESID / GELU modes, row stride ldo elements.
struct GemmOut {
  float* x = nullptr;
  void* xb = nullptr;  // bf16
  int ldo = 0;
};

// A operand of the shared tcgen05 GEMM: one tensor map, or -- the all-gather
// fused into K1 over peer memory -- up to kMaxASrc maps, map s covering rows
// [row0[s], row0[s+1]) of A from its own buffer (another GPU's, mapped over
// NVLink). Source boundaries must be multiples of 128 rows (one M tile, or
// one CTA's half of a CTA-pair tile, reads one source).
constexpr int kMaxASrc = 8;
struct AMaps {
  CUtensorMap m[kMaxASrc + 1];
  int row0[kMaxASrc + 1];
  int n;
  // when *alt_flag != 0 (set on the device by the row statistics) every A
  // tile is read through m[n] -- the mean-shifted copy of the whole matrix
  // written by launch_center_rows -- instead of the source maps m[0..n)
  const int32_t* alt_flag = nullptr;
};
inline AMaps single_amap(const CUtensorMap& t) {
  AMaps a;
  a.m[0] = t;
  a.row0[0] = 0;
  a.row0[1] = 0x7fffffff;
  a.n = 1;
  return a;
}

// Creates a 2D K-major bf16/fp16 tensor map with a {64, box_rows} box and the
// 128-byte swizzle (the K1 operand layout). Returns false on failure.
bool make_tmap_kmajor(CUtensorMap* map, const void* base, uint64_t k, uint64_t rows,
                      uint64_t row_stride_bytes, uint32_t box_rows);
// The same, memoised on (address, shape, stride, box) (bounded cache).
bool make_tmap_kmajor_cached(CUtensorMap* map, const void* base, uint64_t k, uint64_t rows,
                             uint64_t row_stride_bytes, uint32_t box_rows);

// Box rows of the B tensor map for an M x N GEMM (32, 64, 128 or 256). 128
// selects the CTA-pair kernel when the problem fills the SM pairs; 32/64 only
// for a single M tile (decode-sized M), to spread the weight stream over SMs.
int gemm_pick_bn(int64_t M, int N, int num_sms);
// B box rows for a GEMM launched with split_acc (decode-sized M is split over
// K instead of N, so it takes the widest tile).
int gemm_pick_bn_skinny(int64_t M, int N, int num_sms);
// Box rows of the A tensor map (K-major, 64-element K box) every caller of the
// single-CTA GEMM must use for an M-row A operand: 32 / 64 for small M, else 128.
int gemm_a_box(int64_t M);

// K1: KV[M x N] = epilogue(A[M x K] * B[N x K]^T), N = 2*d_kv (K half, V half).
// A is described by tmA (box rows 128), B by tmB (box rows 256 or 128 = bn).
// split_acc: a decode-sized M (<= 128) may split K over CTAs (fp32 partials
// reduced in a fixed order; a different summation order than the fused path).
// Off for every K/V projection, so restored K/V stay bit-identical to the K/V
// a forward wrote.
// The mean-shifted A copy of launch_center_rows and its device flag.
struct AltA {
  CUtensorMap map;
  const int32_t* flag;
};
// m_sched (> M): lay the tiles and K splits out as for m_sched rows and store
// only the first M -- a row-truncated GEMM then sums every element in the
// order of the full one (tensor maps and bn must be those of m_sched rows).
// With split_acc the CTA-pair kernel may also split the K loop of the tiles
// of its last, partial wave over two SM pairs (see tc_gemm_pair_kernel).
cudaError_t launch_restore_kv(const CUtensorMap& tmA, const CUtensorMap& tmB, int bn, int M,
                              int N, int K, bool bf16_in, const KvOut& out, const EpiArgs& epi,
                              int num_sms, cudaStream_t stream, bool split_acc = false,
                              const AltA* alt = nullptr, int m_sched = 0);
// Per-source LayerNorm statistics of a head-sharded layer (the owners'
// slots, mapped over NVLink): rows [row0[s], row0[s+1]) come from
// mean[s] / rstd[s].
struct StatSources {
  const float* mean[kMaxASrc];
  const float* rstd[kMaxASrc];
  int64_t row0[kMaxASrc + 1];
  int n;
};
cudaError_t launch_gather_stats(const StatSources& src, int64_t max_rows, float* mean, float* rstd,
                                cudaStream_t stream);
// Stream-ordered cross-GPU flags: store `value` (system-scope release) into
// each of n flags whose addresses are in device memory; wait until a flag in
// this GPU's memory is >= value (cuStreamWaitValue32 or a polling kernel).
cudaError_t launch_signal_flags(uint32_t* const* d_flag_ptrs, int n, uint32_t value,
                                cudaStream_t stream);
cudaError_t wait_flag_geq(cudaStream_t stream, const uint32_t* d_flag, uint32_t value);

// K1 with a multi-source A (AMaps): the peer-memory all-gather fused in.
cudaError_t launch_restore_kv_multi(const AMaps& am, const CUtensorMap& tmB, int bn, int M, int N,
                                    int K, bool bf16_in, const KvOut& out, const EpiArgs& epi,
                                    int num_sms, cudaStream_t stream);

// The same GEMM with a dense epilogue (mode kEpiResid or kEpiGelu).
cudaError_t launch_gemm_dense(const CUtensorMap& tmA, const CUtensorMap& tmB, int bn, int mode,
                              int M, int N, int K, const GemmOut& g, const EpiArgs& epi,
                              int num_sms, cudaStream_t stream, bool split_acc = false,
                              const AltA* alt = nullptr, int m_sched = 0);

// Causal attention over the paged cache for a prefill from position 0
// (attention_forward, model.cpp:237-288): q [n x n_heads*dh] bf16 (RoPE
// applied), K/V from `kv` (paged or dense, row width kv.d_kv, GQA groups),
// out [n x n_heads*dh] bf16 = softmax(q k^T / sqrt(dh)) v per head.
cudaError_t launch_attention(const void* q, int n, int n_heads, int n_kv_heads, int dh,
                             const KvOut& kv, void* out, cudaStream_t stream);

// Batched continuation (forward_tokens / decode_step, model.cpp:237-288 with
// start_pos > 0): sequence s owns query rows [cu_q[s], cu_q[s+1]) at
// positions seq_start[s] + i and attends to its cached keys [0, position]
// through page-table row s (stride kv.table_stride). max_new = max rows of
// one sequence (grid extent).
cudaError_t launch_attention_extend(const void* q, int n_seqs, int max_new, const int32_t* cu_q,
                                    const int32_t* seq_start, int n_heads, int n_kv_heads,
                                    int dh, const KvOut& kv, void* out, cudaStream_t stream);

// The same attention on tcgen05 (attention_tc.cu): S and O in TMEM, K/V tiles
// gathered from the pages by TMA. kv_rows = rows of the K/V pools (paged:
// num_pages * page_size; page_size a power of two >= 8). dh 64 or 128.
cudaError_t launch_attention_tc(const void* q, int n, int n_heads, int n_kv_heads, int dh,
                                const KvOut& kv, int64_t kv_rows, void* out,
                                cudaStream_t stream);

// The tcgen05 attention for a ragged batch of prefills from position 0:
// sequence s owns query rows [cu[s], cu[s+1]) (device) and page-table row s
// (stride kv.table_stride), attending causally to its own keys 0..; max_len =
// the longest sequence (grid extent).
cudaError_t launch_attention_tc_varlen(const void* q, int64_t total, int n_seqs, int max_len,
                                       const int32_t* cu, int n_heads, int n_kv_heads, int dh,
                                       const KvOut& kv, int64_t kv_rows, void* out,
                                       cudaStream_t stream);

// Embedding gather (model.cpp:82-92): x[i] = E[tokens[i]] (fp32), xb = bf16.
cudaError_t launch_embed(const int32_t* tokens, int64_t n, const void* emb, int d, float* x,
                         void* xb, cudaStream_t stream);

// Greedy next token (argmax_token, model.cpp:67-80): argmax_t E[t] . h.
cudaError_t launch_argmax_logits(const void* emb, int vocab, int d, const float* h,
                                 int32_t* out_token, cudaStream_t stream);

// Greedy next token of every sequence's last row: out[s] = argmax over the
// vocabulary of E . h[cu[s+1]-1] (fp32 h rows of width d).
cudaError_t launch_argmax_rows(const void* emb, int vocab, int d, const float* h,
                               const int32_t* cu, int n_seqs, int32_t* out_tokens,
                               cudaStream_t stream);

// Greedy tokens through the tensor cores: hl = [bf16(h_s); bf16(h_s -
// bf16(h_s))] for each sequence's last row (2*n_seqs x d), logits = E hl^T
// (GEMM, fp32 [vocab x ld]), out[s] = argmax_t logits[t][s] + logits[t][B+s].
cudaError_t launch_hilo_rows(const float* x, const int32_t* cu, int n_seqs, int d, void* hl,
                             cudaStream_t stream);
cudaError_t launch_argmax_pairs(const float* logits, int vocab, int ld, int n_seqs, int32_t* out,
                                cudaStream_t stream);

// Pages -> interleaved [K_row | V_row] rows for positions [pos0, pos0 + n) of
// one sequence (the KV-offload snapshot payload, storage.cpp:67-75).
cudaError_t launch_kv_gather(const KvOut& kv, int pos0, int64_t n_rows, void* rows,
                             cudaStream_t stream);

// Decode-time save, stage 1: row b of a step's layer inputs (layers
// [h0, h0+nh), row stride rows_in_step) -> dsts[b].dst + l * dsts[b].pitch.
struct AppendDst {
  void* dst;
  int64_t pitch;  // bytes between layers in the request's round buffer
};
cudaError_t launch_append_rows(const void* step_rows, int rows_in_step, int h0, int nh, int d,
                               const AppendDst* d_dsts, int n_rows, cudaStream_t stream);

// Session rows in the reference's formats (HC_DTYPE_F32 / HC_DTYPE_F16) ->
// bf16 (round to nearest even); dst may equal src for F16.
cudaError_t launch_convert_to_bf16(const void* src, int src_dtype, void* dst, int64_t n,
                                   cudaStream_t stream);

// Row statistics for the LayerNorm fold: mean and 1/sqrt(var+1e-5) per row
// (the reference's double statistics, model.cpp:43-61, to ~1e-7).
// Rows whose |mean| exceeds this many standard deviations make the LayerNorm
// fold lose precision (H W^T ~ mean * colsum(W) cancels in fp32): the row
// statistics raise a per-matrix flag and the GEMM reads a shifted copy.
constexpr float kCenterRatio = 16.0f;

// Row statistics; flag (nullable, zeroed by the caller) is set when a row has
// |mean| * rstd > kCenterRatio.
cudaError_t launch_row_stats_flagged(const void* x, int64_t rows, int cols, int64_t row_stride,
                                     bool bf16_in, float* mean, float* rstd, int32_t* flag,
                                     cudaStream_t stream);
// HC_LN_CENTER=0 disables the mean shift (A/B measurements only).
bool ln_center_enabled();
// HC_QKV_FUSED=0: the Q and the K/V projections of a recompute layer as two
// GEMMs even when W_q precedes [W_k;W_v] in memory (A/B measurements only).
bool qkv_fusion_enabled();
// When *flag (device) is set: out[r] = bf16(x[r] - c_r), c_r = bf16(mean[r])
// (exact for |x - c| small against c, Sterbenz), and mean[r] -= c_r in place,
// so the LayerNorm fold over `out` is well conditioned. A no-op otherwise.
cudaError_t launch_center_rows(const void* x, int64_t rows, int cols, int64_t row_stride,
                               float* mean, const int32_t* flag, void* out, cudaStream_t stream);
// The same without the flag.
cudaError_t launch_row_stats(const void* x, int64_t rows, int cols, int64_t row_stride,
                             bool bf16_in, float* mean, float* rstd, cudaStream_t stream);

// colsum[n] = sum_k W[n,k] (double accumulation) for the LayerNorm fold.
cudaError_t launch_colsum(const void* w, int64_t rows, int cols, bool bf16_in, float* out,
                          cudaStream_t stream);

// Deterministic synthetic data: dst[i] = Rng(seed)::symmetric(bound) draw
// (offset+i) (reference model.cpp:17-31), stored as bf16/fp16/fp32.
// p[0, n) = 0 as a kernel (stream-ordered memsets stall behind copy-engine work)
cudaError_t launch_zero_i32(int32_t* p, int64_t n, cudaStream_t stream);
// p[i] = i (an identity page table)
cudaError_t launch_iota_i32(int32_t* p, int64_t n, cudaStream_t stream);
cudaError_t launch_fill_symmetric(void* dst, int64_t n, uint64_t seed, uint64_t offset,
                                  float bound, int dtype, cudaStream_t stream);

// Interleaved [K_row | V_row] rows (reference KV chunk payload, storage.cpp:67-75)
// -> K and V (dense or paged, same KvOut addressing as K1). HBM-bound.
cudaError_t launch_kv_scatter(const void* rows, int64_t n_rows, const KvOut& out,
                              cudaStream_t stream);
// Columns [col0, col0 + out.d_kv) of dense all-heads K and V rows ([n_rows x
// src_ld] bf16, row r at position out.start_pos + r) -> out's pages.
cudaError_t launch_kv_slice(const void* k_src, const void* v_src, int src_ld, int col0,
                            int64_t n_rows, const KvOut& out, cudaStream_t stream);

}  // namespace hc
