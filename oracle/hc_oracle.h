/*
 * hc_oracle.h -- CPU restatement of the HCache reference's state-restoration
 * path, used ONLY as a checker.
 *
 * TEST INFRASTRUCTURE. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library, and only to
 * check or time the reference algorithm. The product path
 * (paper_2410_05004_b200/, libhcache_b200.so) never links or calls it.
 *
 * Every routine restates one reference routine (cited file:line, paths
 * relative to the reference tree proj/). Arithmetic order, precision and
 * rounding follow the reference exactly so results are bit-identical to the
 * reference built from source (oracle/_ref, checked in tests/test_oracle.py
 * and pinned by tests/golden/*.json). Compile without -ffast-math and without
 * FMA contraction (see oracle/Makefile).
 */
#ifndef HC_ORACLE_H
#define HC_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- deterministic generators: src/model.cpp:17-31 (splitmix64 Rng) ---- */

/* i-th output (0-based) of Rng(seed).next(); the stream is counter based. */
uint64_t hco_splitmix64_at(uint64_t seed, uint64_t index);
/* Rng::symmetric (model.cpp:27-30) for the index-th draw of Rng(seed). */
float hco_symmetric_at(uint64_t seed, uint64_t index, float bound);
/* out[i] = hco_symmetric_at(seed, offset + i, bound), i in [0, n). */
void hco_fill_symmetric(float* out, size_t n, uint64_t seed, uint64_t offset,
                        float bound);

/* init_model (model.cpp:175-194): flat buffer in reference draw order,
 * [embedding (vocab x d) | per layer: wq wk wv wo (d x d), fc1 (dffn x d),
 * fc2 (d x dffn)]. Returns number of floats written (or needed if out NULL). */
size_t hco_init_model(int n_layers, int d, int d_ffn, int vocab, uint64_t seed,
                      float* out);

/* ---- element codecs ---- */
/* IEEE binary16 RNE: include/hcache/fp16.hpp:10-40, :42-68 */
uint16_t hco_float_to_half(float f);
float hco_half_to_float(uint16_t h);
/* bfloat16 RNE (the build's 2-byte element; deviation from fp16) */
uint16_t hco_float_to_bf16(float f);
float hco_bf16_to_float(uint16_t h);
void hco_round_to_bf16(float* x, size_t n); /* in place x = bf16(x) */

/* ---- hot-path math ---- */
/* layer_norm (model.cpp:43-61): unit scale, zero bias, eps 1e-5. */
void hco_layer_norm(const float* x, int64_t rows, int cols, float* out);
/* matmul_wt (src/matrix.cpp:8-21): y[i,o] = sum_k x[i,k]*w[o,k], float acc in
 * ascending k. Rows are split across nthreads (order per element unchanged). */
void hco_matmul_wt(const float* x, int64_t m, int k, const float* w, int out,
                   float* y, int nthreads);
/* apply_rope (model.cpp:196-217) with positions start_pos + i. */
void hco_apply_rope(float* x, int64_t rows, int cols, int n_heads,
                    int start_pos);
/* RoPE coefficient table exactly as model.cpp:207-209 computes it:
 * cos_out/sin_out[pos * (d_head/2) + t] for pos in [0, n_pos). */
void hco_rope_table(int n_pos, int d_head, float* cos_out, float* sin_out);
/* project_hidden_to_kv (model.cpp:219-235) for one layer. wk/wv are
 * (d_kv x d); n_kv_heads heads of d_kv/n_kv_heads each (GQA: SURVEY 0.7). */
void hco_project_hidden_to_kv(const float* h, int64_t n, int d,
                              const float* wk, const float* wv, int d_kv,
                              int n_kv_heads, int start_pos, int norm_enabled,
                              int rope_enabled, float* k_out, float* v_out,
                              int nthreads);

/* ---- full transformer (RECOMPUTE complement): model.cpp:102-115,237-356 ---- */
typedef struct {
  int n_layers, d_hidden, n_heads, d_ffn, vocab_size, max_seq;
  int norm_enabled, rope_enabled;
} hco_config;

/* prefill (model.cpp:324-330 via forward_tokens :305-322). weights = the
 * hco_init_model layout. layer_inputs (L*n*d), k_out/v_out (L*n*d),
 * final_hidden (n*d) may be NULL. Returns the greedy next token. */
int hco_prefill(const hco_config* cfg, const float* weights, const int* tokens,
                int64_t n, float* layer_inputs, float* k_out, float* v_out,
                float* final_hidden, int nthreads);
/* prefill_layers (model.cpp:349-356): layers [lb, le) over tokens from
 * position 0; writes K/V of those layers into k_out/v_out (L*n*d). */
void hco_prefill_layers(const hco_config* cfg, const float* weights,
                        const int* tokens, int64_t n, int layer_begin,
                        int layer_end, float* k_out, float* v_out,
                        int nthreads);

/* block_forward (model.cpp:102-115) of one layer from explicit weights
 * (row-major out x in), start_pos 0 and an empty cache: x (n x d) is updated
 * in place, the layer's K/V (n x d) written. Lets a parity check walk a
 * large model layer by layer without materialising the whole weight set. */
void hco_block_forward(const hco_config* cfg, const float* wq, const float* wk,
                       const float* wv, const float* wo, const float* fc1,
                       const float* fc2, float* x, int64_t n, float* k_out,
                       float* v_out, int nthreads);

/* hco_fill_symmetric rounded to bf16 (RNE) and widened back, rows split over
 * nthreads (the draws are counter based, so the values do not depend on it). */
void hco_fill_symmetric_bf16(float* out, size_t n, uint64_t seed, uint64_t offset,
                             float bound, int nthreads);

/* ---- chunk indexing: include/hcache/storage.hpp:20, src/storage.cpp:29-31 */
int hco_chunk_tokens(void);
int hco_device_for_chunk(int layer, int chunk_idx, int device_count);
int hco_num_chunks(int n_tokens);

/* ---- planner: src/planner.cpp:34-128 ---- */
typedef struct {
  double io_h, io_kv, c_h, c_token;
  int n_layers;
} hco_timings;
/* complement: 0 NONE, 1 KV_OFFLOAD, 2 RECOMPUTE (planner.hpp:8) */
typedef struct {
  int l_h, l_o, complement;
} hco_plan;
int hco_plan_closed_form(const hco_timings* t, hco_plan* out); /* 0 ok */
double hco_makespan(const hco_plan* p, const hco_timings* t);
int hco_brute_force_plan(const hco_timings* t, hco_plan* out);

/* ---- pipeline timeline: src/pipeline.cpp:33-104 ---- */
typedef struct {
  int layer;
  double io_s, compute_s;
  int has_io, has_compute;
} hco_job;
typedef struct {
  int lane; /* 0 IO, 1 COMPUTE */
  int layer;
  int job; /* index of the job the event belongs to */
  double start_s, end_s;
} hco_event;
/* events must hold 2*n_jobs; returns event count, total_s/fill_s out. */
int hco_simulate_pipeline(const hco_job* jobs, int n_jobs, int prefetch_depth,
                          hco_event* events, double* total_s, double* fill_s);

/* ---- trace lengths: src/trace.cpp:54-100 (Conversation kind) ---- */
/* history_tokens of every request, in generation order (session-major). */
int hco_conversation_history(int n_sessions, int rounds, double mean_input,
                             double mean_output, double arrival_rate,
                             int vocab, uint64_t seed, int* history_out);

/* FNV-1a 64 over bytes (for golden hashes). */
uint64_t hco_fnv1a(const void* data, size_t n);

#ifdef __cplusplus
}
#endif
#endif
