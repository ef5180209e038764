/*
 * hcache_b200.h -- C ABI of the B200-native HCache state-restoration path.
 *
 * This is the drop-in boundary: plain C types, plain pointers and sizes, no
 * torch or C++ types. Each entry point names the reference interface it
 * replaces (paths relative to the reference tree proj/). The C++ facade
 * include/hcache_b200.hpp re-exposes these with the reference's C++
 * signatures and exception types; INTEGRATION.md shows the bindings.
 *
 * Memory ownership: weights and KV pages are caller-owned device
 * memory passed by pointer; the pinned-host chunk arena is owned by hc_store.
 * Device work is stream ordered on the caller's cudaStream_t (passed as
 * void*; NULL = legacy default stream). Errors: every call returns hc_status;
 * hc_last_error() gives a thread-local message. There is no CPU fallback:
 * compute entry points fail with HC_ECUDA when no sm_100 device is present.
 */
#ifndef HCACHE_B200_H
#define HCACHE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HC_ABI_VERSION 1
#define HC_CHUNK_TOKENS 64    /* storage.hpp:20 kChunkTokens */
#define HC_MAX_LAYERS 256
#define HC_MAX_EVENTS (4 * HC_MAX_LAYERS)
#define HC_MAX_SESSION_ID 128

/* Error contract (SURVEY 8b "Errors"): the reference throws
 * std::invalid_argument -> HC_EINVAL; std::runtime_error for a missing
 * manifest/chunk -> HC_ENOENT, for an unfinalized session -> HC_EINCOMPLETE,
 * other runtime_error -> HC_ERUNTIME; snapshot() == false -> HC_EAGAIN;
 * read_layer() == nullopt -> HC_ENOENT. */
typedef enum hc_status {
  HC_OK = 0,
  HC_EINVAL = 1,
  HC_ENOENT = 2,
  HC_EINCOMPLETE = 3,
  HC_EAGAIN = 4,
  HC_ECUDA = 5,
  HC_ENCCL = 6,
  HC_ERUNTIME = 7,
  HC_ENOMEM = 8
} hc_status;

typedef enum hc_dtype { HC_DTYPE_F32 = 0, HC_DTYPE_BF16 = 1, HC_DTYPE_F16 = 2 } hc_dtype;
/* StateKind (storage.hpp:22) */
typedef enum hc_state_kind { HC_STATE_HIDDEN = 0, HC_STATE_KV = 1 } hc_state_kind;
/* LayerMethod / Complement (planner.hpp:8-9); MIXED = three-way B200 plan */
typedef enum hc_layer_method {
  HC_METHOD_HIDDEN = 0,
  HC_METHOD_KV_OFFLOAD = 1,
  HC_METHOD_RECOMPUTE = 2
} hc_layer_method;
typedef enum hc_complement {
  HC_COMPLEMENT_NONE = 0,
  HC_COMPLEMENT_KV_OFFLOAD = 1,
  HC_COMPLEMENT_RECOMPUTE = 2,
  HC_COMPLEMENT_MIXED = 3
} hc_complement;

const char* hc_last_error(void);
const char* hc_version(void);
int32_t hc_abi_version(void);
/* Number of CUDA devices usable by the library (0 on a GPU-less host). */
int32_t hc_device_count(void);

/* ------------------------------------------------------------------ model */
/* ModelConfig (model.hpp:11-25) + n_kv_heads for GQA (0 -> n_heads). */
typedef struct hc_model_config {
  int32_t n_layers;
  int32_t d_hidden;
  int32_t n_heads;
  int32_t n_kv_heads;
  int32_t d_ffn;
  int32_t vocab_size;
  int32_t max_seq;
  int32_t elem_bytes; /* persisted element width: 2 (bf16) or 4 (fp32) */
  int32_t norm_enabled;
  int32_t rope_enabled;
} hc_model_config;

/* ModelConfig::validate (model.cpp:140-150) */
hc_status hc_config_validate(const hc_model_config* cfg);
/* ModelConfig::hash (model.cpp:152-168), FNV-1a over the reference fields */
uint64_t hc_config_hash(const hc_model_config* cfg);

/* Device-resident weights of the restoration path (WeightSet, model.hpp:27-39).
 * kv_head_begin/kv_head_count select the KV heads this GPU projects (head
 * sharding; all heads: 0, n_kv_heads). Weight tensors are
 * caller-owned device memory and must outlive the handle. */
typedef struct hc_weights hc_weights;
hc_status hc_weights_create(const hc_model_config* cfg, int32_t kv_head_begin,
                            int32_t kv_head_count, int32_t device, hc_weights** out);
void hc_weights_destroy(hc_weights* w);
/* [W_k ; W_v] of this GPU's heads: (2*kv_head_count*d_head) x d_hidden bf16,
 * row-major (K-major for the projection), K rows then V rows. Zero copy. */
hc_status hc_weights_set_layer_kv(hc_weights* w, int32_t layer, const void* d_wkv);
/* Full block weights for the RECOMPUTE path (model.hpp:27-32), bf16,
 * row-major (out x in): wq d x d, wkv as above (all heads), wo d x d,
 * fc1 d_ffn x d, fc2 d x d_ffn. When wkv starts right where wq ends
 * (one [W_q ; W_k ; W_v] allocation, the reference's own draw order,
 * model.cpp:185-188) and d_hidden % 256 == 0, a recompute layer projects Q,
 * K and V with one GEMM (HC_QKV_FUSED=0 turns this off); the K/V it writes
 * are bit-identical either way. */
hc_status hc_weights_set_layer_full(hc_weights* w, int32_t layer, const void* d_wq,
                                   const void* d_wkv, const void* d_wo, const void* d_fc1,
                                   const void* d_fc2);
/* Embedding (vocab x d bf16), model.hpp:36. */
hc_status hc_weights_set_embedding(hc_weights* w, const void* d_embedding);

/* ---------------------------------------------------------- paged KV cache */
/* Per layer a pool of num_pages pages, each page_size rows of d_kv elements
 * (local heads x d_head, NHD). k_layers/v_layers: host arrays of n_layers
 * device pointers. Token p of a sequence lives in page
 * page_table[seq*table_stride + p/page_size], slot p%page_size. */
typedef struct hc_kv_pages {
  int32_t n_layers;
  int32_t page_size;
  int32_t num_pages;
  int32_t d_kv;
  int32_t dtype; /* HC_DTYPE_BF16 (HC_DTYPE_F32 accepted for parity) */
  void* const* k_layers;
  void* const* v_layers;
} hc_kv_pages;

/* ------------------------------------------------------- K1: projection */
/* project_hidden_to_kv (model.hpp:95-96, model.cpp:219-235) for one layer:
 * LN -> [W_k;W_v] GEMM -> RoPE(K) at start_pos.. -> dense K, V
 * ([n_rows x d_kv] each, out_dtype bf16 or f32). d_hidden: n_rows x d bf16. */
hc_status hc_project_hidden_to_kv(const hc_weights* w, int32_t layer, const void* d_hidden,
                                  int64_t n_rows, int32_t start_pos, void* d_k, void* d_v,
                                  int32_t out_dtype, void* stream);
/* Same projection written straight into the paged cache. Rows of several
 * sequences may be concatenated (d_cu_seqlens: n_seqs+1 device offsets, or
 * NULL for one sequence); positions restart at 0 per sequence
 * (restore.cpp:73). */
hc_status hc_project_to_pages(const hc_weights* w, int32_t layer, const void* d_hidden,
                              int64_t n_rows, const int32_t* d_cu_seqlens, int32_t n_seqs,
                              const hc_kv_pages* pages, const int32_t* d_page_table,
                              int32_t table_stride, void* stream);

/* split_kv (storage.cpp:77-86) into pages: d_rows n_rows x (2*d_kv) bf16
 * interleaved [K_row | V_row] -> paged K and V (K4, HBM-bound). */
hc_status hc_kv_scatter_to_pages(const void* d_rows, int64_t n_rows, int32_t layer,
                                 const int32_t* d_cu_seqlens, int32_t n_seqs,
                                 const hc_kv_pages* pages, const int32_t* d_page_table,
                                 int32_t table_stride, void* stream);

/* Deterministic synthetic data on the device: dst[i] = the (offset+i)-th
 * draw of the reference Rng(seed).symmetric(bound) (model.cpp:17-31), stored
 * as dtype. Reproducible element by element on the CPU. */
hc_status hc_fill_symmetric(void* d_dst, int64_t n, uint64_t seed, uint64_t offset, float bound,
                            int32_t dtype, void* stream);

/* ------------------------------------------------------ chunk indexing */
int32_t hc_chunk_tokens(void);
/* device_for_chunk (storage.hpp:45, storage.cpp:29-31) */
int32_t hc_device_for_chunk(int32_t layer, int32_t chunk_idx, int32_t device_count);

/* ---------------------------------------------------------------- planner */
/* RestorationPlan (planner.hpp:29-40). The reference has one complement per
 * plan; MIXED plans (l_re recompute prefix, l_h hidden, l_kv KV suffix) are
 * the B200 three-way extension. layer_assignment holds hc_layer_method. */
typedef struct hc_plan {
  int32_t n_layers;
  int32_t l_h;
  int32_t l_o;
  int32_t complement;
  int32_t l_kv;
  int32_t l_re;
  uint8_t layer_assignment[HC_MAX_LAYERS];
} hc_plan;

/* ProfiledTimings (planner.hpp:16-24), seconds per layer. */
typedef struct hc_timings {
  double io_h;
  double io_kv;
  double c_h;
  double c_token;
  int32_t n_layers;
} hc_timings;

hc_status hc_timings_validate(const hc_timings* t);
/* RestorationPlan::make (planner.cpp:34-51) */
hc_status hc_plan_make(int32_t n_layers, int32_t l_h, int32_t complement, hc_plan* out);
/* three-way plan: layers [0,l_re) RECOMPUTE, then l_h HIDDEN, then l_kv KV */
hc_status hc_plan_make_mixed(int32_t l_re, int32_t l_h, int32_t l_kv, hc_plan* out);
/* serialize / parse (planner.cpp:53-73): "l_h=.. l_o=.. complement=.." */
hc_status hc_plan_serialize(const hc_plan* p, char* buf, int32_t cap);
hc_status hc_plan_parse(const char* record, hc_plan* out);
/* plan (planner.cpp:75-90), makespan (:92-107), brute_force_plan (:109-128) */
hc_status hc_plan_closed_form(const hc_timings* t, hc_plan* out);
hc_status hc_makespan(const hc_plan* p, const hc_timings* t, double* out);
hc_status hc_brute_force_plan(const hc_timings* t, hc_plan* out);
/* B200 planner: exhaustive over (l_re, l_h, l_kv), costed by the bounded
 * staging pipeline (simulate_pipeline at prefetch_depth) so the plan is
 * bubble-free under the executor's real buffer bound. The
 * RECOMPUTE prefix's last layer is costed c_h: the executor stops it after
 * its K/V projection (its output is the next layer's stored input).
 * c_token >= HC_RECOMPUTE_UNAVAILABLE means no RECOMPUTE layers at all. */
#define HC_RECOMPUTE_UNAVAILABLE 1e9
hc_status hc_plan_three_way(const hc_timings* t, int32_t prefetch_depth, hc_plan* out,
                            double* makespan_out);
/* B200 extension: the token split of the plan's first layer after the
 * recompute prefix (hc_restore_opts.split_tokens) that minimises the pipeline
 * makespan; 0 when no split helps or the layer is not HIDDEN. */
hc_status hc_plan_token_split(const hc_timings* t, int32_t prefetch_depth, const hc_plan* plan,
                              int32_t n_tokens, int32_t* split_out, double* makespan_out);

/* --------------------------------------------------------------- timeline */
typedef enum hc_lane { HC_LANE_IO = 0, HC_LANE_COMPUTE = 1 } hc_lane;
typedef enum hc_event_kind {
  HC_EV_FETCH_HIDDEN = 0,
  HC_EV_FETCH_KV = 1,
  HC_EV_PROJECT = 2,
  HC_EV_RECOMPUTE = 3,
  HC_EV_SCATTER = 4,
  HC_EV_GATHER = 5,
  HC_EV_FETCH = 6,
  HC_EV_COMPUTE = 7
} hc_event_kind;
/* TimelineEvent / Timeline (pipeline.hpp:18-28) */
typedef struct hc_event {
  int32_t lane;
  int32_t layer;
  int32_t kind;
  int32_t pad_;
  double start_s;
  double end_s;
} hc_event;
typedef struct hc_timeline {
  int32_t n_events;
  int32_t pad_;
  double total_s;
  double fill_s;
  hc_event events[HC_MAX_EVENTS];
} hc_timeline;
/* PipelineJob (pipeline.hpp:30-41) */
typedef struct hc_pipeline_job {
  int32_t layer;
  int32_t has_io;
  int32_t has_compute;
  int32_t io_kind;
  int32_t compute_kind;
  int32_t pad_;
  double io_s;
  double compute_s;
} hc_pipeline_job;

double hc_timeline_lane_busy(const hc_timeline* tl, int32_t lane);
/* B200 extension of profile_hardware (harness.cpp:431-490): refine timings
 * from a measured restore's timeline. io_h / io_kv / c_h / c_token become the
 * per-event busy time of that kind (union of its intervals / event count;
 * RECOMPUTE without the prefix's last, projection-only layer, and only when
 * the prefix has >= 2 layers); kinds without events keep their value. */
hc_status hc_timings_from_timeline(const hc_timeline* tl, hc_timings* io);
hc_status hc_timeline_bubble_fraction(const hc_timeline* tl, double* out);
/* simulate_pipeline (pipeline.cpp:33-104) */
hc_status hc_simulate_pipeline(const hc_pipeline_job* jobs, int32_t n_jobs,
                               int32_t prefetch_depth, hc_timeline* out);

/* ------------------------------------------------------------------ store */
/* DevicePool (storage.hpp:27-34). The B200 store keeps chunks in pinned host
 * memory; "devices" are separate pinned arenas (stand-ins for SSDs) that
 * chunks are striped over exactly as the reference stripes files. bw/latency
 * feed the simulated read-time model only. */
typedef struct hc_pool_desc {
  int32_t device_count;
  int32_t pad_;
  double bw_bytes_per_s;
  double read_latency_s;
} hc_pool_desc;

/* SessionSeed (storage.hpp:71-79) + d_kv (GQA KV row width / 2; 0 -> d_hidden)
 * and dtype of 2-byte elements (bf16 default; fp16 = the reference codec). */
typedef struct hc_session_seed {
  const char* session_id;
  uint64_t config_hash;
  int32_t n_layers;
  int32_t d_hidden;
  int32_t d_kv;
  int32_t elem_bytes;
  int32_t dtype;
  int32_t pad_;
  const hc_plan* plan;
  const int32_t* tokens;
  int64_t n_tokens;
} hc_session_seed;

/* SessionManifest (storage.hpp:54-69) */
typedef struct hc_manifest {
  char session_id[HC_MAX_SESSION_ID];
  uint64_t config_hash;
  int32_t n_tokens;
  int32_t n_layers;
  int32_t d_hidden;
  int32_t d_kv;
  int32_t elem_bytes;
  int32_t dtype;
  int32_t device_count;
  int32_t chunk_tokens;
  int32_t finalized;
  int32_t pad_;
  int64_t n_token_ids;
  hc_plan plan;
} hc_manifest;

typedef struct hc_store hc_store;
/* StorageManager(DevicePool, buffer_capacity) (storage.hpp:86-87) */
hc_status hc_store_create(const hc_pool_desc* pool, size_t buffer_capacity_bytes,
                          hc_store** out);
void hc_store_destroy(hc_store* s);
/* B200 extension: page-lock `bytes` of pinned arena now (cudaHostAlloc pins
 * page by page, ~0.1 s per 256 MiB), so later snapshots and chunk extents are
 * carved from it without pinning on the save path (a serving host reserves
 * its whole save volume at start-up). */
hc_status hc_store_reserve(hc_store* s, size_t bytes);
/* create_session (storage.hpp:90): HC_EINVAL/ HC_ERUNTIME on duplicate id */
hc_status hc_store_create_session(hc_store* s, const hc_session_seed* seed);
/* reopen_for_append (storage.hpp:91) */
hc_status hc_store_reopen_for_append(hc_store* s, const char* sid, const int32_t* new_tokens,
                                     int64_t n);
/* snapshot (storage.hpp:96-97): stage 1, bulk copy of n_rows rows (width d
 * for HIDDEN, 2*d_kv for KV) into the bounded pinned FIFO. rows may be host
 * (src_dtype f32/bf16/f16) or device memory (must already be the session
 * dtype; copied D2H asynchronously on `stream`, a side stream). row_width
 * must be d_hidden (HIDDEN) or 2*d_kv (KV), as the reference checks. Returns
 * HC_EAGAIN on backpressure with nothing enqueued. */
hc_status hc_store_snapshot(hc_store* s, const char* sid, int32_t layer, int32_t kind,
                            const void* rows, int64_t n_rows, int32_t row_width,
                            int32_t src_dtype, int32_t src_on_device, void* stream);
/* snapshot of tokens [tok_begin, tok_begin + n_rows) of a layer (tok_begin
 * a multiple of 64): the save path of a head-sharded context, where every
 * rank persists only its own token range of each hidden layer (chunk index,
 * striping and payload stay the reference's; chunks below tok_begin are held
 * by the other ranks' stores). Further rows of the layer append after it.
 * B200 extension of snapshot (storage.hpp:96-97). */
hc_status hc_store_snapshot_range(hc_store* s, const char* sid, int32_t layer, int32_t kind,
                                  int64_t tok_begin, const void* rows, int64_t n_rows,
                                  int32_t row_width, int32_t src_dtype, int32_t src_on_device,
                                  void* stream);
/* drain / drain_all (storage.hpp:101-102): stage 2, chunk assembly. */
hc_status hc_store_drain(hc_store* s, int64_t max_chunks, int64_t* flushed);
hc_status hc_store_drain_all(hc_store* s);
/* finalize (storage.hpp:105), idempotent */
hc_status hc_store_finalize(hc_store* s, const char* sid);
/* open (storage.hpp:107): HC_ENOENT unknown, HC_EINCOMPLETE not finalized */
hc_status hc_store_open(hc_store* s, const char* sid, hc_manifest* out);
/* manifest.find(layer, kind) (storage.hpp:68): HC_ENOENT when absent */
hc_status hc_store_layer_info(hc_store* s, const char* sid, int32_t layer, int32_t kind,
                              int32_t* n_chunks, int32_t* n_tokens);
/* manifest.tokens (storage.hpp:64) */
hc_status hc_store_tokens(hc_store* s, const char* sid, int32_t* out, int64_t cap,
                          int64_t* n_out);
/* read_layer (storage.hpp:111-112): token-ordered reassembly into dst
 * (n_tokens x width elements of the session dtype). dst on device: chunk
 * groups are gathered H2D on `stream` by the copy engine. HC_ENOENT when the
 * layer/kind was never stored. */
hc_status hc_store_read_layer(hc_store* s, const char* sid, int32_t layer, int32_t kind,
                              void* dst, int64_t dst_bytes, int32_t dst_on_device, void* stream);
/* Like read_layer for the token range [tok_begin, tok_end) (chunk aligned
 * begin), used by the head-sharded multi-GPU fetch. */
hc_status hc_store_read_layer_range(hc_store* s, const char* sid, int32_t layer, int32_t kind,
                                    int32_t tok_begin, int32_t tok_end, void* dst,
                                    int64_t dst_bytes, int32_t dst_on_device, void* stream);
/* Where chunk c of (sid, layer, kind) lives: device index (device_for_chunk)
 * and host pointer/bytes of its payload (tests of bit-exact placement). */
hc_status hc_store_chunk_info(hc_store* s, const char* sid, int32_t layer, int32_t kind,
                              int32_t chunk_idx, int32_t* device, const void** payload,
                              int64_t* bytes);
/* Chunks currently stored on each device (out[device_count]). */
hc_status hc_store_device_chunk_counts(hc_store* s, int64_t* out, int32_t cap);
hc_status hc_store_start_daemon(hc_store* s);
hc_status hc_store_stop_daemon(hc_store* s);
size_t hc_store_buffer_bytes(hc_store* s);
/* 1 when the arenas are page-locked (cudaHostAlloc), 0 on a GPU-less host. */
int32_t hc_store_pinned(hc_store* s);
size_t hc_store_buffer_capacity(hc_store* s);
uint64_t hc_store_backpressure_events(hc_store* s);
/* simulated_read_seconds_tokens (storage.cpp:348-365) */
double hc_store_simulated_read_seconds_tokens(hc_store* s, int32_t n_tokens, int32_t width,
                                              int32_t elem_bytes);

/* ---------------------------------------------------------------- restore */
/* ThrottleConfig (restore.hpp:14-29) for the device engine. */
typedef struct hc_restore_opts {
  int32_t prefetch_depth; /* staged hidden layers in flight beyond the one in use (>=1) */
  int32_t timeline;       /* 1: record per-layer CUDA events into the timeline */
  /* B200 extension (0 = off): the first layer after the RECOMPUTE prefix must be
   * HIDDEN; its first split_tokens tokens (a multiple of 64) are recomputed
   * with the prefix and only tokens [split_tokens, n) are fetched and
   * projected (hc_plan_token_split picks the value that balances the lanes). */
  int32_t split_tokens;
  /* hc_restore_sharded only: 0 = K1 reads every owner's staging slot in
   * place over NVLink (the all-gather fused into the GEMM); 1 = the owners'
   * ranges are first gathered by the copy engines into a local buffer (the
   * all-gather-then-GEMM baseline; also taken automatically for a layer whose
   * peer slots the driver cannot describe with a TMA tensor map). */
  int32_t peer_gather;
} hc_restore_opts;

/* restore (restore.hpp:40-42): executes the plan over a finalized session
 * into the paged cache. HIDDEN layers: chunk H2D on a copy stream into an HBM
 * staging ring -> K1. KV_OFFLOAD layers: chunk H2D -> K4 scatter. RECOMPUTE
 * prefix: K6 from the manifest tokens (needs full weights). The plan must
 * equal the manifest's (HC_EINVAL otherwise, restore.cpp:230-231). Blocks
 * until done when `timeline` is non-NULL (fills it), else returns with the
 * work queued on `stream`. */
hc_status hc_restore(hc_store* s, const char* sid, const hc_weights* w, const hc_plan* plan,
                     const hc_restore_opts* opts, const hc_kv_pages* pages,
                     const int32_t* d_page_table, void* stream, hc_timeline* timeline);
/* Several finalized sessions restored concurrently (config 4). The sessions
 * must share one plan (HC_EINVAL otherwise); it is executed like hc_restore's:
 * the RECOMPUTE prefix as one ragged forward over all sessions (each from
 * position 0, token ids from the manifests), per HIDDEN layer all sessions'
 * chunks land in one concatenated staging buffer and one grouped K1 launch
 * projects them (per-row sequence/position/page indirection), per KV layer
 * one K4 scatter. bf16 sessions only. d_page_tables: n_sessions x table_stride. */
hc_status hc_restore_batch(hc_store* s, const char* const* sids, int32_t n_sessions,
                           const hc_weights* w, const hc_restore_opts* opts,
                           const hc_kv_pages* pages, const int32_t* d_page_tables,
                           int32_t table_stride, void* stream, hc_timeline* timeline);
/* restore_token_wise (restore.hpp:47-49), the token-wise partition ablation:
 * at every layer tokens [0, hidden_tokens) are projected from hidden states
 * and tokens [hidden_tokens, n) spliced from the stored KV rows (every KV
 * chunk overlapping them is fetched). Both HIDDEN and KV must be stored for
 * every layer; HC_EINVAL for a split outside [0, n]. */
hc_status hc_restore_token_wise(hc_store* s, const char* sid, const hc_weights* w,
                                int32_t hidden_tokens, const hc_kv_pages* pages,
                                const int32_t* d_page_table, void* stream, hc_timeline* timeline);
/* Hidden states already resident in HBM (per layer device pointers, rows
 * concatenated per d_cu_seqlens): K1 over every layer. The kernel-bound leg. */
hc_status hc_restore_resident(const hc_weights* w, const void* const* d_hidden_layers,
                              int64_t n_rows, const int32_t* d_cu_seqlens, int32_t n_seqs,
                              const hc_kv_pages* pages, const int32_t* d_page_table,
                              int32_t table_stride, void* stream);

/* forward_tokens / decode_step (model.cpp:305-347, model.hpp:115-120) batched
 * over sequences with paged caches: sequence s appends new_lens[s] tokens
 * (host array) at positions start_pos[s].. (host array; its cached keys
 * [0, start_pos[s]) are attended to). d_tokens: all sequences' tokens
 * concatenated (device). Page-table row s at d_page_tables + s*table_stride.
 * d_layer_inputs (optional, n_layers x T x d_hidden bf16, T = sum new_lens)
 * receives each layer's input hidden state (the rows the save path persists);
 * d_next_tokens[s] (device) the greedy next token after sequence s. */
hc_status hc_forward_batch(const hc_weights* w, const int32_t* d_tokens, int32_t n_seqs,
                           const int32_t* new_lens, const int32_t* start_pos,
                           const hc_kv_pages* pages, const int32_t* d_page_tables,
                           int32_t table_stride, void* d_layer_inputs, int32_t* d_next_tokens,
                           void* stream);
/* Pages -> interleaved [K_row | V_row] rows (the KV chunk payload,
 * storage.cpp:67-75) for positions [pos0, pos0 + n_rows) of one layer. */
hc_status hc_kv_gather_rows(const hc_kv_pages* pages, int32_t layer, const int32_t* d_page_table,
                            int32_t pos0, int64_t n_rows, void* d_rows, void* stream);

/* ------------------------------------------------------ recompute (K6) */
/* prefill_layers (model.hpp:124-125, model.cpp:349-356): embeds d_tokens and
 * runs layers [lb, le) from position 0, writing their K/V into the pages. */
hc_status hc_prefill_layers(const hc_weights* w, const int32_t* d_tokens, int64_t n,
                            int32_t layer_begin, int32_t layer_end, const hc_kv_pages* pages,
                            const int32_t* d_page_table, void* stream);
/* prefill (model.hpp:115-116): all layers; also writes each layer's input
 * hidden state H_L (bf16, n x d at d_layer_inputs + L*n*d, may be NULL) --
 * the states the save path snapshots. Returns the greedy next token via
 * next_token (may be NULL). */
hc_status hc_prefill(const hc_weights* w, const int32_t* d_tokens, int64_t n,
                     const hc_kv_pages* pages, const int32_t* d_page_table,
                     void* d_layer_inputs, int32_t* next_token, void* stream);

/* Building blocks of K6, exposed for parity tests against fp32 references:
 * causal attention over dense K/V (n x d_kv rows, GQA groups) and the shared
 * tcgen05 GEMM C = A B^T (A M x K, B N x K, bf16) with the RESID epilogue
 * (x[M x N] fp32 += C, xb = bf16(x)) or the GELU epilogue (xb = bf16(gelu(
 * LN-fold(C)))), mean/rstd/colsum may be NULL (no fold). */
hc_status hc_attention_dense(const void* d_q, int32_t n, int32_t n_heads, int32_t n_kv_heads,
                             int32_t d_head, const void* d_k, const void* d_v, int32_t d_kv,
                             void* d_out, void* stream);
/* mode | HC_GEMM_SPLIT_K: allow the decode-shape path (M <= 128: K split over
 * CTAs, fp32 partials reduced in a fixed order by a second kernel). */
#define HC_GEMM_SPLIT_K 0x100
hc_status hc_gemm_epilogue(int32_t mode, const void* d_a, const void* d_b, int32_t m, int32_t n,
                           int32_t k, float* d_x, void* d_xb, const float* d_mean,
                           const float* d_rstd, const float* d_colsum, int32_t device,
                           void* stream);

/* -------------------------------------------------------------- profiling */
/* profile_hardware (harness.hpp:76-77), measured on the device: io_h / io_kv
 * = pinned H2D time of one layer's hidden / KV rows for n_tokens, c_h = K1
 * time, c_token = K6 full-layer time (0 if full weights are absent). */
hc_status hc_profile(const hc_weights* w, int32_t n_tokens, hc_timings* out);
/* Measurement entry point (bench/profiling): runs the row-stats kernel and
 * K1 for `layer` on n_rows resident rows `iters` times, each bracketed by
 * CUDA events on `stream`; returns the mean milliseconds of each kernel. */
hc_status hc_bench_project(const hc_weights* w, int32_t layer, const void* d_hidden,
                           int64_t n_rows, int32_t iters, void* stream, double* stats_ms,
                           double* k1_ms);
/* Pinned host->device copy bandwidth (bytes/s) for a `bytes` transfer. */
hc_status hc_measure_h2d(int32_t device, size_t bytes, int32_t reps, double* bytes_per_s);

/* ------------------------------------- multi-GPU: peer-memory all-gather */
/* Head-sharded restore with the all-gather fused into K1: rows
 * [row_begin[s], row_begin[s+1]) of one layer's hidden states live in
 * d_src[s] -- typically another GPU's staging buffer mapped into this process
 * (CUDA IPC over NVLink). The row statistics and the K1 A tiles are read
 * straight from the owning buffers; K/V for this GPU's heads land in `pages`
 * (positions start_pos..). Interior boundaries must be multiples of 128 rows;
 * up to 8 sources. Results are bit-identical to hc_project_to_pages on the
 * concatenated rows. Replaces hc_store_read_layer_range + all-gather +
 * hc_project_to_pages of the NCCL pipeline. */
hc_status hc_project_multi_source(const hc_weights* w, int32_t layer, int32_t n_src,
                                  const void* const* d_src, const int64_t* row_begin,
                                  const hc_kv_pages* pages, const int32_t* d_page_table,
                                  int32_t start_pos, void* stream);
/* Stream-ordered cross-GPU flags: wait until *d_flag >= value (d_flag in this
 * GPU's memory; cuStreamWaitValue32, or a polling kernel), and store `value`
 * into each of n flags (any GPU's memory, system-scope release) after all
 * prior work on the stream. */
hc_status hc_stream_wait_flag(void* stream, const uint32_t* d_flag, uint32_t value);
hc_status hc_stream_signal_flags(void* stream, uint32_t* const* d_flag_ptrs, int32_t n,
                                 uint32_t value);

/* ------------------------------------- multi-GPU: head-sharded restore */
/* restore (restore.hpp:40-42) of a context whose KV heads are sharded over
 * `world` GPUs, one process per GPU (north star (4)). Rank r owns
 * KV heads hc_shard_heads(r) and the 128-row aligned token range
 * hc_shard_range(r) of every HIDDEN layer: it fetches only that range over
 * its own PCIe link into a small ring of HBM slots that every other rank has
 * mapped (CUDA IPC over NVLink / NVSwitch), computes the range's LayerNorm
 * statistics (and the mean shift of rows with |mean| >> sigma) in place,
 * and announces the slot through flags in the peers' memory. Every rank's
 * K1 then reads all ranges' A tiles straight from the owners' slots -- the
 * all-gather fused into the GEMM, no gathered n x d copy -- and projects
 * only its own heads into its paged cache; it reads the owners' statistics
 * (8 B per row), not their rows. KV_OFFLOAD layers fetch this rank's heads'
 * [K|V] rows only. RECOMPUTE layers need the whole model on one GPU: with
 * world > 1 they are rejected (HC_EINVAL); with world == 1 the call is
 * hc_restore. Every rank must call with the same session plan, in the same
 * order of calls. */
typedef struct hc_peer_group hc_peer_group;
/* Chunk-aligned (128-row) contiguous token range [*begin, *end) of `rank`. */
hc_status hc_shard_range(int64_t n_tokens, int32_t world, int32_t rank, int64_t* begin,
                         int64_t* end);
/* KV heads [*begin, *begin + *count) of `rank` (n_kv_heads % world == 0). */
hc_status hc_shard_heads(int32_t n_kv_heads, int32_t world, int32_t rank, int32_t* begin,
                         int32_t* count);
/* This rank's member: `depth` staging slots of max_rows x d_hidden bf16 rows
 * (+ their statistics) and the flag arrays, on `device`. */
hc_status hc_peer_group_create(int32_t world, int32_t rank, int32_t device, int32_t d_hidden,
                               int64_t max_rows, int32_t depth, hc_peer_group** out);
void hc_peer_group_destroy(hc_peer_group* g);
/* The member's CUDA IPC handles as an opaque blob of hc_peer_group_blob_size()
 * bytes, to be handed to every other rank by any transport (MPI, sockets,
 * torch.distributed). */
size_t hc_peer_group_blob_size(void);
hc_status hc_peer_group_export(const hc_peer_group* g, void* blob, size_t cap);
/* Maps every peer: blobs[r] = rank r's blob (blobs[rank] is ignored). */
hc_status hc_peer_group_import(hc_peer_group* g, const void* const* blobs);
/* Reads back the peers' view of this rank after import (tests): 1 when every
 * peer is mapped. */
int32_t hc_peer_group_ready(const hc_peer_group* g);
hc_status hc_restore_sharded(hc_peer_group* g, hc_store* s, const char* sid,
                             const hc_weights* w, const hc_plan* plan,
                             const hc_restore_opts* opts, const hc_kv_pages* pages,
                             const int32_t* d_page_table, void* stream, hc_timeline* timeline);

/* ---------------------------------------------------------- serving loop */
/* Strategy / SavingMode (harness.hpp:14-17). */
typedef enum hc_strategy {
  HC_STRATEGY_HCACHE = 0,
  HC_STRATEGY_KV_OFFLOAD = 1,
  HC_STRATEGY_RECOMPUTE = 2,
  HC_STRATEGY_IDEAL = 3
} hc_strategy;
typedef enum hc_saving_mode {
  HC_SAVING_TWO_STAGE = 0, /* D2H on a side stream into the store FIFO, chunking by the daemon */
  HC_SAVING_DIRECT = 1,    /* synchronous copies and persistence on the serving thread */
  HC_SAVING_OFF = 2        /* persisted, but outside the clock (reference: cost 0) */
} hc_saving_mode;

/* Request (trace.hpp:11-19). */
typedef struct hc_request {
  const char* session_id;
  int32_t round;
  int32_t n_context; /* long-context pre-ingested tokens (0 for conversations) */
  const int32_t* context;
  int32_t n_prompt;
  int32_t output_budget;
  const int32_t* prompt;
  double arrival_s;
} hc_request;

/* RunOptions (harness.hpp:60-65) for the device engine. */
typedef struct hc_serve_opts {
  int32_t strategy;     /* hc_strategy */
  int32_t saving;       /* hc_saving_mode */
  hc_plan plan;         /* HC_STRATEGY_HCACHE's per-layer plan */
  int32_t page_size;    /* KV page size (tokens), 0 -> 64 */
  int32_t num_pages;    /* KV page pool (pages of page_size tokens, all layers) */
  int32_t max_batch;    /* decode batch cap, 0 -> unbounded */
  int32_t pad_;
} hc_serve_opts;

/* RequestMetrics (harness.hpp:27-36); times in seconds of the engine clock. */
typedef struct hc_request_metrics {
  int32_t round;
  int32_t history_tokens;
  int32_t generated;
  int32_t pad_;
  double arrival_s;
  double restore_s;
  double ttft_s;
  double tbt_s;
} hc_request_metrics;

/* Metrics aggregates (harness.hpp:38-55) + engine extras. */
typedef struct hc_serve_metrics {
  double ttft_p50, ttft_p95;
  double tbt_mean, tbt_p50, tbt_p95;
  double restore_tokens_per_s;
  double storage_bytes_per_token;
  uint64_t saved_bytes, saved_tokens, backpressure_stalls;
  double busy_s;          /* restore + prefill + decode + charged saving time */
  double save_stall_s;    /* charged saving time (DIRECT copies, backpressure waits) */
  double persist_wait_s;  /* uncharged waits for a previous round's persistence */
  int64_t decode_steps;
  int64_t decode_tokens;
} hc_serve_metrics;

/* run (harness.hpp:67-72, harness.cpp:189-429) on the GPU: restore -> prefill
 * -> continuous-batching decode per request, one restoration+prefill in flight
 * (strict phase ordering), saving each round's states per the strategy's plan
 * into `store`. The clock advances by the measured duration of every phase
 * (host wall time with the stream synchronised: restore, prompt prefill,
 * decode steps, charged saving); idle gaps jump to the next arrival.
 * Requests must be sorted by arrival. outputs: sum(output_budget) token ids,
 * request order. per_request: n_requests entries. Weights need the full
 * blocks and the embedding. */
hc_status hc_serve_run(hc_store* store, const hc_weights* w, const hc_request* requests,
                       int32_t n_requests, const hc_serve_opts* opts,
                       hc_request_metrics* per_request, int32_t* outputs, hc_serve_metrics* out,
                       void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HCACHE_B200_H */
