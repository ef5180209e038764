// hcache_b200.hpp -- header-only C++ facade over the C ABI (hcache_b200.h)
// with the reference's C++ restoration API (proj/include/hcache/*.hpp):
// same type and function names, argument meaning and exception types, so a
// reference-based caller switches namespaces (hcache -> hcache_b200) and
// passes device weights / KV pages where the reference took host matrices.
//
//   planner.hpp   Complement, LayerMethod, ProfiledTimings, RestorationPlan,
//                 plan, makespan, brute_force_plan (+ plan_three_way)
//   pipeline.hpp  Lane, TimelineEvent, Timeline, PipelineJob, simulate_pipeline
//   storage.hpp   kChunkTokens, StateKind, DevicePool, ChunkKey,
//                 device_for_chunk, LayerChunks, SessionManifest, SessionSeed,
//                 StorageManager, interleave_kv, split_kv
//   restore.hpp   ThrottleConfig, RestoreResult, restore (device engine)
//   model.hpp     ModelConfig, Matrix (host rows), DeviceWeights (hc_weights)
//
// Errors follow the reference: std::invalid_argument for HC_EINVAL, a
// std::runtime_error for every other failure; snapshot() returns false on
// backpressure and read_layer() returns std::nullopt for absent layers.
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "hcache_b200.h"

namespace hcache_b200 {

inline void check(hc_status s) {
  if (s == HC_OK) return;
  const std::string msg = hc_last_error();
  if (s == HC_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

// ------------------------------------------------------------------ model.hpp
struct ModelConfig {
  int n_layers = 4;
  int d_hidden = 256;
  int n_heads = 8;
  int d_ffn = 1024;
  int vocab_size = 1024;
  int max_seq = 4096;
  int elem_bytes = 4;
  bool norm_enabled = true;
  bool rope_enabled = true;
  int n_kv_heads = 0;  // 0 = n_heads (MHA); B200 extension for GQA

  int d_head() const { return d_hidden / n_heads; }
  hc_model_config c() const {
    return hc_model_config{n_layers, d_hidden, n_heads, n_kv_heads, d_ffn, vocab_size,
                           max_seq, elem_bytes, norm_enabled ? 1 : 0, rope_enabled ? 1 : 0};
  }
  void validate() const {
    hc_model_config x = c();
    check(hc_config_validate(&x));
  }
  std::uint64_t hash() const {
    hc_model_config x = c();
    return hc_config_hash(&x);
  }
};

// Row-major float matrix (matrix.hpp:11-30), the host-side row container.
struct Matrix {
  std::size_t rows = 0;
  std::size_t cols = 0;
  std::vector<float> v;
  Matrix() = default;
  Matrix(std::size_t r, std::size_t c) : rows(r), cols(c), v(r * c, 0.0f) {}
  float& at(std::size_t r, std::size_t c) { return v[r * cols + c]; }
  float at(std::size_t r, std::size_t c) const { return v[r * cols + c]; }
  float* row(std::size_t r) { return v.data() + r * cols; }
  const float* row(std::size_t r) const { return v.data() + r * cols; }
  bool operator==(const Matrix& o) const { return rows == o.rows && cols == o.cols && v == o.v; }
};

// Device weights of the restoration path (WeightSet, model.hpp:34-39).
class DeviceWeights {
 public:
  DeviceWeights(const ModelConfig& cfg, int kv_head_begin = 0, int kv_head_count = 0,
                int device = 0) {
    hc_model_config c = cfg.c();
    const int kvh = cfg.n_kv_heads ? cfg.n_kv_heads : cfg.n_heads;
    check(hc_weights_create(&c, kv_head_begin, kv_head_count ? kv_head_count : kvh - kv_head_begin,
                            device, &w_));
  }
  ~DeviceWeights() { hc_weights_destroy(w_); }
  DeviceWeights(const DeviceWeights&) = delete;
  DeviceWeights& operator=(const DeviceWeights&) = delete;
  void set_layer_kv(int layer, const void* d_wkv) { check(hc_weights_set_layer_kv(w_, layer, d_wkv)); }
  void set_layer_full(int layer, const void* wq, const void* wkv, const void* wo, const void* fc1,
                      const void* fc2) {
    check(hc_weights_set_layer_full(w_, layer, wq, wkv, wo, fc1, fc2));
  }
  void set_embedding(const void* emb) { check(hc_weights_set_embedding(w_, emb)); }
  hc_weights* get() const { return w_; }

 private:
  hc_weights* w_ = nullptr;
};

// ---------------------------------------------------------------- planner.hpp
enum class Complement { None, KvOffload, Recompute, Mixed };
enum class LayerMethod { Hidden, KvOffload, Recompute };

inline const char* to_string(Complement c) {
  switch (c) {
    case Complement::None: return "NONE";
    case Complement::KvOffload: return "KV_OFFLOAD";
    case Complement::Recompute: return "RECOMPUTE";
    case Complement::Mixed: return "MIXED";
  }
  return "?";
}

struct ProfiledTimings {
  double io_h = 0, io_kv = 0, c_h = 0, c_token = 0;
  int n_layers = 0;
  hc_timings c() const { return hc_timings{io_h, io_kv, c_h, c_token, n_layers}; }
  void validate() const {
    hc_timings t = c();
    check(hc_timings_validate(&t));
  }
};

struct RestorationPlan {
  int l_h = 0;
  int l_o = 0;
  Complement complement = Complement::None;
  std::vector<LayerMethod> layer_assignment;
  hc_plan raw{};

  int n_layers() const { return l_h + l_o; }
  static RestorationPlan from(const hc_plan& p) {
    RestorationPlan r;
    r.raw = p;
    r.l_h = p.l_h;
    r.l_o = p.l_o;
    r.complement = Complement(p.complement);
    for (int i = 0; i < p.n_layers; ++i) r.layer_assignment.push_back(LayerMethod(p.layer_assignment[i]));
    return r;
  }
  static RestorationPlan make(int n_layers, int l_h, Complement c) {
    hc_plan p;
    check(hc_plan_make(n_layers, l_h, int(c), &p));
    return from(p);
  }
  static RestorationPlan make_mixed(int l_re, int l_h, int l_kv) {
    hc_plan p;
    check(hc_plan_make_mixed(l_re, l_h, l_kv, &p));
    return from(p);
  }
  std::string serialize() const {
    char buf[256];
    check(hc_plan_serialize(&raw, buf, sizeof buf));
    return buf;
  }
  static RestorationPlan parse(const std::string& record) {
    hc_plan p;
    check(hc_plan_parse(record.c_str(), &p));
    return from(p);
  }
};

inline RestorationPlan plan(const ProfiledTimings& t) {
  hc_timings c = t.c();
  hc_plan p;
  check(hc_plan_closed_form(&c, &p));
  return RestorationPlan::from(p);
}
inline double makespan(const RestorationPlan& p, const ProfiledTimings& t) {
  hc_timings c = t.c();
  double out = 0;
  check(hc_makespan(&p.raw, &c, &out));
  return out;
}
inline RestorationPlan brute_force_plan(const ProfiledTimings& t) {
  hc_timings c = t.c();
  hc_plan p;
  check(hc_brute_force_plan(&c, &p));
  return RestorationPlan::from(p);
}
// B200 planner (bounded staging, three-way split); makespan via *out.
inline RestorationPlan plan_three_way(const ProfiledTimings& t, int prefetch_depth,
                                      double* out = nullptr) {
  hc_timings c = t.c();
  hc_plan p;
  double ms = 0;
  check(hc_plan_three_way(&c, prefetch_depth, &p, &ms));
  if (out) *out = ms;
  return RestorationPlan::from(p);
}

// --------------------------------------------------------------- pipeline.hpp
enum class Lane { Io, Compute };

struct TimelineEvent {
  Lane lane;
  int layer = -1;
  std::string kind;
  double start_s = 0;
  double end_s = 0;
};

struct Timeline {
  std::vector<TimelineEvent> events;
  double total_s = 0;
  double fill_s = 0;

  static Timeline from(const hc_timeline& t) {
    static const char* kinds[] = {"fetch_hidden", "fetch_kv", "project", "recompute",
                                  "scatter",      "gather",   "fetch",   "compute"};
    Timeline r;
    r.total_s = t.total_s;
    r.fill_s = t.fill_s;
    for (int i = 0; i < t.n_events; ++i)
      r.events.push_back({Lane(t.events[i].lane), t.events[i].layer, kinds[t.events[i].kind],
                          t.events[i].start_s, t.events[i].end_s});
    return r;
  }
  double lane_busy(Lane lane) const {
    double b = 0;
    for (const auto& e : events)
      if (e.lane == lane) b += e.end_s - e.start_s;
    return b;
  }
  double bubble_fraction() const {
    if (events.empty()) throw std::invalid_argument("bubble_fraction: empty timeline");
    if (total_s <= 0) return 0;
    const double io = lane_busy(Lane::Io), comp = lane_busy(Lane::Compute);
    const double f = ((io > comp ? io : comp) - (io < comp ? io : comp)) / total_s;
    return f < 0 ? 0 : (f > 1 ? 1 : f);
  }
};

struct PipelineJob {
  int layer = -1;
  double io_s = 0;
  double compute_s = 0;
  bool has_io = false;
  bool has_compute = false;
  hc_event_kind io_kind = HC_EV_FETCH;
  hc_event_kind compute_kind = HC_EV_COMPUTE;
};

inline Timeline simulate_pipeline(const std::vector<PipelineJob>& jobs, int prefetch_depth) {
  std::vector<hc_pipeline_job> c;
  for (const auto& j : jobs)
    c.push_back(hc_pipeline_job{j.layer, j.has_io ? 1 : 0, j.has_compute ? 1 : 0, j.io_kind,
                                j.compute_kind, 0, j.io_s, j.compute_s});
  std::vector<hc_timeline> tl(1);
  check(hc_simulate_pipeline(c.data(), int(c.size()), prefetch_depth, tl.data()));
  return Timeline::from(tl[0]);
}

// ---------------------------------------------------------------- storage.hpp
constexpr int kChunkTokens = HC_CHUNK_TOKENS;
enum class StateKind { Hidden, Kv };

struct DevicePool {
  int devices = 1;  // pinned host arenas standing in for the SSD roots
  double bw_bytes_per_s = 0;
  double read_latency_s = 0;
  int count() const { return devices; }
};

struct ChunkKey {
  std::string session_id;
  int layer = 0;
  StateKind kind = StateKind::Hidden;
  int chunk_idx = 0;
};

inline int device_for_chunk(const ChunkKey& key, int device_count) {
  return hc_device_for_chunk(key.layer, key.chunk_idx, device_count);
}

struct LayerChunks {
  int layer = 0;
  StateKind kind = StateKind::Hidden;
  int n_chunks = 0;
  int n_tokens = 0;
};

struct SessionSeed {
  std::string session_id;
  std::uint64_t config_hash = 0;
  int n_layers = 0;
  int d_hidden = 0;
  int elem_bytes = 2;
  RestorationPlan plan;
  std::vector<int> tokens;
  int d_kv = 0;                 // GQA: KV rows are 2*d_kv wide (0 = d_hidden)
  int dtype = HC_DTYPE_BF16;    // 2-byte element codec (HC_DTYPE_F16 = reference fp16)
};

struct SessionManifest {
  std::string session_id;
  std::uint64_t config_hash = 0;
  int n_tokens = 0;
  int n_layers = 0;
  int d_hidden = 0;
  int d_kv = 0;
  int elem_bytes = 2;
  int dtype = HC_DTYPE_BF16;
  int device_count = 0;
  int chunk_tokens = kChunkTokens;
  RestorationPlan plan;
  std::vector<int> tokens;
  std::vector<LayerChunks> layers;
  bool finalized = false;

  const LayerChunks* find(int layer, StateKind kind) const {
    for (const auto& lc : layers)
      if (lc.layer == layer && lc.kind == kind) return &lc;
    return nullptr;
  }
};

class StorageManager {
 public:
  explicit StorageManager(DevicePool pool, std::size_t buffer_capacity_bytes = 256ull << 20)
      : pool_(pool) {
    hc_pool_desc d{pool.devices, 0, pool.bw_bytes_per_s, pool.read_latency_s};
    check(hc_store_create(&d, buffer_capacity_bytes, &s_));
  }
  ~StorageManager() { hc_store_destroy(s_); }
  StorageManager(const StorageManager&) = delete;
  StorageManager& operator=(const StorageManager&) = delete;

  // B200 extension: page-lock arena now, off the save path (hc_store_reserve)
  void reserve(std::size_t bytes) { check(hc_store_reserve(s_, bytes)); }

  void create_session(const SessionSeed& seed) {
    std::vector<int32_t> toks(seed.tokens.begin(), seed.tokens.end());
    hc_session_seed c{seed.session_id.c_str(), seed.config_hash, seed.n_layers, seed.d_hidden,
                      seed.d_kv, seed.elem_bytes, seed.dtype, 0,
                      seed.plan.n_layers() ? &seed.plan.raw : nullptr, toks.data(),
                      int64_t(toks.size())};
    check(hc_store_create_session(s_, &c));
  }
  void reopen_for_append(const std::string& sid, const std::vector<int>& new_tokens) {
    std::vector<int32_t> t(new_tokens.begin(), new_tokens.end());
    check(hc_store_reopen_for_append(s_, sid.c_str(), t.data(), int64_t(t.size())));
  }
  // Host rows (fp32): false on backpressure (storage.cpp:139-142).
  bool snapshot(const std::string& sid, int layer, StateKind kind, const Matrix& rows) {
    hc_status st = hc_store_snapshot(s_, sid.c_str(), layer, int(kind), rows.v.data(),
                                     int64_t(rows.rows), int32_t(rows.cols), HC_DTYPE_F32, 0,
                                     nullptr);
    if (st == HC_EAGAIN) return false;
    check(st);
    return true;
  }
  // Device rows in the session dtype, D2H on `stream` (stage-1 side stream).
  bool snapshot_device(const std::string& sid, int layer, StateKind kind, const void* d_rows,
                       int64_t n_rows, int row_width, int dtype, void* stream) {
    hc_status st = hc_store_snapshot(s_, sid.c_str(), layer, int(kind), d_rows, n_rows,
                                     row_width, dtype, 1, stream);
    if (st == HC_EAGAIN) return false;
    check(st);
    return true;
  }
  // B200 extension: device rows that are tokens [tok_begin, ..) of the layer
  // (a head-sharded rank's own range, hc_store_snapshot_range).
  bool snapshot_device_range(const std::string& sid, int layer, StateKind kind, int64_t tok_begin,
                             const void* d_rows, int64_t n_rows, int row_width, int dtype,
                             void* stream) {
    hc_status st = hc_store_snapshot_range(s_, sid.c_str(), layer, int(kind), tok_begin, d_rows,
                                           n_rows, row_width, dtype, 1, stream);
    if (st == HC_EAGAIN) return false;
    check(st);
    return true;
  }
  std::size_t drain(std::size_t max_chunks = std::size_t(-1)) {
    int64_t f = 0;
    check(hc_store_drain(s_, max_chunks == std::size_t(-1) ? -1 : int64_t(max_chunks), &f));
    return std::size_t(f);
  }
  void drain_all() { check(hc_store_drain_all(s_)); }
  void finalize(const std::string& sid) { check(hc_store_finalize(s_, sid.c_str())); }

  SessionManifest open(const std::string& sid) const {
    hc_manifest m;
    check(hc_store_open(s_, sid.c_str(), &m));
    SessionManifest r;
    r.session_id = m.session_id;
    r.config_hash = m.config_hash;
    r.n_tokens = m.n_tokens;
    r.n_layers = m.n_layers;
    r.d_hidden = m.d_hidden;
    r.d_kv = m.d_kv;
    r.elem_bytes = m.elem_bytes;
    r.dtype = m.dtype;
    r.device_count = m.device_count;
    r.chunk_tokens = m.chunk_tokens;
    r.plan = RestorationPlan::from(m.plan);
    r.finalized = m.finalized != 0;
    std::vector<int32_t> t(size_t(m.n_token_ids));
    int64_t n = 0;
    check(hc_store_tokens(s_, sid.c_str(), t.data(), int64_t(t.size()), &n));
    r.tokens.assign(t.begin(), t.end());
    for (int layer = 0; layer < m.n_layers; ++layer)
      for (StateKind k : {StateKind::Hidden, StateKind::Kv}) {
        int32_t nc = 0, nt = 0;
        if (hc_store_layer_info(s_, sid.c_str(), layer, int(k), &nc, &nt) == HC_OK)
          r.layers.push_back({layer, k, nc, nt});
      }
    return r;
  }

  // Token-ordered reassembly decoded to fp32 (storage.cpp:324-346).
  std::optional<Matrix> read_layer(const SessionManifest& m, int layer, StateKind kind) const {
    const LayerChunks* lc = m.find(layer, kind);
    if (!lc || lc->n_tokens == 0) return std::nullopt;
    const int width = kind == StateKind::Hidden ? m.d_hidden : 2 * m.d_kv;
    const size_t n = size_t(lc->n_tokens) * size_t(width);
    std::vector<uint8_t> raw(n * size_t(m.elem_bytes));
    check(hc_store_read_layer(s_, m.session_id.c_str(), layer, int(kind), raw.data(),
                              int64_t(raw.size()), 0, nullptr));
    Matrix out(size_t(lc->n_tokens), size_t(width));
    for (size_t i = 0; i < n; ++i) out.v[i] = decode(raw.data(), i, m.dtype);
    return out;
  }
  // Device gather of one layer (H2D on `stream`).
  void read_layer_device(const std::string& sid, int layer, StateKind kind, void* d_dst,
                         int64_t bytes, void* stream) const {
    check(hc_store_read_layer(s_, sid.c_str(), layer, int(kind), d_dst, bytes, 1, stream));
  }

  double simulated_read_seconds_tokens(int n_tokens, int width, int elem_bytes) const {
    return hc_store_simulated_read_seconds_tokens(s_, n_tokens, width, elem_bytes);
  }
  void start_daemon() { check(hc_store_start_daemon(s_)); }
  void stop_daemon() { check(hc_store_stop_daemon(s_)); }
  std::size_t buffer_bytes() const { return hc_store_buffer_bytes(s_); }
  std::size_t buffer_capacity() const { return hc_store_buffer_capacity(s_); }
  std::uint64_t backpressure_events() const { return hc_store_backpressure_events(s_); }
  const DevicePool& pool() const { return pool_; }
  hc_store* get() const { return s_; }

 private:
  static float decode(const uint8_t* raw, size_t i, int dtype) {
    if (dtype == HC_DTYPE_F32) {
      float f;
      std::memcpy(&f, raw + 4 * i, 4);
      return f;
    }
    uint16_t h;
    std::memcpy(&h, raw + 2 * i, 2);
    uint32_t x;
    if (dtype == HC_DTYPE_BF16) {
      x = uint32_t(h) << 16;
    } else {  // IEEE binary16 (fp16.hpp:42-68)
      uint32_t sign = (uint32_t(h) & 0x8000u) << 16, exp = (h >> 10) & 0x1Fu, man = h & 0x3FFu;
      if (exp == 0) {
        if (man == 0) {
          x = sign;
        } else {
          int e = -1;
          do {
            ++e;
            man <<= 1;
          } while (!(man & 0x400u));
          x = sign | uint32_t(127 - 15 - e) << 23 | ((man & 0x3FFu) << 13);
        }
      } else if (exp == 31) {
        x = sign | 0x7F800000u | (man << 13);
      } else {
        x = sign | ((exp - 15 + 127) << 23) | (man << 13);
      }
    }
    float f;
    std::memcpy(&f, &x, 4);
    return f;
  }
  DevicePool pool_;
  hc_store* s_ = nullptr;
};

// n x 2d interleaved rows (K then V per token) <-> (K, V) (storage.cpp:67-86).
inline Matrix interleave_kv(const Matrix& k, const Matrix& v) {
  if (k.rows != v.rows || k.cols != v.cols) throw std::invalid_argument("interleave_kv: K/V shape mismatch");
  Matrix rows(k.rows, k.cols * 2);
  for (size_t i = 0; i < k.rows; ++i) {
    std::memcpy(rows.row(i), k.row(i), k.cols * sizeof(float));
    std::memcpy(rows.row(i) + k.cols, v.row(i), k.cols * sizeof(float));
  }
  return rows;
}
inline std::pair<Matrix, Matrix> split_kv(const Matrix& rows) {
  if (rows.cols % 2 != 0) throw std::invalid_argument("split_kv: odd width");
  const size_t d = rows.cols / 2;
  Matrix k(rows.rows, d), v(rows.rows, d);
  for (size_t i = 0; i < rows.rows; ++i) {
    std::memcpy(k.row(i), rows.row(i), d * sizeof(float));
    std::memcpy(v.row(i), rows.row(i) + d, d * sizeof(float));
  }
  return {k, v};
}

// ---------------------------------------------------------------- restore.hpp
struct ThrottleConfig {
  int prefetch_depth = 0;  // 0 = auto (stage every hidden layer within 8 GiB)
  bool timeline = true;
  int split_tokens = 0;    // B200 extension (hc_restore_opts.split_tokens)
  int peer_gather = 0;     // restore_sharded: 0 fused peer-memory K1, 1 copy-engine gather
};

struct RestoreResult {
  Timeline timeline;  // the restored KV lives in the caller's pages
};

// Paged KV cache descriptor: per-layer device pools [num_pages][page_size][d_kv].
struct KvPages {
  hc_kv_pages desc{};
  std::vector<void*> k, v;
  KvPages(int n_layers, int page_size, int num_pages, int d_kv, std::vector<void*> k_layers,
          std::vector<void*> v_layers, int dtype = HC_DTYPE_BF16)
      : k(std::move(k_layers)), v(std::move(v_layers)) {
    desc = hc_kv_pages{n_layers, page_size, num_pages, d_kv, dtype, k.data(), v.data()};
  }
};

// restore (restore.hpp:40-42) on the device: the plan must equal the
// session manifest's (std::invalid_argument otherwise).
inline RestoreResult restore(StorageManager& store, const std::string& session_id,
                             const DeviceWeights& w, const RestorationPlan& plan,
                             const ThrottleConfig& throttle, const KvPages& pages,
                             const int32_t* d_page_table, void* stream = nullptr) {
  hc_restore_opts o{throttle.prefetch_depth, throttle.timeline ? 1 : 0, throttle.split_tokens,
                    0};
  std::vector<hc_timeline> tl(1);
  check(hc_restore(store.get(), session_id.c_str(), w.get(), &plan.raw, &o, &pages.desc,
                   d_page_table, stream, throttle.timeline ? tl.data() : nullptr));
  RestoreResult r;
  if (throttle.timeline) r.timeline = Timeline::from(tl[0]);
  return r;
}

// ------------------------------------------ multi-GPU head-sharded restore
// One rank's member of a head-sharded restore (hc_peer_group): its staging
// slots and flags, exported as an opaque blob that the host hands to every
// other rank by any transport, then import of every rank's blob.
class PeerGroup {
 public:
  PeerGroup(int world, int rank, int device, int d_hidden, int64_t max_rows, int depth = 2) {
    check(hc_peer_group_create(world, rank, device, d_hidden, max_rows, depth, &g_));
  }
  ~PeerGroup() { hc_peer_group_destroy(g_); }
  PeerGroup(const PeerGroup&) = delete;
  PeerGroup& operator=(const PeerGroup&) = delete;
  std::vector<uint8_t> export_blob() const {
    std::vector<uint8_t> b(hc_peer_group_blob_size());
    check(hc_peer_group_export(g_, b.data(), b.size()));
    return b;
  }
  void import_blobs(const std::vector<std::vector<uint8_t>>& blobs) {
    std::vector<const void*> p;
    for (const auto& b : blobs) p.push_back(b.data());
    check(hc_peer_group_import(g_, p.data()));
  }
  hc_peer_group* get() const { return g_; }

 private:
  hc_peer_group* g_ = nullptr;
};

inline std::pair<int64_t, int64_t> shard_range(int64_t n_tokens, int world, int rank) {
  int64_t b = 0, e = 0;
  check(hc_shard_range(n_tokens, world, rank, &b, &e));
  return {b, e};
}
inline std::pair<int, int> shard_heads(int n_kv_heads, int world, int rank) {
  int32_t b = 0, c = 0;
  check(hc_shard_heads(n_kv_heads, world, rank, &b, &c));
  return {b, c};
}

// restore (restore.hpp:40-42) of this rank's KV heads of a head-sharded
// context; every rank calls it with the same plan.
inline RestoreResult restore_sharded(PeerGroup& group, StorageManager& store,
                                     const std::string& session_id, const DeviceWeights& w,
                                     const RestorationPlan& plan, const ThrottleConfig& throttle,
                                     const KvPages& pages, const int32_t* d_page_table,
                                     void* stream = nullptr) {
  hc_restore_opts o{throttle.prefetch_depth, throttle.timeline ? 1 : 0, 0, throttle.peer_gather};
  std::vector<hc_timeline> tl(1);
  check(hc_restore_sharded(group.get(), store.get(), session_id.c_str(), w.get(), &plan.raw, &o,
                           &pages.desc, d_page_table, stream,
                           throttle.timeline ? tl.data() : nullptr));
  RestoreResult r;
  if (throttle.timeline) r.timeline = Timeline::from(tl[0]);
  return r;
}

// profile_hardware (harness.hpp:76-77), measured on the device.
inline ProfiledTimings profile_hardware(const DeviceWeights& w, int n_tokens) {
  hc_timings t{};
  check(hc_profile(w.get(), n_tokens, &t));
  return ProfiledTimings{t.io_h, t.io_kv, t.c_h, t.c_token, t.n_layers};
}


// restore_token_wise (restore.hpp:47-49), the token-wise partition ablation.
inline RestoreResult restore_token_wise(StorageManager& store, const std::string& session_id,
                                        const DeviceWeights& w, int hidden_tokens,
                                        const KvPages& pages, const int32_t* d_page_table,
                                        void* stream = nullptr) {
  std::vector<hc_timeline> tl(1);
  check(hc_restore_token_wise(store.get(), session_id.c_str(), w.get(), hidden_tokens,
                              &pages.desc, d_page_table, stream, tl.data()));
  RestoreResult r;
  r.timeline = Timeline::from(tl[0]);
  return r;
}

// forward_tokens / decode_step (model.hpp:115-120) for a batch of sequences
// continuing their paged caches; next tokens stay on the device.
inline void forward_batch(const DeviceWeights& w, const int32_t* d_tokens,
                          const std::vector<int32_t>& new_lens,
                          const std::vector<int32_t>& start_pos, const KvPages& pages,
                          const int32_t* d_page_tables, int table_stride,
                          void* d_layer_inputs, int32_t* d_next_tokens, void* stream = nullptr) {
  if (new_lens.size() != start_pos.size())
    throw std::invalid_argument("forward_batch: new_lens / start_pos size mismatch");
  check(hc_forward_batch(w.get(), d_tokens, int32_t(new_lens.size()), new_lens.data(),
                         start_pos.data(), &pages.desc, d_page_tables, table_stride,
                         d_layer_inputs, d_next_tokens, stream));
}

// ---------------------------------------------------------------- serving
// Strategy / SavingMode / Request / RequestMetrics / Metrics / RunOptions /
// run (harness.hpp:14-72, trace.hpp:11-19) on the device engine.
enum class Strategy { HCache = HC_STRATEGY_HCACHE, KvOffload = HC_STRATEGY_KV_OFFLOAD,
                      Recompute = HC_STRATEGY_RECOMPUTE, Ideal = HC_STRATEGY_IDEAL };
enum class SavingMode { TwoStage = HC_SAVING_TWO_STAGE, Direct = HC_SAVING_DIRECT,
                        Off = HC_SAVING_OFF };

struct Request {
  std::string session_id;
  int round = 1;
  int history_tokens = 0;
  std::vector<int32_t> context;
  std::vector<int32_t> prompt;
  int output_budget = 1;
  double arrival_s = 0;
};

struct RequestMetrics {
  std::string session_id;
  int round = 1;
  double arrival_s = 0;
  int history_tokens = 0;
  double restore_s = 0, ttft_s = 0, tbt_s = 0;
  int generated = 0;
};

struct Metrics {
  Strategy strategy = Strategy::Ideal;
  std::vector<RequestMetrics> per_request;
  std::vector<std::vector<int32_t>> outputs;
  hc_serve_metrics agg{};  // ttft_p50/p95, tbt_mean/p50/p95, restore tok/s, bytes/token, ...
};

struct RunOptions {
  Strategy strategy = Strategy::HCache;
  SavingMode saving = SavingMode::TwoStage;
  RestorationPlan hcache_plan;  // required for Strategy::HCache
  int page_size = 64;
  int num_pages = 0;  // KV page pool (all layers); 0: sized for the whole trace
  int max_batch = 0;
};

inline Metrics run(const std::vector<Request>& trace, const DeviceWeights& w,
                   StorageManager& store, const RunOptions& opt, void* stream = nullptr) {
  std::vector<hc_request> reqs(trace.size());
  long pages_needed = 0;
  for (size_t i = 0; i < trace.size(); ++i) {
    const Request& r = trace[i];
    reqs[i] = hc_request{r.session_id.c_str(), r.round, int32_t(r.context.size()),
                         r.context.data(), int32_t(r.prompt.size()), r.output_budget,
                         r.prompt.data(), r.arrival_s};
    pages_needed += (r.history_tokens + long(r.context.size()) + long(r.prompt.size()) +
                     r.output_budget + opt.page_size - 1) / opt.page_size;
  }
  hc_serve_opts o{};
  o.strategy = int32_t(opt.strategy);
  o.saving = int32_t(opt.saving);
  o.plan = opt.hcache_plan.raw;
  o.page_size = opt.page_size;
  o.num_pages = opt.num_pages > 0 ? opt.num_pages : int32_t(std::max(1L, pages_needed));
  o.max_batch = opt.max_batch;
  std::vector<hc_request_metrics> per(std::max<size_t>(1, trace.size()));
  size_t total_out = 0;
  for (const auto& r : trace) total_out += size_t(r.output_budget);
  std::vector<int32_t> outs(std::max<size_t>(1, total_out));
  Metrics m;
  m.strategy = opt.strategy;
  check(hc_serve_run(store.get(), w.get(), reqs.data(), int32_t(reqs.size()), &o, per.data(),
                     outs.data(), &m.agg, stream));
  size_t off = 0;
  for (size_t i = 0; i < trace.size(); ++i) {
    const hc_request_metrics& q = per[i];
    m.per_request.push_back(RequestMetrics{trace[i].session_id, q.round, q.arrival_s,
                                           q.history_tokens, q.restore_s, q.ttft_s, q.tbt_s,
                                           q.generated});
    m.outputs.emplace_back(outs.begin() + long(off),
                           outs.begin() + long(off) + trace[i].output_budget);
    off += size_t(trace[i].output_budget);
  }
  return m;
}

}  // namespace hcache_b200
