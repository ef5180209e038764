// capi_core.cpp -- C ABI: errors, config, weights, K1 projection entry points,
// KV scatter, synthetic fill, chunk indexing.
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.h"
#include "kernels.h"
#include "weights.h"

namespace hc {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& m) { g_last_error = m; }
void clear_last_error() { g_last_error.clear(); }

int device_sm_count(int dev) {
  static std::mutex mu;
  static std::vector<int> cache;
  std::lock_guard<std::mutex> lk(mu);
  if (dev >= int(cache.size())) cache.resize(size_t(dev) + 1, 0);
  if (!cache[size_t(dev)]) {
    int v = 0;
    HC_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
    cache[size_t(dev)] = v;
    // every compute path passes here first: keep freed stream-ordered scratch
    // in the pool instead of returning it to the driver at each synchronize
    cudaMemPool_t pool;
    HC_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t thresh = UINT64_MAX;
    HC_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thresh));
  }
  return cache[size_t(dev)];
}

void require_sm100(int dev) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
    fail(HC_ECUDA, "no CUDA device: the B200 restoration path has no CPU fallback");
  if (dev < 0 || dev >= n) fail(HC_EINVAL, "device index out of range");
  int major = 0;
  HC_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  if (major != 10) fail(HC_ECUDA, "sm_100-class (B200) GPU required");
}

static void validate_config(const hc_model_config* c) {
  // ModelConfig::validate (model.cpp:140-150) + GQA
  if (!c) fail(HC_EINVAL, "ModelConfig: null");
  if (c->n_layers < 1 || c->d_hidden < 1 || c->n_heads < 1 || c->d_ffn < 1 ||
      c->vocab_size < 1 || c->max_seq < 1)
    fail(HC_EINVAL, "ModelConfig: all counts must be >= 1");
  if (c->d_hidden % c->n_heads != 0)
    fail(HC_EINVAL, "ModelConfig: d_hidden not divisible by n_heads");
  if (c->rope_enabled && (c->d_hidden / c->n_heads) % 2 != 0)
    fail(HC_EINVAL, "ModelConfig: rope needs even d_head");
  if (c->elem_bytes != 2 && c->elem_bytes != 4)
    fail(HC_EINVAL, "ModelConfig: elem_bytes must be 2 or 4");
  int kvh = c->n_kv_heads ? c->n_kv_heads : c->n_heads;
  if (kvh < 1 || c->n_heads % kvh != 0)
    fail(HC_EINVAL, "ModelConfig: n_heads not divisible by n_kv_heads");
  if (c->n_layers > HC_MAX_LAYERS) fail(HC_EINVAL, "ModelConfig: too many layers");
}

EpiArgs epi_for(const hc_weights* w, const float* colsum, const float* mean, const float* rstd) {
  EpiArgs e;
  if (w->cfg.norm_enabled) {
    e.row_mean = mean;
    e.row_rstd = rstd;
    e.colsum = colsum;
  }
  if (w->cfg.rope_enabled) {
    e.rope = w->rope;
    e.d_head = w->d_head;
    e.rope_rows = w->rope_rows;
  }
  return e;
}

// [W_k;W_v] tensor map with a bn-row box: the cached 256/128-row maps, else
// encoded for the narrow decode-sized tiles.
CUtensorMap weight_map(const hc_weights::Layer& L, int bn, int d, int rows) {
  if (bn == 256) return L.tm256;
  if (bn == 128) return L.tm128;
  CUtensorMap m;
  if (!make_tmap_kmajor_cached(&m, L.wkv, uint64_t(d), uint64_t(rows), uint64_t(d) * 2,
                               uint32_t(bn)))
    fail(HC_ECUDA, "cuTensorMapEncodeTiled failed for the weight operand");
  return m;
}

void project_rows(const hc_weights* w, int layer, const void* d_hidden, int64_t n_rows,
                  const KvOut& out, cudaStream_t stream, const float* pre_stats,
                  const int32_t* pre_flag, const void* pre_centered) {
  if (layer < 0 || layer >= w->cfg.n_layers) fail(HC_EINVAL, "project: layer out of range");
  const auto& L = w->layers[size_t(layer)];
  if (!L.ready) fail(HC_EINVAL, "project: layer weights not set");
  if (n_rows <= 0) return;
  if (!d_hidden) fail(HC_EINVAL, "project: null hidden states");
  if ((reinterpret_cast<uintptr_t>(d_hidden) & 15) != 0)
    fail(HC_EINVAL, "project: hidden states must be 16-byte aligned");
  const int d = w->cfg.d_hidden;
  const int N = 2 * w->d_kv;
  if (w->cfg.rope_enabled && !out.cu_seqlens && int64_t(out.start_pos) + n_rows > w->rope_rows)
    fail(HC_EINVAL, "project: positions exceed max_seq");
  const bool norm = w->cfg.norm_enabled != 0;
  const bool need = norm && !pre_stats;
  if (!ln_center_enabled()) pre_flag = nullptr;
  // statistics (+ the centering flag) unless the caller computed them
  StreamScratch stats(need ? size_t(n_rows) * 2 * sizeof(float) + 16 : 0, stream);
  float* mean = need ? static_cast<float*>(stats.ptr) : const_cast<float*>(pre_stats);
  const float* rstd = mean ? mean + n_rows : nullptr;
  const int32_t* flag =
      need && ln_center_enabled() ? reinterpret_cast<int32_t*>(mean + 2 * n_rows) : pre_flag;
  if (need && flag) {
    HC_CUDA(launch_zero_i32(const_cast<int32_t*>(flag), 1, stream));
    HC_CUDA(launch_row_stats_flagged(d_hidden, n_rows, d, d, true, mean, mean + n_rows,
                                     const_cast<int32_t*>(flag), stream));
  } else if (need) {
    HC_CUDA(launch_row_stats(d_hidden, n_rows, d, d, true, mean, mean + n_rows, stream));
  }
  const uint32_t abox = uint32_t(gemm_a_box(n_rows));
  CUtensorMap tmA;
  if (!make_tmap_kmajor_cached(&tmA, d_hidden, uint64_t(d), uint64_t(n_rows), uint64_t(d) * 2,
                               abox))
    fail(HC_ECUDA, "cuTensorMapEncodeTiled failed for the hidden-state operand");
  // rows with |mean| >> sigma: K1 reads a mean-shifted copy (a no-op kernel
  // and an unused map unless the statistics raised the flag)
  const bool own_center = norm && flag && !(pre_flag && pre_centered);
  StreamScratch centered(own_center ? size_t(n_rows) * size_t(d) * 2 : 0, stream);
  AltA alt;
  if (norm && flag) {
    const void* cbuf = own_center ? centered.ptr : pre_centered;
    if (own_center)
      HC_CUDA(launch_center_rows(d_hidden, n_rows, d, d, mean, flag, centered.ptr, stream));
    if (!make_tmap_kmajor_cached(&alt.map, cbuf, uint64_t(d), uint64_t(n_rows), uint64_t(d) * 2,
                                 abox))
      fail(HC_ECUDA, "cuTensorMapEncodeTiled failed for the centered operand");
    alt.flag = flag;
  }
  const int sms = device_sm_count(w->device);
  const int bn = gemm_pick_bn(n_rows, N, sms);
  HC_CUDA(launch_restore_kv(tmA, weight_map(L, bn, d, N), bn, int(n_rows), N, d, true, out,
                            epi_for(w, L.colsum, mean, rstd), sms, stream, false,
                            norm && flag ? &alt : nullptr));
}

KvOut kv_out_pages(const hc_kv_pages* pages, int layer, const int32_t* page_table,
                   int table_stride, const int32_t* cu_seqlens, int n_seqs) {
  KvOut o;
  o.k_base = pages->k_layers[layer];
  o.v_base = pages->v_layers[layer];
  o.d_kv = pages->d_kv;
  o.page_size = pages->page_size;
  o.page_table = page_table;
  o.table_stride = table_stride;
  o.cu_seqlens = cu_seqlens;
  o.n_seqs = cu_seqlens ? n_seqs : 1;
  o.out_f32 = pages->dtype == HC_DTYPE_F32 ? 1 : 0;
  return o;
}

void validate_pages(const hc_weights* w, const hc_kv_pages* pages, int d_kv_expected) {
  if (!pages || !pages->k_layers || !pages->v_layers) fail(HC_EINVAL, "kv pages: null");
  if (pages->n_layers != w->cfg.n_layers) fail(HC_EINVAL, "kv pages: layer count mismatch");
  if (pages->d_kv != d_kv_expected) fail(HC_EINVAL, "kv pages: d_kv mismatch");
  if (pages->page_size < 1 || pages->num_pages < 1) fail(HC_EINVAL, "kv pages: bad geometry");
  if (pages->dtype != HC_DTYPE_BF16 && pages->dtype != HC_DTYPE_F32)
    fail(HC_EINVAL, "kv pages: dtype must be bf16 or f32");
}

}  // namespace hc

using namespace hc;

extern "C" {

const char* hc_last_error(void) { return g_last_error.c_str(); }
const char* hc_version(void) { return "hcache-b200 0.1 (sm_100a)"; }
int32_t hc_abi_version(void) { return HC_ABI_VERSION; }

int32_t hc_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

hc_status hc_config_validate(const hc_model_config* cfg) {
  return guard([&] { validate_config(cfg); });
}

uint64_t hc_config_hash(const hc_model_config* c) {
  // ModelConfig::hash (model.cpp:152-168); n_kv_heads mixed only for GQA so
  // MHA hashes equal the reference's.
  uint64_t h = 1469598103934665603ull;
  auto mix = [&h](uint64_t x) {
    h ^= x;
    h *= 1099511628211ull;
  };
  mix(uint64_t(c->n_layers));
  mix(uint64_t(c->d_hidden));
  mix(uint64_t(c->n_heads));
  mix(uint64_t(c->d_ffn));
  mix(uint64_t(c->vocab_size));
  mix(uint64_t(c->max_seq));
  mix(uint64_t(c->elem_bytes));
  mix(uint64_t(c->norm_enabled ? 1 : 2));
  mix(uint64_t(c->rope_enabled ? 1 : 2));
  if (c->n_kv_heads && c->n_kv_heads != c->n_heads) mix(uint64_t(c->n_kv_heads) + 1000);
  return h;
}

hc_status hc_weights_create(const hc_model_config* cfg, int32_t kv_head_begin,
                            int32_t kv_head_count, int32_t device, hc_weights** out) {
  return guard([&] {
    if (!out) fail(HC_EINVAL, "weights: null out");
    *out = nullptr;
    validate_config(cfg);
    const int kvh = cfg->n_kv_heads ? cfg->n_kv_heads : cfg->n_heads;
    if (kv_head_begin < 0 || kv_head_count < 1 || kv_head_begin + kv_head_count > kvh)
      fail(HC_EINVAL, "weights: KV head range out of bounds");
    const int d_head = cfg->d_hidden / cfg->n_heads;
    if ((kv_head_count * d_head) % 32 != 0)
      fail(HC_EINVAL, "weights: local KV width must be a multiple of 32");
    if (cfg->d_hidden % 8 != 0) fail(HC_EINVAL, "weights: d_hidden must be a multiple of 8");
    require_sm100(device);
    DeviceGuard dg(device);
    auto* w = new hc_weights();
    w->cfg = *cfg;
    w->cfg.n_kv_heads = kvh;
    w->device = device;
    w->head_begin = kv_head_begin;
    w->head_count = kv_head_count;
    w->d_head = d_head;
    w->d_kv = kv_head_count * d_head;
    w->d_kv_all = kvh * d_head;
    w->layers.resize(size_t(cfg->n_layers));
    try {
      if (cfg->rope_enabled) {
        // coefficients exactly as apply_rope computes them (model.cpp:207-209)
        const int half = d_head / 2;
        std::vector<double> freq(static_cast<size_t>(half));
        for (int t = 0; t < half; ++t)
          freq[size_t(t)] = std::pow(10000.0, -2.0 * double(t) / double(d_head));
        std::vector<float2> tab(static_cast<size_t>(cfg->max_seq) * static_cast<size_t>(half));
        for (int p = 0; p < cfg->max_seq; ++p)
          for (int t = 0; t < half; ++t) {
            double a = double(p) * freq[size_t(t)];
            tab[size_t(p) * half + t] = make_float2(float(std::cos(a)), float(std::sin(a)));
          }
        HC_CUDA(cudaMalloc(&w->rope, tab.size() * sizeof(float2)));
        HC_CUDA(cudaMemcpy(w->rope, tab.data(), tab.size() * sizeof(float2),
                           cudaMemcpyHostToDevice));
        w->rope_rows = cfg->max_seq;
      }
    } catch (...) {
      hc_weights_destroy(w);
      throw;
    }
    *out = w;
  });
}

void hc_weights_destroy(hc_weights* w) {
  if (!w) return;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(w->device);
  for (auto& L : w->layers) {
    if (L.colsum) cudaFree(L.colsum);
    if (L.colsum_all) cudaFree(L.colsum_all);
    if (L.colsum_q) cudaFree(L.colsum_q);
    if (L.colsum_fc1) cudaFree(L.colsum_fc1);
    if (L.colsum_qkv) cudaFree(L.colsum_qkv);
  }
  if (w->rope) cudaFree(w->rope);
  if (prev >= 0) cudaSetDevice(prev);
  delete w;
}

hc_status hc_weights_set_layer_kv(hc_weights* w, int32_t layer, const void* d_wkv) {
  return guard([&] {
    if (!w || !d_wkv) fail(HC_EINVAL, "set_layer_kv: null argument");
    if (layer < 0 || layer >= w->cfg.n_layers) fail(HC_EINVAL, "set_layer_kv: bad layer");
    if ((reinterpret_cast<uintptr_t>(d_wkv) & 15) != 0)
      fail(HC_EINVAL, "set_layer_kv: weights must be 16-byte aligned");
    DeviceGuard dg(w->device);
    auto& L = w->layers[size_t(layer)];
    const int rows = 2 * w->d_kv, d = w->cfg.d_hidden;
    if (!L.colsum) HC_CUDA(cudaMalloc(&L.colsum, size_t(rows) * sizeof(float)));
    HC_CUDA(launch_colsum(d_wkv, rows, d, true, L.colsum, nullptr));
    HC_CUDA(cudaStreamSynchronize(nullptr));
    if (!make_tmap_kmajor(&L.tm256, d_wkv, uint64_t(d), uint64_t(rows), uint64_t(d) * 2, 256) ||
        !make_tmap_kmajor(&L.tm128, d_wkv, uint64_t(d), uint64_t(rows), uint64_t(d) * 2, 128))
      fail(HC_ECUDA, "cuTensorMapEncodeTiled failed for the weight operand");
    L.wkv = d_wkv;
    L.ready = true;
  });
}

hc_status hc_weights_set_layer_full(hc_weights* w, int32_t layer, const void* d_wq,
                                   const void* d_wkv, const void* d_wo, const void* d_fc1,
                                   const void* d_fc2) {
  return guard([&] {
    if (!w || !d_wq || !d_wkv || !d_wo || !d_fc1 || !d_fc2)
      fail(HC_EINVAL, "set_layer_full: null argument");
    if (layer < 0 || layer >= w->cfg.n_layers) fail(HC_EINVAL, "set_layer_full: bad layer");
    DeviceGuard dg(w->device);
    auto& L = w->layers[size_t(layer)];
    const int rows = 2 * w->d_kv_all, d = w->cfg.d_hidden;
    for (auto p : {d_wq, d_wkv, d_wo, d_fc1, d_fc2})
      if ((reinterpret_cast<uintptr_t>(p) & 15) != 0)
        fail(HC_EINVAL, "set_layer_full: weights must be 16-byte aligned");
    if (!L.colsum_all) HC_CUDA(cudaMalloc(&L.colsum_all, size_t(rows) * sizeof(float)));
    if (!L.colsum_q) HC_CUDA(cudaMalloc(&L.colsum_q, size_t(d) * sizeof(float)));
    if (!L.colsum_fc1) HC_CUDA(cudaMalloc(&L.colsum_fc1, size_t(w->cfg.d_ffn) * sizeof(float)));
    HC_CUDA(launch_colsum(d_wkv, rows, d, true, L.colsum_all, nullptr));
    HC_CUDA(launch_colsum(d_wq, d, d, true, L.colsum_q, nullptr));
    HC_CUDA(launch_colsum(d_fc1, w->cfg.d_ffn, d, true, L.colsum_fc1, nullptr));
    // [W_q ; W_k ; W_v] contiguous: one fused Q/K/V GEMM per recompute layer
    // (tiles of 256 columns never straddle the Q | K boundary)
    L.wqkv = nullptr;
    if (static_cast<const char*>(d_wkv) == static_cast<const char*>(d_wq) + size_t(d) * d * 2 &&
        d % 256 == 0 && qkv_fusion_enabled()) {
      if (!L.colsum_qkv)
        HC_CUDA(cudaMalloc(&L.colsum_qkv, size_t(d + rows) * sizeof(float)));
      HC_CUDA(cudaMemcpy(L.colsum_qkv, L.colsum_q, size_t(d) * sizeof(float),
                         cudaMemcpyDeviceToDevice));
      HC_CUDA(cudaMemcpy(L.colsum_qkv + d, L.colsum_all, size_t(rows) * sizeof(float),
                         cudaMemcpyDeviceToDevice));
      L.wqkv = d_wq;
    }
    HC_CUDA(cudaStreamSynchronize(nullptr));
    L.wq = d_wq;
    L.wkv_all = d_wkv;
    L.wo = d_wo;
    L.fc1 = d_fc1;
    L.fc2 = d_fc2;
    L.full = true;
  });
}

hc_status hc_weights_set_embedding(hc_weights* w, const void* d_embedding) {
  return guard([&] {
    if (!w || !d_embedding) fail(HC_EINVAL, "set_embedding: null argument");
    w->embedding = d_embedding;
  });
}

hc_status hc_project_hidden_to_kv(const hc_weights* w, int32_t layer, const void* d_hidden,
                                  int64_t n_rows, int32_t start_pos, void* d_k, void* d_v,
                                  int32_t out_dtype, void* stream) {
  return guard([&] {
    if (!w || !d_k || !d_v) fail(HC_EINVAL, "project: null argument");
    if (out_dtype != HC_DTYPE_BF16 && out_dtype != HC_DTYPE_F32)
      fail(HC_EINVAL, "project: out_dtype must be bf16 or f32");
    if (start_pos < 0) fail(HC_EINVAL, "project: negative start_pos");
    DeviceGuard dg(w->device);
    KvOut o;
    o.k_base = d_k;
    o.v_base = d_v;
    o.d_kv = w->d_kv;
    o.start_pos = start_pos;
    o.out_f32 = out_dtype == HC_DTYPE_F32;
    project_rows(w, layer, d_hidden, n_rows, o, as_stream(stream));
  });
}

}  // extern "C"

namespace hc {
// Ragged batches restart positions at 0 per sequence, so K1's RoPE rows are
// bounded by the longest sequence. Only when the concatenated rows exceed the
// table can a sequence do so; then the offsets are read back (synchronously)
// and checked, so no launch reads past the RoPE table.
void check_seq_positions(const hc_weights* w, const int32_t* d_cu_seqlens, int n_seqs,
                         int64_t n_rows, cudaStream_t stream) {
  if (!w->cfg.rope_enabled || !d_cu_seqlens || n_rows <= w->rope_rows) return;
  std::vector<int32_t> cu(size_t(n_seqs) + 1);
  HC_CUDA(cudaMemcpyAsync(cu.data(), d_cu_seqlens, sizeof(int32_t) * cu.size(),
                          cudaMemcpyDeviceToHost, stream));
  HC_CUDA(cudaStreamSynchronize(stream));
  for (int i = 0; i < n_seqs; ++i)
    if (cu[size_t(i) + 1] - cu[size_t(i)] > w->rope_rows)
      fail(HC_EINVAL, "project: a sequence exceeds max_seq (RoPE table)");
}
}  // namespace hc

extern "C" {

hc_status hc_project_to_pages(const hc_weights* w, int32_t layer, const void* d_hidden,
                              int64_t n_rows, const int32_t* d_cu_seqlens, int32_t n_seqs,
                              const hc_kv_pages* pages, const int32_t* d_page_table,
                              int32_t table_stride, void* stream) {
  return guard([&] {
    if (!w || !d_page_table) fail(HC_EINVAL, "project_to_pages: null argument");
    validate_pages(w, pages, w->d_kv);
    if (d_cu_seqlens && n_seqs < 1) fail(HC_EINVAL, "project_to_pages: n_seqs < 1");
    DeviceGuard dg(w->device);
    check_seq_positions(w, d_cu_seqlens, n_seqs, n_rows, as_stream(stream));
    project_rows(w, layer, d_hidden, n_rows,
                 kv_out_pages(pages, layer, d_page_table, table_stride, d_cu_seqlens, n_seqs),
                 as_stream(stream));
  });
}

hc_status hc_kv_scatter_to_pages(const void* d_rows, int64_t n_rows, int32_t layer,
                                 const int32_t* d_cu_seqlens, int32_t n_seqs,
                                 const hc_kv_pages* pages, const int32_t* d_page_table,
                                 int32_t table_stride, void* stream) {
  return guard([&] {
    if (!d_rows || !pages || !d_page_table) fail(HC_EINVAL, "kv_scatter: null argument");
    if (layer < 0 || layer >= pages->n_layers) fail(HC_EINVAL, "kv_scatter: bad layer");
    if (pages->dtype != HC_DTYPE_BF16 || pages->d_kv % 8 != 0)
      fail(HC_EINVAL, "kv_scatter: bf16 pages with d_kv % 8 == 0 required");
    KvOut o = kv_out_pages(pages, layer, d_page_table, table_stride, d_cu_seqlens, n_seqs);
    HC_CUDA(launch_kv_scatter(d_rows, n_rows, o, as_stream(stream)));
  });
}

hc_status hc_fill_symmetric(void* d_dst, int64_t n, uint64_t seed, uint64_t offset, float bound,
                            int32_t dtype, void* stream) {
  return guard([&] {
    if (!d_dst && n > 0) fail(HC_EINVAL, "fill_symmetric: null destination");
    if (dtype < 0 || dtype > 2) fail(HC_EINVAL, "fill_symmetric: bad dtype");
    HC_CUDA(launch_fill_symmetric(d_dst, n, seed, offset, bound, dtype, as_stream(stream)));
  });
}

hc_status hc_bench_project(const hc_weights* w, int32_t layer, const void* d_hidden,
                           int64_t n_rows, int32_t iters, void* stream, double* stats_ms,
                           double* k1_ms) {
  return guard([&] {
    if (!w || !d_hidden || iters < 1 || n_rows < 1) fail(HC_EINVAL, "bench_project: bad argument");
    if (layer < 0 || layer >= w->cfg.n_layers || !w->layers[size_t(layer)].ready)
      fail(HC_EINVAL, "bench_project: layer weights not set");
    DeviceGuard dg(w->device);
    cudaStream_t s = as_stream(stream);
    const auto& L = w->layers[size_t(layer)];
    const int d = w->cfg.d_hidden, N = 2 * w->d_kv;
    StreamScratch stats(size_t(n_rows) * 2 * sizeof(float), s);
    StreamScratch kv(size_t(n_rows) * size_t(N) * 2, s);
    float* mean = static_cast<float*>(stats.ptr);
    KvOut o;
    o.k_base = kv.ptr;
    o.v_base = static_cast<char*>(kv.ptr) + size_t(n_rows) * size_t(w->d_kv) * 2;
    o.d_kv = w->d_kv;
    CUtensorMap tmA;
    if (!make_tmap_kmajor(&tmA, d_hidden, uint64_t(d), uint64_t(n_rows), uint64_t(d) * 2,
                          uint32_t(gemm_a_box(n_rows))))
      fail(HC_ECUDA, "cuTensorMapEncodeTiled failed");
    const int sms = device_sm_count(w->device);
    const int bn = gemm_pick_bn(n_rows, N, sms);
    const CUtensorMap tmB = weight_map(L, bn, d, N);
    std::vector<cudaEvent_t> ev(size_t(3 * iters));
    for (auto& e : ev) HC_CUDA(cudaEventCreate(&e));
    for (int i = 0; i < iters; ++i) {
      HC_CUDA(cudaEventRecord(ev[size_t(3 * i)], s));
      HC_CUDA(launch_row_stats(d_hidden, n_rows, d, d, true, mean, mean + n_rows, s));
      HC_CUDA(cudaEventRecord(ev[size_t(3 * i + 1)], s));
      HC_CUDA(launch_restore_kv(tmA, tmB, bn, int(n_rows), N, d, true, o,
                                epi_for(w, L.colsum, mean, mean + n_rows), sms, s));
      HC_CUDA(cudaEventRecord(ev[size_t(3 * i + 2)], s));
    }
    HC_CUDA(cudaStreamSynchronize(s));
    double a = 0, b = 0;
    for (int i = 0; i < iters; ++i) {
      float x = 0, y = 0;
      HC_CUDA(cudaEventElapsedTime(&x, ev[size_t(3 * i)], ev[size_t(3 * i + 1)]));
      HC_CUDA(cudaEventElapsedTime(&y, ev[size_t(3 * i + 1)], ev[size_t(3 * i + 2)]));
      a += x;
      b += y;
    }
    for (auto& e : ev) cudaEventDestroy(e);
    if (stats_ms) *stats_ms = a / iters;
    if (k1_ms) *k1_ms = b / iters;
  });
}

int32_t hc_chunk_tokens(void) { return HC_CHUNK_TOKENS; }

int32_t hc_device_for_chunk(int32_t layer, int32_t chunk_idx, int32_t device_count) {
  // storage.cpp:29-31: round robin, start device rotated per layer
  if (device_count <= 0) return -1;
  return (layer + chunk_idx) % device_count;
}

}  // extern "C"
