// recompute.cu -- K6: the RECOMPUTE complement (prefill_layers,
// proj/src/model.cpp:349-356) and full prefill (model.cpp:305-330) on B200.
//
// Per layer (block_forward, model.cpp:102-115), all GEMMs on the shared
// tcgen05 kernel with LayerNorm folded into the epilogue:
//   stats(xb)                         row mean / rstd of the residual stream
//   K1  [W_k;W_v]  LN -> K, V (RoPE K) straight into the paged cache
//   Q   W_q        LN -> Q (RoPE) dense bf16
//   attention      causal, paged K/V (attention.cu)
//   O   W_o        x += mix W_o^T (fp32 residual), xb = bf16(x)
//   stats(xb)
//   FC1 fc1        xb1 = bf16(gelu(LN(x) fc1^T))
//   FC2 fc2        x += xb1 fc2^T, xb = bf16(x)
// x is the fp32 residual stream; xb its bf16 copy feeds the next GEMM and is
// the H_L the save path snapshots.
#include <algorithm>
#include <chrono>
#include <map>
#include <mutex>
#include <tuple>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "kernels.h"
#include "recompute.h"

namespace hc {

namespace {

CUtensorMap tmap(const void* base, int k, int64_t rows, int box_rows) {
  CUtensorMap m;
  if (!make_tmap_kmajor(&m, base, uint64_t(k), uint64_t(rows), uint64_t(k) * 2, uint32_t(box_rows)))
    fail(HC_ECUDA, "cuTensorMapEncodeTiled failed (recompute)");
  return m;
}

int pick_bn(int64_t M, int N, int sms) { return gemm_pick_bn(M, N, sms); }

// HC_HOST_PROFILE=1: host-side enqueue time per forward section, printed at
// exit (diagnostics for the launch-bound decode step).
struct HostProf {
  static constexpr int kN = 12;
  const char* names[kN] = {"setup", "embed", "inputs_copy", "stats", "kv_gemm", "q_gemm",
                           "attention", "o_gemm", "stats2", "fc1", "fc2", "argmax"};
  double t[kN] = {};
  long calls = 0;
  bool on = getenv("HC_HOST_PROFILE") != nullptr;
  ~HostProf() {
    if (!on || !calls) return;
    fprintf(stderr, "[hc host profile] %ld forward calls, us per call:\n", calls);
    for (int i = 0; i < kN; ++i) fprintf(stderr, "  %-12s %9.1f\n", names[i], t[i] * 1e6 / calls);
  }
};
HostProf g_prof;
struct ProfMark {
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  void lap(int i) {
    if (!g_prof.on) return;
    const auto t1 = std::chrono::steady_clock::now();
    g_prof.t[i] += std::chrono::duration<double>(t1 - t0).count();
    t0 = t1;
  }
};

// Weight operands: their tensor maps depend only on (address, shape, box), so
// they are encoded once and reused by every forward / decode step.
CUtensorMap wmap(const void* base, int k, int64_t rows, int box_rows) {
  struct Key {
    const void* base;
    int k;
    int64_t rows;
    int box;
    bool operator<(const Key& o) const {
      return std::tie(base, k, rows, box) < std::tie(o.base, o.k, o.rows, o.box);
    }
  };
  static std::mutex mu;
  static std::map<Key, CUtensorMap> cache;
  const Key key{base, k, rows, box_rows};
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  const CUtensorMap m = tmap(base, k, rows, box_rows);
  std::lock_guard<std::mutex> lk(mu);
  cache.emplace(key, m);
  return m;
}

// tcgen05 attention (default) or the mma.sync kernel (HC_ATTN_TC=0, or page
// sizes the TMA gather cannot express)
bool attention_tc_ok(const KvOut& kv) {
  static const int tc = [] {
    const char* e = getenv("HC_ATTN_TC");
    return e ? atoi(e) : 1;
  }();
  const bool pow2 = !kv.page_table || (kv.page_size >= 8 && (kv.page_size & (kv.page_size - 1)) == 0);
  return tc && pow2;
}

cudaError_t attention(const void* q, int n, int n_heads, int n_kv_heads, int dh, const KvOut& kv,
                      int64_t kv_rows, void* out, cudaStream_t stream) {
  if (attention_tc_ok(kv)) return launch_attention_tc(q, n, n_heads, n_kv_heads, dh, kv, kv_rows, out, stream);
  return launch_attention(q, n, n_heads, n_kv_heads, dh, kv, out, stream);
}

}  // namespace

void forward_impl(const hc_weights* w, const int32_t* d_tokens, int64_t n, int lb, int le,
                  const hc_kv_pages* pages, const int32_t* d_page_table, cudaStream_t stream,
                  const std::function<void(int, bool)>& hook, void* d_layer_inputs,
                  int32_t* next_token, const SeqBatch& sb, int32_t* d_next_tokens,
                  int64_t n_last = 0, bool kv_only_last = false) {
  if (!w || !d_tokens || !pages || !d_page_table) fail(HC_EINVAL, "prefill_layers: null argument");
  const auto& c = w->cfg;
  if (lb < 0 || le > c.n_layers || lb > le) fail(HC_EINVAL, "prefill_layers: bad layer range");
  if (n < 1) fail(HC_EINVAL, "forward: empty sequence");
  if (n_last < 0 || n_last > n || (n_last > 0 && (sb.cu || next_token || d_next_tokens)))
    fail(HC_EINVAL, "forward: bad last-layer row count");
  if (kv_only_last && (next_token || d_next_tokens))
    fail(HC_EINVAL, "forward: the next token needs the last layer's output");
  if (!sb.cu && n > c.max_seq) fail(HC_EINVAL, "forward: sequence exceeds max_seq");
  if (!w->embedding) fail(HC_EINVAL, "prefill_layers: embedding not set");
  // (a head-sharded weight set may run the forward too -- its full block
  // weights hold every head -- into pages of all heads, validated below)
  for (int L = lb; L < le; ++L)
    if (!w->layers[size_t(L)].full) fail(HC_EINVAL, "prefill_layers: full block weights not set");
  validate_pages(w, pages, w->d_kv_all);
  if (pages->dtype != HC_DTYPE_BF16) fail(HC_EINVAL, "prefill_layers: bf16 pages required");
  if (w->d_head != 64 && w->d_head != 128)
    fail(HC_EINVAL, "prefill_layers: attention supports d_head 64 or 128");
  if (c.d_ffn % 32 != 0 || c.d_hidden % 32 != 0)
    fail(HC_EINVAL, "prefill_layers: d_hidden and d_ffn must be multiples of 32");
  ProfMark pm;
  if (g_prof.on) ++g_prof.calls;
  DeviceGuard dg(w->device);
  const int d = c.d_hidden, dffn = c.d_ffn, sms = device_sm_count(w->device);
  const size_t nd = size_t(n) * size_t(d);
  StreamScratch x_buf(nd * 4, stream), xb_buf(nd * 2, stream), q_buf(nd * 2, stream),
      mix_buf(nd * 2, stream), h1_buf(size_t(n) * size_t(dffn) * 2, stream),
      stats(size_t(n) * 2 * 4 + size_t(2 * (le - lb) + 4) * 4, stream),
      xc_buf(c.norm_enabled ? nd * 2 : 0, stream);
  float* x = static_cast<float*>(x_buf.ptr);
  float* mean = static_cast<float*>(stats.ptr);
  float* rstd = mean + n;
  // one mean-shift flag per statistics call (two per layer), zeroed once
  int32_t* flags = reinterpret_cast<int32_t*>(mean + 2 * n);
  int n_flag = 0;
  pm.lap(0);
  HC_CUDA(launch_embed(d_tokens, n, w->embedding, d, x, xb_buf.ptr, stream));
  if (c.norm_enabled && ln_center_enabled())
    HC_CUDA(launch_zero_i32(flags, 2 * (le - lb), stream));
  // LayerNorm statistics of xb + the mean-shifted operand for rows with
  // |mean| >> sigma (launch_center_rows; a no-op unless flagged)
  AltA alt;
  const AltA* altp = nullptr;
  const bool center = c.norm_enabled && ln_center_enabled();
  if (center) altp = &alt;
  // tensor maps and tile widths of the GEMMs over the first `rows` rows
  // (every GEMM of an M-row operand uses the A box and tiles M picks)
  struct Maps {
    int64_t rows = -1;
    CUtensorMap xb, mix, h1, xc;
    int bn_kv = 0, bn_d = 0, bn_f = 0;
  };
  auto make_maps = [&](int64_t rows) {
    Maps mp;
    mp.rows = rows;
    const int ab = gemm_a_box(rows);
    mp.xb = tmap(xb_buf.ptr, d, n, ab);
    mp.mix = tmap(mix_buf.ptr, d, n, ab);
    mp.h1 = tmap(h1_buf.ptr, dffn, n, ab);
    if (center) mp.xc = tmap(xc_buf.ptr, d, n, ab);
    // K/V: the exact path (restores must reproduce these K/V bit for bit);
    // the other projections may split K when the rows are decode-sized
    mp.bn_kv = pick_bn(rows, 2 * w->d_kv_all, sms);
    mp.bn_d = gemm_pick_bn_skinny(rows, d, sms);
    mp.bn_f = gemm_pick_bn_skinny(rows, dffn, sms);
    return mp;
  };
  const Maps full_maps = make_maps(n);
  Maps part_maps;
  auto maps = [&](int64_t rows) -> const Maps* {
    if (rows == n) return &full_maps;
    if (part_maps.rows != rows) part_maps = make_maps(rows);
    return &part_maps;
  };
  auto ln_stats = [&](int64_t rows) {
    if (!center) {
      HC_CUDA(launch_row_stats(xb_buf.ptr, rows, d, d, true, mean, rstd, stream));
      return;
    }
    int32_t* flag = flags + n_flag++;
    alt.flag = flag;  // the GEMMs that follow read this call's flag
    HC_CUDA(launch_row_stats_flagged(xb_buf.ptr, rows, d, d, true, mean, rstd, flag, stream));
    HC_CUDA(launch_center_rows(xb_buf.ptr, rows, d, d, mean, flag, xc_buf.ptr, stream));
  };
  pm.lap(1);
  for (int L = lb; L < le; ++L) {
    const auto& lw = w->layers[size_t(L)];
    // rows of this layer: all n, or only the first n_last tokens of the last
    // layer (a restore recomputing part of its first hidden layer)
    const int64_t m = (L == le - 1 && n_last > 0) ? n_last : n;
    // rows of this layer's output the next layer reads. A restore's
    // RECOMPUTE prefix (kv_only_last) needs only the K/V of its last layer
    // -- the layer after it is restored from its stored input -- so that
    // layer stops after its K/V projection, and when that layer is shortened
    // to n_last rows the layer before it computes only those rows' output
    // (causal: rows [0, n_last) depend on rows [0, n_last) only). Its
    // GEMMs keep the m-row schedule (m_sched), so every element is summed in
    // the full layer's order.
    int64_t mo = m;
    if (kv_only_last && L == le - 1) mo = 0;
    else if (kv_only_last && L == le - 2 && n_last > 0) mo = n_last;
    hook(L, true);
    if (d_layer_inputs)
      HC_CUDA(cudaMemcpyAsync(static_cast<char*>(d_layer_inputs) + size_t(L) * nd * 2, xb_buf.ptr,
                              nd * 2, cudaMemcpyDeviceToDevice, stream));
    // attention block: LN(x) -> K/V (paged) and Q
    pm.lap(2);
    ln_stats(m);
    pm.lap(3);
    KvOut kv = kv_out_pages(pages, L, d_page_table, sb.table_stride, sb.cu, sb.n_seqs);
    kv.seq_start = sb.seq_start;
    // Q, K and V as one GEMM over [W_q;W_k;W_v] when the caller laid the
    // weights out that way (the K/V columns see the same per-element
    // arithmetic as the separate K/V GEMM, so restores stay bit-identical);
    // not for the K/V-only last layer of a restore's prefix, nor for
    // decode-sized steps (there the Q GEMM splits K over the SMs instead)
    const bool fused = lw.wqkv != nullptr && mo > 0 && m > 128;
    {
      const Maps& mk = *maps(m);
      if (center) alt.map = mk.xc;
      if (fused) {
        KvOut kq = kv;
        kq.q_base = q_buf.ptr;
        kq.q_cols = d;
        const int nq = d + 2 * w->d_kv_all;
        const int bn = pick_bn(m, nq, sms);
        HC_CUDA(launch_restore_kv(mk.xb, wmap(lw.wqkv, d, nq, bn), bn, int(m), nq, d, true, kq,
                                  epi_for(w, lw.colsum_qkv, mean, rstd), sms, stream, false,
                                  altp));
      } else {
        HC_CUDA(launch_restore_kv(mk.xb, wmap(lw.wkv_all, d, 2 * w->d_kv_all, mk.bn_kv), mk.bn_kv,
                                  int(m), 2 * w->d_kv_all, d, true, kv,
                                  epi_for(w, lw.colsum_all, mean, rstd), sms, stream, false, altp));
      }
    }
    pm.lap(4);
    if (mo == 0) {  // only this layer's K/V was needed
      hook(L, false);
      pm.lap(10);
      continue;
    }
    // the GEMMs below store mo rows but keep the m-row schedule (m_sched):
    // every element is summed in the order of the full layer's GEMMs
    const Maps& mp = *maps(m);
    if (center) alt.map = mp.xc;
    if (!fused) {
      KvOut qo;
      qo.k_base = q_buf.ptr;
      qo.v_base = q_buf.ptr;
      qo.d_kv = d;  // every column is "K": RoPE applies to all of Q
      qo.cu_seqlens = sb.cu;
      qo.n_seqs = sb.cu ? sb.n_seqs : 1;
      qo.seq_start = sb.seq_start;
      HC_CUDA(launch_restore_kv(mp.xb, wmap(lw.wq, d, d, mp.bn_d), mp.bn_d, int(mo), d, d, true, qo,
                                epi_for(w, lw.colsum_q, mean, rstd), sms, stream, true, altp,
                                int(m)));
    }
    pm.lap(5);
    if (sb.cu && sb.from_zero && attention_tc_ok(kv))
      HC_CUDA(launch_attention_tc_varlen(q_buf.ptr, n, sb.n_seqs, sb.max_new, sb.cu, c.n_heads,
                                         c.n_kv_heads, w->d_head, kv,
                                         int64_t(pages->num_pages) * pages->page_size,
                                         mix_buf.ptr, stream));
    else if (sb.cu)
      HC_CUDA(launch_attention_extend(q_buf.ptr, sb.n_seqs, sb.max_new, sb.cu, sb.seq_start,
                                      c.n_heads, c.n_kv_heads, w->d_head, kv, mix_buf.ptr,
                                      stream));
    else
      HC_CUDA(attention(q_buf.ptr, int(mo), c.n_heads, c.n_kv_heads, w->d_head, kv,
                        int64_t(pages->num_pages) * pages->page_size, mix_buf.ptr, stream));
    pm.lap(6);
    GemmOut resid;
    resid.x = x;
    resid.xb = xb_buf.ptr;
    resid.ldo = d;
    HC_CUDA(launch_gemm_dense(mp.mix, wmap(lw.wo, d, d, mp.bn_d), mp.bn_d, kEpiResid, int(mo), d,
                              d, resid, EpiArgs{}, sms, stream, true, nullptr, int(m)));
    pm.lap(7);
    // FFN block (ffn_forward, model.cpp:290-303)
    ln_stats(mo);
    pm.lap(8);
    GemmOut g1;
    g1.xb = h1_buf.ptr;
    g1.ldo = dffn;
    EpiArgs fold;
    if (c.norm_enabled) {
      fold.row_mean = mean;
      fold.row_rstd = rstd;
      fold.colsum = lw.colsum_fc1;
    }
    HC_CUDA(launch_gemm_dense(mp.xb, wmap(lw.fc1, d, dffn, mp.bn_f), mp.bn_f, kEpiGelu, int(mo),
                              dffn, d, g1, fold, sms, stream, true, altp, int(m)));
    pm.lap(9);
    HC_CUDA(launch_gemm_dense(mp.h1, wmap(lw.fc2, dffn, d, mp.bn_d), mp.bn_d, kEpiResid, int(mo),
                              d, dffn, resid, EpiArgs{}, sms, stream, true, nullptr, int(m)));
    hook(L, false);
    pm.lap(10);
  }
  if (d_next_tokens && sb.cu) {
    // logits on the tensor cores: E [vocab x d] x [hi; lo]^T, fp32 accumulate
    const int B = sb.n_seqs;
    if (2 * B <= 256) {
      const int npad = 2 * B <= 32 ? 32 : 2 * B <= 64 ? 64 : 2 * B <= 128 ? 128 : 256;
      const int vocab = c.vocab_size;
      StreamScratch hl(size_t(2 * B) * size_t(d) * 2, stream),
          lg(size_t(vocab) * size_t(npad) * 4, stream), lgb(size_t(vocab) * size_t(npad) * 2, stream);
      HC_CUDA(launch_hilo_rows(x, sb.cu, B, d, hl.ptr, stream));
      HC_CUDA(cudaMemsetAsync(lg.ptr, 0, size_t(vocab) * size_t(npad) * 4, stream));
      GemmOut go;
      go.x = static_cast<float*>(lg.ptr);
      go.xb = lgb.ptr;
      go.ldo = npad;
      HC_CUDA(launch_gemm_dense(wmap(w->embedding, d, vocab, gemm_a_box(vocab)),
                                tmap(hl.ptr, d, 2 * B, npad), npad, kEpiResid, vocab, npad, d, go,
                                EpiArgs{}, sms, stream));
      HC_CUDA(launch_argmax_pairs(static_cast<float*>(lg.ptr), vocab, npad, B, d_next_tokens,
                                  stream));
    } else {
      HC_CUDA(launch_argmax_rows(w->embedding, c.vocab_size, d, x, sb.cu, sb.n_seqs,
                                 d_next_tokens, stream));
    }
  }
  pm.lap(11);
  if (next_token) {
    StreamScratch tok(sizeof(int32_t), stream);
    HC_CUDA(launch_argmax_logits(w->embedding, c.vocab_size, d, x + size_t(n - 1) * d,
                                 static_cast<int32_t*>(tok.ptr), stream));
    HC_CUDA(cudaMemcpyAsync(next_token, tok.ptr, sizeof(int32_t), cudaMemcpyDeviceToHost, stream));
    HC_CUDA(cudaStreamSynchronize(stream));
  }
}

void prefill_layers_impl(const hc_weights* w, const int32_t* d_tokens, int64_t n, int lb, int le,
                         const hc_kv_pages* pages, const int32_t* d_page_table,
                         cudaStream_t stream, const std::function<void(int, bool)>& hook,
                         void* d_layer_inputs, int32_t* next_token, int64_t n_last,
                         bool kv_only_last) {
  forward_impl(w, d_tokens, n, lb, le, pages, d_page_table, stream, hook, d_layer_inputs,
               next_token, SeqBatch{}, nullptr, n_last, kv_only_last);
}

void forward_batch_dev(const hc_weights* w, const int32_t* d_tokens, int n_seqs, int64_t total,
                       int max_new, const int32_t* d_cu, const int32_t* d_starts,
                       const hc_kv_pages* pages, const int32_t* d_page_tables, int table_stride,
                       void* d_layer_inputs, int32_t* d_next_tokens, cudaStream_t stream) {
  if (!w || n_seqs < 1 || total < 1 || max_new < 1 || !d_cu || !d_starts)
    fail(HC_EINVAL, "forward_batch: bad argument");
  SeqBatch sb;
  sb.n_seqs = n_seqs;
  sb.cu = d_cu;
  sb.seq_start = d_starts;
  sb.max_new = max_new;
  sb.table_stride = table_stride;
  forward_impl(w, d_tokens, total, 0, w->cfg.n_layers, pages, d_page_tables, stream,
               [](int, bool) {}, d_layer_inputs, nullptr, sb, d_next_tokens);
}

void forward_batch_layers(const hc_weights* w, const int32_t* d_tokens, int n_seqs, int64_t total,
                          int max_new, const int32_t* d_cu, const int32_t* d_starts,
                          const hc_kv_pages* pages, const int32_t* d_page_tables,
                          int table_stride, int lb, int le, cudaStream_t stream,
                          const std::function<void(int, bool)>& hook, bool kv_only_last) {
  if (!w || n_seqs < 1 || total < 1 || max_new < 1 || !d_cu || !d_starts)
    fail(HC_EINVAL, "forward_batch: bad argument");
  SeqBatch sb;
  sb.n_seqs = n_seqs;
  sb.cu = d_cu;
  sb.seq_start = d_starts;
  sb.max_new = max_new;
  sb.table_stride = table_stride;
  sb.from_zero = true;  // the RECOMPUTE prefix of a restore: every session from position 0
  forward_impl(w, d_tokens, total, lb, le, pages, d_page_tables, stream, hook, nullptr, nullptr,
               sb, nullptr, 0, kv_only_last);
}

void forward_batch(const hc_weights* w, const int32_t* d_tokens, int n_seqs,
                   const int32_t* new_lens, const int32_t* start_pos, const hc_kv_pages* pages,
                   const int32_t* d_page_tables, int table_stride, void* d_layer_inputs,
                   int32_t* d_next_tokens, cudaStream_t stream) {
  if (!w || n_seqs < 1 || !new_lens || !start_pos) fail(HC_EINVAL, "forward_batch: bad argument");
  if (!pages) fail(HC_EINVAL, "forward_batch: null pages");
  std::vector<int32_t> meta(size_t(2 * n_seqs + 1));
  int64_t total = 0;
  int max_new = 0;
  for (int s = 0; s < n_seqs; ++s) {
    if (new_lens[s] < 1) fail(HC_EINVAL, "forward: empty sequence");
    if (start_pos[s] < 0) fail(HC_EINVAL, "forward_batch: negative start position");
    if (int64_t(start_pos[s]) + new_lens[s] > w->cfg.max_seq)
      fail(HC_EINVAL, "forward: sequence exceeds max_seq");
    if (int64_t(start_pos[s]) + new_lens[s] > int64_t(table_stride) * pages->page_size)
      fail(HC_EINVAL, "forward_batch: page table row too short");
    meta[size_t(s)] = int32_t(total);
    meta[size_t(n_seqs + 1 + s)] = start_pos[s];
    total += new_lens[s];
    max_new = std::max(max_new, new_lens[s]);
  }
  meta[size_t(n_seqs)] = int32_t(total);
  DeviceGuard dg(w->device);
  StreamScratch dmeta(meta.size() * sizeof(int32_t), stream);
  HC_CUDA(cudaMemcpyAsync(dmeta.ptr, meta.data(), meta.size() * sizeof(int32_t),
                          cudaMemcpyHostToDevice, stream));
  SeqBatch sb;
  sb.n_seqs = n_seqs;
  sb.cu = static_cast<int32_t*>(dmeta.ptr);
  sb.seq_start = sb.cu + n_seqs + 1;
  sb.max_new = max_new;
  sb.table_stride = table_stride;
  sb.from_zero = std::all_of(start_pos, start_pos + n_seqs, [](int32_t p) { return p == 0; });
  forward_impl(w, d_tokens, total, 0, w->cfg.n_layers, pages, d_page_tables, stream,
               [](int, bool) {}, d_layer_inputs, nullptr, sb, d_next_tokens);
}

double recompute_layer_seconds(const hc_weights* w, int n, double warm_s) {
  if (!w || !w->embedding || n < 1) return 0.0;
  int layer = -1;
  for (int l = 0; l < w->cfg.n_layers; ++l)
    if (w->layers[size_t(l)].full) {
      layer = l;
      break;
    }
  if (layer < 0 || (w->d_head != 64 && w->d_head != 128)) return 0.0;
  // up to 4 consecutive layers per call, as a restore's prefix runs them:
  // the per-call embedding and setup are not part of a layer's cost
  int nl = 1;
  while (nl < 4 && layer + nl < w->cfg.n_layers && w->layers[size_t(layer + nl)].full) ++nl;
  DeviceGuard dg(w->device);
  cudaStream_t s = nullptr;
  const size_t kvb = size_t(n) * size_t(w->d_kv_all) * 2;
  StreamScratch kbuf(kvb, s), vbuf(kvb, s), tok(sizeof(int32_t) * size_t(n), s),
      table(sizeof(int32_t), s);
  HC_CUDA(cudaMemsetAsync(tok.ptr, 0, sizeof(int32_t) * size_t(n), s));
  HC_CUDA(cudaMemsetAsync(table.ptr, 0, sizeof(int32_t), s));
  std::vector<void*> kp(size_t(w->cfg.n_layers), kbuf.ptr), vp(size_t(w->cfg.n_layers), vbuf.ptr);
  hc_kv_pages pages{w->cfg.n_layers, n, 1, w->d_kv_all, HC_DTYPE_BF16, kp.data(), vp.data()};
  cudaEvent_t a, b;
  HC_CUDA(cudaEventCreate(&a));
  HC_CUDA(cudaEventCreate(&b));
  auto one = [&] {
    prefill_layers_impl(w, static_cast<int32_t*>(tok.ptr), n, layer, layer + nl, &pages,
                        static_cast<int32_t*>(table.ptr), s, [](int, bool) {});
  };
  auto timed = [&](int reps) {
    HC_CUDA(cudaEventRecord(a, s));
    for (int i = 0; i < reps; ++i) one();
    HC_CUDA(cudaEventRecord(b, s));
    HC_CUDA(cudaEventSynchronize(b));
    float ms = 0;
    HC_CUDA(cudaEventElapsedTime(&ms, a, b));
    return double(ms) * 1e-3;
  };
  one();  // pool allocations, tensor-map encodes
  // run back to back until the clocks settle (a restore keeps the tensor
  // cores busy for tens of ms; its power-capped clock, not the boost clock,
  // sets the recompute cost), then take the mean of the next launches
  double warm = 0;
  while (warm < warm_s) warm += timed(8);
  const int reps = 16;
  const double sec = timed(reps) / reps / nl;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return sec;
}

}  // namespace hc

using namespace hc;

extern "C" {

hc_status hc_prefill_layers(const hc_weights* w, const int32_t* d_tokens, int64_t n,
                            int32_t layer_begin, int32_t layer_end, const hc_kv_pages* pages,
                            const int32_t* d_page_table, void* stream) {
  return guard([&] {
    NvtxRange r("hc_prefill_layers");
    // prefill_layers (model.cpp:349-356) discards the last block's output:
    // only the K/V of its last layer are observable
    prefill_layers_impl(w, d_tokens, n, layer_begin, layer_end, pages, d_page_table,
                        as_stream(stream), [](int, bool) {}, nullptr, nullptr, 0, true);
  });
}

hc_status hc_attention_dense(const void* d_q, int32_t n, int32_t n_heads, int32_t n_kv_heads,
                             int32_t d_head, const void* d_k, const void* d_v, int32_t d_kv,
                             void* d_out, void* stream) {
  return guard([&] {
    if (!d_q || !d_k || !d_v || !d_out) fail(HC_EINVAL, "attention: null argument");
    if (n_kv_heads < 1 || n_heads % n_kv_heads || d_kv != n_kv_heads * d_head)
      fail(HC_EINVAL, "attention: bad head geometry");
    KvOut kv;
    kv.k_base = const_cast<void*>(d_k);
    kv.v_base = const_cast<void*>(d_v);
    kv.d_kv = d_kv;
    HC_CUDA(attention(d_q, n, n_heads, n_kv_heads, d_head, kv, n, d_out, as_stream(stream)));
  });
}

hc_status hc_gemm_epilogue(int32_t mode, const void* d_a, const void* d_b, int32_t m, int32_t n,
                           int32_t k, float* d_x, void* d_xb, const float* d_mean,
                           const float* d_rstd, const float* d_colsum, int32_t device,
                           void* stream) {
  return guard([&] {
    const bool split_k = (mode & HC_GEMM_SPLIT_K) != 0;  // decode-shape K split (tests)
    mode &= ~HC_GEMM_SPLIT_K;
    if (mode != kEpiResid && mode != kEpiGelu) fail(HC_EINVAL, "gemm: mode must be 1 or 2");
    if (!d_a || !d_b || !d_xb || (mode == kEpiResid && !d_x)) fail(HC_EINVAL, "gemm: null argument");
    if (n % 32 || k % 8) fail(HC_EINVAL, "gemm: n % 32 and k % 8 must be 0");
    require_sm100(device);
    DeviceGuard dg(device);
    const bool split = split_k || getenv("HC_GEMM_SPLIT") != nullptr;
    const int sms = device_sm_count(device);
    const int bn = split ? gemm_pick_bn_skinny(m, n, sms) : pick_bn(m, n, sms);
    GemmOut g;
    g.x = d_x;
    g.xb = d_xb;
    g.ldo = n;
    EpiArgs e;
    if (d_mean && d_rstd && d_colsum) {
      e.row_mean = d_mean;
      e.row_rstd = d_rstd;
      e.colsum = d_colsum;
    }
    HC_CUDA(launch_gemm_dense(tmap(d_a, k, m, gemm_a_box(m)), tmap(d_b, k, n, bn), bn, mode, m, n, k, g, e,
                              sms, as_stream(stream), split));
  });
}

hc_status hc_forward_batch(const hc_weights* w, const int32_t* d_tokens, int32_t n_seqs,
                           const int32_t* new_lens, const int32_t* start_pos,
                           const hc_kv_pages* pages, const int32_t* d_page_tables,
                           int32_t table_stride, void* d_layer_inputs, int32_t* d_next_tokens,
                           void* stream) {
  return guard([&] {
    forward_batch(w, d_tokens, n_seqs, new_lens, start_pos, pages, d_page_tables, table_stride,
                  d_layer_inputs, d_next_tokens, as_stream(stream));
  });
}

hc_status hc_kv_gather_rows(const hc_kv_pages* pages, int32_t layer, const int32_t* d_page_table,
                            int32_t pos0, int64_t n_rows, void* d_rows, void* stream) {
  return guard([&] {
    if (!pages || !d_page_table || !d_rows || pos0 < 0 || n_rows < 0)
      fail(HC_EINVAL, "kv_gather_rows: bad argument");
    if (layer < 0 || layer >= pages->n_layers) fail(HC_EINVAL, "kv_gather_rows: bad layer");
    if (pages->dtype != HC_DTYPE_BF16 || pages->d_kv % 8)
      fail(HC_EINVAL, "kv_gather_rows: bf16 pages with d_kv % 8 == 0 required");
    KvOut kv;
    kv.k_base = pages->k_layers[layer];
    kv.v_base = pages->v_layers[layer];
    kv.d_kv = pages->d_kv;
    kv.page_size = pages->page_size;
    kv.page_table = d_page_table;
    HC_CUDA(launch_kv_gather(kv, pos0, n_rows, d_rows, as_stream(stream)));
  });
}

hc_status hc_prefill(const hc_weights* w, const int32_t* d_tokens, int64_t n,
                     const hc_kv_pages* pages, const int32_t* d_page_table, void* d_layer_inputs,
                     int32_t* next_token, void* stream) {
  return guard([&] {
    NvtxRange r("hc_prefill");
    if (!w) fail(HC_EINVAL, "prefill: null weights");
    prefill_layers_impl(w, d_tokens, n, 0, w->cfg.n_layers, pages, d_page_table,
                        as_stream(stream), [](int, bool) {}, d_layer_inputs, next_token);
  });
}

}  // extern "C"
