// ref_shim.cpp -- extern "C" entry points over the UNMODIFIED reference
// library (compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libhcache_ref.so). TEST INFRASTRUCTURE: used to pin the oracle
// restatement (tests/test_oracle.py), to generate tests/golden/*, and as the
// CPU baseline timed by bench.py (--impl reference / cpu_baseline).
// This file is our own glue; no reference source is copied into the repo.
#include <chrono>
#include <cstring>
#include <filesystem>
#include <thread>
#include <vector>

#include "hcache/harness.hpp"
#include "hcache/model.hpp"
#include "hcache/pipeline.hpp"
#include "hcache/planner.hpp"
#include "hcache/restore.hpp"
#include "hcache/storage.hpp"
#include "hcache/trace.hpp"
#include "hcache/fp16.hpp"

using namespace hcache;

namespace {

ModelConfig make_cfg(int n_layers, int d, int n_heads, int d_ffn, int vocab,
                     int max_seq, int norm, int rope) {
  ModelConfig c;
  c.n_layers = n_layers;
  c.d_hidden = d;
  c.n_heads = n_heads;
  c.d_ffn = d_ffn;
  c.vocab_size = vocab;
  c.max_seq = max_seq;
  c.norm_enabled = norm != 0;
  c.rope_enabled = rope != 0;
  return c;
}

void put(float*& dst, const Matrix& m) {
  std::memcpy(dst, m.v.data(), m.v.size() * sizeof(float));
  dst += m.v.size();
}

Matrix from(const float* p, std::size_t r, std::size_t c) {
  Matrix m(r, c);
  std::memcpy(m.v.data(), p, r * c * sizeof(float));
  return m;
}

// One-layer WeightSet carrying only wk/wv: project_hidden_to_kv reads nothing
// else (model.cpp:219-235). n_heads := n_kv_heads gives the GQA projection.
WeightSet kv_only(const float* wk, const float* wv, int d, int d_kv, int n_kv_heads,
                  int norm, int rope) {
  WeightSet ws;
  ws.config.n_layers = 1;
  ws.config.d_hidden = d;
  ws.config.n_heads = n_kv_heads;
  ws.config.norm_enabled = norm != 0;
  ws.config.rope_enabled = rope != 0;
  ws.layers.resize(1);
  ws.layers[0].wk = from(wk, std::size_t(d_kv), std::size_t(d));
  ws.layers[0].wv = from(wv, std::size_t(d_kv), std::size_t(d));
  return ws;
}

}  // namespace

extern "C" {

int ref_init_model(int n_layers, int d, int n_heads, int d_ffn, int vocab,
                   unsigned long long seed, float* out) {
  try {
    WeightSet ws = init_model(make_cfg(n_layers, d, n_heads, d_ffn, vocab, 4096, 1, 1), seed);
    put(out, ws.embedding);
    for (const auto& lw : ws.layers) {
      put(out, lw.wq);
      put(out, lw.wk);
      put(out, lw.wv);
      put(out, lw.wo);
      put(out, lw.fc1);
      put(out, lw.fc2);
    }
    return 0;
  } catch (...) {
    return -1;
  }
}

// prefill with init_model(seed) weights; outputs may be null.
int ref_prefill(int n_layers, int d, int n_heads, int d_ffn, int vocab, int max_seq,
                int norm, int rope, unsigned long long seed, const int* tokens, int n,
                float* layer_inputs, float* k_out, float* v_out, float* final_hidden) {
  try {
    WeightSet ws = init_model(make_cfg(n_layers, d, n_heads, d_ffn, vocab, max_seq, norm, rope), seed);
    PrefillResult pr = prefill(ws, TokenSeq{std::vector<int>(tokens, tokens + n)});
    for (int L = 0; L < n_layers; ++L) {
      if (layer_inputs) {
        float* p = layer_inputs + std::size_t(L) * n * d;
        put(p, pr.layer_inputs[std::size_t(L)]);
      }
      if (k_out) {
        float* p = k_out + std::size_t(L) * n * d;
        put(p, pr.kv.layers[std::size_t(L)].k);
      }
      if (v_out) {
        float* p = v_out + std::size_t(L) * n * d;
        put(p, pr.kv.layers[std::size_t(L)].v);
      }
    }
    if (final_hidden) put(final_hidden, pr.final_hidden);
    return pr.next_token;
  } catch (...) {
    return -1;
  }
}

int ref_prefill_layers(int n_layers, int d, int n_heads, int d_ffn, int vocab, int max_seq,
                       int norm, int rope, unsigned long long seed, const int* tokens, int n,
                       int lb, int le, float* k_out, float* v_out) {
  try {
    WeightSet ws = init_model(make_cfg(n_layers, d, n_heads, d_ffn, vocab, max_seq, norm, rope), seed);
    KVCache kv;
    prefill_layers(ws, TokenSeq{std::vector<int>(tokens, tokens + n)}, lb, le, kv);
    for (int L = lb; L < le; ++L) {
      float* pk = k_out + std::size_t(L) * n * d;
      float* pv = v_out + std::size_t(L) * n * d;
      put(pk, kv.layers[std::size_t(L)].k);
      put(pv, kv.layers[std::size_t(L)].v);
    }
    return 0;
  } catch (...) {
    return -1;
  }
}

int ref_project(const float* h, int n, int d, const float* wk, const float* wv, int d_kv,
                int n_kv_heads, int start_pos, int norm, int rope, float* k_out,
                float* v_out) {
  try {
    WeightSet ws = kv_only(wk, wv, d, d_kv, n_kv_heads, norm, rope);
    LayerKV kv = project_hidden_to_kv(ws, 0, from(h, std::size_t(n), std::size_t(d)), start_pos);
    std::memcpy(k_out, kv.k.v.data(), kv.k.v.size() * sizeof(float));
    std::memcpy(v_out, kv.v.v.data(), kv.v.v.size() * sizeof(float));
    return 0;
  } catch (...) {
    return -1;
  }
}

// The reference projection fanned out over row slices on nthreads host
// threads (legal: the function is pure). Returns seconds.
double ref_project_timed(const float* h, int n, int d, const float* wk, const float* wv,
                         int d_kv, int n_kv_heads, int start_pos, int norm, int rope,
                         float* k_out, float* v_out, int nthreads) {
  WeightSet ws = kv_only(wk, wv, d, d_kv, n_kv_heads, norm, rope);
  if (nthreads < 1) nthreads = 1;
  std::vector<Matrix> slices;
  std::vector<int> begins;
  int per = (n + nthreads - 1) / nthreads;
  for (int b = 0; b < n; b += per) {
    int e = std::min(n, b + per);
    slices.push_back(from(h + std::size_t(b) * d, std::size_t(e - b), std::size_t(d)));
    begins.push_back(b);
  }
  std::vector<LayerKV> outs(slices.size());
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> th;
  for (std::size_t i = 0; i < slices.size(); ++i)
    th.emplace_back([&, i] { outs[i] = project_hidden_to_kv(ws, 0, slices[i], start_pos + begins[i]); });
  for (auto& t : th) t.join();
  double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (k_out && v_out) {
    for (std::size_t i = 0; i < slices.size(); ++i) {
      std::size_t off = std::size_t(begins[i]) * std::size_t(d_kv);
      std::memcpy(k_out + off, outs[i].k.v.data(), outs[i].k.v.size() * sizeof(float));
      std::memcpy(v_out + off, outs[i].v.v.data(), outs[i].v.v.size() * sizeof(float));
    }
  }
  return dt;
}

int ref_apply_rope(float* x, int rows, int cols, int n_heads, int start_pos) {
  try {
    Matrix m = from(x, std::size_t(rows), std::size_t(cols));
    std::vector<int> pos(static_cast<std::size_t>(rows));
    for (int i = 0; i < rows; ++i) pos[std::size_t(i)] = start_pos + i;
    apply_rope(m, pos, n_heads);
    std::memcpy(x, m.v.data(), m.v.size() * sizeof(float));
    return 0;
  } catch (...) {
    return -1;
  }
}

unsigned short ref_float_to_half(float f) { return float_to_half(f); }
float ref_half_to_float(unsigned short h) { return half_to_float(h); }

int ref_device_for_chunk(int layer, int chunk_idx, int device_count) {
  return device_for_chunk(ChunkKey{"s", layer, StateKind::Hidden, chunk_idx}, device_count);
}

// planner: complement 0 NONE, 1 KV_OFFLOAD, 2 RECOMPUTE
static int comp_code(Complement c) {
  return c == Complement::None ? 0 : (c == Complement::KvOffload ? 1 : 2);
}
static Complement comp_of(int c) {
  return c == 0 ? Complement::None : (c == 1 ? Complement::KvOffload : Complement::Recompute);
}

int ref_plan(double io_h, double io_kv, double c_h, double c_token, int n_layers, int brute,
             int* l_h, int* l_o, int* comp, double* makespan_out) {
  try {
    ProfiledTimings t{io_h, io_kv, c_h, c_token, n_layers};
    RestorationPlan p = brute ? brute_force_plan(t) : plan(t);
    *l_h = p.l_h;
    *l_o = p.l_o;
    *comp = comp_code(p.complement);
    *makespan_out = makespan(p, t);
    return 0;
  } catch (...) {
    return -1;
  }
}

int ref_plan_serialize(int n_layers, int l_h, int comp, char* buf, int cap) {
  try {
    std::string s = RestorationPlan::make(n_layers, l_h, comp_of(comp)).serialize();
    std::snprintf(buf, std::size_t(cap), "%s", s.c_str());
    return 0;
  } catch (...) {
    return -1;
  }
}

// simulate_pipeline: events out as (lane, layer, start, end) after the
// reference's stable sort. Returns event count (or -1).
int ref_simulate_pipeline(int n_jobs, const int* layer, const double* io_s,
                          const double* compute_s, const int* has_io, const int* has_compute,
                          int depth, int* ev_lane, int* ev_layer, double* ev_start,
                          double* ev_end, double* total_s, double* fill_s) {
  try {
    std::vector<PipelineJob> jobs(static_cast<std::size_t>(n_jobs));
    for (int j = 0; j < n_jobs; ++j) {
      jobs[std::size_t(j)].layer = layer[j];
      jobs[std::size_t(j)].io_s = io_s[j];
      jobs[std::size_t(j)].compute_s = compute_s[j];
      jobs[std::size_t(j)].has_io = has_io[j] != 0;
      jobs[std::size_t(j)].has_compute = has_compute[j] != 0;
    }
    Timeline tl = simulate_pipeline(jobs, depth);
    int k = 0;
    for (const auto& e : tl.events) {
      ev_lane[k] = e.lane == Lane::Io ? 0 : 1;
      ev_layer[k] = e.layer;
      ev_start[k] = e.start_s;
      ev_end[k] = e.end_s;
      ++k;
    }
    *total_s = tl.total_s;
    *fill_s = tl.fill_s;
    return k;
  } catch (...) {
    return -1;
  }
}

int ref_conversation_history(int n_sessions, int rounds, unsigned long long seed, int* out) {
  try {
    TraceParams p;
    p.n_sessions = n_sessions;
    p.rounds = rounds;
    Trace tr = gen_trace(TraceKind::Conversation, p, seed);
    // requests are stable-sorted by arrival; report in (session, round) order
    int k = 0;
    for (int s = 0; s < n_sessions; ++s)
      for (const auto& r : tr.requests)
        if (r.session_id == "sess" + std::to_string(s)) out[k++] = r.history_tokens;
    return k;
  } catch (...) {
    return -1;
  }
}

// gen_trace (trace.cpp:55-100) in arrival order: per request
// meta[6*i..] = {session index, round, history, n_context, n_prompt, budget},
// arrival[i], hash[i] = FNV-1a over the context then prompt token ids (int32).
int ref_gen_trace(int kind, int n_sessions, int rounds, unsigned long long seed, int max_out,
                  int* meta, double* arrival, unsigned long long* hash) {
  try {
    TraceParams p;
    p.n_sessions = n_sessions;
    p.rounds = rounds;
    Trace tr = gen_trace(kind == 0 ? TraceKind::Conversation : TraceKind::LongContext, p, seed);
    int k = 0;
    for (const auto& r : tr.requests) {
      if (k >= max_out) return -1;
      meta[6 * k + 0] = std::stoi(r.session_id.substr(4));
      meta[6 * k + 1] = r.round;
      meta[6 * k + 2] = r.history_tokens;
      meta[6 * k + 3] = int(r.context.size());
      meta[6 * k + 4] = int(r.prompt.size());
      meta[6 * k + 5] = r.output_budget;
      arrival[k] = r.arrival_s;
      unsigned long long h = 1469598103934665603ull;
      auto mix = [&](const std::vector<int>& v) {
        for (int t : v) {
          const int32_t x = t;
          const unsigned char* b = reinterpret_cast<const unsigned char*>(&x);
          for (int j = 0; j < 4; ++j) {
            h ^= b[j];
            h *= 1099511628211ull;
          }
        }
      };
      mix(r.context);
      mix(r.prompt);
      hash[k] = h;
      ++k;
    }
    return k;
  } catch (...) {
    return -1;
  }
}

// The reference restore() as shipped: WallClock mode, one compute thread and
// one IO thread, store on `root` (use tmpfs). Config and seed as given, plan
// all-hidden, tokens (i*11+1)%vocab. Returns timeline.total_s (or -1).
double ref_restore_wall(int n_layers, int d, int n_heads, int d_ffn, int vocab, int n,
                        int elem_bytes, unsigned long long seed, const char* root,
                        double* max_abs_diff_out) {
  try {
    ModelConfig c = make_cfg(n_layers, d, n_heads, d_ffn, vocab, std::max(4096, n), 1, 1);
    c.elem_bytes = elem_bytes;
    WeightSet ws = init_model(c, seed);
    std::vector<int> toks(static_cast<std::size_t>(n));
    for (int i = 0; i < n; ++i) toks[std::size_t(i)] = (i * 11 + 1) % vocab;
    PrefillResult pr = prefill(ws, TokenSeq{toks});
    DevicePool pool;
    std::filesystem::path base(root);
    std::filesystem::remove_all(base);
    pool.roots.push_back(base / "dev0");
    StorageManager store(pool);
    RestorationPlan p = RestorationPlan::make(n_layers, n_layers, Complement::None);
    SessionSeed s{"bench", c.hash(), n_layers, d, elem_bytes, p, toks};
    store.create_session(s);
    for (int L = 0; L < n_layers; ++L)
      while (!store.snapshot("bench", L, StateKind::Hidden, pr.layer_inputs[std::size_t(L)]))
        store.drain();
    store.finalize("bench");
    ThrottleConfig th;
    th.mode = ThrottleConfig::Mode::WallClock;
    RestoreResult r = restore(store, "bench", ws, p, th);
    double worst = 0;
    for (int L = 0; L < n_layers; ++L) {
      worst = std::max(worst, max_abs_diff(r.kv.layers[std::size_t(L)].k, pr.kv.layers[std::size_t(L)].k));
      worst = std::max(worst, max_abs_diff(r.kv.layers[std::size_t(L)].v, pr.kv.layers[std::size_t(L)].v));
    }
    if (max_abs_diff_out) *max_abs_diff_out = worst;
    std::filesystem::remove_all(base);
    return r.timeline.total_s;
  } catch (...) {
    return -1;
  }
}

}  // extern "C"
