// C++ facade tests: the reference's own test cases (proj/tests/test_planner.cpp,
// test_storage.cpp, test_restore.cpp timeline arithmetic) written against
// hcache_b200.hpp exactly as they are written against hcache::, plus a device
// restore when a B200 is present ("gpu" argument).
#include <cuda_runtime.h>

#include <sys/wait.h>
#include <unistd.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <ctime>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "hcache_b200.hpp"

using namespace hcache_b200;

static int g_fail = 0, g_checks = 0;
#define CHECK(x)                                                          \
  do {                                                                    \
    ++g_checks;                                                           \
    if (!(x)) {                                                           \
      ++g_fail;                                                           \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #x);            \
    }                                                                     \
  } while (0)
#define CHECK_THROWS_AS(expr, T)                                          \
  do {                                                                    \
    ++g_checks;                                                           \
    bool ok = false;                                                      \
    try {                                                                 \
      expr;                                                               \
    } catch (const T&) {                                                  \
      ok = true;                                                          \
    } catch (...) {                                                       \
    }                                                                     \
    if (!ok) {                                                            \
      ++g_fail;                                                           \
      std::printf("FAIL %s:%d: %s does not throw %s\n", __FILE__, __LINE__, #expr, #T); \
    }                                                                     \
  } while (0)
static bool approx(double a, double b, double eps = 1e-12) {
  return std::fabs(a - b) <= eps * std::max(1.0, std::fabs(b));
}

static ProfiledTimings timings(double io_h, double io_kv, double c_h, double c_token, int n) {
  ProfiledTimings t;
  t.io_h = io_h;
  t.io_kv = io_kv;
  t.c_h = c_h;
  t.c_token = c_token;
  t.n_layers = n;
  return t;
}

static void planner_tests() {
  // test_planner.cpp:24-36
  ProfiledTimings t = timings(0.26, 0.52, 0.28, 1.9, 32);
  RestorationPlan p = plan(t);
  CHECK(p.l_h == 31 && p.l_o == 1 && p.complement == Complement::KvOffload);
  CHECK(approx(makespan(p, t), 8.68));
  CHECK(p.layer_assignment.front() == LayerMethod::Hidden);
  CHECK(p.layer_assignment.back() == LayerMethod::KvOffload);
  // :38-49
  t = timings(0.5, 1.0, 0.3, 1.0, 48);
  p = plan(t);
  CHECK(p.l_h == 40 && p.l_o == 8 && p.complement == Complement::Recompute);
  CHECK(p.layer_assignment[8] == LayerMethod::Hidden);
  CHECK(approx(makespan(p, t), 20.0));
  // :60-79
  std::mt19937_64 rng(12345);
  std::uniform_real_distribution<double> u(0.05, 2.0);
  std::uniform_int_distribution<int> layers(1, 60);
  for (int it = 0; it < 1000; ++it) {
    double io_h = u(rng);
    ProfiledTimings r = timings(io_h, 2 * io_h, u(rng), u(rng), layers(rng));
    r.c_token = std::max(r.c_token, r.c_h);
    double mc = makespan(plan(r), r), mb = makespan(brute_force_plan(r), r);
    double stage = std::max({r.io_h, r.io_kv, r.c_h, r.c_token});
    CHECK(mb <= mc + 1e-12 && mc <= mb + stage + 1e-9);
  }
  // :91-99, :101-105
  RestorationPlan q = RestorationPlan::parse(RestorationPlan::make(48, 40, Complement::Recompute).serialize());
  CHECK(q.l_h == 40 && q.l_o == 8 && q.complement == Complement::Recompute);
  CHECK_THROWS_AS(RestorationPlan::parse("garbage"), std::runtime_error);
  CHECK_THROWS_AS(timings(0, 1, 1, 1, 4).validate(), std::invalid_argument);
  CHECK_THROWS_AS(RestorationPlan::make(4, 2, Complement::None), std::invalid_argument);
  // B200 three-way planner never loses to the closed form at unbounded depth
  double ms = 0;
  RestorationPlan tw = plan_three_way(timings(0.61e-3, 1.22e-3, 0.20e-3, 1.27e-3, 32), 32, &ms);
  CHECK(ms <= makespan(plan(timings(0.61e-3, 1.22e-3, 0.20e-3, 1.27e-3, 32)),
                       timings(0.61e-3, 1.22e-3, 0.20e-3, 1.27e-3, 32)) * 1.0001);
  CHECK(tw.n_layers() == 32);
}

static void pipeline_tests() {
  // test_restore.cpp:90-126 timeline arithmetic via simulate_pipeline
  const double io = 256.0 * 64 * 4 / 1e9;
  auto jobs = [&](double c) {
    std::vector<PipelineJob> j;
    for (int L = 0; L < 4; ++L) j.push_back({L, io, c, true, true, HC_EV_FETCH_HIDDEN, HC_EV_PROJECT});
    return j;
  };
  Timeline a = simulate_pipeline(jobs(io), 1);
  CHECK(approx(a.total_s, 5 * io, 1e-9) && approx(a.fill_s, io, 1e-9));
  CHECK(a.bubble_fraction() < 0.25);
  Timeline b = simulate_pipeline(jobs(io / 2), 1);
  CHECK(approx(b.total_s, 4.5 * io, 1e-9) && approx(b.bubble_fraction(), 4.0 / 9.0, 1e-9));
}

static Matrix pattern(int rows, int cols, float scale = 1e-3f, float shift = 0.0f) {
  Matrix m(static_cast<size_t>(rows), static_cast<size_t>(cols));
  for (size_t i = 0; i < m.v.size(); ++i) m.v[i] = scale * float(int(i % 2001) - 1000) + shift;
  return m;
}

static SessionSeed seed(const std::string& id, int d, int n_layers, int eb = 4) {
  SessionSeed s;
  s.session_id = id;
  s.config_hash = 99;
  s.n_layers = n_layers;
  s.d_hidden = d;
  s.elem_bytes = eb;
  s.plan = RestorationPlan::make(n_layers, n_layers, Complement::None);
  s.tokens = {1, 2, 3};
  return s;
}

static void storage_tests() {
  {  // test_storage.cpp:69-86
    StorageManager store(DevicePool{3});
    store.create_session(seed("s", 32, 1));
    store.snapshot("s", 0, StateKind::Hidden, pattern(130, 32));
    store.finalize("s");
    SessionManifest m = store.open("s");
    const LayerChunks* lc = m.find(0, StateKind::Hidden);
    CHECK(lc && lc->n_tokens == 130 && lc->n_chunks == 3 && m.n_tokens == 130);
  }
  {  // :101-121 fp32 round trip, hidden + KV
    StorageManager store(DevicePool{2});
    store.create_session(seed("s", 48, 2));
    Matrix h = pattern(200, 48), k = pattern(200, 48, 2e-3f), v = pattern(200, 48, -1e-3f);
    store.snapshot("s", 0, StateKind::Hidden, h);
    store.snapshot("s", 1, StateKind::Kv, interleave_kv(k, v));
    store.finalize("s");
    SessionManifest m = store.open("s");
    auto h2 = store.read_layer(m, 0, StateKind::Hidden);
    CHECK(h2.has_value() && *h2 == h);
    auto kv2 = store.read_layer(m, 1, StateKind::Kv);
    CHECK(kv2.has_value());
    auto back = split_kv(*kv2);
    CHECK(back.first == k && back.second == v);
    CHECK(m.tokens == std::vector<int>({1, 2, 3}));
  }
  {  // :123-134 fp16 (the reference codec)
    StorageManager store(DevicePool{2});
    SessionSeed s = seed("s", 32, 1, 2);
    s.dtype = HC_DTYPE_F16;
    store.create_session(s);
    Matrix h = pattern(100, 32);
    store.snapshot("s", 0, StateKind::Hidden, h);
    store.finalize("s");
    auto h2 = store.read_layer(store.open("s"), 0, StateKind::Hidden);
    double err = 0;
    for (size_t i = 0; i < h.v.size(); ++i) err = std::max(err, double(std::fabs(h2->v[i] - h.v[i])));
    CHECK(err > 0 && err < 1e-3);
  }
  {  // :154-177 finalize idempotent, open before finalize throws, absent layer
    StorageManager store(DevicePool{1});
    store.create_session(seed("s", 16, 3));
    store.snapshot("s", 1, StateKind::Hidden, pattern(10, 16));
    store.drain_all();
    CHECK_THROWS_AS(store.open("s"), std::runtime_error);
    store.finalize("s");
    store.finalize("s");
    SessionManifest m = store.open("s");
    CHECK(m.finalized && m.n_tokens == 10);
    CHECK(!store.read_layer(m, 0, StateKind::Hidden).has_value());
    CHECK(!store.read_layer(m, 1, StateKind::Kv).has_value());
  }
  {  // :199-216 append
    StorageManager store(DevicePool{2});
    Matrix all = pattern(150, 32);
    Matrix a(90, 32), b(60, 32);
    std::memcpy(a.v.data(), all.v.data(), a.v.size() * 4);
    std::memcpy(b.v.data(), all.v.data() + a.v.size(), b.v.size() * 4);
    store.create_session(seed("s", 32, 1));
    store.snapshot("s", 0, StateKind::Hidden, a);
    store.finalize("s");
    store.reopen_for_append("s", {7, 8});
    CHECK_THROWS_AS(store.open("s"), std::runtime_error);
    store.snapshot("s", 0, StateKind::Hidden, b);
    store.finalize("s");
    SessionManifest m = store.open("s");
    CHECK(m.n_tokens == 150 && m.tokens == std::vector<int>({1, 2, 3, 7, 8}));
    CHECK(*store.read_layer(m, 0, StateKind::Hidden) == all);
  }
  {  // :218-230 backpressure
    StorageManager store(DevicePool{1}, 4 * 1024);
    store.create_session(seed("s", 16, 1));
    CHECK(store.snapshot("s", 0, StateKind::Hidden, pattern(40, 16)));
    CHECK(!store.snapshot("s", 0, StateKind::Hidden, pattern(40, 16)));
    CHECK(store.backpressure_events() == 1);
    store.drain();
    CHECK(store.snapshot("s", 0, StateKind::Hidden, pattern(40, 16)));
  }
  {  // :579-588 validation
    StorageManager store(DevicePool{1});
    store.create_session(seed("s", 16, 1));
    CHECK_THROWS_AS(store.snapshot("nope", 0, StateKind::Hidden, pattern(4, 16)), std::runtime_error);
    CHECK_THROWS_AS(store.snapshot("s", 0, StateKind::Hidden, pattern(4, 8)), std::invalid_argument);
    CHECK_THROWS_AS(store.create_session(seed("s", 16, 1)), std::runtime_error);
  }
  // chunk placement (storage.cpp:29-31)
  for (int L = 0; L < 3; ++L)
    for (int c = 0; c < 20; ++c) CHECK(device_for_chunk({"s", L, StateKind::Hidden, c}, 4) == (L + c) % 4);
}

static void gpu_tests() {
  // all-hidden restore into pages == dense projection, bit for bit
  const int L = 2, d = 256, heads = 4, n = 300, page = 32;
  ModelConfig cfg;
  cfg.n_layers = L;
  cfg.d_hidden = d;
  cfg.n_heads = heads;
  cfg.elem_bytes = 2;
  DeviceWeights w(cfg);
  std::vector<void*> wkv(L), hid(L), kp(L), vp(L);
  const int n_pages = (n + page - 1) / page;
  for (int l = 0; l < L; ++l) {
    cudaMalloc(&wkv[l], size_t(2 * d) * d * 2);
    cudaMalloc(&hid[l], size_t(n) * d * 2);
    cudaMalloc(&kp[l], size_t(n_pages) * page * d * 2);
    cudaMalloc(&vp[l], size_t(n_pages) * page * d * 2);
    check(hc_fill_symmetric(wkv[l], int64_t(2 * d) * d, 1234 + l, 0, 0.0625f, HC_DTYPE_BF16, nullptr));
    check(hc_fill_symmetric(hid[l], int64_t(n) * d, 7 + l, 0, 1.7320508f, HC_DTYPE_BF16, nullptr));
    w.set_layer_kv(l, wkv[l]);
  }
  StorageManager store(DevicePool{2});
  SessionSeed s = seed("g", d, L, 2);
  store.create_session(s);
  for (int l = 0; l < L; ++l)
    CHECK(store.snapshot_device("g", l, StateKind::Hidden, hid[l], n, d, HC_DTYPE_BF16, nullptr));
  store.finalize("g");
  std::vector<int32_t> table(n_pages);
  for (int i = 0; i < n_pages; ++i) table[size_t(i)] = n_pages - 1 - i;  // reversed pages
  int32_t* d_table = nullptr;
  cudaMalloc(&d_table, table.size() * 4);
  cudaMemcpy(d_table, table.data(), table.size() * 4, cudaMemcpyHostToDevice);
  KvPages pages(L, page, n_pages, d, kp, vp);
  RestoreResult r = restore(store, "g", w, s.plan, ThrottleConfig{}, pages, d_table);
  CHECK(r.timeline.total_s > 0 && !r.timeline.events.empty());
  std::vector<uint16_t> kd(size_t(n) * d), vd(kd.size()), kpg(size_t(n_pages) * page * d);
  void *dk = nullptr, *dv = nullptr;
  cudaMalloc(&dk, kd.size() * 2);
  cudaMalloc(&dv, vd.size() * 2);
  for (int l = 0; l < L; ++l) {
    check(hc_project_hidden_to_kv(w.get(), l, hid[l], n, 0, dk, dv, HC_DTYPE_BF16, nullptr));
    cudaMemcpy(kd.data(), dk, kd.size() * 2, cudaMemcpyDeviceToHost);
    cudaMemcpy(kpg.data(), kp[l], kpg.size() * 2, cudaMemcpyDeviceToHost);
    bool same = true;
    for (int t = 0; t < n && same; ++t) {
      const int pg = table[size_t(t / page)], slot = t % page;
      same = std::memcmp(&kd[size_t(t) * d], &kpg[(size_t(pg) * page + slot) * d], size_t(d) * 2) == 0;
    }
    CHECK(same);
  }
  // plan mismatch -> std::invalid_argument (test_restore.cpp:199-207)
  CHECK_THROWS_AS(restore(store, "g", w, RestorationPlan::make(L, 1, Complement::KvOffload),
                          ThrottleConfig{}, pages, d_table),
                  std::invalid_argument);
  for (int l = 0; l < L; ++l) {
    cudaFree(wkv[l]);
    cudaFree(hid[l]);
    cudaFree(kp[l]);
    cudaFree(vp[l]);
  }
  cudaFree(dk);
  cudaFree(dv);
  cudaFree(d_table);
}

// serving loop through the facade (harness.hpp run): HCACHE and KV_OFFLOAD
// rebuild the live K/V exactly, so they generate the same tokens; RECOMPUTE
// and IDEAL both re-prefill and agree with each other.
static void serve_tests() {
  const int L = 2, d = 256, heads = 4, dffn = 1024, vocab = 512;
  ModelConfig cfg;
  cfg.n_layers = L;
  cfg.d_hidden = d;
  cfg.n_heads = heads;
  cfg.d_ffn = dffn;
  cfg.vocab_size = vocab;
  cfg.max_seq = 1024;
  cfg.elem_bytes = 2;
  DeviceWeights w(cfg);
  std::vector<void*> bufs;
  auto fill = [&](size_t elems, uint64_t seed) {
    void* p = nullptr;
    cudaMalloc(&p, elems * 2);
    check(hc_fill_symmetric(p, int64_t(elems), seed, 0, 0.0625f, HC_DTYPE_BF16, nullptr));
    bufs.push_back(p);
    return p;
  };
  w.set_embedding(fill(size_t(vocab) * d, 1));
  for (int l = 0; l < L; ++l) {
    void* wkv = fill(size_t(2 * d) * d, 10 + l);
    w.set_layer_kv(l, wkv);
    w.set_layer_full(l, fill(size_t(d) * d, 20 + l), wkv, fill(size_t(d) * d, 30 + l),
                     fill(size_t(dffn) * d, 40 + l), fill(size_t(d) * dffn, 50 + l));
  }
  std::vector<Request> trace;
  for (int r = 1; r <= 2; ++r)
    for (int s = 0; s < 2; ++s) {
      Request q;
      q.session_id = "s" + std::to_string(s);
      q.round = r;
      for (int i = 0; i < 20; ++i) q.prompt.push_back((i * 7 + s * 13 + r) % vocab);
      q.output_budget = 6;
      q.arrival_s = (r - 1) * 1000.0 + s * 0.001;
      trace.push_back(q);
    }
  auto one = [&](Strategy st) {
    StorageManager store(DevicePool{2});
    RunOptions o;
    o.strategy = st;
    o.hcache_plan = RestorationPlan::make(L, L, Complement::None);
    return run(trace, w, store, o);
  };
  Metrics hc = one(Strategy::HCache), kvo = one(Strategy::KvOffload),
          re = one(Strategy::Recompute), id = one(Strategy::Ideal);
  CHECK(hc.outputs.size() == trace.size() && hc.outputs[0].size() == 6);
  CHECK(hc.outputs == kvo.outputs);
  CHECK(re.outputs == id.outputs);
  CHECK(hc.per_request[2].history_tokens == 26 && hc.per_request[2].restore_s > 0);
  CHECK(id.per_request[2].restore_s == 0);
  CHECK(hc.agg.storage_bytes_per_token == double(L * d * 2));
  for (void* p : bufs) cudaFree(p);
}

// Head-sharded restore driven from C++ alone (no Python, no torch): `world`
// processes forked on one GPU, IPC blobs exchanged through files; each rank
// stores only its token range, restores its heads, and must equal a local K1
// over the whole rows bit for bit.
static int sharded_rank(int world, int rank, const std::string& dir) {
  const int L = 2, d = 512, heads = 8, n = 900, page = 64, dh = d / heads;
  ModelConfig cfg;
  cfg.n_layers = L;
  cfg.d_hidden = d;
  cfg.n_heads = heads;
  cfg.d_ffn = 4 * d;
  cfg.max_seq = 2048;
  cfg.elem_bytes = 2;
  const auto hs = shard_heads(heads, world, rank);
  const int d_kv = hs.second * dh;
  DeviceWeights w(cfg, hs.first, hs.second);
  std::vector<void*> full_w(L), wkv(L), hid(L), kp(L), vp(L);
  const int n_pages = (n + page - 1) / page;
  for (int l = 0; l < L; ++l) {
    cudaMalloc(&full_w[l], size_t(2 * d) * d * 2);
    cudaMalloc(&wkv[l], size_t(2 * d_kv) * d * 2);
    cudaMalloc(&hid[l], size_t(n) * d * 2);
    cudaMalloc(&kp[l], size_t(n_pages) * page * d_kv * 2);
    cudaMalloc(&vp[l], size_t(n_pages) * page * d_kv * 2);
    check(hc_fill_symmetric(full_w[l], int64_t(2 * d) * d, 1234 + l, 0, 0.0625f, HC_DTYPE_BF16,
                            nullptr));
    // this rank's heads: K rows [h0*dh, (h0+hc)*dh) then the same V rows
    const size_t row = size_t(d) * 2, k0 = size_t(hs.first) * dh;
    cudaMemcpy(wkv[l], static_cast<char*>(full_w[l]) + k0 * row, size_t(d_kv) * row,
               cudaMemcpyDeviceToDevice);
    cudaMemcpy(static_cast<char*>(wkv[l]) + size_t(d_kv) * row,
               static_cast<char*>(full_w[l]) + (size_t(d) + k0) * row, size_t(d_kv) * row,
               cudaMemcpyDeviceToDevice);
    check(hc_fill_symmetric(hid[l], int64_t(n) * d, 7 + l, 0, 1.7320508f, HC_DTYPE_BF16, nullptr));
    w.set_layer_kv(l, wkv[l]);
  }
  const auto rg = shard_range(n, world, rank);
  StorageManager store(DevicePool{2});
  SessionSeed s = seed("sh", d, L, 2);
  s.tokens.assign(size_t(n), 1);
  s.d_kv = d_kv;
  store.create_session(s);
  for (int l = 0; l < L && rg.second > rg.first; ++l)
    CHECK(store.snapshot_device_range("sh", l, StateKind::Hidden, rg.first,
                                      static_cast<char*>(hid[l]) + size_t(rg.first) * d * 2,
                                      rg.second - rg.first, d, HC_DTYPE_BF16, nullptr));
  store.finalize("sh");
  int64_t rows_max = 0;
  for (int r = 0; r < world; ++r) {
    auto x = shard_range(n, world, r);
    rows_max = std::max(rows_max, x.second - x.first);
  }
  PeerGroup g(world, rank, 0, d, rows_max, 2);
  {  // blob exchange through files (any transport works)
    auto mine = g.export_blob();
    const std::string tmp = dir + "/r" + std::to_string(rank) + ".tmp";
    FILE* f = std::fopen(tmp.c_str(), "wb");
    std::fwrite(mine.data(), 1, mine.size(), f);
    std::fclose(f);
    std::rename(tmp.c_str(), (dir + "/r" + std::to_string(rank) + ".blob").c_str());
    std::vector<std::vector<uint8_t>> all(static_cast<size_t>(world));
    for (int r = 0; r < world; ++r) {
      const std::string path = dir + "/r" + std::to_string(r) + ".blob";
      for (int tries = 0; tries < 6000; ++tries) {
        FILE* x = std::fopen(path.c_str(), "rb");
        if (x) {
          all[size_t(r)].resize(mine.size());
          const size_t got = std::fread(all[size_t(r)].data(), 1, mine.size(), x);
          std::fclose(x);
          if (got == mine.size()) break;
        }
        struct timespec ts{0, 10000000};
        nanosleep(&ts, nullptr);
      }
    }
    g.import_blobs(all);
  }
  std::vector<int32_t> table(static_cast<size_t>(n_pages));
  for (int i = 0; i < n_pages; ++i) table[size_t(i)] = n_pages - 1 - i;
  int32_t* d_table = nullptr;
  cudaMalloc(&d_table, table.size() * 4);
  cudaMemcpy(d_table, table.data(), table.size() * 4, cudaMemcpyHostToDevice);
  KvPages pages(L, page, n_pages, d_kv, kp, vp);
  RestorationPlan plan = s.plan;
  RestoreResult r{};
  for (int it = 0; it < 3; ++it)  // wraps the 2-slot ring
    r = restore_sharded(g, store, "sh", w, plan, ThrottleConfig{}, pages, d_table);
  CHECK(r.timeline.total_s > 0);
  std::vector<uint16_t> kd(size_t(n) * d_kv), kpg(size_t(n_pages) * page * d_kv);
  void *dk = nullptr, *dv = nullptr;
  cudaMalloc(&dk, kd.size() * 2);
  cudaMalloc(&dv, kd.size() * 2);
  for (int l = 0; l < L; ++l) {
    check(hc_project_hidden_to_kv(w.get(), l, hid[l], n, 0, dk, dv, HC_DTYPE_BF16, nullptr));
    cudaMemcpy(kd.data(), dk, kd.size() * 2, cudaMemcpyDeviceToHost);
    cudaMemcpy(kpg.data(), kp[l], kpg.size() * 2, cudaMemcpyDeviceToHost);
    bool same = true;
    for (int t = 0; t < n && same; ++t) {
      const int pg = table[size_t(t / page)], slot = t % page;
      same = std::memcmp(&kd[size_t(t) * d_kv], &kpg[(size_t(pg) * page + slot) * d_kv],
                         size_t(d_kv) * 2) == 0;
    }
    CHECK(same);
  }
  // every rank done with the peers' slots before any of them unmaps / exits
  {
    const std::string done = dir + "/done" + std::to_string(rank);
    FILE* f = std::fopen(done.c_str(), "wb");
    std::fclose(f);
    for (int q = 0; q < world; ++q)
      for (int tries = 0; tries < 6000; ++tries) {
        FILE* x = std::fopen((dir + "/done" + std::to_string(q)).c_str(), "rb");
        if (x) {
          std::fclose(x);
          break;
        }
        struct timespec ts{0, 10000000};
        nanosleep(&ts, nullptr);
      }
  }
  std::printf("rank %d: %d checks, %d failures\n", rank, g_checks, g_fail);
  return g_fail ? 1 : 0;
}

static int sharded_tests(int world) {
  char tmpl[] = "/tmp/hc_facade_XXXXXX";
  const std::string dir = mkdtemp(tmpl);
  std::vector<pid_t> kids;
  for (int r = 0; r < world; ++r) {
    pid_t pid = fork();
    if (pid == 0) {
      int rc = 1;
      try {
        rc = sharded_rank(world, r, dir);
      } catch (const std::exception& e) {
        std::printf("rank %d: exception %s\n", r, e.what());
      }
      std::fflush(stdout);
      _exit(rc);
    }
    kids.push_back(pid);
  }
  int bad = 0;
  for (pid_t k : kids) {
    int st = 0;
    waitpid(k, &st, 0);
    if (!WIFEXITED(st) || WEXITSTATUS(st) != 0) ++bad;
  }
  std::printf("sharded (%d ranks): %d failed ranks\n", world, bad);
  return bad;
}

int main(int argc, char** argv) {
  // forked before this process touches CUDA
  if (argc > 2 && std::string(argv[1]) == "gpu-sharded") {
    const int bad = sharded_tests(std::atoi(argv[2]));
    std::printf("%d checks, %d failures\n", bad ? 1 : 0, bad);
    return bad ? 1 : 0;
  }
  const bool gpu = argc > 1 && std::string(argv[1]) == "gpu";
  planner_tests();
  pipeline_tests();
  storage_tests();
  if (gpu) {
    if (hc_device_count() < 1) {
      std::printf("no GPU\n");
      return 2;
    }
    gpu_tests();
    serve_tests();
  }
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
