// serve.cpp -- the serving loop on the GPU (harness run, proj/src/harness.cpp:
// 189-429): per request restore -> prompt prefill -> continuous-batching
// decode, saving every round's states for the next one.
//
// Differences from the reference by design: the clock advances by MEASURED
// durations (host wall time around each phase with the stream synchronised)
// instead of the simulated cost model; the forward passes run on the tensor
// cores (hc_forward_batch, one launch sequence per decode step for the whole
// batch); saving is the paper's two-stage scheme on B200 terms:
//   stage 1  every step's layer inputs (the H_L rows of the plan's HIDDEN
//            layers) are appended device-to-device into a per-request HBM
//            buffer inside the step; at completion they leave by async D2H on
//            a side stream into the store's pinned FIFO (hc_store snapshot
//            from device), KV-offload layers gathered from the pages likewise;
//   stage 2  the store daemon assembles 64-token chunks as copies land; a
//            persist worker finalizes the session off the serving thread.
// Nothing of stage 1/2 sits on the decode critical path except the D2D
// append (B x L_H rows per step). SavingMode::Direct instead copies each
// step's rows to the host synchronously and persists inline (charged).
#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "common.h"
#include "kernels.h"
#include "recompute.h"
#include "store.h"
#include "weights.h"

namespace hc {

void restore_session(hc_store* st, const char* sid_c, const hc_weights* w, const hc_plan* plan,
                     const hc_restore_opts* opts, const hc_kv_pages* pages,
                     const int32_t* d_page_table, cudaStream_t stream, hc_timeline* tl);

namespace {

using Clock = std::chrono::steady_clock;
double since(Clock::time_point t0) {
  return std::chrono::duration<double>(Clock::now() - t0).count();
}

// percentile (harness.cpp:36-44): linear interpolation between order stats
double percentile(std::vector<double> xs, double p) {
  if (xs.empty()) return 0;
  std::sort(xs.begin(), xs.end());
  const double idx = p * double(xs.size() - 1);
  const size_t lo = size_t(idx);
  const size_t hi = std::min(lo + 1, xs.size() - 1);
  const double frac = idx - double(lo);
  return xs[lo] * (1 - frac) + xs[hi] * frac;
}

// Contiguous layer range of one method in a plan (plans are prefix / middle /
// suffix by construction, planner.cpp:34-51).
struct Range {
  int begin = 0, count = 0;
};
Range method_range(const hc_plan& p, int method) {
  Range r;
  int last = -2;
  for (int L = 0; L < p.n_layers; ++L)
    if (p.layer_assignment[L] == method) {
      if (r.count == 0) r.begin = L;
      else if (last != L - 1) fail(HC_EINVAL, "serve: plan layers of one method must be contiguous");
      ++r.count;
      last = L;
    }
  return r;
}

// Finalizes sessions off the serving thread once their D2H copies landed.
class PersistWorker {
 public:
  explicit PersistWorker(Store& st) : st_(st), th_([this] { loop(); }) {}
  ~PersistWorker() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    th_.join();
  }
  void submit(const std::string& sid, cudaEvent_t ready) {
    std::lock_guard<std::mutex> lk(mu_);
    pending_.insert(sid);
    jobs_.push_back({sid, ready});
    cv_.notify_all();
  }
  // Blocks until `sid` has no persistence in flight; rethrows worker errors.
  void wait(const std::string& sid) {
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [&] { return !pending_.count(sid) || !error_.empty(); });
    if (!error_.empty()) fail(HC_ERUNTIME, "persist worker: " + error_);
  }
  void wait_all() {
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [&] { return pending_.empty() || !error_.empty(); });
    if (!error_.empty()) fail(HC_ERUNTIME, "persist worker: " + error_);
  }

 private:
  struct Job {
    std::string sid;
    cudaEvent_t ready;
  };
  void loop() {
    for (;;) {
      Job j;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || !jobs_.empty(); });
        if (jobs_.empty()) return;
        j = jobs_.front();
        jobs_.pop_front();
      }
      std::string err;
      try {
        if (j.ready) {
          check_cuda(cudaEventSynchronize(j.ready), "persist wait");
          cudaEventDestroy(j.ready);
        }
        st_.finalize(j.sid);
      } catch (const std::exception& e) {
        err = e.what();
      }
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (!err.empty()) error_ = err;
        // the same session may be queued again only after wait(sid)
        pending_.erase(j.sid);
      }
      cv_.notify_all();
    }
  }
  Store& st_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<Job> jobs_;
  std::set<std::string> pending_;
  std::string error_;
  bool stop_ = false;
  std::thread th_;
};

struct Active {
  size_t idx = 0;
  int kv_len = 0;        // cached positions
  int last_token = -1;
  std::vector<int32_t> out;
  int hist_before = 0;
  int budget = 1;
  bool flushed = false;
  double first_emit_t = 0, last_emit_t = 0;
  hc_request_metrics rm{};
  std::vector<int32_t> pages;
  int saved_rows = 0;            // rows appended to the round buffer
  void* acc = nullptr;           // HBM round buffer [n_hidden][cap][d] (two-stage / off)
  std::vector<uint16_t> host_acc;  // host round buffer (direct)
  int cap = 0;
};

class Engine {
 public:
  Engine(hc_store* store, const hc_weights* w, const hc_request* reqs, int n_reqs,
         const hc_serve_opts& o, cudaStream_t stream)
      : st_(store->impl), store_(store), w_(w), reqs_(reqs), n_(n_reqs), o_(o), s_(stream) {}

  void run(hc_request_metrics* per_request, int32_t* outputs, hc_serve_metrics* out);

 private:
  // setup / teardown
  void setup();
  void teardown();
  std::vector<int32_t> alloc_pages(int tokens);
  void upload_table(const std::vector<int32_t>& pages);
  // phases
  void admit(size_t idx);
  void decode_batch(std::vector<Active*>& batch);
  void complete(Active& a);
  void ingest_context(size_t idx, Active& a);
  void prefill_from_zero(const std::vector<int32_t>& toks, const Active& a, void* layer_inputs);
  void append_rows(Active& a, const void* step_rows, int rows_in_step, int row, int n_rows);
  void persist(const std::string& sid, bool exists, const std::vector<int32_t>& round_tokens,
               Active& a, int row_begin, int n_rows, const void* dev_hidden_rows, int hid_pitch,
               bool charged);
  bool persisting() const {
    return o_.strategy == HC_STRATEGY_HCACHE || o_.strategy == HC_STRATEGY_KV_OFFLOAD;
  }
  void charge(double dt) {
    t_ += dt;
    busy_ += dt;
  }

  Store& st_;
  hc_store* store_;
  const hc_weights* w_;
  const hc_request* reqs_;
  int n_;
  hc_serve_opts o_;
  cudaStream_t s_;
  cudaStream_t save_ = nullptr;
  hc_plan plan_{};
  Range hid_, kvr_;
  int L_ = 0, d_ = 0, dkv_ = 0, page_ = 64, stride_ = 1;
  // page pool
  std::vector<void*> kp_, vp_;
  hc_kv_pages pages_{};
  std::vector<int32_t> free_pages_;
  // staging
  int max_rows_ = 1, max_batch_ = 1;
  int32_t* h_tok_ = nullptr;    // pinned: tokens
  int32_t* h_table_ = nullptr;  // pinned: batch page tables
  int32_t* h_next_ = nullptr;   // pinned: next tokens
  int32_t* h_meta_ = nullptr;   // pinned: decode cu_seqlens + positions
  AppendDst* h_app_ = nullptr;  // pinned: per-sequence round-buffer rows (stage 1)
  AppendDst* d_app_ = nullptr;
  int32_t* d_tok_ = nullptr;
  int32_t* d_table_ = nullptr;
  int32_t* d_next_ = nullptr;
  int32_t* d_meta_ = nullptr;
  // decode steps as CUDA graphs, one per batch size (launch-bound otherwise)
  cudaStream_t cap_ = nullptr;
  std::map<int, cudaGraphExec_t> graphs_;
  std::map<int, int> eager_runs_;
  bool use_graphs_ = true;
  void* d_step_ = nullptr;      // [L][max_rows][d] layer inputs of one step
  std::unique_ptr<PersistWorker> worker_;
  bool started_daemon_ = false;
  // state
  std::map<std::string, std::vector<int32_t>> history_;
  std::vector<Active> dec_;
  std::vector<hc_request_metrics> per_;
  std::vector<std::vector<int32_t>> outs_;
  double t_ = 0, busy_ = 0, stall_ = 0, persist_wait_ = 0;
  uint64_t saved_bytes_ = 0, saved_tokens_ = 0, backpressure_ = 0;
  int64_t steps_ = 0, step_tokens_ = 0;
};

void Engine::setup() {
  const auto& c = w_->cfg;
  L_ = c.n_layers;
  d_ = c.d_hidden;
  dkv_ = w_->d_kv_all;
  if (!w_->embedding) fail(HC_EINVAL, "serve: embedding not set");
  for (int L = 0; L < L_; ++L)
    if (!w_->layers[size_t(L)].full) fail(HC_EINVAL, "serve: full block weights not set");
  if (w_->d_kv != w_->d_kv_all) fail(HC_EINVAL, "serve: needs all KV heads on this GPU");
  if (o_.strategy < HC_STRATEGY_HCACHE || o_.strategy > HC_STRATEGY_IDEAL)
    fail(HC_EINVAL, "serve: bad strategy");
  if (o_.saving < HC_SAVING_TWO_STAGE || o_.saving > HC_SAVING_OFF)
    fail(HC_EINVAL, "serve: bad saving mode");
  page_ = o_.page_size > 0 ? o_.page_size : 64;
  if (o_.num_pages < 1) fail(HC_EINVAL, "serve: num_pages must be >= 1");
  // run_plan (harness.cpp:194-197)
  if (o_.strategy == HC_STRATEGY_HCACHE) {
    plan_ = o_.plan;
  } else {
    if (hc_plan_make(L_, 0, HC_COMPLEMENT_KV_OFFLOAD, &plan_) != HC_OK)
      fail(HC_EINVAL, "serve: plan");
  }
  if (persisting() && plan_.n_layers != L_)
    fail(HC_EINVAL, "run: plan does not cover the model's layers");
  hid_ = method_range(plan_, HC_METHOD_HIDDEN);
  kvr_ = method_range(plan_, HC_METHOD_KV_OFFLOAD);
  // request validation and staging sizes
  int max_need = 1, max_rows = 1, max_hist = 0;
  std::map<std::string, int> hist;
  for (int i = 0; i < n_; ++i) {
    const hc_request& r = reqs_[i];
    if (!r.session_id || r.n_prompt < 1 || !r.prompt || r.output_budget < 1)
      fail(HC_EINVAL, "serve: request needs a session id, a prompt and a budget >= 1");
    if (i > 0 && r.arrival_s < reqs_[i - 1].arrival_s)
      fail(HC_EINVAL, "serve: requests must be sorted by arrival");
    int& h = hist[r.session_id];
    if (r.n_context > 0 && h == 0) h = r.n_context;
    max_hist = std::max(max_hist, h);
    const int need = h + r.n_prompt + r.output_budget;
    if (need > c.max_seq) fail(HC_EINVAL, "serve: request exceeds max_seq");
    max_need = std::max(max_need, need);
    max_rows = std::max({max_rows, r.n_prompt, r.n_context});
    h = need;
  }
  stride_ = (max_need + page_ - 1) / page_;
  if (persisting()) {
    // the run's save volume, page-locked outside the clock: per session and
    // stored layer the chunk extents it can grow to (first extent >= 8 slots
    // per arena, later ones doubling: <= 2x the final chunk count) -- an
    // under-estimate would pin a new slab (~0.1 s of cudaHostAlloc) under the
    // store lock in the middle of a restore
    const size_t ch = size_t(HC_CHUNK_TOKENS);
    const size_t cb_h = ch * size_t(d_) * 2, cb_kv = ch * size_t(2 * dkv_) * 2;
    size_t bytes = 0;
    for (const auto& kv : hist) {
      const size_t chunks = (size_t(kv.second) + ch - 1) / ch;
      const size_t slots = std::max(2 * chunks, size_t(8) * size_t(st_.device_count())) + size_t(st_.device_count());
      bytes += slots * (size_t(hid_.count) * cb_h + size_t(kvr_.count) * cb_kv);
    }
    st_.reserve_pinned(std::min<size_t>(size_t(96) << 30, bytes));
  }
  max_batch_ = o_.max_batch > 0 ? std::min(o_.max_batch, n_) : n_;
  max_rows_ = std::max(max_rows, max_batch_);
  // page pool: per layer K and V [num_pages][page][d_kv] bf16
  const size_t pool_bytes = size_t(o_.num_pages) * size_t(page_) * size_t(dkv_) * 2;
  kp_.assign(size_t(L_), nullptr);
  vp_.assign(size_t(L_), nullptr);
  for (int L = 0; L < L_; ++L) {
    HC_CUDA(cudaMalloc(&kp_[size_t(L)], pool_bytes));
    HC_CUDA(cudaMalloc(&vp_[size_t(L)], pool_bytes));
  }
  pages_ = hc_kv_pages{L_, page_, o_.num_pages, dkv_, HC_DTYPE_BF16, kp_.data(), vp_.data()};
  free_pages_.resize(size_t(o_.num_pages));
  for (int p = 0; p < o_.num_pages; ++p) free_pages_[size_t(p)] = o_.num_pages - 1 - p;
  HC_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h_tok_), sizeof(int32_t) * size_t(max_rows_),
                        cudaHostAllocDefault));
  HC_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h_table_),
                        sizeof(int32_t) * size_t(max_batch_) * size_t(stride_),
                        cudaHostAllocDefault));
  HC_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h_next_), sizeof(int32_t) * size_t(max_batch_),
                        cudaHostAllocDefault));
  HC_CUDA(cudaMalloc(&d_tok_, sizeof(int32_t) * size_t(max_rows_)));
  HC_CUDA(cudaMalloc(&d_table_, sizeof(int32_t) * size_t(max_batch_) * size_t(stride_)));
  HC_CUDA(cudaMalloc(&d_next_, sizeof(int32_t) * size_t(max_batch_)));
  HC_CUDA(cudaMalloc(&d_step_, size_t(L_) * size_t(max_rows_) * size_t(d_) * 2));
  HC_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h_meta_),
                        sizeof(int32_t) * size_t(2 * max_batch_ + 1), cudaHostAllocDefault));
  HC_CUDA(cudaMalloc(&d_meta_, sizeof(int32_t) * size_t(2 * max_batch_ + 1)));
  HC_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h_app_), sizeof(AppendDst) * size_t(max_batch_),
                        cudaHostAllocDefault));
  HC_CUDA(cudaMalloc(&d_app_, sizeof(AppendDst) * size_t(max_batch_)));
  HC_CUDA(cudaStreamCreateWithFlags(&save_, cudaStreamNonBlocking));
  HC_CUDA(cudaStreamCreateWithFlags(&cap_, cudaStreamNonBlocking));
  {
    const char* e = getenv("HC_SERVE_GRAPHS");
    use_graphs_ = !(e && atoi(e) == 0);
  }
  // grow the stream-ordered pool once to what the largest restore stages
  // (its ring of hidden-state layers + K/V rows), outside the clock, so the
  // first large restore does not pay for the pool's growth
  if (persisting() && max_hist > 0) {
    const size_t warm = std::min<size_t>(size_t(16) << 30,
                                         size_t(max_hist) * size_t(d_) * 2 * size_t(L_) +
                                             size_t(max_hist) * size_t(4 * dkv_) * 2);
    void* p = nullptr;
    if (cudaMallocAsync(&p, warm, s_) == cudaSuccess) {
      HC_CUDA(cudaFreeAsync(p, s_));
      HC_CUDA(cudaStreamSynchronize(s_));
    } else {
      cudaGetLastError();
    }
  }
  per_.assign(size_t(n_), hc_request_metrics{});
  outs_.assign(size_t(n_), {});
  if (persisting()) {
    worker_.reset(new PersistWorker(st_));
    if (o_.saving == HC_SAVING_TWO_STAGE && !st_.daemon_running()) {
      st_.start_daemon();
      started_daemon_ = true;
    }
  }
}

void Engine::teardown() {
  if (worker_) {
    try {
      worker_->wait_all();
    } catch (...) {
    }
    worker_.reset();
  }
  if (save_) cudaStreamSynchronize(save_);
  cudaStreamSynchronize(s_);
  if (started_daemon_) st_.stop_daemon();
  for (auto& a : dec_)
    if (a.acc) cudaFree(a.acc);
  for (void* p : kp_) cudaFree(p);
  for (void* p : vp_) cudaFree(p);
  cudaFreeHost(h_tok_);
  cudaFreeHost(h_table_);
  cudaFreeHost(h_next_);
  cudaFree(d_tok_);
  cudaFree(d_table_);
  cudaFree(d_next_);
  cudaFree(d_step_);
  cudaFreeHost(h_meta_);
  cudaFree(d_meta_);
  cudaFreeHost(h_app_);
  cudaFree(d_app_);
  for (auto& g : graphs_) cudaGraphExecDestroy(g.second);
  graphs_.clear();
  if (cap_) cudaStreamDestroy(cap_);
  if (save_) cudaStreamDestroy(save_);
}

std::vector<int32_t> Engine::alloc_pages(int tokens) {
  const size_t need = size_t((tokens + page_ - 1) / page_);
  if (need > free_pages_.size())
    fail(HC_ENOMEM, "serve: KV page pool exhausted (raise num_pages)");
  std::vector<int32_t> p(free_pages_.end() - std::ptrdiff_t(need), free_pages_.end());
  free_pages_.resize(free_pages_.size() - need);
  return p;
}

void Engine::upload_table(const std::vector<int32_t>& pages) {
  HC_CUDA(cudaStreamSynchronize(s_));  // h_table_ may still feed an earlier copy
  std::memcpy(h_table_, pages.data(), pages.size() * sizeof(int32_t));
  HC_CUDA(cudaMemcpyAsync(d_table_, h_table_, pages.size() * sizeof(int32_t),
                          cudaMemcpyHostToDevice, s_));
}

void Engine::prefill_from_zero(const std::vector<int32_t>& toks, const Active& a,
                               void* layer_inputs) {
  HC_CUDA(cudaStreamSynchronize(s_));
  StreamScratch dt(toks.size() * sizeof(int32_t), s_);
  HC_CUDA(cudaMemcpyAsync(dt.ptr, toks.data(), toks.size() * sizeof(int32_t),
                          cudaMemcpyHostToDevice, s_));
  upload_table(a.pages);
  prefill_layers_impl(w_, static_cast<int32_t*>(dt.ptr), int64_t(toks.size()), 0, L_, &pages_,
                      d_table_, s_, [](int, bool) {}, layer_inputs);
  HC_CUDA(cudaStreamSynchronize(s_));
}

// Stage 1: rows [row, row + n_rows) of this step's layer inputs (row stride
// rows_in_step within each layer) -> the request's round buffer.
void Engine::append_rows(Active& a, const void* step_rows, int rows_in_step, int row, int n_rows) {
  if (!persisting() || hid_.count == 0) {
    a.saved_rows += n_rows;
    return;
  }
  const size_t rb = size_t(d_) * 2;
  const char* src = static_cast<const char*>(step_rows) +
                    (size_t(hid_.begin) * size_t(rows_in_step) + size_t(row)) * rb;
  if (o_.saving == HC_SAVING_DIRECT) {
    // synchronous copy on the serving thread (charged by the caller's timer)
    std::vector<uint16_t> tmp(size_t(hid_.count) * size_t(n_rows) * size_t(d_));
    HC_CUDA(cudaMemcpy2DAsync(tmp.data(), rb * size_t(n_rows), src, rb * size_t(rows_in_step),
                              rb * size_t(n_rows), size_t(hid_.count), cudaMemcpyDeviceToHost, s_));
    HC_CUDA(cudaStreamSynchronize(s_));
    for (int l = 0; l < hid_.count; ++l)
      std::memcpy(a.host_acc.data() + (size_t(l) * size_t(a.cap) + size_t(a.saved_rows)) * size_t(d_),
                  tmp.data() + size_t(l) * size_t(n_rows) * size_t(d_), rb * size_t(n_rows));
  } else {
    char* dst = static_cast<char*>(a.acc) + size_t(a.saved_rows) * rb;
    HC_CUDA(cudaMemcpy2DAsync(dst, rb * size_t(a.cap), src, rb * size_t(rows_in_step),
                              rb * size_t(n_rows), size_t(hid_.count), cudaMemcpyDeviceToDevice,
                              s_));
  }
  a.saved_rows += n_rows;
}

// persist_states + finalize (harness.cpp:216-242, 258-276) for rows
// [row_begin, row_begin + n_rows) of the session.
void Engine::persist(const std::string& sid, bool exists, const std::vector<int32_t>& round_tokens,
                     Active& a, int row_begin, int n_rows, const void* dev_hidden_rows,
                     int hid_pitch, bool charged) {
  const auto t0 = Clock::now();
  worker_->wait(sid);  // the previous round's chunks are in place
  if (exists) {
    st_.reopen_for_append(sid, round_tokens.data(), int64_t(round_tokens.size()));
  } else {
    hc_session_seed seed{};
    seed.session_id = sid.c_str();
    seed.config_hash = hc_config_hash(&w_->cfg);
    seed.n_layers = L_;
    seed.d_hidden = d_;
    seed.d_kv = dkv_;
    seed.elem_bytes = 2;
    seed.dtype = HC_DTYPE_BF16;
    seed.plan = &plan_;
    seed.tokens = round_tokens.data();
    seed.n_tokens = int64_t(round_tokens.size());
    st_.create_session(seed);
  }
  // KV-offload layers: gather the rows out of the pages on the compute
  // stream, so the gather is ordered before any later work on s_ that
  // reuses these pages (complete() returns them to the free list right after
  // this call); the save stream then only reads the private gathered buffer.
  void* kvbuf = nullptr;
  const size_t kvb = size_t(n_rows) * size_t(2 * dkv_) * 2;
  if (kvr_.count > 0) {
    HC_CUDA(cudaMallocAsync(&kvbuf, kvb * size_t(kvr_.count), s_));
    StreamScratch table(a.pages.size() * sizeof(int32_t), s_);
    HC_CUDA(cudaMemcpyAsync(table.ptr, a.pages.data(), a.pages.size() * sizeof(int32_t),
                            cudaMemcpyHostToDevice, s_));
    // (pageable source: staged by the driver before the call returns)
    for (int l = 0; l < kvr_.count; ++l)
      if (hc_kv_gather_rows(&pages_, kvr_.begin + l, static_cast<int32_t*>(table.ptr), row_begin,
                            n_rows, static_cast<char*>(kvbuf) + kvb * size_t(l), s_) != HC_OK)
        fail(HC_ECUDA, std::string("serve: kv gather: ") + hc_last_error());
  }
  // the save stream picks up everything the compute stream produced so far
  cudaEvent_t produced;
  HC_CUDA(cudaEventCreateWithFlags(&produced, cudaEventDisableTiming));
  HC_CUDA(cudaEventRecord(produced, s_));
  HC_CUDA(cudaStreamWaitEvent(save_, produced, 0));
  HC_CUDA(cudaEventDestroy(produced));
  double stall = 0;
  auto put = [&](int layer, int kind, const void* rows, bool on_device, int width) {
    while (!st_.snapshot(sid, layer, kind, rows, n_rows, width, HC_DTYPE_BF16, on_device, save_)) {
      ++backpressure_;
      const auto tb = Clock::now();
      st_.drain(-1);
      stall += since(tb);
    }
    saved_bytes_ += uint64_t(n_rows) * uint64_t(width) * 2;
  };
  const size_t rb = size_t(d_) * 2;
  for (int l = 0; l < hid_.count; ++l) {
    if (o_.saving == HC_SAVING_DIRECT && !dev_hidden_rows)
      put(hid_.begin + l, HC_STATE_HIDDEN,
          a.host_acc.data() + size_t(l) * size_t(a.cap) * size_t(d_), false, d_);
    else
      put(hid_.begin + l, HC_STATE_HIDDEN,
          static_cast<const char*>(dev_hidden_rows ? dev_hidden_rows : a.acc) +
              size_t(l) * size_t(dev_hidden_rows ? hid_pitch : a.cap) * rb,
          true, d_);
  }
  for (int l = 0; l < kvr_.count; ++l)
    put(kvr_.begin + l, HC_STATE_KV, static_cast<char*>(kvbuf) + kvb * size_t(l), true, 2 * dkv_);
  if (kvbuf) HC_CUDA(cudaFreeAsync(kvbuf, save_));
  if (a.acc) {
    HC_CUDA(cudaFreeAsync(a.acc, save_));
    a.acc = nullptr;
  }
  saved_tokens_ += uint64_t(n_rows);
  if (o_.saving == HC_SAVING_TWO_STAGE) {
    cudaEvent_t ready;
    HC_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    HC_CUDA(cudaEventRecord(ready, save_));
    worker_->submit(sid, ready);
  } else {
    HC_CUDA(cudaStreamSynchronize(save_));
    st_.finalize(sid);
  }
  if (charged) {
    const double dt = o_.saving == HC_SAVING_OFF ? 0.0
                      : o_.saving == HC_SAVING_DIRECT ? since(t0)
                                                      : stall;
    charge(dt);
    stall_ += dt;
  }
}

void Engine::ingest_context(size_t idx, Active& a) {
  // long-context sessions were ingested offline (harness.cpp:325-341): not charged
  const hc_request& rq = reqs_[idx];
  std::vector<int32_t> ctx(rq.context, rq.context + rq.n_context);
  void* inputs = nullptr;
  if (persisting() && hid_.count > 0)
    HC_CUDA(cudaMalloc(&inputs, size_t(L_) * size_t(rq.n_context) * size_t(d_) * 2));
  prefill_from_zero(ctx, a, inputs);
  if (persisting()) {
    const char* hrows = inputs ? static_cast<const char*>(inputs) +
                                     size_t(hid_.begin) * size_t(rq.n_context) * size_t(d_) * 2
                               : nullptr;
    Active tmp;
    tmp.pages = a.pages;
    persist(rq.session_id, false, ctx, tmp, 0, rq.n_context, hrows, rq.n_context, false);
    worker_->wait(rq.session_id);
    HC_CUDA(cudaStreamSynchronize(save_));
  }
  if (inputs) cudaFree(inputs);
  history_[rq.session_id] = ctx;
}

void Engine::admit(size_t idx) {
  const hc_request& rq = reqs_[idx];
  const std::string sid(rq.session_id);
  auto& hist = history_[sid];
  Active a;
  a.idx = idx;
  a.budget = rq.output_budget;
  const int hist_now = hist.empty() && rq.n_context > 0 ? rq.n_context : int(hist.size());
  a.pages = alloc_pages(hist_now + rq.n_prompt + rq.output_budget);
  bool kv_present = false;
  if (rq.n_context > 0 && hist.empty()) {
    ingest_context(idx, a);
    kv_present = true;
  }
  a.hist_before = int(hist.size());
  a.rm.round = rq.round;
  a.rm.arrival_s = rq.arrival_s;
  a.rm.history_tokens = a.hist_before;
  a.cap = rq.n_prompt + rq.output_budget;
  if (persisting() && hid_.count > 0) {
    if (o_.saving == HC_SAVING_DIRECT)
      a.host_acc.assign(size_t(hid_.count) * size_t(a.cap) * size_t(d_), 0);
    else
      HC_CUDA(cudaMallocAsync(&a.acc, size_t(hid_.count) * size_t(a.cap) * size_t(d_) * 2, s_));
  }

  double restore_s = 0;
  if (!hist.empty()) {
    switch (o_.strategy) {
      case HC_STRATEGY_IDEAL:
        if (!kv_present) prefill_from_zero(hist, a, nullptr);
        break;
      case HC_STRATEGY_RECOMPUTE: {
        const auto t0 = Clock::now();
        prefill_from_zero(hist, a, nullptr);
        restore_s = since(t0);
        break;
      }
      default: {
        const auto tw = Clock::now();
        worker_->wait(sid);  // previous round still persisting: not the request's cost
        persist_wait_ += since(tw);
        HC_CUDA(cudaStreamSynchronize(s_));
        const auto t0 = Clock::now();
        upload_table(a.pages);
        hc_restore_opts ro{};
        restore_session(store_, sid.c_str(), w_, &plan_, &ro, &pages_, d_table_, s_, nullptr);
        HC_CUDA(cudaStreamSynchronize(s_));
        restore_s = since(t0);
      }
    }
  }
  charge(restore_s);
  a.rm.restore_s = restore_s;

  // prompt prefill at positions hist.. (harness.cpp:380-390)
  const auto t0 = Clock::now();
  std::memcpy(h_tok_, rq.prompt, sizeof(int32_t) * size_t(rq.n_prompt));
  HC_CUDA(cudaMemcpyAsync(d_tok_, h_tok_, sizeof(int32_t) * size_t(rq.n_prompt),
                          cudaMemcpyHostToDevice, s_));
  upload_table(a.pages);
  const int32_t np = rq.n_prompt, start = a.hist_before;
  forward_batch(w_, d_tok_, 1, &np, &start, &pages_, d_table_, stride_, d_step_, d_next_, s_);
  HC_CUDA(cudaMemcpyAsync(h_next_, d_next_, sizeof(int32_t), cudaMemcpyDeviceToHost, s_));
  append_rows(a, d_step_, np, 0, np);
  HC_CUDA(cudaStreamSynchronize(s_));
  charge(since(t0));

  a.kv_len = a.hist_before + np;
  a.rm.ttft_s = t_ - rq.arrival_s;
  a.first_emit_t = a.last_emit_t = t_;
  a.out.push_back(h_next_[0]);
  a.last_token = h_next_[0];
  if (a.budget == 1) {
    dec_.push_back(std::move(a));
    std::vector<Active*> one{&dec_.back()};
    decode_batch(one);  // flush the single emitted token's state
    complete(dec_.back());
    dec_.pop_back();
  } else {
    dec_.push_back(std::move(a));
  }
}

void Engine::decode_batch(std::vector<Active*>& batch) {
  // one batched decode step (harness.cpp:294-318): every member's pending token
  const auto t0 = Clock::now();
  const int B = int(batch.size());
  std::vector<int32_t> starts(static_cast<size_t>(B));
  HC_CUDA(cudaStreamSynchronize(s_));  // pinned staging reuse
  for (int b = 0; b < B; ++b) {
    Active& a = *batch[size_t(b)];
    h_tok_[b] = a.last_token;
    starts[size_t(b)] = a.kv_len;
    std::memcpy(h_table_ + size_t(b) * size_t(stride_), a.pages.data(),
                a.pages.size() * sizeof(int32_t));
  }
  for (int b = 0; b <= B; ++b) h_meta_[b] = b;  // one row per sequence
  for (int b = 0; b < B; ++b) {
    if (starts[size_t(b)] + 1 > w_->cfg.max_seq) fail(HC_EINVAL, "forward: sequence exceeds max_seq");
    h_meta_[B + 1 + b] = starts[size_t(b)];
  }
  HC_CUDA(cudaMemcpyAsync(d_tok_, h_tok_, sizeof(int32_t) * size_t(B), cudaMemcpyHostToDevice, s_));
  HC_CUDA(cudaMemcpyAsync(d_table_, h_table_, sizeof(int32_t) * size_t(B) * size_t(stride_),
                          cudaMemcpyHostToDevice, s_));
  HC_CUDA(cudaMemcpyAsync(d_meta_, h_meta_, sizeof(int32_t) * size_t(2 * B + 1),
                          cudaMemcpyHostToDevice, s_));
  // stage 1 of the two-stage save rides inside the step: one kernel appends
  // every sequence's new row of each HIDDEN layer to its round buffer
  const bool fused_append = persisting() && hid_.count > 0 && o_.saving != HC_SAVING_DIRECT;
  if (fused_append) {
    const size_t rb = size_t(d_) * 2;
    for (int b = 0; b < B; ++b) {
      Active& a = *batch[size_t(b)];
      h_app_[b].dst = static_cast<char*>(a.acc) + size_t(a.saved_rows) * rb;
      h_app_[b].pitch = int64_t(a.cap) * int64_t(rb);
    }
    HC_CUDA(cudaMemcpyAsync(d_app_, h_app_, sizeof(AppendDst) * size_t(B), cudaMemcpyHostToDevice,
                            s_));
  }
  auto step = [&](cudaStream_t st) {
    forward_batch_dev(w_, d_tok_, B, B, 1, d_meta_, d_meta_ + B + 1, &pages_, d_table_, stride_,
                      d_step_, d_next_, st);
    if (fused_append)
      HC_CUDA(launch_append_rows(d_step_, B, hid_.begin, hid_.count, d_, d_app_, B, st));
  };
  auto it = graphs_.find(B);
  if (it != graphs_.end()) {
    HC_CUDA(cudaGraphLaunch(it->second, s_));
  } else if (use_graphs_ && eager_runs_[B] >= 1) {
    // capture once per batch size (after one eager run set every kernel up)
    cudaGraph_t graph = nullptr;
    HC_CUDA(cudaStreamBeginCapture(cap_, cudaStreamCaptureModeThreadLocal));
    try {
      step(cap_);
    } catch (...) {
      cudaStreamEndCapture(cap_, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    HC_CUDA(cudaStreamEndCapture(cap_, &graph));
    cudaGraphExec_t exec = nullptr;
    HC_CUDA(cudaGraphInstantiate(&exec, graph, 0));
    cudaGraphDestroy(graph);
    graphs_[B] = exec;
    HC_CUDA(cudaGraphLaunch(exec, s_));
  } else {
    step(s_);
    ++eager_runs_[B];
  }
  HC_CUDA(cudaMemcpyAsync(h_next_, d_next_, sizeof(int32_t) * size_t(B), cudaMemcpyDeviceToHost,
                          s_));
  for (int b = 0; b < B; ++b) {
    if (fused_append) ++batch[size_t(b)]->saved_rows;
    else append_rows(*batch[size_t(b)], d_step_, B, b, 1);
  }
  HC_CUDA(cudaStreamSynchronize(s_));
  charge(since(t0));
  ++steps_;
  step_tokens_ += B;
  for (int b = 0; b < B; ++b) {
    Active& a = *batch[size_t(b)];
    ++a.kv_len;
    if (int(a.out.size()) < a.budget) {
      a.out.push_back(h_next_[b]);
      a.last_token = h_next_[b];
      a.last_emit_t = t_;
    } else {
      a.flushed = true;
    }
  }
}

void Engine::complete(Active& a) {
  const hc_request& rq = reqs_[a.idx];
  const std::string sid(rq.session_id);
  std::vector<int32_t> round_tokens(rq.prompt, rq.prompt + rq.n_prompt);
  round_tokens.insert(round_tokens.end(), a.out.begin(), a.out.end());
  if (a.saved_rows != int(round_tokens.size()))
    fail(HC_ERUNTIME, "serve: saved rows do not match the round's tokens");
  if (persisting()) {
    const bool exists = rq.round > 1 || rq.n_context > 0;
    persist(sid, exists, round_tokens, a, a.hist_before, int(round_tokens.size()), nullptr, 0,
            true);
  } else if (a.acc) {
    HC_CUDA(cudaFreeAsync(a.acc, s_));
    a.acc = nullptr;
  }
  auto& hist = history_[sid];
  hist.insert(hist.end(), round_tokens.begin(), round_tokens.end());
  free_pages_.insert(free_pages_.end(), a.pages.begin(), a.pages.end());
  a.pages.clear();
  a.rm.generated = int(a.out.size());
  a.rm.tbt_s = a.out.size() > 1 ? (a.last_emit_t - a.first_emit_t) / double(a.out.size() - 1) : 0;
  per_[a.idx] = a.rm;
  outs_[a.idx] = a.out;
}

void Engine::run(hc_request_metrics* per_request, int32_t* outputs, hc_serve_metrics* out) {
  setup();
  try {
    std::deque<size_t> waiting;
    size_t next_arr = 0;
    while (next_arr < size_t(n_) || !waiting.empty() || !dec_.empty()) {
      while (next_arr < size_t(n_) && reqs_[next_arr].arrival_s <= t_ + 1e-12)
        waiting.push_back(next_arr++);
      if (waiting.empty() && dec_.empty()) {
        t_ = std::max(t_, reqs_[next_arr].arrival_s);
        continue;
      }
      const bool room = o_.max_batch <= 0 || int(dec_.size()) < o_.max_batch;
      if (!waiting.empty() && room) {
        // strict phase ordering: a pending restoration+prefill pauses decode
        const size_t idx = waiting.front();
        waiting.pop_front();
        admit(idx);
        continue;
      }
      std::vector<Active*> batch;
      for (auto& a : dec_) batch.push_back(&a);
      decode_batch(batch);
      for (auto it = dec_.begin(); it != dec_.end();) {
        if (it->flushed) {
          complete(*it);
          it = dec_.erase(it);
        } else {
          ++it;
        }
      }
    }
    if (worker_) worker_->wait_all();
  } catch (...) {
    teardown();
    throw;
  }
  teardown();
  // aggregates (Metrics::finalize_aggregates, harness.cpp:133-151)
  std::vector<double> ttft, tbt;
  double hist_sum = 0, restore_sum = 0, tbt_mean = 0;
  size_t off = 0;
  for (int i = 0; i < n_; ++i) {
    const auto& r = per_[size_t(i)];
    per_request[i] = r;
    ttft.push_back(r.ttft_s);
    if (r.generated > 1) tbt.push_back(r.tbt_s);
    hist_sum += r.history_tokens;
    restore_sum += r.restore_s;
    if (outputs)
      for (int32_t tok : outs_[size_t(i)]) outputs[off++] = tok;
  }
  for (double x : tbt) tbt_mean += x;
  hc_serve_metrics m{};
  m.ttft_p50 = percentile(ttft, 0.50);
  m.ttft_p95 = percentile(ttft, 0.95);
  m.tbt_p50 = percentile(tbt, 0.50);
  m.tbt_p95 = percentile(tbt, 0.95);
  m.tbt_mean = tbt.empty() ? 0 : tbt_mean / double(tbt.size());
  m.restore_tokens_per_s = restore_sum > 0 ? hist_sum / restore_sum : 0;
  m.saved_bytes = saved_bytes_;
  m.saved_tokens = saved_tokens_;
  m.storage_bytes_per_token = saved_tokens_ > 0 ? double(saved_bytes_) / double(saved_tokens_) : 0;
  m.backpressure_stalls = backpressure_;
  m.busy_s = busy_;
  m.save_stall_s = stall_;
  m.persist_wait_s = persist_wait_;
  m.decode_steps = steps_;
  m.decode_tokens = step_tokens_;
  *out = m;
}

}  // namespace
}  // namespace hc

using namespace hc;

extern "C" hc_status hc_serve_run(hc_store* store, const hc_weights* w, const hc_request* requests,
                                  int32_t n_requests, const hc_serve_opts* opts,
                                  hc_request_metrics* per_request, int32_t* outputs,
                                  hc_serve_metrics* out, void* stream) {
  return guard([&] {
    if (!store || !w || !opts || !per_request || !out || (n_requests > 0 && !requests))
      fail(HC_EINVAL, "serve: null argument");
    if (n_requests < 0) fail(HC_EINVAL, "serve: negative request count");
    DeviceGuard dg(w->device);
    Engine e(store, w, requests, n_requests, *opts, as_stream(stream));
    e.run(per_request, outputs, out);
  });
}
