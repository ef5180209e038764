// sharded.cpp -- head-sharded multi-GPU restore behind the C ABI
// (hc_peer_group_*, hc_restore_sharded, north star (4)).
//
// One process per GPU. Every HIDDEN layer's hidden state is needed in full by
// every GPU (each KV head contracts over all of d), while the projection
// output shards by KV head. Per HIDDEN layer, on rank r of N:
//
//   IO lane  (copy stream)  wait until every consumer released the staging
//            slot (flags in this GPU's memory), fetch this rank's 128-row
//            aligned token range over its own PCIe link into the slot;
//   owner    (aux stream)   LayerNorm statistics of the range (and the mean
//            shift of rows with |mean| >> sigma, in place) into the slot, then
//            store the slot's epoch into every rank's `ready` flag
//            (system-scope release stores over NVLink);
//   compute  (caller stream) wait for every owner's `ready` flag, copy the
//            owners' statistics (8 B per row) into one array, run K1 with one
//            TMA tensor map per owner's slot -- the A tiles stream straight
//            from the peers' HBM, the all-gather is fused into the GEMM -- for
//            this rank's KV heads only, then store the epoch into every
//            owner's `consumed` flag.
//
// KV_OFFLOAD layers fetch this rank's heads' [K|V] rows (its own store holds
// exactly those) and scatter them locally (K4). The slots and flags are
// cudaMalloc'ed and exported with CUDA IPC; the host transports the handles
// (MPI, sockets, torch.distributed -- anything). Every rank must issue the
// same sequence of restores; a step counter numbers the slot hand-offs.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "common.h"
#include "engine.h"
#include "kernels.h"
#include "recompute.h"
#include "store.h"
#include "weights.h"

namespace hc {
CUtensorMap weight_map(const hc_weights::Layer& L, int bn, int d, int rows);
void restore_session(hc_store* st, const char* sid_c, const hc_weights* w, const hc_plan* plan,
                     const hc_restore_opts* opts, const hc_kv_pages* pages,
                     const int32_t* d_page_table, cudaStream_t stream, hc_timeline* tl);
std::string plan_serialize(const hc_plan* p);

namespace {

constexpr uint32_t kBlobMagic = 0x48435047u;  // "HCPG"

struct Blob {
  uint32_t magic;
  int32_t world, rank, d;
  int64_t max_rows;
  int32_t depth, pad_;
  uint64_t slot_bytes;
  cudaIpcMemHandle_t slab, flags;
};

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

void shard_range(int64_t n, int world, int rank, int64_t* b, int64_t* e) {
  // 128-row aligned contiguous ranges (one K1 M tile reads one owner)
  const int64_t blocks = (n + 127) / 128;
  const int64_t per = (blocks + world - 1) / world;
  *b = std::min(n, int64_t(rank) * per * 128);
  *e = std::min(n, int64_t(rank + 1) * per * 128);
}

}  // namespace
}  // namespace hc

struct hc_peer_group {
  int world = 1, rank = 0, device = 0, d = 0, depth = 2;
  int64_t max_rows = 0;
  size_t data_bytes = 0, slot_bytes = 0;
  void* slab = nullptr;            // this rank's slots: [depth][data | mean | rstd | flag]
  uint32_t* flags = nullptr;       // [2][world][depth]: 0 = ready (by owner), 1 = consumed (by consumer)
  std::vector<char*> peer_slab;    // every rank's slab mapped here (own = slab)
  std::vector<uint32_t*> peer_flags;
  uint32_t** d_ready = nullptr;    // [depth][world]: &peer_flags[r][0][rank][slot]
  uint32_t** d_consumed = nullptr; // [depth][world]: &peer_flags[r][1][rank][slot]
  uint64_t step = 0;               // HIDDEN-layer hand-offs so far
  bool imported = false;

  char* slot_data(int r, int s) const { return peer_slab[size_t(r)] + size_t(s) * slot_bytes; }
  float* slot_mean(int r, int s) const {
    return reinterpret_cast<float*>(slot_data(r, s) + data_bytes);
  }
  float* slot_rstd(int r, int s) const { return slot_mean(r, s) + max_rows; }
  int32_t* slot_flag(int r, int s) const {
    return reinterpret_cast<int32_t*>(slot_rstd(r, s) + max_rows);
  }
  uint32_t* my_flag(int kind, int who, int s) const {
    return flags + (size_t(kind) * size_t(world) + size_t(who)) * size_t(depth) + size_t(s);
  }
};

using namespace hc;

namespace {

void release_group(hc_peer_group* g) {
  if (!g) return;
  DeviceGuard dg(g->device);
  cudaDeviceSynchronize();
  for (int r = 0; r < int(g->peer_slab.size()); ++r) {
    if (r == g->rank) continue;
    if (g->peer_slab[size_t(r)]) cudaIpcCloseMemHandle(g->peer_slab[size_t(r)]);
    if (g->peer_flags[size_t(r)]) cudaIpcCloseMemHandle(g->peer_flags[size_t(r)]);
  }
  if (g->d_ready) cudaFree(g->d_ready);
  if (g->d_consumed) cudaFree(g->d_consumed);
  if (g->slab) cudaFree(g->slab);
  if (g->flags) cudaFree(g->flags);
}

// One rank's share of a head-sharded restore (see the file comment).
void restore_sharded(hc_peer_group* g, hc_store* st, const char* sid_c, const hc_weights* w,
                     const hc_plan* plan_arg, const hc_restore_opts* opts,
                     const hc_kv_pages* pages, const int32_t* d_page_table, cudaStream_t stream,
                     hc_timeline* tl) {
  auto bad = [](const std::string& m) { fail(HC_EINVAL, "restore_sharded: " + m); };
  if (!g || !st || !sid_c || !w || !plan_arg || !pages || !d_page_table) bad("null argument");
  if (g->world == 1) {  // nothing to shard: the single-GPU executor
    restore_session(st, sid_c, w, plan_arg, opts, pages, d_page_table, stream, tl);
    return;
  }
  if (!g->imported) bad("peer group not imported (hc_peer_group_import)");
  if (opts && opts->split_tokens) bad("split_tokens is not supported at world > 1");
  if (w->device != g->device) bad("weights and peer group on different devices");
  Store& store = st->impl;
  const std::string sid(sid_c);
  const hc_manifest m = store.open(sid);  // HC_ENOENT / HC_EINCOMPLETE
  if (plan_serialize(&m.plan) != plan_serialize(plan_arg)) bad("plan does not match session manifest");
  const hc_plan& plan = m.plan;
  if (m.n_layers != w->cfg.n_layers || plan.n_layers != w->cfg.n_layers) bad("layer count mismatch");
  if (m.d_hidden != w->cfg.d_hidden || m.d_hidden != g->d) bad("d_hidden mismatch");
  if (m.elem_bytes != 2 || m.dtype != HC_DTYPE_BF16) bad("bf16 sessions required");
  const int64_t n = m.n_token_ids;  // the context (a shard stores part of it)
  if (n <= 0) fail(HC_ENOENT, "restore_sharded: missing hidden chunks (empty session)");
  validate_pages(w, pages, w->d_kv);
  if (n > int64_t(pages->num_pages) * pages->page_size) bad("KV pages too small for the session");
  if (w->cfg.rope_enabled && n > w->rope_rows) bad("session longer than max_seq (RoPE table)");
  const auto order = compute_order(plan);
  int n_hidden = 0, n_kv = 0, n_re = 0;
  for (const auto& j : order) {
    if (j.method == HC_METHOD_RECOMPUTE) {
      // replicated prefix: every rank runs layers [0, n_re) for all heads
      // (the attention of a layer needs every head) and keeps its own heads
      if (j.layer != n_re) bad("RECOMPUTE layers must form a prefix");
      ++n_re;
      if (!w->layers[size_t(j.layer)].full) bad("RECOMPUTE prefix needs full block weights");
      continue;
    }
    if (j.method == HC_METHOD_HIDDEN) {
      ++n_hidden;
      if (!w->layers[size_t(j.layer)].ready) bad("layer weights not set for a HIDDEN layer");
    } else {
      ++n_kv;
    }
  }
  if (n_kv && (m.d_kv != w->d_kv)) bad("KV rows of this rank's heads expected (session d_kv)");
  if (n_kv && pages->dtype != HC_DTYPE_BF16) bad("KV-offload layers need bf16 pages");
  const int32_t* host_tokens = nullptr;
  if (n_re) {
    if (!w->embedding) bad("RECOMPUTE prefix needs the embedding");
    if (pages->dtype != HC_DTYPE_BF16) bad("RECOMPUTE prefix needs bf16 pages");
    int64_t n_ids = 0;
    host_tokens = store.pinned_tokens(sid, &n_ids);
    if (!host_tokens || n_ids < n) bad("manifest has fewer token ids than tokens");
  }
  const int W = g->world, me = g->rank, d = g->d;
  std::vector<int64_t> r0(size_t(W) + 1);
  for (int r = 0; r < W; ++r) {
    int64_t b, e;
    shard_range(n, W, r, &b, &e);
    r0[size_t(r)] = b;
    if (e - b > g->max_rows) bad("a rank's token range exceeds the peer group's slot rows");
  }
  r0[size_t(W)] = n;
  const int64_t mb = r0[size_t(me)], me_e = r0[size_t(me) + 1], my_rows = me_e - mb;
  // gather plans (throw before anything is queued)
  std::vector<std::vector<CopySeg>> segs(order.size());
  for (size_t i = 0; i < order.size(); ++i) {
    const auto& j = order[i];
    if (j.method == HC_METHOD_RECOMPUTE) continue;
    if (j.method == HC_METHOD_HIDDEN) {
      if (my_rows > 0)
        segs[i] = store.gather_plan(sid, j.layer, HC_STATE_HIDDEN, int(mb), int(me_e), nullptr);
    } else {
      size_t got = 0;
      segs[i] = store.gather_plan(sid, j.layer, HC_STATE_KV, 0, int(n), &got);
      if (got != size_t(n) * size_t(2 * m.d_kv) * 2) bad("KV layer has a short token count");
    }
  }

  DeviceGuard dg(w->device);
  Engine& eng = engine(w->device);
  const bool timed = tl != nullptr || (opts && opts->timeline);
  EventPool evp(timed);
  std::vector<TimedOp> ops;
  const bool norm = w->cfg.norm_enabled != 0;
  const bool center = norm && ln_center_enabled();
  const int sms = device_sm_count(w->device);
  const int N = 2 * w->d_kv;
  const size_t kv_bytes = size_t(n) * size_t(2 * m.d_kv) * 2;
  const int nbuf_kv = std::min(std::max(n_kv, 1), 2);
  StreamScratch ring_kv(n_kv ? kv_bytes * size_t(nbuf_kv) : 0, stream);
  StreamScratch stats(norm && n_hidden ? size_t(n) * 2 * sizeof(float) : 0, stream);
  float* mean = static_cast<float*>(stats.ptr);
  float* rstd = mean ? mean + n : nullptr;
  LaneJoin unwind_join(stream, {eng.copy, eng.aux});

  cudaEvent_t t0 = evp.get();
  HC_CUDA(cudaEventRecord(t0, stream));
  HC_CUDA(cudaStreamWaitEvent(eng.copy, t0, 0));
  HC_CUDA(cudaStreamWaitEvent(eng.aux, t0, 0));
  std::vector<cudaEvent_t> joins, consumed_kv(size_t(nbuf_kv), nullptr);
  const uint32_t abox = uint32_t(gemm_a_box(n));
  // opts->peer_gather == 1 (or HC_SHARDED_GATHER=copy): gather every
  // owner's range with the copy engines into a local buffer and run K1 over
  // it (the all-gather-then-GEMM baseline); default: K1 reads the owners'
  // slots in place (fused)
  static const bool copy_gather_env = [] {
    const char* e = getenv("HC_SHARDED_GATHER");
    return e && std::string(e) == "copy";
  }();
  const bool copy_gather = copy_gather_env || (opts && opts->peer_gather == 1);
  std::unique_ptr<StreamScratch> gathered;  // [n x d], allocated on first use

  // Replicated RECOMPUTE prefix on the compute lane (restore.cpp:177-182):
  // the IO lane fetches the hidden layers' ranges meanwhile, as far as the
  // peer group's slot ring reaches. All heads' K/V of a prefix layer go to a
  // one-layer dense scratch (64-row pages, identity table) that the layer's
  // attention reads; this rank's head columns are then copied into its pages.
  const int64_t re_pages = (n + 63) / 64;
  StreamScratch re_tok(n_re ? sizeof(int32_t) * size_t(n) : 0, stream),
      re_table(n_re ? sizeof(int32_t) * size_t(re_pages) : 0, stream),
      re_k(n_re ? size_t(re_pages) * 64 * size_t(w->d_kv_all) * 2 : 0, stream),
      re_v(n_re ? size_t(re_pages) * 64 * size_t(w->d_kv_all) * 2 : 0, stream);
  bool prefix_done = n_re == 0;
  std::vector<cudaEvent_t> marks;
  std::vector<void*> kp(size_t(w->cfg.n_layers), re_k.ptr), vp(size_t(w->cfg.n_layers), re_v.ptr);
  // enqueued once the first layer's fetch is on the IO lane, so the link
  // starts while the host enqueues the prefix
  auto run_prefix = [&] {
    if (prefix_done) return;
    prefix_done = true;
    HC_CUDA(cudaMemcpyAsync(re_tok.ptr, host_tokens, sizeof(int32_t) * size_t(n),
                            cudaMemcpyHostToDevice, stream));
    HC_CUDA(launch_iota_i32(static_cast<int32_t*>(re_table.ptr), re_pages, stream));
    const hc_kv_pages scratch{w->cfg.n_layers, 64, int32_t(re_pages), w->d_kv_all, HC_DTYPE_BF16,
                              kp.data(), vp.data()};
    auto hook = [&](int layer, bool start) {
      if (start) {
        if (timed) {
          marks.push_back(evp.get());
          HC_CUDA(cudaEventRecord(marks.back(), stream));
        }
        return;
      }
      HC_CUDA(launch_kv_slice(re_k.ptr, re_v.ptr, w->d_kv_all, w->head_begin * w->d_head, n,
                              kv_out_pages(pages, layer, d_page_table, 0, nullptr, 1), stream));
      if (timed) {
        cudaEvent_t e = evp.get();
        HC_CUDA(cudaEventRecord(e, stream));
        ops.push_back({HC_LANE_COMPUTE, layer, HC_EV_RECOMPUTE, marks.back(), e});
      }
    };
    prefill_layers_impl(w, static_cast<const int32_t*>(re_tok.ptr), n, 0, n_re, &scratch,
                        static_cast<const int32_t*>(re_table.ptr), stream, hook, nullptr, nullptr,
                        0, true);
  };
  int ikv = 0;
  for (size_t i = 0; i < order.size(); ++i) {
    const auto& j = order[i];
    const auto& L = w->layers[size_t(j.layer)];
    if (j.method == HC_METHOD_RECOMPUTE) continue;  // (the prefix above)
    if (j.method == HC_METHOD_HIDDEN) {
      const uint64_t stp = g->step++;
      const int slot = int(stp % uint64_t(g->depth));
      const uint32_t ep = uint32_t(stp / uint64_t(g->depth) + 1);
      // IO lane: the slot is free once every consumer released epoch ep-1
      if (ep > 1)
        for (int c = 0; c < W; ++c) HC_CUDA(wait_flag_geq(eng.copy, g->my_flag(1, c, slot), ep - 1));
      cudaEvent_t fs = timed ? evp.get() : nullptr;
      if (fs) HC_CUDA(cudaEventRecord(fs, eng.copy));
      char* data = g->slot_data(me, slot);
      if (my_rows > 0)
        issue_gather(segs[i], reinterpret_cast<uint8_t*>(data), eng, joins, &EventPool::make, &evp);
      cudaEvent_t fetched = evp.get();
      HC_CUDA(cudaEventRecord(fetched, eng.copy));
      if (timed) ops.push_back({HC_LANE_IO, j.layer, HC_EV_FETCH_HIDDEN, fs, fetched});
      // owner: statistics (+ in-place mean shift) of the range, then publish
      HC_CUDA(cudaStreamWaitEvent(eng.aux, fetched, 0));
      if (norm && my_rows > 0) {
        float* om = g->slot_mean(me, slot);
        float* orr = g->slot_rstd(me, slot);
        if (center) {
          int32_t* fl = g->slot_flag(me, slot);
          HC_CUDA(launch_zero_i32(fl, 1, eng.aux));
          HC_CUDA(launch_row_stats_flagged(data, my_rows, d, d, true, om, orr, fl, eng.aux));
          HC_CUDA(launch_center_rows(data, my_rows, d, d, om, fl, data, eng.aux));
        } else {
          HC_CUDA(launch_row_stats(data, my_rows, d, d, true, om, orr, eng.aux));
        }
      }
      HC_CUDA(launch_signal_flags(g->d_ready + size_t(slot) * size_t(W), W, ep, eng.aux));
      run_prefix();  // (first layer only)
      // compute lane: every owner's range of this layer is in place
      for (int r = 0; r < W; ++r) HC_CUDA(wait_flag_geq(stream, g->my_flag(0, r, slot), ep));
      cudaEvent_t cs = timed ? evp.get() : nullptr;
      if (cs) HC_CUDA(cudaEventRecord(cs, stream));
      AMaps am;
      am.n = 0;
      StatSources ss;
      ss.n = 0;
      int64_t max_range = 0;
      bool fused = !copy_gather;
      for (int r = 0; r < W && fused; ++r) {
        const int64_t rows = r0[size_t(r) + 1] - r0[size_t(r)];
        if (rows == 0) continue;
        // a tensor map over another GPU's slot; should the driver refuse it,
        // this layer falls back to the copy-engine gather below
        fused = make_tmap_kmajor_cached(&am.m[am.n], g->slot_data(r, slot), uint64_t(d),
                                        uint64_t(rows), uint64_t(d) * 2, abox);
        am.row0[am.n] = int(r0[size_t(r)]);
        ++am.n;
      }
      if (!fused) {
        // all-gather by the copy engines over NVLink into a local [n x d]
        // buffer, then K1 over it (one map): the non-fused baseline, and the
        // fallback where TMA cannot address peer memory
        if (!gathered) gathered.reset(new StreamScratch(size_t(n) * size_t(d) * 2, stream));
        char* gbuf = static_cast<char*>(gathered->ptr);
        for (int r = 0; r < W; ++r) {
          const int64_t rows = r0[size_t(r) + 1] - r0[size_t(r)];
          if (rows > 0)
            HC_CUDA(cudaMemcpyAsync(gbuf + size_t(r0[size_t(r)]) * size_t(d) * 2,
                                    g->slot_data(r, slot), size_t(rows) * size_t(d) * 2,
                                    cudaMemcpyDefault, stream));
        }
        CUtensorMap gm;
        if (!make_tmap_kmajor_cached(&gm, gbuf, uint64_t(d), uint64_t(n), uint64_t(d) * 2, abox))
          fail(HC_ECUDA, "cuTensorMapEncodeTiled failed for the gathered hidden rows");
        am = single_amap(gm);
      }
      for (int r = 0; r < W; ++r) {
        const int64_t rows = r0[size_t(r) + 1] - r0[size_t(r)];
        if (rows == 0) continue;
        ss.mean[ss.n] = g->slot_mean(r, slot);
        ss.rstd[ss.n] = g->slot_rstd(r, slot);
        ss.row0[ss.n] = r0[size_t(r)];
        ++ss.n;
        max_range = std::max(max_range, rows);
      }
      if (fused) am.row0[am.n] = 0x7fffffff;
      ss.row0[ss.n] = n;
      if (norm) HC_CUDA(launch_gather_stats(ss, max_range, mean, rstd, stream));
      const int bn = gemm_pick_bn(n, N, sms);
      KvOut out = kv_out_pages(pages, j.layer, d_page_table, 0, nullptr, 1);
      HC_CUDA(launch_restore_kv_multi(am, weight_map(L, bn, d, N), bn, int(n), N, d, true, out,
                                      epi_for(w, L.colsum, mean, rstd), sms, stream));
      HC_CUDA(launch_signal_flags(g->d_consumed + size_t(slot) * size_t(W), W, ep, stream));
      cudaEvent_t done = timed ? evp.get() : nullptr;
      if (done) HC_CUDA(cudaEventRecord(done, stream));
      if (timed) ops.push_back({HC_LANE_COMPUTE, j.layer, HC_EV_PROJECT, cs, done});
      continue;
    }
    // KV_OFFLOAD: this rank's heads' rows, local ring + scatter
    const int slot = ikv % nbuf_kv;
    const bool reuse = ikv >= nbuf_kv;
    ++ikv;
    uint8_t* buf = static_cast<uint8_t*>(ring_kv.ptr) + kv_bytes * size_t(slot);
    if (reuse) HC_CUDA(cudaStreamWaitEvent(eng.copy, consumed_kv[size_t(slot)], 0));
    cudaEvent_t fs = timed ? evp.get() : nullptr;
    if (fs) HC_CUDA(cudaEventRecord(fs, eng.copy));
    issue_gather(segs[i], buf, eng, joins, &EventPool::make, &evp);
    cudaEvent_t fetched = evp.get();
    HC_CUDA(cudaEventRecord(fetched, eng.copy));
    if (timed) ops.push_back({HC_LANE_IO, j.layer, HC_EV_FETCH_KV, fs, fetched});
    run_prefix();  // (first layer only)
    HC_CUDA(cudaStreamWaitEvent(stream, fetched, 0));
    cudaEvent_t cs = timed ? evp.get() : nullptr;
    if (cs) HC_CUDA(cudaEventRecord(cs, stream));
    HC_CUDA(launch_kv_scatter(buf, n, kv_out_pages(pages, j.layer, d_page_table, 0, nullptr, 1),
                              stream));
    cudaEvent_t done = evp.get();
    HC_CUDA(cudaEventRecord(done, stream));
    consumed_kv[size_t(slot)] = done;
    if (timed) ops.push_back({HC_LANE_COMPUTE, j.layer, HC_EV_SCATTER, cs, done});
  }
  run_prefix();  // an all-RECOMPUTE plan
  // join the owner lane and the IO lane into the caller stream
  for (cudaStream_t lane : {eng.aux, eng.copy}) {
    cudaEvent_t e = evp.get();
    HC_CUDA(cudaEventRecord(e, lane));
    HC_CUDA(cudaStreamWaitEvent(stream, e, 0));
  }
  if (timed) {
    HC_CUDA(cudaStreamSynchronize(stream));
    if (tl) fill_timeline(tl, t0, ops);
  }
}

}  // namespace

extern "C" {

hc_status hc_shard_range(int64_t n_tokens, int32_t world, int32_t rank, int64_t* begin,
                         int64_t* end) {
  return guard([&] {
    if (n_tokens < 0 || world < 1 || rank < 0 || rank >= world || !begin || !end)
      fail(HC_EINVAL, "shard_range: bad argument");
    shard_range(n_tokens, world, rank, begin, end);
  });
}

hc_status hc_shard_heads(int32_t n_kv_heads, int32_t world, int32_t rank, int32_t* begin,
                         int32_t* count) {
  return guard([&] {
    if (n_kv_heads < 1 || world < 1 || rank < 0 || rank >= world || !begin || !count)
      fail(HC_EINVAL, "shard_heads: bad argument");
    if (n_kv_heads % world)
      fail(HC_EINVAL, "shard_heads: head sharding needs n_kv_heads % world == 0");
    *count = n_kv_heads / world;
    *begin = rank * *count;
  });
}

hc_status hc_peer_group_create(int32_t world, int32_t rank, int32_t device, int32_t d_hidden,
                               int64_t max_rows, int32_t depth, hc_peer_group** out) {
  return guard([&] {
    if (!out) fail(HC_EINVAL, "peer_group_create: null out");
    *out = nullptr;
    if (world < 1 || world > kMaxASrc || rank < 0 || rank >= world)
      fail(HC_EINVAL, "peer_group_create: 1..8 ranks");
    if (d_hidden < 8 || d_hidden % 8 || max_rows < 1 || depth < 1 || depth > 64)
      fail(HC_EINVAL, "peer_group_create: bad shape");
    auto* g = new hc_peer_group;
    g->world = world;
    g->rank = rank;
    g->device = device;
    g->d = d_hidden;
    g->depth = depth;
    g->max_rows = max_rows;
    g->data_bytes = align_up(size_t(max_rows) * size_t(d_hidden) * 2, 256);
    g->slot_bytes = align_up(g->data_bytes + size_t(max_rows) * 8 + 16, 256);
    try {
      DeviceGuard dg(device);
      HC_CUDA(cudaMalloc(&g->slab, g->slot_bytes * size_t(depth)));
      HC_CUDA(cudaMalloc(&g->flags, sizeof(uint32_t) * 2 * size_t(world) * size_t(depth)));
      HC_CUDA(cudaMemset(g->flags, 0, sizeof(uint32_t) * 2 * size_t(world) * size_t(depth)));
      HC_CUDA(cudaDeviceSynchronize());
    } catch (...) {
      release_group(g);
      delete g;
      throw;
    }
    *out = g;
  });
}

void hc_peer_group_destroy(hc_peer_group* g) {
  if (!g) return;
  release_group(g);
  delete g;
}

size_t hc_peer_group_blob_size(void) { return sizeof(Blob); }

hc_status hc_peer_group_export(const hc_peer_group* g, void* blob, size_t cap) {
  return guard([&] {
    if (!g || !blob || cap < sizeof(Blob)) fail(HC_EINVAL, "peer_group_export: bad argument");
    DeviceGuard dg(g->device);
    Blob b;
    std::memset(&b, 0, sizeof b);
    b.magic = kBlobMagic;
    b.world = g->world;
    b.rank = g->rank;
    b.d = g->d;
    b.max_rows = g->max_rows;
    b.depth = g->depth;
    b.slot_bytes = g->slot_bytes;
    HC_CUDA(cudaIpcGetMemHandle(&b.slab, g->slab));
    HC_CUDA(cudaIpcGetMemHandle(&b.flags, g->flags));
    std::memcpy(blob, &b, sizeof b);
  });
}

hc_status hc_peer_group_import(hc_peer_group* g, const void* const* blobs) {
  return guard([&] {
    if (!g || !blobs) fail(HC_EINVAL, "peer_group_import: null argument");
    if (g->imported) fail(HC_EINVAL, "peer_group_import: already imported");
    DeviceGuard dg(g->device);
    g->peer_slab.assign(size_t(g->world), nullptr);
    g->peer_flags.assign(size_t(g->world), nullptr);
    g->peer_slab[size_t(g->rank)] = static_cast<char*>(g->slab);
    g->peer_flags[size_t(g->rank)] = g->flags;
    try {
      for (int r = 0; r < g->world; ++r) {
        if (r == g->rank) continue;
        if (!blobs[r]) fail(HC_EINVAL, "peer_group_import: missing blob");
        Blob b;
        std::memcpy(&b, blobs[r], sizeof b);
        if (b.magic != kBlobMagic || b.world != g->world || b.rank != r || b.d != g->d ||
            b.max_rows != g->max_rows || b.depth != g->depth || b.slot_bytes != g->slot_bytes)
          fail(HC_EINVAL, "peer_group_import: rank " + std::to_string(r) +
                              " has a different group shape");
        void* p = nullptr;
        HC_CUDA(cudaIpcOpenMemHandle(&p, b.slab, cudaIpcMemLazyEnablePeerAccess));
        g->peer_slab[size_t(r)] = static_cast<char*>(p);
        HC_CUDA(cudaIpcOpenMemHandle(&p, b.flags, cudaIpcMemLazyEnablePeerAccess));
        g->peer_flags[size_t(r)] = static_cast<uint32_t*>(p);
      }
      // signal tables: slot s, target rank r
      std::vector<uint32_t*> ready(size_t(g->depth) * size_t(g->world)),
          consumed(size_t(g->depth) * size_t(g->world));
      for (int s = 0; s < g->depth; ++s)
        for (int r = 0; r < g->world; ++r) {
          uint32_t* f = g->peer_flags[size_t(r)];
          const size_t at = size_t(s) * size_t(g->world) + size_t(r);
          ready[at] = f + (size_t(0) * size_t(g->world) + size_t(g->rank)) * size_t(g->depth) + size_t(s);
          consumed[at] = f + (size_t(1) * size_t(g->world) + size_t(g->rank)) * size_t(g->depth) + size_t(s);
        }
      HC_CUDA(cudaMalloc(&g->d_ready, sizeof(uint32_t*) * ready.size()));
      HC_CUDA(cudaMalloc(&g->d_consumed, sizeof(uint32_t*) * consumed.size()));
      HC_CUDA(cudaMemcpy(g->d_ready, ready.data(), sizeof(uint32_t*) * ready.size(),
                         cudaMemcpyHostToDevice));
      HC_CUDA(cudaMemcpy(g->d_consumed, consumed.data(), sizeof(uint32_t*) * consumed.size(),
                         cudaMemcpyHostToDevice));
    } catch (...) {
      for (int r = 0; r < g->world; ++r) {
        if (r == g->rank) continue;
        if (g->peer_slab[size_t(r)]) cudaIpcCloseMemHandle(g->peer_slab[size_t(r)]);
        if (g->peer_flags[size_t(r)]) cudaIpcCloseMemHandle(g->peer_flags[size_t(r)]);
      }
      g->peer_slab.clear();
      g->peer_flags.clear();
      throw;
    }
    g->imported = true;
  });
}

int32_t hc_peer_group_ready(const hc_peer_group* g) { return g && g->imported ? 1 : 0; }

hc_status hc_restore_sharded(hc_peer_group* g, hc_store* s, const char* sid,
                             const hc_weights* w, const hc_plan* plan,
                             const hc_restore_opts* opts, const hc_kv_pages* pages,
                             const int32_t* d_page_table, void* stream, hc_timeline* timeline) {
  return guard([&] {
    NvtxRange r("hc_restore_sharded");
    restore_sharded(g, s, sid, w, plan, opts, pages, d_page_table, as_stream(stream), timeline);
  });
}

}  // extern "C"
