// store.cpp -- pinned-host chunk store (StorageManager, proj/src/storage.cpp).
#include "store.h"

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>

namespace hc {

// ------------------------------------------------------------ element codecs
namespace {

inline uint16_t f32_to_bf16(float f) {
  uint32_t x;
  std::memcpy(&x, &f, 4);
  if ((x & 0x7F800000u) == 0x7F800000u && (x & 0x7FFFFFu)) return uint16_t((x >> 16) | 0x40u);
  x += 0x7FFFu + ((x >> 16) & 1u);
  return uint16_t(x >> 16);
}
inline float bf16_to_f32(uint16_t h) {
  uint32_t x = uint32_t(h) << 16;
  float f;
  std::memcpy(&f, &x, 4);
  return f;
}
// IEEE binary16 RNE, include/hcache/fp16.hpp:10-40 (the reference codec)
inline uint16_t f32_to_f16(float f) {
  uint32_t x;
  std::memcpy(&x, &f, 4);
  uint32_t sign = (x >> 16) & 0x8000u, exp = (x >> 23) & 0xFFu, man = x & 0x7FFFFFu;
  if (exp == 0xFF) return uint16_t(sign | 0x7C00u | (man ? 0x200u : 0));
  int e = int(exp) - 127 + 15;
  if (e >= 31) return uint16_t(sign | 0x7C00u);
  if (e <= 0) {
    if (e < -10) return uint16_t(sign);
    man |= 0x800000u;
    int shift = 14 - e;
    uint32_t hm = man >> shift, rem = man & ((1u << shift) - 1), halfway = 1u << (shift - 1);
    if (rem > halfway || (rem == halfway && (hm & 1))) ++hm;
    return uint16_t(sign | hm);
  }
  uint32_t hm = man >> 13, rem = man & 0x1FFFu;
  if (rem > 0x1000u || (rem == 0x1000u && (hm & 1))) {
    if (++hm == 0x400u) {
      hm = 0;
      if (++e >= 31) return uint16_t(sign | 0x7C00u);
    }
  }
  return uint16_t(sign | (uint32_t(e) << 10) | hm);
}
// fp16.hpp:42-68
inline float f16_to_f32(uint16_t h) {
  uint32_t sign = (uint32_t(h) & 0x8000u) << 16, exp = (h >> 10) & 0x1Fu, man = h & 0x3FFu, x;
  if (exp == 0) {
    if (man == 0) {
      x = sign;
    } else {
      int e = -1;
      do {
        ++e;
        man <<= 1;
      } while (!(man & 0x400u));
      man &= 0x3FFu;
      x = sign | uint32_t(127 - 15 - e) << 23 | (man << 13);
    }
  } else if (exp == 31) {
    x = sign | 0x7F800000u | (man << 13);
  } else {
    x = sign | ((exp - 15 + 127) << 23) | (man << 13);
  }
  float f;
  std::memcpy(&f, &x, 4);
  return f;
}

inline size_t dtype_bytes(int dt) { return dt == HC_DTYPE_F32 ? 4 : 2; }

void convert(const void* src, int src_dt, void* dst, int dst_dt, size_t n) {
  if (src_dt == dst_dt) {
    std::memcpy(dst, src, n * dtype_bytes(src_dt));
    return;
  }
  for (size_t i = 0; i < n; ++i) {
    float f;
    if (src_dt == HC_DTYPE_F32) f = static_cast<const float*>(src)[i];
    else if (src_dt == HC_DTYPE_BF16) f = bf16_to_f32(static_cast<const uint16_t*>(src)[i]);
    else f = f16_to_f32(static_cast<const uint16_t*>(src)[i]);
    if (dst_dt == HC_DTYPE_F32) static_cast<float*>(dst)[i] = f;
    else if (dst_dt == HC_DTYPE_BF16) static_cast<uint16_t*>(dst)[i] = f32_to_bf16(f);
    else static_cast<uint16_t*>(dst)[i] = f32_to_f16(f);
  }
}

}  // namespace

// ------------------------------------------------------------ PinnedPool
PinnedPool::~PinnedPool() {
  for (auto& b : blocks_) {
    if (b.second) cudaFreeHost(b.first);
    else std::free(b.first);
  }
}

size_t PinnedPool::size_class(size_t bytes) {
  size_t c = 4096;
  while (c < bytes) c <<= 1;
  return c;
}

void PinnedPool::probe() {
  if (!probed_) {
    int n = 0;
    pinned_ = cudaGetDeviceCount(&n) == cudaSuccess && n > 0;
    if (!pinned_) cudaGetLastError();
    probed_ = true;
  }
}

uint8_t* PinnedPool::new_block(size_t bytes) {
  void* p = nullptr;
  if (pinned_) {
    if (cudaHostAlloc(&p, bytes, cudaHostAllocPortable) != cudaSuccess) {
      cudaGetLastError();
      fail(HC_ENOMEM, "cudaHostAlloc failed for the pinned chunk arena");
    }
    blocks_.push_back({p, true});
  } else {
    p = std::aligned_alloc(4096, bytes);
    if (!p) fail(HC_ENOMEM, "host allocation failed");
    blocks_.push_back({p, false});
  }
  return static_cast<uint8_t*>(p);
}

namespace {
constexpr size_t kSlabBytes = size_t(256) << 20;
}

void* PinnedPool::alloc_raw(size_t bytes) {
  std::lock_guard<std::mutex> lk(mu_);
  probe();
  const size_t r = std::max<size_t>(4096, (bytes + 4095) & ~size_t(4095));
  if (r > left_) {
    // the next reserved slab that fits, else a new one
    auto it = std::find_if(slabs_.begin(), slabs_.end(),
                           [&](const std::pair<uint8_t*, size_t>& sl) { return sl.second >= r; });
    if (it != slabs_.end()) {
      cur_ = it->first;
      left_ = it->second;
      slabs_.erase(it);
    } else {
      const size_t sz = std::max(r, kSlabBytes);
      cur_ = new_block(sz);
      left_ = sz;
    }
  }
  void* p = cur_;
  cur_ += r;
  left_ -= r;
  return p;
}

void PinnedPool::reserve(size_t bytes) {
  std::lock_guard<std::mutex> lk(mu_);
  probe();
  size_t have = left_;
  for (const auto& sl : slabs_) have += sl.second;
  while (have < bytes) {
    slabs_.push_back({new_block(kSlabBytes), kSlabBytes});
    have += kSlabBytes;
  }
}

void* PinnedPool::alloc(size_t bytes) {
  const size_t c = size_class(bytes);
  {
    std::lock_guard<std::mutex> lk(mu_);
    auto it = free_.find(c);
    if (it != free_.end() && !it->second.empty()) {
      void* p = it->second.back();
      it->second.pop_back();
      return p;
    }
  }
  return alloc_raw(c);
}

void PinnedPool::release(void* p, size_t bytes) {
  std::lock_guard<std::mutex> lk(mu_);
  free_[size_class(bytes)].push_back(p);
}

// ------------------------------------------------------------ Store
Store::Store(const hc_pool_desc& pool, size_t capacity)
    : ndev_(pool.device_count), bw_(pool.bw_bytes_per_s), lat_(pool.read_latency_s),
      capacity_(capacity) {
  // DevicePool::validate (storage.cpp:22-27)
  if (ndev_ < 1) fail(HC_EINVAL, "DevicePool: needs >= 1 device");
  if (bw_ < 0 || lat_ < 0) fail(HC_EINVAL, "DevicePool: negative throttle");
  dev_chunks_.assign(size_t(ndev_), 0);
}

Store::~Store() {
  stop_daemon();
  for (auto& r : fifo_)
    if (r.ready) cudaEventDestroy(r.ready);
}

Session& Store::find_open(const std::string& sid) {
  auto it = sessions_.find(sid);
  if (it == sessions_.end()) fail(HC_ERUNTIME, "unknown session: " + sid);
  return it->second;
}

const Session& Store::session_locked(const std::string& sid) const {
  auto it = sessions_.find(sid);
  if (it == sessions_.end()) fail(HC_ENOENT, "no manifest for session: " + sid);
  return it->second;
}

void Store::create_session(const hc_session_seed& seed) {
  // create_session (storage.cpp:118-127)
  if (!seed.session_id || !*seed.session_id) fail(HC_EINVAL, "create_session: empty id");
  if (std::strlen(seed.session_id) >= HC_MAX_SESSION_ID)
    fail(HC_EINVAL, "create_session: id too long");
  if (seed.n_layers < 1 || seed.n_layers > HC_MAX_LAYERS || seed.d_hidden < 1)
    fail(HC_EINVAL, "create_session: bad shape");
  if (seed.elem_bytes != 2 && seed.elem_bytes != 4)
    fail(HC_EINVAL, "create_session: elem_bytes must be 2 or 4");
  Session s;
  s.id = seed.session_id;
  s.config_hash = seed.config_hash;
  s.n_layers = seed.n_layers;
  s.d_hidden = seed.d_hidden;
  s.d_kv = seed.d_kv > 0 ? seed.d_kv : seed.d_hidden;
  s.elem_bytes = seed.elem_bytes;
  s.dtype = seed.elem_bytes == 4 ? HC_DTYPE_F32
                                 : (seed.dtype == HC_DTYPE_F16 ? HC_DTYPE_F16 : HC_DTYPE_BF16);
  if (seed.plan) {
    if (seed.plan->n_layers != seed.n_layers)
      fail(HC_EINVAL, "create_session: plan layer count mismatch");
    s.plan = *seed.plan;
  } else {
    std::memset(&s.plan, 0, sizeof s.plan);
    s.plan.n_layers = seed.n_layers;
    s.plan.l_h = seed.n_layers;
  }
  if (seed.tokens && seed.n_tokens > 0) s.tokens.assign(seed.tokens, seed.tokens + seed.n_tokens);
  std::lock_guard<std::mutex> lk(mu_);
  if (sessions_.count(s.id)) fail(HC_ERUNTIME, "duplicate session id: " + s.id);
  sessions_.emplace(s.id, std::move(s));
}

void Store::reopen_for_append(const std::string& sid, const int32_t* toks, int64_t n) {
  // reopen_for_append (storage.cpp:284-322): the partial tail chunk stays in
  // its slot and keeps filling.
  std::lock_guard<std::mutex> lk(mu_);
  auto it = sessions_.find(sid);
  if (it == sessions_.end()) fail(HC_ENOENT, "no manifest for session: " + sid);
  Session& s = it->second;
  if (!s.finalized) {
    if (s.ever_finalized) fail(HC_ERUNTIME, "session already open: " + sid);
    fail(HC_EINCOMPLETE, "session incomplete (not finalized): " + sid);
  }
  if (toks && n > 0) s.tokens.insert(s.tokens.end(), toks, toks + n);
  s.finalized = false;
}

bool Store::snapshot(const std::string& sid, int layer, int kind, const void* rows,
                     int64_t n_rows, int row_width, int src_dtype, bool src_on_device,
                     cudaStream_t stream, int64_t tok_begin) {
  // snapshot (storage.cpp:129-149)
  std::lock_guard<std::mutex> lk(mu_);
  Session& s = find_open(sid);
  if (tok_begin >= 0 && tok_begin % HC_CHUNK_TOKENS != 0)
    fail(HC_EINVAL, "snapshot_range: tok_begin must be a multiple of 64");
  if (tok_begin > int64_t(s.tokens.size()))
    fail(HC_EINVAL, "snapshot_range: tok_begin beyond the session's tokens");
  if (s.finalized) fail(HC_ERUNTIME, "snapshot after finalize: " + sid);
  if (kind != HC_STATE_HIDDEN && kind != HC_STATE_KV) fail(HC_EINVAL, "snapshot: bad kind");
  if (row_width != s.width(kind)) fail(HC_EINVAL, "snapshot: bad row width");
  if (layer < 0 || layer >= s.n_layers) fail(HC_EINVAL, "snapshot: layer out of range");
  if (n_rows < 0 || (n_rows > 0 && !rows)) fail(HC_EINVAL, "snapshot: bad rows");
  if (src_dtype < HC_DTYPE_F32 || src_dtype > HC_DTYPE_F16)
    fail(HC_EINVAL, "snapshot: bad source dtype");
  const size_t n_elems = size_t(n_rows) * size_t(row_width);
  const size_t bytes = n_elems * size_t(s.elem_bytes);
  if (fifo_bytes_ + bytes > capacity_) {
    ++backpressure_;
    return false;
  }
  Record rec;
  rec.sid = sid;
  rec.layer = layer;
  rec.kind = kind;
  rec.bytes = bytes;
  rec.tok_begin = tok_begin;
  // Device rows appended at a chunk boundary of a stream with nothing pending
  // in stage 1: copy them device->host straight into their chunk slots (the
  // layer-before-token chunk layout, north star (1)) -- one copy-engine run
  // per extent run of consecutive slots, no host memcpy -- and keep only the
  // copy's event in stage 1 (the same byte budget and backpressure).
  if (src_on_device && bytes && src_dtype == s.dtype) {
    LayerStream& ls = s.streams[{layer, kind}];
    ls.kind = kind;
    const size_t cb = s.chunk_bytes(kind), tb = s.token_bytes(kind);
    // range snapshots (a head-sharded rank's token range): a fresh stream
    // starts at tok_begin, or the range continues the stored one
    const bool fresh = ls.n_tokens == 0 && ls.chunks.empty();
    const bool range_ok = tok_begin < 0 || tok_begin == ls.n_tokens || fresh;
    if (range_ok && ls.partial_bytes == 0 && ls.pending_fifo == 0 &&
        int(ls.chunks.size()) == ls.next_chunk_idx) {
      int expect = int((s.tokens.size() + HC_CHUNK_TOKENS - 1) / HC_CHUNK_TOKENS);
      if (tok_begin >= 0) {
        if (fresh && tok_begin > 0) {  // chunks [0, tok_begin/64) are held by other ranks
          const int c0 = int(tok_begin / HC_CHUNK_TOKENS);
          for (int c = 0; c < c0; ++c)
            ls.chunks.push_back(ChunkRef{(layer + c) % ndev_, nullptr, -1});
          ls.next_chunk_idx = ls.first_stored = c0;
          ls.n_tokens = int(tok_begin);
        }
        expect = int((bytes + cb - 1) / cb);  // (flush_record's sizing for range records)
      }
      const uint8_t* src = static_cast<const uint8_t*>(rows);
      uint8_t* run_dst = nullptr;
      size_t run_src = 0, run_len = 0, off = 0;
      auto flush_run = [&] {
        if (run_len)
          check_cuda(cudaMemcpyAsync(run_dst, src + run_src, run_len, cudaMemcpyDeviceToHost,
                                     stream),
                     "snapshot D2H");
        run_len = 0;
      };
      while (off < bytes) {
        uint8_t* slot = new_slot(s, ls, layer, ls.next_chunk_idx, expect);
        const size_t take = std::min(cb, bytes - off);
        if (run_len && run_dst + run_len == slot) {
          run_len += take;
        } else {
          flush_run();
          run_dst = slot;
          run_src = off;
          run_len = take;
        }
        ls.n_tokens += int(take / tb);
        if (take == cb) {
          ++ls.next_chunk_idx;
          ++rec.chunks;
        } else {
          ls.partial_bytes = take;
        }
        off += take;
      }
      flush_run();
      check_cuda(cudaEventCreateWithFlags(&rec.ready, cudaEventDisableTiming), "event create");
      check_cuda(cudaEventRecord(rec.ready, stream), "event record");
      rec.direct = true;
      fifo_bytes_ += bytes;
      fifo_.push_back(rec);
      cv_.notify_all();
      return true;
    }
  }
  rec.buf = static_cast<uint8_t*>(pool_mem_.alloc(bytes ? bytes : 1));
  if (src_on_device) {
    if (src_dtype != s.dtype) {
      pool_mem_.release(rec.buf, bytes ? bytes : 1);
      fail(HC_EINVAL, "snapshot: device rows must already be in the session dtype");
    }
    if (bytes) {
      check_cuda(cudaMemcpyAsync(rec.buf, rows, bytes, cudaMemcpyDeviceToHost, stream),
                 "snapshot D2H");
      check_cuda(cudaEventCreateWithFlags(&rec.ready, cudaEventDisableTiming), "event create");
      check_cuda(cudaEventRecord(rec.ready, stream), "event record");
    }
  } else {
    convert(rows, src_dtype, rec.buf, s.dtype, n_elems);
  }
  fifo_bytes_ += bytes;
  ++s.streams[{layer, kind}].pending_fifo;
  fifo_.push_back(rec);
  cv_.notify_all();
  return true;
}

uint8_t* Store::new_slot(Session& s, LayerStream& ls, int layer, int chunk_idx,
                         int expect_chunks) {
  const int dev = (layer + chunk_idx) % ndev_;  // device_for_chunk (storage.cpp:29-31)
  if (ls.extents.empty()) ls.extents.resize(size_t(ndev_));
  auto& ex = ls.extents[size_t(dev)];
  const size_t cb = s.chunk_bytes(ls.kind);
  if (ex.used == ex.cap) {
    // next extent of consecutive slots. The first one is sized for every
    // chunk this device will hold when the session's token count is known
    // (one copy-engine run per layer and device at restore); later ones grow
    // geometrically. <= 256 MiB each.
    const int max_slots = std::max<int>(1, int((size_t(256) << 20) / cb));
    int cap;
    if (ex.cap == 0) {
      cap = std::max(8, (expect_chunks + ndev_ - 1) / ndev_);
    } else {
      cap = ex.cap * 2;
    }
    cap = std::min(cap, max_slots);
    ex.base = static_cast<uint8_t*>(pool_mem_.alloc_raw(cb * size_t(cap)));
    ex.cap = cap;
    ex.used = 0;
    ex.id = ++next_extent_id_;
  }
  uint8_t* p = ex.base + cb * size_t(ex.used++);
  ls.chunks.push_back(ChunkRef{dev, p, ex.id});
  ++dev_chunks_[size_t(dev)];
  return p;
}

int64_t Store::flush_record(Record& rec) {
  // one stage-1 record into its chunk slots (the body of drain_locked)
  fifo_bytes_ -= rec.bytes;
  if (rec.ready) {
    check_cuda(cudaEventSynchronize(rec.ready), "snapshot D2H wait");
    cudaEventDestroy(rec.ready);
  }
  if (rec.direct) return rec.chunks;  // already in its slots (see snapshot)
  int64_t flushed = 0;
  Session& s = sessions_.at(rec.sid);
  LayerStream& ls = s.streams[{rec.layer, rec.kind}];
  ls.kind = rec.kind;
  --ls.pending_fifo;
  const size_t cb = s.chunk_bytes(rec.kind), tb = s.token_bytes(rec.kind);
  // first extent per device: sized for the chunks this stream will hold -- a
  // whole session, or (range snapshots) this record's own chunks
  int expect_chunks =
      int((s.tokens.size() + HC_CHUNK_TOKENS - 1) / HC_CHUNK_TOKENS);
  if (rec.tok_begin >= 0) {
    if (rec.tok_begin != ls.n_tokens) {
      if (ls.n_tokens != 0 || !ls.chunks.empty()) {
        pool_mem_.release(rec.buf, rec.bytes ? rec.bytes : 1);
        fail(HC_EINVAL, "snapshot_range: tokens must continue the layer's stored range");
      }
      // a shard stream: chunks [0, tok_begin/64) are held by other ranks
      const int c0 = int(rec.tok_begin / HC_CHUNK_TOKENS);
      for (int c = 0; c < c0; ++c)
        ls.chunks.push_back(ChunkRef{(rec.layer + c) % ndev_, nullptr, -1});
      ls.next_chunk_idx = ls.first_stored = c0;
      ls.n_tokens = int(rec.tok_begin);
    }
    expect_chunks = int((rec.bytes + cb - 1) / cb);
  }
  size_t off = 0;
  while (off < rec.bytes) {
    if (ls.partial_bytes == 0 && int(ls.chunks.size()) == ls.next_chunk_idx)
      new_slot(s, ls, rec.layer, ls.next_chunk_idx, expect_chunks);
    const size_t take = std::min(cb - ls.partial_bytes, rec.bytes - off);
    std::memcpy(ls.chunks[size_t(ls.next_chunk_idx)].ptr + ls.partial_bytes, rec.buf + off, take);
    off += take;
    ls.partial_bytes += take;
    ls.n_tokens += int(take / tb);
    if (ls.partial_bytes == cb) {
      ls.partial_bytes = 0;
      ++ls.next_chunk_idx;
      ++flushed;
    }
  }
  pool_mem_.release(rec.buf, rec.bytes ? rec.bytes : 1);
  return flushed;
}

int64_t Store::drain_locked(int64_t max_chunks, bool block) {
  // drain_locked (storage.cpp:162-191)
  int64_t flushed = 0;
  while (!fifo_.empty() && flushed < max_chunks) {
    if (!block && fifo_.front().ready && cudaEventQuery(fifo_.front().ready) == cudaErrorNotReady)
      break;
    Record rec = fifo_.front();
    fifo_.pop_front();
    flushed += flush_record(rec);
  }
  return flushed;
}

int64_t Store::drain(int64_t max_chunks) {
  std::lock_guard<std::mutex> lk(mu_);
  return drain_locked(max_chunks < 0 ? INT64_MAX : max_chunks);
}

void Store::finalize(const std::string& sid) {
  // finalize (storage.cpp:200-217): drains first; idempotent; partial tails
  // are already in place (length implies token count)
  std::lock_guard<std::mutex> lk(mu_);
  // every record whose copy has landed, then this session's own records in
  // order (the serving engine finalizes after its last D2H completed, so these
  // do not block). Records of other sessions still in flight stay queued for
  // the daemon / the next drain: waiting on them here would hold the store
  // lock across unrelated D2H copies and stall concurrent restores.
  drain_locked(INT64_MAX, false);
  for (auto it = fifo_.begin(); it != fifo_.end();) {
    if (it->sid == sid) {
      Record rec = *it;
      it = fifo_.erase(it);
      flush_record(rec);
    } else {
      ++it;
    }
  }
  Session& s = find_open(sid);
  if (s.finalized) return;
  if (!s.tokens.empty()) {
    const size_t need = s.tokens.size() * sizeof(int32_t);
    if (need > s.pinned_tokens_cap) {
      if (s.pinned_tokens) pool_mem_.release(s.pinned_tokens, s.pinned_tokens_cap);
      s.pinned_tokens = static_cast<int32_t*>(pool_mem_.alloc(need));
      s.pinned_tokens_cap = need;
    }
    std::memcpy(s.pinned_tokens, s.tokens.data(), need);
  }
  s.finalized = true;
  s.ever_finalized = true;
}

const int32_t* Store::pinned_tokens(const std::string& sid, int64_t* n_out) const {
  std::lock_guard<std::mutex> lk(mu_);
  const Session& s = session_locked(sid);
  if (!s.finalized) fail(HC_EINCOMPLETE, "session incomplete (not finalized): " + sid);
  if (n_out) *n_out = int64_t(s.tokens.size());
  return s.pinned_tokens;
}

hc_manifest Store::open(const std::string& sid) const {
  // open (storage.cpp:247-282)
  std::lock_guard<std::mutex> lk(mu_);
  const Session& s = session_locked(sid);
  if (!s.finalized) fail(HC_EINCOMPLETE, "session incomplete (not finalized): " + sid);
  hc_manifest m;
  std::memset(&m, 0, sizeof m);
  std::snprintf(m.session_id, sizeof m.session_id, "%s", s.id.c_str());
  m.config_hash = s.config_hash;
  m.n_layers = s.n_layers;
  m.d_hidden = s.d_hidden;
  m.d_kv = s.d_kv;
  m.elem_bytes = s.elem_bytes;
  m.dtype = s.dtype;
  m.device_count = ndev_;
  m.chunk_tokens = HC_CHUNK_TOKENS;
  m.finalized = 1;
  m.n_token_ids = int64_t(s.tokens.size());
  m.plan = s.plan;
  int n_tokens = 0;
  for (const auto& kv : s.streams) n_tokens = std::max(n_tokens, kv.second.n_tokens);
  m.n_tokens = n_tokens;
  return m;
}

bool Store::layer_info(const std::string& sid, int layer, int kind, int* n_chunks,
                       int* n_tokens) const {
  std::lock_guard<std::mutex> lk(mu_);
  const Session& s = session_locked(sid);
  auto it = s.streams.find({layer, kind});
  if (it == s.streams.end()) return false;
  const LayerStream& ls = it->second;
  if (n_chunks) *n_chunks = ls.next_chunk_idx + (ls.partial_bytes ? 1 : 0);
  if (n_tokens) *n_tokens = ls.n_tokens;
  return true;
}

std::vector<int32_t> Store::tokens(const std::string& sid) const {
  std::lock_guard<std::mutex> lk(mu_);
  return session_locked(sid).tokens;
}

std::vector<CopySeg> Store::gather_plan(const std::string& sid, int layer, int kind, int b,
                                        int e, size_t* bytes_out) const {
  // read_layer (storage.cpp:324-346) as copy-engine segments: per device,
  // runs of chunks in consecutive slots become one strided transfer.
  std::lock_guard<std::mutex> lk(mu_);
  const Session& s = session_locked(sid);
  if (!s.finalized) fail(HC_EINCOMPLETE, "session incomplete (not finalized): " + sid);
  auto it = s.streams.find({layer, kind});
  if (it == s.streams.end() || it->second.n_tokens == 0)
    fail(HC_ENOENT, "layer " + std::to_string(layer) + " (" +
                        (kind == HC_STATE_HIDDEN ? "HIDDEN" : "KV") + ") not stored");
  const LayerStream& ls = it->second;
  if (e < 0) e = ls.n_tokens;
  if (b < 0 || b >= e || e > ls.n_tokens || b % HC_CHUNK_TOKENS != 0)
    fail(HC_EINVAL, "read_layer: bad token range");
  if (b < ls.first_stored * HC_CHUNK_TOKENS)
    fail(HC_ENOENT, "layer " + std::to_string(layer) + ": tokens below " +
                        std::to_string(ls.first_stored * HC_CHUNK_TOKENS) +
                        " are not held by this shard");
  const int64_t cb = int64_t(s.chunk_bytes(kind)), tb = int64_t(s.token_bytes(kind));
  const int c_first = b / HC_CHUNK_TOKENS, c_last = (e - 1) / HC_CHUNK_TOKENS;
  auto chunk_len = [&](int c) {  // tokens of chunk c inside [b, e)
    return std::min(c * HC_CHUNK_TOKENS + HC_CHUNK_TOKENS, e) - c * HC_CHUNK_TOKENS;
  };
  std::vector<CopySeg> segs;
  for (int dev = 0; dev < ndev_; ++dev) {
    int c = c_first;
    while (c <= c_last && (layer + c) % ndev_ != dev) ++c;
    while (c <= c_last) {
      const int len = chunk_len(c);
      if (len < HC_CHUNK_TOKENS) {  // partial tail: exact bytes
        segs.push_back(CopySeg{ls.chunks[size_t(c)].ptr, int64_t(c * HC_CHUNK_TOKENS - b) * tb,
                               int64_t(len) * tb, 1, cb, cb});
        c += ndev_;
        continue;
      }
      int run = 1;
      while (c + run * ndev_ <= c_last && chunk_len(c + run * ndev_) == HC_CHUNK_TOKENS &&
             ls.chunks[size_t(c + run * ndev_)].extent == ls.chunks[size_t(c)].extent &&
             ls.chunks[size_t(c + run * ndev_)].ptr ==
                 ls.chunks[size_t(c + (run - 1) * ndev_)].ptr + cb)
        ++run;
      segs.push_back(CopySeg{ls.chunks[size_t(c)].ptr, int64_t(c * HC_CHUNK_TOKENS - b) * tb, cb,
                             run, cb, cb * ndev_});
      c += run * ndev_;
    }
  }
  if (bytes_out) *bytes_out = size_t(e - b) * size_t(tb);
  return segs;
}

void Store::chunk_info(const std::string& sid, int layer, int kind, int c, int* dev,
                       const void** payload, int64_t* bytes) const {
  std::lock_guard<std::mutex> lk(mu_);
  const Session& s = session_locked(sid);
  auto it = s.streams.find({layer, kind});
  if (it == s.streams.end()) fail(HC_ENOENT, "chunk_info: layer not stored");
  const LayerStream& ls = it->second;
  const int n_chunks = ls.next_chunk_idx + (ls.partial_bytes ? 1 : 0);
  if (c < 0 || c >= n_chunks || !ls.chunks[size_t(c)].ptr)
    fail(HC_ENOENT, "chunk_info: no such chunk");
  if (dev) *dev = ls.chunks[size_t(c)].device;
  if (payload) *payload = ls.chunks[size_t(c)].ptr;
  if (bytes)
    *bytes = c < ls.next_chunk_idx ? int64_t(s.chunk_bytes(kind)) : int64_t(ls.partial_bytes);
}

std::vector<int64_t> Store::device_chunk_counts() const {
  // chunk "files" on each device: full chunks, plus partial tails once the
  // session is finalized (storage.cpp:206-213)
  std::lock_guard<std::mutex> lk(mu_);
  std::vector<int64_t> out(size_t(ndev_), 0);
  for (const auto& kv : sessions_)
    for (const auto& st : kv.second.streams) {
      const LayerStream& ls = st.second;
      for (int c = ls.first_stored; c < int(ls.chunks.size()); ++c)
        if (c < ls.next_chunk_idx || kv.second.finalized || kv.second.ever_finalized)
          ++out[size_t(ls.chunks[size_t(c)].device)];
    }
  return out;
}

void Store::start_daemon() {
  // start_daemon (storage.cpp:375-387)
  std::lock_guard<std::mutex> lk(mu_);
  if (daemon_run_) return;
  daemon_run_ = true;
  daemon_ = std::thread([this] {
    std::unique_lock<std::mutex> lk(mu_);
    while (daemon_run_) {
      cv_.wait_for(lk, std::chrono::milliseconds(5),
                   [this] { return !fifo_.empty() || !daemon_run_; });
      try {
        drain_locked(INT64_MAX, false);
      } catch (...) {
      }
      if (!fifo_.empty() && daemon_run_)  // a D2H still in flight: poll without holding mu_
        cv_.wait_for(lk, std::chrono::microseconds(200));
    }
  });
}

bool Store::daemon_running() const {
  std::lock_guard<std::mutex> lk(mu_);
  return daemon_run_;
}

void Store::stop_daemon() {
  {
    std::lock_guard<std::mutex> lk(mu_);
    if (!daemon_run_) return;
    daemon_run_ = false;
  }
  cv_.notify_all();
  if (daemon_.joinable()) daemon_.join();
}

size_t Store::buffer_bytes() const {
  std::lock_guard<std::mutex> lk(mu_);
  return fifo_bytes_;
}

uint64_t Store::backpressure_events() const {
  std::lock_guard<std::mutex> lk(mu_);
  return backpressure_;
}

double Store::simulated_read_seconds_tokens(int n_tokens, int width, int elem_bytes) const {
  // simulated_read_seconds_tokens (storage.cpp:348-365)
  if (n_tokens <= 0) return 0.0;
  const int n_chunks = (n_tokens + HC_CHUNK_TOKENS - 1) / HC_CHUNK_TOKENS;
  std::vector<double> per_device(size_t(ndev_), 0.0);
  int token = 0;
  for (int ci = 0; ci < n_chunks; ++ci) {
    const int len = std::min(HC_CHUNK_TOKENS, n_tokens - token);
    token += len;
    const double bytes = double(len) * double(width) * double(elem_bytes);
    double t = lat_;
    if (bw_ > 0) t += bytes / bw_;
    per_device[size_t(ci % ndev_)] += t;
  }
  double worst = 0;
  for (double t : per_device) worst = std::max(worst, t);
  return worst;
}

}  // namespace hc

using namespace hc;

namespace {
Store& S(hc_store* s) {
  if (!s) fail(HC_EINVAL, "null store");
  return s->impl;
}
std::string SID(const char* sid) {
  if (!sid) fail(HC_EINVAL, "null session id");
  return sid;
}
}  // namespace

extern "C" {

hc_status hc_store_create(const hc_pool_desc* pool, size_t buffer_capacity_bytes,
                          hc_store** out) {
  return guard([&] {
    if (!pool || !out) fail(HC_EINVAL, "store_create: null argument");
    *out = nullptr;
    *out = new hc_store(*pool, buffer_capacity_bytes);
  });
}

void hc_store_destroy(hc_store* s) { delete s; }

hc_status hc_store_reserve(hc_store* s, size_t bytes) {
  return guard([&] {
    if (!s) fail(HC_EINVAL, "store_reserve: null store");
    S(s).reserve_pinned(bytes);
  });
}

hc_status hc_store_create_session(hc_store* s, const hc_session_seed* seed) {
  return guard([&] {
    if (!seed) fail(HC_EINVAL, "create_session: null seed");
    S(s).create_session(*seed);
  });
}

hc_status hc_store_reopen_for_append(hc_store* s, const char* sid, const int32_t* new_tokens,
                                     int64_t n) {
  return guard([&] { S(s).reopen_for_append(SID(sid), new_tokens, n); });
}

hc_status hc_store_snapshot(hc_store* s, const char* sid, int32_t layer, int32_t kind,
                            const void* rows, int64_t n_rows, int32_t row_width,
                            int32_t src_dtype, int32_t src_on_device, void* stream) {
  hc_status st = HC_OK;
  hc_status g = guard([&] {
    NvtxRange r("hc_store_snapshot");
    if (!S(s).snapshot(SID(sid), layer, kind, rows, n_rows, row_width, src_dtype,
                       src_on_device != 0, as_stream(stream)))
      st = HC_EAGAIN;
  });
  if (g == HC_OK && st == HC_EAGAIN) set_last_error("snapshot: buffer full (backpressure)");
  return g != HC_OK ? g : st;
}

hc_status hc_store_snapshot_range(hc_store* s, const char* sid, int32_t layer, int32_t kind,
                                  int64_t tok_begin, const void* rows, int64_t n_rows,
                                  int32_t row_width, int32_t src_dtype, int32_t src_on_device,
                                  void* stream) {
  hc_status st = HC_OK;
  hc_status g = guard([&] {
    if (tok_begin < 0) fail(HC_EINVAL, "snapshot_range: negative tok_begin");
    if (!S(s).snapshot(SID(sid), layer, kind, rows, n_rows, row_width, src_dtype,
                       src_on_device != 0, as_stream(stream), tok_begin))
      st = HC_EAGAIN;
  });
  if (g == HC_OK && st == HC_EAGAIN) set_last_error("snapshot: buffer full (backpressure)");
  return g != HC_OK ? g : st;
}

hc_status hc_store_drain(hc_store* s, int64_t max_chunks, int64_t* flushed) {
  return guard([&] {
    int64_t f = S(s).drain(max_chunks);
    if (flushed) *flushed = f;
  });
}

hc_status hc_store_drain_all(hc_store* s) {
  return guard([&] { S(s).drain(-1); });
}

hc_status hc_store_finalize(hc_store* s, const char* sid) {
  return guard([&] { S(s).finalize(SID(sid)); });
}

hc_status hc_store_open(hc_store* s, const char* sid, hc_manifest* out) {
  return guard([&] {
    if (!out) fail(HC_EINVAL, "open: null out");
    *out = S(s).open(SID(sid));
  });
}

hc_status hc_store_layer_info(hc_store* s, const char* sid, int32_t layer, int32_t kind,
                              int32_t* n_chunks, int32_t* n_tokens) {
  return guard([&] {
    int c = 0, t = 0;
    if (!S(s).layer_info(SID(sid), layer, kind, &c, &t))
      fail(HC_ENOENT, "layer/kind not stored");
    if (n_chunks) *n_chunks = c;
    if (n_tokens) *n_tokens = t;
  });
}

hc_status hc_store_tokens(hc_store* s, const char* sid, int32_t* out, int64_t cap,
                          int64_t* n_out) {
  return guard([&] {
    auto t = S(s).tokens(SID(sid));
    if (n_out) *n_out = int64_t(t.size());
    if (out) std::memcpy(out, t.data(), sizeof(int32_t) * size_t(std::min<int64_t>(cap, int64_t(t.size()))));
  });
}

static void read_range(hc_store* s, const char* sid, int32_t layer, int32_t kind, int b, int e,
                       void* dst, int64_t dst_bytes, int32_t on_device, void* stream) {
  size_t need = 0;
  auto segs = S(s).gather_plan(SID(sid), layer, kind, b, e, &need);
  if (!dst || dst_bytes < int64_t(need)) fail(HC_EINVAL, "read_layer: destination too small");
  auto* d = static_cast<uint8_t*>(dst);
  for (const auto& g : segs) {
    if (on_device) {
      if (g.height == 1 || g.dpitch == g.width)
        check_cuda(cudaMemcpyAsync(d + g.dst_off, g.src, size_t(g.width * g.height),
                                   cudaMemcpyHostToDevice, as_stream(stream)),
                   "read_layer H2D");
      else
        check_cuda(cudaMemcpy2DAsync(d + g.dst_off, size_t(g.dpitch), g.src, size_t(g.spitch),
                                     size_t(g.width), size_t(g.height), cudaMemcpyHostToDevice,
                                     as_stream(stream)),
                   "read_layer H2D");
    } else {
      for (int64_t r = 0; r < g.height; ++r)
        std::memcpy(d + g.dst_off + r * g.dpitch, g.src + r * g.spitch, size_t(g.width));
    }
  }
}

hc_status hc_store_read_layer(hc_store* s, const char* sid, int32_t layer, int32_t kind,
                              void* dst, int64_t dst_bytes, int32_t dst_on_device, void* stream) {
  return guard([&] { read_range(s, sid, layer, kind, 0, -1, dst, dst_bytes, dst_on_device, stream); });
}

hc_status hc_store_read_layer_range(hc_store* s, const char* sid, int32_t layer, int32_t kind,
                                    int32_t tok_begin, int32_t tok_end, void* dst,
                                    int64_t dst_bytes, int32_t dst_on_device, void* stream) {
  return guard([&] {
    read_range(s, sid, layer, kind, tok_begin, tok_end, dst, dst_bytes, dst_on_device, stream);
  });
}

hc_status hc_store_chunk_info(hc_store* s, const char* sid, int32_t layer, int32_t kind,
                              int32_t chunk_idx, int32_t* device, const void** payload,
                              int64_t* bytes) {
  return guard([&] {
    int dev = 0;
    S(s).chunk_info(SID(sid), layer, kind, chunk_idx, &dev, payload, bytes);
    if (device) *device = dev;
  });
}

hc_status hc_store_device_chunk_counts(hc_store* s, int64_t* out, int32_t cap) {
  return guard([&] {
    auto v = S(s).device_chunk_counts();
    if (!out || cap < int32_t(v.size())) fail(HC_EINVAL, "device_chunk_counts: buffer too small");
    std::copy(v.begin(), v.end(), out);
  });
}

hc_status hc_store_start_daemon(hc_store* s) {
  return guard([&] { S(s).start_daemon(); });
}
hc_status hc_store_stop_daemon(hc_store* s) {
  return guard([&] { S(s).stop_daemon(); });
}
size_t hc_store_buffer_bytes(hc_store* s) { return s ? s->impl.buffer_bytes() : 0; }
size_t hc_store_buffer_capacity(hc_store* s) { return s ? s->impl.capacity() : 0; }
uint64_t hc_store_backpressure_events(hc_store* s) {
  return s ? s->impl.backpressure_events() : 0;
}
double hc_store_simulated_read_seconds_tokens(hc_store* s, int32_t n_tokens, int32_t width,
                                              int32_t elem_bytes) {
  return s ? s->impl.simulated_read_seconds_tokens(n_tokens, width, elem_bytes) : 0.0;
}
int32_t hc_store_pinned(hc_store* s) { return s && s->impl.pinned() ? 1 : 0; }

}  // extern "C"
