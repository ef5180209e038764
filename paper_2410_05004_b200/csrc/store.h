// store.h -- pinned-host chunk store behind hc_store (internal).
//
// The reference StorageManager (proj/include/hcache/storage.hpp:84-165) keeps
// 64-token chunks as files striped over directory "devices". Here the devices
// are pinned host arenas (stand-ins for SSDs, north star (1)); chunk keys,
// striping (device_for_chunk), payload layout (tokens consecutive, d elements
// each, or [K_row|V_row] for KV) and manifest semantics are the reference's.
// Stage 1 (snapshot) is a bulk copy -- D2H on the caller's side stream when
// the rows are on the GPU -- into a bounded pinned FIFO; stage 2 (drain)
// assembles chunks into the arenas. Chunks of one (session, layer, kind) on
// one device are allocated in consecutive slots of growing extents, so a
// restore gathers a layer with one strided copy-engine transfer per run.
#pragma once

#include <condition_variable>
#include <cstdint>
#include <deque>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "common.h"

namespace hc {

// Pinned (cudaHostAlloc, portable) memory with size-class free lists; falls
// back to aligned host memory on GPU-less hosts (store logic tests).
class PinnedPool {
 public:
  ~PinnedPool();
  void* alloc(size_t bytes);
  void release(void* p, size_t bytes);
  // Never returned before destruction: carved from 256 MiB page-locked slabs
  // (cudaHostAlloc pins page by page -- tens of ms per slab -- and is
  // best kept off a restore's critical path).
  void* alloc_raw(size_t bytes);
  // Page-lock slabs for `bytes` of future alloc_raw calls now.
  void reserve(size_t bytes);
  bool pinned() const { return pinned_; }

 private:
  static size_t size_class(size_t bytes);
  void probe();
  uint8_t* new_block(size_t bytes);
  std::mutex mu_;
  std::map<size_t, std::vector<void*>> free_;
  std::vector<std::pair<void*, bool>> blocks_;  // (ptr, is_cuda_host)
  std::vector<std::pair<uint8_t*, size_t>> slabs_;  // reserved, not yet in use
  uint8_t* cur_ = nullptr;  // bump pointer into the current slab
  size_t left_ = 0;
  bool pinned_ = false;
  bool probed_ = false;
};

struct ChunkRef {
  int device = 0;
  uint8_t* ptr = nullptr;  // slot start (slot_bytes capacity)
  int64_t extent = 0;      // id of the pinned allocation holding the slot
};

struct LayerStream {
  int kind = 0;
  int n_tokens = 0;         // tokens stored so far
  int next_chunk_idx = 0;   // index of the chunk being filled (== full chunks)
  int first_stored = 0;     // shard streams: chunks [0, first_stored) are held elsewhere
  size_t partial_bytes = 0; // bytes in the chunk being filled
  std::vector<ChunkRef> chunks;  // every started chunk, in chunk order
  int pending_fifo = 0;     // stage-1 records of this stream awaiting assembly
  // per device: current extent (consecutive slots)
  struct Extent {
    uint8_t* base = nullptr;
    int cap = 0;
    int used = 0;
    int64_t id = 0;
  };
  std::vector<Extent> extents;
};

struct Session {
  std::string id;
  uint64_t config_hash = 0;
  int n_layers = 0, d_hidden = 0, d_kv = 0, elem_bytes = 2, dtype = HC_DTYPE_BF16;
  hc_plan plan{};
  std::vector<int32_t> tokens;
  int32_t* pinned_tokens = nullptr;  // page-locked copy made at finalize (restore H2D)
  size_t pinned_tokens_cap = 0;
  std::map<std::pair<int, int>, LayerStream> streams;  // (layer, kind)
  bool finalized = false;
  bool ever_finalized = false;
  int width(int kind) const { return kind == HC_STATE_HIDDEN ? d_hidden : 2 * d_kv; }
  size_t token_bytes(int kind) const { return size_t(width(kind)) * size_t(elem_bytes); }
  size_t chunk_bytes(int kind) const { return size_t(HC_CHUNK_TOKENS) * token_bytes(kind); }
};

// One contiguous source run of a gather: `height` slots of `width` bytes,
// src pitch `spitch`, landing at dst offset `dst_off` with pitch `dpitch`.
struct CopySeg {
  const uint8_t* src;
  int64_t dst_off;
  int64_t width;
  int64_t height;
  int64_t spitch;
  int64_t dpitch;
};

class Store {
 public:
  Store(const hc_pool_desc& pool, size_t capacity);
  ~Store();

  void create_session(const hc_session_seed& seed);
  void reopen_for_append(const std::string& sid, const int32_t* toks, int64_t n);
  // tok_begin >= 0 (chunk aligned): the rows are tokens [tok_begin, ..) of
  // the layer -- a head-sharded rank stores only its own token range; the
  // stream's earlier chunks then belong to other ranks. -1: append.
  bool snapshot(const std::string& sid, int layer, int kind, const void* rows, int64_t n_rows,
                int row_width, int src_dtype, bool src_on_device, cudaStream_t stream,
                int64_t tok_begin = -1);
  int64_t drain(int64_t max_chunks);
  void finalize(const std::string& sid);
  hc_manifest open(const std::string& sid) const;
  bool layer_info(const std::string& sid, int layer, int kind, int* n_chunks, int* n_tokens) const;
  std::vector<int32_t> tokens(const std::string& sid) const;
  // Page-locked token ids of a finalized session (valid until the next
  // reopen/finalize); n_out = count.
  const int32_t* pinned_tokens(const std::string& sid, int64_t* n_out) const;
  // Gather plan for tokens [b, e) of (sid, layer, kind) into a dst buffer that
  // starts at token b. Requires a finalized session; b chunk aligned.
  std::vector<CopySeg> gather_plan(const std::string& sid, int layer, int kind, int b, int e,
                                   size_t* bytes_out) const;
  void chunk_info(const std::string& sid, int layer, int kind, int c, int* dev,
                  const void** payload, int64_t* bytes) const;
  std::vector<int64_t> device_chunk_counts() const;
  // Page-lock `bytes` of chunk arena now (e.g. a serving run's whole save
  // volume at start-up), so later extents are carved without cudaHostAlloc.
  void reserve_pinned(size_t bytes) { pool_mem_.reserve(bytes); }
  void start_daemon();
  bool daemon_running() const;
  void stop_daemon();
  size_t buffer_bytes() const;
  size_t capacity() const { return capacity_; }
  uint64_t backpressure_events() const;
  double simulated_read_seconds_tokens(int n_tokens, int width, int elem_bytes) const;
  int device_count() const { return ndev_; }
  bool pinned() const { return pool_mem_.pinned(); }
  const Session& session_locked(const std::string& sid) const;  // caller holds no lock
  std::mutex& mutex() const { return mu_; }

 private:
  struct Record {
    std::string sid;
    int layer = 0, kind = 0;
    uint8_t* buf = nullptr;
    size_t bytes = 0;
    cudaEvent_t ready = nullptr;  // D2H completion (device-sourced rows)
    int64_t tok_begin = -1;       // range snapshot (shard sessions)
    // direct: the rows were copied device->host straight into their chunk
    // slots at snapshot time (the stream's bookkeeping is already advanced);
    // the record only holds the copy's event and its stage-1 byte budget
    bool direct = false;
    int64_t chunks = 0;
  };
  // block=false stops at the first record whose device->host copy is still
  // in flight (the daemon never waits on the GPU while holding mu_).
  int64_t drain_locked(int64_t max_chunks, bool block = true);
  int64_t flush_record(Record& rec);
  uint8_t* new_slot(Session& s, LayerStream& ls, int layer, int chunk_idx, int expect_chunks);
  Session& find_open(const std::string& sid);

  int ndev_;
  double bw_, lat_;
  size_t capacity_;
  mutable PinnedPool pool_mem_;
  mutable std::mutex mu_;
  std::condition_variable cv_;
  std::deque<Record> fifo_;
  size_t fifo_bytes_ = 0;
  uint64_t backpressure_ = 0;
  std::map<std::string, Session> sessions_;
  std::vector<int64_t> dev_chunks_;
  int64_t next_extent_id_ = 0;
  std::thread daemon_;
  bool daemon_run_ = false;
};

}  // namespace hc

struct hc_store {
  hc::Store impl;
  hc_store(const hc_pool_desc& p, size_t cap) : impl(p, cap) {}
};
