"""Python mirror of the reference's restoration API, over the C ABI.

Names, argument meaning and error behaviour follow the reference
(proj/include/hcache/{planner,pipeline,storage,restore,model}.hpp) so the
parity tests read like the reference's own tests:

* ``RestorationPlan`` / ``ProfiledTimings`` / ``plan`` / ``makespan`` /
  ``brute_force_plan`` (planner.hpp) + ``plan_three_way`` (B200 extension)
* ``PipelineJob`` / ``Timeline`` / ``simulate_pipeline`` (pipeline.hpp)
* ``DevicePool`` / ``SessionSeed`` / ``StorageManager`` / ``interleave_kv`` /
  ``split_kv`` / ``device_for_chunk`` / ``kChunkTokens`` (storage.hpp)
* ``Weights`` / ``KvCache`` / ``project_hidden_to_kv`` / ``restore`` /
  ``restore_batch`` / ``ThrottleConfig`` (model.hpp, restore.hpp) -- device
  side, CUDA tensors via torch for allocation only.

Reference exceptions map as: std::invalid_argument -> ``InvalidArgument``
(a ``ValueError``); std::runtime_error -> ``HCacheError`` subclasses.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from enum import IntEnum
from typing import List, Optional, Sequence

import numpy as np

from . import capi
from .capi import check, lib

kChunkTokens = capi.HC_CHUNK_TOKENS


class Complement(IntEnum):
    NONE = capi.HC_COMPLEMENT_NONE
    KV_OFFLOAD = capi.HC_COMPLEMENT_KV_OFFLOAD
    RECOMPUTE = capi.HC_COMPLEMENT_RECOMPUTE
    MIXED = capi.HC_COMPLEMENT_MIXED


class LayerMethod(IntEnum):
    HIDDEN = capi.HC_METHOD_HIDDEN
    KV_OFFLOAD = capi.HC_METHOD_KV_OFFLOAD
    RECOMPUTE = capi.HC_METHOD_RECOMPUTE


class StateKind(IntEnum):
    HIDDEN = capi.HC_STATE_HIDDEN
    KV = capi.HC_STATE_KV


class Lane(IntEnum):
    IO = capi.HC_LANE_IO
    COMPUTE = capi.HC_LANE_COMPUTE


def device_for_chunk(layer: int, chunk_idx: int, device_count: int) -> int:
    """storage.cpp:29-31."""
    return lib().hc_device_for_chunk(layer, chunk_idx, device_count)


# --------------------------------------------------------------------- planner
class RestorationPlan:
    """planner.hpp:29-40 (+ MIXED three-way plans)."""

    def __init__(self, c: capi.PlanC):
        self._c = c

    @staticmethod
    def make(n_layers: int, l_h: int, complement: Complement) -> "RestorationPlan":
        p = capi.PlanC()
        check(lib().hc_plan_make(n_layers, l_h, int(complement), C.byref(p)))
        return RestorationPlan(p)

    @staticmethod
    def make_mixed(l_re: int, l_h: int, l_kv: int) -> "RestorationPlan":
        p = capi.PlanC()
        check(lib().hc_plan_make_mixed(l_re, l_h, l_kv, C.byref(p)))
        return RestorationPlan(p)

    @staticmethod
    def parse(record: str) -> "RestorationPlan":
        p = capi.PlanC()
        check(lib().hc_plan_parse(record.encode(), C.byref(p)))
        return RestorationPlan(p)

    def serialize(self) -> str:
        buf = C.create_string_buffer(256)
        check(lib().hc_plan_serialize(C.byref(self._c), buf, 256))
        return buf.value.decode()

    l_h = property(lambda self: self._c.l_h)
    l_o = property(lambda self: self._c.l_o)
    l_kv = property(lambda self: self._c.l_kv)
    l_re = property(lambda self: self._c.l_re)
    complement = property(lambda self: Complement(self._c.complement))

    def n_layers(self) -> int:
        return self._c.n_layers

    @property
    def layer_assignment(self) -> List[LayerMethod]:
        return [LayerMethod(self._c.layer_assignment[i]) for i in range(self._c.n_layers)]

    def __eq__(self, other):
        return isinstance(other, RestorationPlan) and self.serialize() == other.serialize()

    def __repr__(self):
        return f"RestorationPlan({self.serialize()})"


# c_token at or above this: no RECOMPUTE layers (no full block weights, or the
# model is not whole on this GPU) -- include/hcache_b200.h HC_RECOMPUTE_UNAVAILABLE
RECOMPUTE_UNAVAILABLE = 1e9


@dataclass
class ProfiledTimings:
    """planner.hpp:16-24 (seconds per layer)."""
    io_h: float = 0.0
    io_kv: float = 0.0
    c_h: float = 0.0
    c_token: float = 0.0
    n_layers: int = 0

    def _c(self):
        return capi.TimingsC(self.io_h, self.io_kv, self.c_h, self.c_token, self.n_layers)

    def validate(self):
        check(lib().hc_timings_validate(C.byref(self._c())))


def plan(t: ProfiledTimings) -> RestorationPlan:
    p = capi.PlanC()
    check(lib().hc_plan_closed_form(C.byref(t._c()), C.byref(p)))
    return RestorationPlan(p)


def brute_force_plan(t: ProfiledTimings) -> RestorationPlan:
    p = capi.PlanC()
    check(lib().hc_brute_force_plan(C.byref(t._c()), C.byref(p)))
    return RestorationPlan(p)


def makespan(p: RestorationPlan, t: ProfiledTimings) -> float:
    out = C.c_double()
    check(lib().hc_makespan(C.byref(p._c), C.byref(t._c()), C.byref(out)))
    return out.value


def executor_depth(n_layers: int, layer_bytes: Optional[int] = None) -> int:
    """The staging depth restore() uses by default (ThrottleConfig
    prefetch_depth 0, restore.cpp auto_depth): every hidden layer staged, up
    to an 8 GiB ring; without `layer_bytes` (one layer's staged hidden bytes)
    the budget is assumed to hold all of them."""
    if not layer_bytes:
        return max(1, n_layers)
    fit = max(2, (8 << 30) // max(1, int(layer_bytes)))
    return max(1, min(n_layers, fit) - 1)


def plan_three_way(t: ProfiledTimings, prefetch_depth: Optional[int] = None,
                   layer_bytes: Optional[int] = None):
    """B200 planner: (plan, bounded-staging makespan). prefetch_depth
    defaults to the executor's own (executor_depth), so the plan is costed
    under the staging bound restore() will actually run with."""
    if prefetch_depth is None:
        prefetch_depth = executor_depth(t.n_layers, layer_bytes)
    p = capi.PlanC()
    out = C.c_double()
    check(lib().hc_plan_three_way(C.byref(t._c()), prefetch_depth, C.byref(p), C.byref(out)))
    return RestorationPlan(p), out.value


def plan_token_split(t: ProfiledTimings, plan: "RestorationPlan", n_tokens: int,
                     prefetch_depth: Optional[int] = None, layer_bytes: Optional[int] = None):
    """B200 extension: (split_tokens, makespan) -- how many tokens of the
    plan's first layer after the recompute prefix to recompute instead of
    fetching (ThrottleConfig.split_tokens); 0 when no split helps."""
    if prefetch_depth is None:
        prefetch_depth = executor_depth(t.n_layers, layer_bytes)
    sp = C.c_int32()
    out = C.c_double()
    check(lib().hc_plan_token_split(C.byref(t._c()), prefetch_depth, C.byref(plan._c), n_tokens,
                                    C.byref(sp), C.byref(out)))
    return sp.value, out.value


# -------------------------------------------------------------------- timeline
@dataclass
class TimelineEvent:
    lane: Lane
    layer: int
    kind: str
    start_s: float
    end_s: float


@dataclass
class Timeline:
    """pipeline.hpp:18-28."""
    events: List[TimelineEvent] = field(default_factory=list)
    total_s: float = 0.0
    fill_s: float = 0.0
    _c: Optional[capi.TimelineC] = None

    @staticmethod
    def from_c(tc: capi.TimelineC) -> "Timeline":
        ev = [TimelineEvent(Lane(e.lane), e.layer, capi.EVENT_KINDS[e.kind], e.start_s, e.end_s)
              for e in tc.events[: tc.n_events]]
        return Timeline(ev, tc.total_s, tc.fill_s, tc)

    def lane_busy(self, lane: Lane) -> float:
        """Time the lane was busy: the union of its event intervals (the
        reference's sum, pipeline.cpp:9-14, whenever events do not overlap)."""
        if self._c is not None:
            return lib().hc_timeline_lane_busy(C.byref(self._c), int(lane))
        iv = sorted((e.start_s, e.end_s) for e in self.events
                    if e.lane == lane and e.end_s > e.start_s)
        busy, cur = 0.0, None
        for a, b in iv:
            if cur is not None and a < cur[1]:
                cur[1] = max(cur[1], b)
                continue
            if cur is not None:
                busy += cur[1] - cur[0]
            cur = [a, b]
        return busy + (cur[1] - cur[0] if cur is not None else 0.0)

    def bubble_fraction(self) -> float:
        out = C.c_double()
        check(lib().hc_timeline_bubble_fraction(C.byref(self._c), C.byref(out)))
        return out.value

    def export_text(self) -> str:
        lines = ["# lane layer kind start_s end_s"]
        for e in self.events:
            lines.append(f"{'IO' if e.lane == Lane.IO else 'COMPUTE'} {e.layer} {e.kind} "
                         f"{e.start_s} {e.end_s}")
        return "\n".join(lines) + "\n"


@dataclass
class PipelineJob:
    """pipeline.hpp:30-41."""
    layer: int = -1
    io_s: float = 0.0
    compute_s: float = 0.0
    has_io: bool = False
    has_compute: bool = False
    io_kind: str = "fetch"
    compute_kind: str = "compute"


def simulate_pipeline(jobs: Sequence[PipelineJob], prefetch_depth: int) -> Timeline:
    arr = (capi.PipelineJobC * max(1, len(jobs)))()
    for i, j in enumerate(jobs):
        arr[i] = capi.PipelineJobC(j.layer, int(j.has_io), int(j.has_compute),
                                   capi.EVENT_KINDS.index(j.io_kind),
                                   capi.EVENT_KINDS.index(j.compute_kind), 0, j.io_s,
                                   j.compute_s)
    tc = capi.TimelineC()
    check(lib().hc_simulate_pipeline(arr, len(jobs), prefetch_depth, C.byref(tc)))
    return Timeline.from_c(tc)


# ----------------------------------------------------------------------- store
@dataclass
class DevicePool:
    """storage.hpp:27-34: `count` pinned arenas stand in for the SSD roots."""
    count: int = 1
    bw_bytes_per_s: float = 0.0
    read_latency_s: float = 0.0


@dataclass
class SessionSeed:
    """storage.hpp:71-79 (+ d_kv for GQA, dtype of 2-byte elements)."""
    session_id: str
    config_hash: int = 0
    n_layers: int = 0
    d_hidden: int = 0
    elem_bytes: int = 2
    plan: Optional[RestorationPlan] = None
    tokens: Sequence[int] = ()
    d_kv: int = 0
    dtype: int = capi.HC_DTYPE_BF16


@dataclass
class LayerChunks:
    layer: int
    kind: StateKind
    n_chunks: int
    n_tokens: int


@dataclass
class SessionManifest:
    """storage.hpp:54-69."""
    session_id: str
    config_hash: int
    n_tokens: int
    n_layers: int
    d_hidden: int
    d_kv: int
    elem_bytes: int
    dtype: int
    device_count: int
    chunk_tokens: int
    plan: RestorationPlan
    tokens: List[int]
    finalized: bool
    _store: "StorageManager" = None

    def find(self, layer: int, kind: StateKind) -> Optional[LayerChunks]:
        nc, nt = C.c_int32(), C.c_int32()
        st = lib().hc_store_layer_info(self._store._h, self.session_id.encode(), layer, int(kind),
                                       C.byref(nc), C.byref(nt))
        if st == capi.HC_ENOENT:
            return None
        check(st)
        return LayerChunks(layer, kind, nc.value, nt.value)


_NP_OF = {capi.HC_DTYPE_F32: np.float32, capi.HC_DTYPE_BF16: np.uint16,
          capi.HC_DTYPE_F16: np.uint16}


class StorageManager:
    """storage.hpp:84-165 over pinned host arenas."""

    def __init__(self, pool: DevicePool, buffer_capacity_bytes: int = 256 << 20):
        d = capi.PoolDescC(pool.count, 0, pool.bw_bytes_per_s, pool.read_latency_s)
        h = C.c_void_p()
        check(lib().hc_store_create(C.byref(d), buffer_capacity_bytes, C.byref(h)))
        self._h = h
        self.pool = pool

    def close(self):
        if getattr(self, "_h", None):
            try:
                lib().hc_store_destroy(self._h)
            except Exception:  # interpreter shutdown
                pass
            self._h = None

    __del__ = close

    def reserve(self, nbytes: int):
        """Page-lock nbytes of arena now (hc_store_reserve), off the save path."""
        check(lib().hc_store_reserve(self._h, int(nbytes)))

    def create_session(self, seed: SessionSeed):
        toks = (C.c_int32 * max(1, len(seed.tokens)))(*seed.tokens)
        p = seed.plan._c if seed.plan is not None else None
        c = capi.SessionSeedC(seed.session_id.encode(), seed.config_hash, seed.n_layers,
                              seed.d_hidden, seed.d_kv, seed.elem_bytes, seed.dtype, 0,
                              C.pointer(p) if p is not None else None, toks, len(seed.tokens))
        check(lib().hc_store_create_session(self._h, C.byref(c)))

    def reopen_for_append(self, sid: str, new_tokens: Sequence[int]):
        toks = (C.c_int32 * max(1, len(new_tokens)))(*new_tokens)
        check(lib().hc_store_reopen_for_append(self._h, sid.encode(), toks, len(new_tokens)))

    def snapshot(self, sid: str, layer: int, kind: StateKind, rows, dtype: int = None,
                 stream=None, tok_begin: Optional[int] = None) -> bool:
        """Host numpy rows (float32, or uint16 bf16 bits with dtype) or a CUDA
        torch tensor (session dtype; copied D2H on `stream`). False on
        backpressure, like the reference. tok_begin: the rows are tokens
        [tok_begin, ...) of the layer (hc_store_snapshot_range: a head-sharded
        rank's own token range)."""
        if hasattr(rows, "is_cuda") and rows.is_cuda:
            import torch
            assert rows.is_contiguous()
            src_dtype = {torch.bfloat16: capi.HC_DTYPE_BF16, torch.float16: capi.HC_DTYPE_F16,
                         torch.float32: capi.HC_DTYPE_F32}[rows.dtype]
            s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
            args = (rows.data_ptr(), rows.shape[0], rows.shape[1], src_dtype, 1, s)
        else:
            rows = np.ascontiguousarray(rows)
            if dtype is None:
                rows = rows.astype(np.float32, copy=False)
                src_dtype = capi.HC_DTYPE_F32
            else:
                src_dtype = dtype
            args = (rows.ctypes.data, rows.shape[0], rows.shape[1], src_dtype, 0, None)
        if tok_begin is None:
            st = lib().hc_store_snapshot(self._h, sid.encode(), layer, int(kind), *args)
        else:
            st = lib().hc_store_snapshot_range(self._h, sid.encode(), layer, int(kind),
                                               int(tok_begin), *args)
        if st == capi.HC_EAGAIN:
            return False
        check(st)
        return True

    def drain(self, max_chunks: int = -1) -> int:
        out = C.c_int64()
        check(lib().hc_store_drain(self._h, max_chunks, C.byref(out)))
        return out.value

    def drain_all(self):
        check(lib().hc_store_drain_all(self._h))

    def finalize(self, sid: str):
        check(lib().hc_store_finalize(self._h, sid.encode()))

    def open(self, sid: str) -> SessionManifest:
        m = capi.ManifestC()
        check(lib().hc_store_open(self._h, sid.encode(), C.byref(m)))
        n = C.c_int64()
        check(lib().hc_store_tokens(self._h, sid.encode(), None, 0, C.byref(n)))
        toks = (C.c_int32 * max(1, n.value))()
        check(lib().hc_store_tokens(self._h, sid.encode(), toks, n.value, C.byref(n)))
        return SessionManifest(m.session_id.decode(), m.config_hash, m.n_tokens, m.n_layers,
                               m.d_hidden, m.d_kv, m.elem_bytes, m.dtype, m.device_count,
                               m.chunk_tokens, RestorationPlan(m.plan), list(toks[: n.value]),
                               bool(m.finalized), self)

    def read_layer(self, m: SessionManifest, layer: int, kind: StateKind):
        """Token-ordered reassembly (storage.cpp:324-346) as a host array
        (float32 for fp32 sessions, else uint16 element bits); None when the
        layer/kind was never stored."""
        lc = m.find(layer, kind)
        if lc is None or lc.n_tokens == 0:
            return None
        width = m.d_hidden if kind == StateKind.HIDDEN else 2 * m.d_kv
        out = np.empty((lc.n_tokens, width), _NP_OF[m.dtype])
        check(lib().hc_store_read_layer(self._h, m.session_id.encode(), layer, int(kind),
                                        out.ctypes.data, out.nbytes, 0, None))
        return out

    def read_layer_device(self, sid: str, layer: int, kind: StateKind, dst, stream=None):
        import torch
        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        check(lib().hc_store_read_layer(self._h, sid.encode(), layer, int(kind), dst.data_ptr(),
                                        dst.numel() * dst.element_size(), 1, s))

    def chunk_info(self, sid: str, layer: int, kind: StateKind, chunk_idx: int):
        dev, ptr, nb = C.c_int32(), C.c_void_p(), C.c_int64()
        check(lib().hc_store_chunk_info(self._h, sid.encode(), layer, int(kind), chunk_idx,
                                        C.byref(dev), C.byref(ptr), C.byref(nb)))
        return dev.value, ptr.value, nb.value

    def device_chunk_counts(self) -> List[int]:
        out = (C.c_int64 * self.pool.count)()
        check(lib().hc_store_device_chunk_counts(self._h, out, self.pool.count))
        return list(out)

    def simulated_read_seconds_tokens(self, n_tokens: int, width: int, elem_bytes: int) -> float:
        return lib().hc_store_simulated_read_seconds_tokens(self._h, n_tokens, width, elem_bytes)

    def start_daemon(self):
        check(lib().hc_store_start_daemon(self._h))

    def stop_daemon(self):
        check(lib().hc_store_stop_daemon(self._h))

    def buffer_bytes(self) -> int:
        return lib().hc_store_buffer_bytes(self._h)

    def buffer_capacity(self) -> int:
        return lib().hc_store_buffer_capacity(self._h)

    def backpressure_events(self) -> int:
        return lib().hc_store_backpressure_events(self._h)

    def pinned(self) -> bool:
        return bool(lib().hc_store_pinned(self._h))


def interleave_kv(k: np.ndarray, v: np.ndarray) -> np.ndarray:
    """storage.cpp:67-75: n x 2d rows, K row then V row per token."""
    if k.shape != v.shape:
        raise ValueError("interleave_kv: K/V shape mismatch")
    return np.concatenate([k, v], axis=1)


def split_kv(rows: np.ndarray):
    """storage.cpp:77-86."""
    if rows.shape[1] % 2:
        raise ValueError("split_kv: odd width")
    d = rows.shape[1] // 2
    return rows[:, :d].copy(), rows[:, d:].copy()


# ---------------------------------------------------------------------- device
@dataclass
class ModelConfig:
    """model.hpp:11-25 (+ n_kv_heads for GQA)."""
    n_layers: int = 4
    d_hidden: int = 256
    n_heads: int = 8
    d_ffn: int = 1024
    vocab_size: int = 1024
    max_seq: int = 4096
    elem_bytes: int = 2
    norm_enabled: bool = True
    rope_enabled: bool = True
    n_kv_heads: int = 0

    def _c(self):
        return capi.ModelConfigC(self.n_layers, self.d_hidden, self.n_heads, self.n_kv_heads,
                                 self.d_ffn, self.vocab_size, self.max_seq, self.elem_bytes,
                                 int(self.norm_enabled), int(self.rope_enabled))

    def d_head(self):
        return self.d_hidden // self.n_heads

    def kv_heads(self):
        return self.n_kv_heads or self.n_heads

    def validate(self):
        check(lib().hc_config_validate(C.byref(self._c())))

    def hash(self) -> int:
        return lib().hc_config_hash(C.byref(self._c()))


def _stream(stream):
    if stream is not None:
        return stream
    import torch
    return torch.cuda.current_stream().cuda_stream


class Weights:
    """Device weight set of the restoration path (hc_weights). Tensors are
    torch CUDA bf16, kept alive by this object."""

    def __init__(self, cfg: ModelConfig, kv_head_begin: int = 0, kv_head_count: int = 0,
                 device: int = 0):
        self.cfg = cfg
        self.kv_head_begin = kv_head_begin
        self.kv_head_count = kv_head_count or (cfg.kv_heads() - kv_head_begin)
        self.d_kv = self.kv_head_count * cfg.d_head()
        h = C.c_void_p()
        check(lib().hc_weights_create(C.byref(cfg._c()), kv_head_begin, self.kv_head_count,
                                      device, C.byref(h)))
        self._h = h
        self._keep = {}

    def close(self):
        if getattr(self, "_h", None):
            try:
                lib().hc_weights_destroy(self._h)
            except Exception:  # interpreter shutdown
                pass
            self._h = None

    __del__ = close

    def set_layer_kv(self, layer: int, wkv):
        """wkv: (2*d_kv x d) bf16 CUDA tensor, K rows then V rows."""
        assert wkv.is_contiguous() and wkv.shape == (2 * self.d_kv, self.cfg.d_hidden)
        self._keep[("kv", layer)] = wkv
        check(lib().hc_weights_set_layer_kv(self._h, layer, wkv.data_ptr()))

    def set_layer_full(self, layer: int, wq, wkv, wo, fc1, fc2):
        for name, t in (("wq", wq), ("wkv_all", wkv), ("wo", wo), ("fc1", fc1), ("fc2", fc2)):
            assert t.is_contiguous()
            self._keep[(name, layer)] = t
        check(lib().hc_weights_set_layer_full(self._h, layer, wq.data_ptr(), wkv.data_ptr(),
                                              wo.data_ptr(), fc1.data_ptr(), fc2.data_ptr()))

    def set_embedding(self, emb):
        assert emb.is_contiguous()
        self._keep["embedding"] = emb
        check(lib().hc_weights_set_embedding(self._h, emb.data_ptr()))


def project_hidden_to_kv(w: Weights, layer: int, h, start_pos: int = 0, out_dtype=None,
                         stream=None):
    """model.cpp:219-235 on the GPU: h (n x d bf16 CUDA) -> (K, V) dense."""
    import torch
    out_dtype = out_dtype or torch.bfloat16
    n = h.shape[0]
    k = torch.empty((n, w.d_kv), dtype=out_dtype, device=h.device)
    v = torch.empty_like(k)
    dt = capi.HC_DTYPE_F32 if out_dtype == torch.float32 else capi.HC_DTYPE_BF16
    check(lib().hc_project_hidden_to_kv(w._h, layer, h.data_ptr(), n, start_pos, k.data_ptr(),
                                        v.data_ptr(), dt, _stream(stream)))
    return k, v


class KvCache:
    """Paged KV cache: per layer a pool [num_pages, page_size, d_kv] for K
    and V (torch CUDA tensors) plus the C descriptor."""

    def __init__(self, n_layers: int, num_pages: int, page_size: int, d_kv: int, dtype=None,
                 device="cuda"):
        import torch
        dtype = dtype or torch.bfloat16
        self.n_layers, self.num_pages, self.page_size, self.d_kv = n_layers, num_pages, page_size, d_kv
        self.k = [torch.zeros((num_pages, page_size, d_kv), dtype=dtype, device=device)
                  for _ in range(n_layers)]
        self.v = [torch.zeros_like(t) for t in self.k]
        self._kp = (C.c_void_p * n_layers)(*[t.data_ptr() for t in self.k])
        self._vp = (C.c_void_p * n_layers)(*[t.data_ptr() for t in self.v])
        self.desc = capi.KvPagesC(n_layers, page_size, num_pages, d_kv,
                                  capi.HC_DTYPE_F32 if dtype == torch.float32 else
                                  capi.HC_DTYPE_BF16, self._kp, self._vp)

    def gather(self, layer: int, page_table, n_tokens: int):
        """Dense (K, V) [n_tokens x d_kv] of one sequence through its page table."""
        import torch
        pt = torch.as_tensor(page_table, device=self.k[layer].device).long()
        pos = torch.arange(n_tokens, device=pt.device)
        pages = pt[pos // self.page_size]
        slots = pos % self.page_size
        return self.k[layer][pages, slots], self.v[layer][pages, slots]


# ------------------------------------------------- multi-GPU (head sharded)
def shard_range(n_tokens: int, world: int, rank: int):
    """[begin, end) token range rank `rank` fetches (128-row aligned)."""
    b, e = C.c_int64(), C.c_int64()
    check(lib().hc_shard_range(n_tokens, world, rank, C.byref(b), C.byref(e)))
    return b.value, e.value


def shard_heads(n_kv_heads: int, world: int, rank: int):
    """(first KV head, count) projected by `rank`."""
    b, c = C.c_int32(), C.c_int32()
    check(lib().hc_shard_heads(n_kv_heads, world, rank, C.byref(b), C.byref(c)))
    return b.value, c.value


class PeerGroup:
    """This rank's member of a head-sharded restore (hc_peer_group): staging
    slots + flags in HBM, exported with CUDA IPC. `exchange(blob) -> list of
    every rank's blob` is any all-gather of bytes (torch.distributed
    all_gather_object on gloo or NCCL here; MPI / sockets in a C++ host)."""

    def __init__(self, world: int, rank: int, d_hidden: int, max_rows: int, depth: int = 2,
                 device: int = 0, exchange=None):
        self.world, self.rank, self.device = world, rank, device
        h = C.c_void_p()
        check(lib().hc_peer_group_create(world, rank, device, d_hidden, max_rows, depth,
                                         C.byref(h)))
        self._h = h
        if world > 1:
            n = lib().hc_peer_group_blob_size()
            buf = C.create_string_buffer(n)
            check(lib().hc_peer_group_export(self._h, buf, n))
            blobs = exchange(bytes(buf.raw))
            keep = [C.create_string_buffer(b, len(b)) for b in blobs]
            arr = (C.c_void_p * world)(*[C.cast(k, C.c_void_p) for k in keep])
            check(lib().hc_peer_group_import(self._h, arr))

    @staticmethod
    def torch_exchange(group=None):
        import torch.distributed as dist

        def ex(blob: bytes):
            out = [None] * dist.get_world_size(group)
            dist.all_gather_object(out, blob, group=group)
            return out
        return ex

    def close(self):
        if self._h:
            lib().hc_peer_group_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def restore_sharded(group: PeerGroup, store: "StorageManager", sid: str, w: "Weights",
                    plan: "RestorationPlan", throttle: "ThrottleConfig", kv: "KvCache",
                    page_table, stream=None, timeline: bool = False):
    """hc_restore_sharded: this rank's share of a head-sharded restore (all
    ranks call it with the same session plan). Returns a Timeline when
    `timeline`, else the work is queued on `stream`."""
    import torch
    s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    tl = capi.TimelineC() if timeline else None
    check(lib().hc_restore_sharded(group._h, store._h, sid.encode(), w._h, C.byref(plan._c),
                                   C.byref(throttle._c()), C.byref(kv.desc),
                                   page_table.data_ptr(), s, C.byref(tl) if tl else None))
    return Timeline.from_c(tl) if tl else None


@dataclass
class ThrottleConfig:
    """restore.hpp:14-29 for the device engine: prefetch_depth bounds the
    staged hidden layers (0 = auto: stage every hidden layer within 8 GiB)."""
    prefetch_depth: int = 0
    timeline: bool = True
    split_tokens: int = 0  # B200 extension (hc_restore_opts.split_tokens)
    peer_gather: int = 0   # restore_sharded: 0 fused peer-memory K1, 1 copy-engine gather

    def _c(self):
        return capi.RestoreOptsC(self.prefetch_depth, int(self.timeline), self.split_tokens,
                                 self.peer_gather)


@dataclass
class RestoreResult:
    kv: KvCache
    timeline: Timeline


def restore(store: StorageManager, session_id: str, w: Weights, p: RestorationPlan,
            throttle: ThrottleConfig, kv: KvCache, page_table, stream=None) -> RestoreResult:
    """restore.hpp:40-42 on the GPU. page_table: int32 CUDA tensor."""
    tc = capi.TimelineC() if throttle.timeline else None
    check(lib().hc_restore(store._h, session_id.encode(), w._h, C.byref(p._c),
                           C.byref(throttle._c()), C.byref(kv.desc), page_table.data_ptr(),
                           _stream(stream), C.byref(tc) if tc is not None else None))
    return RestoreResult(kv, Timeline.from_c(tc) if tc is not None else None)


def restore_batch(store: StorageManager, session_ids: Sequence[str], w: Weights,
                  throttle: ThrottleConfig, kv: KvCache, page_tables, stream=None):
    """Concurrent restore of several sessions sharing one plan (config 4):
    RECOMPUTE prefix as one ragged forward, grouped K1 per HIDDEN layer, one
    K4 scatter per KV layer. page_tables: (n_sessions x table_stride) int32
    CUDA tensor."""
    ids = (C.c_char_p * len(session_ids))(*[s.encode() for s in session_ids])
    tc = capi.TimelineC() if throttle.timeline else None
    check(lib().hc_restore_batch(store._h, ids, len(session_ids), w._h, C.byref(throttle._c()),
                                 C.byref(kv.desc), page_tables.data_ptr(), page_tables.shape[1],
                                 _stream(stream), C.byref(tc) if tc is not None else None))
    return RestoreResult(kv, Timeline.from_c(tc) if tc is not None else None)


def restore_token_wise(store: StorageManager, session_id: str, w: Weights, hidden_tokens: int,
                       kv: KvCache, page_table, stream=None) -> RestoreResult:
    """restore.hpp:47-49 (ablation) on the GPU."""
    tc = capi.TimelineC()
    check(lib().hc_restore_token_wise(store._h, session_id.encode(), w._h, hidden_tokens,
                                      C.byref(kv.desc), page_table.data_ptr(), _stream(stream),
                                      C.byref(tc)))
    return RestoreResult(kv, Timeline.from_c(tc))


def forward_batch(w: Weights, tokens, new_lens: Sequence[int], start_pos: Sequence[int],
                  kv: KvCache, page_tables, layer_inputs=None, stream=None):
    """forward_tokens / decode_step (model.cpp:305-347) batched over sequences
    continuing their paged caches. tokens: int32 CUDA (sum(new_lens)),
    page_tables: int32 CUDA [n_seqs x stride]. Returns the next tokens (int32
    CUDA [n_seqs])."""
    import torch
    n = len(new_lens)
    nl = (C.c_int32 * n)(*new_lens)
    sp = (C.c_int32 * n)(*start_pos)
    nxt = torch.empty(n, dtype=torch.int32, device=tokens.device)
    tables = page_tables if page_tables.dim() == 2 else page_tables.view(1, -1)
    check(lib().hc_forward_batch(w._h, tokens.data_ptr(), n, nl, sp, C.byref(kv.desc),
                                 tables.data_ptr(), tables.shape[1],
                                 None if layer_inputs is None else layer_inputs.data_ptr(),
                                 nxt.data_ptr(), _stream(stream)))
    return nxt


def kv_gather_rows(kv: KvCache, layer: int, page_table, pos0: int, n: int, stream=None):
    """Interleaved [K_row | V_row] rows of positions [pos0, pos0+n) (device)."""
    import torch
    rows = torch.empty((n, 2 * kv.d_kv), dtype=torch.bfloat16, device=page_table.device)
    check(lib().hc_kv_gather_rows(C.byref(kv.desc), layer, page_table.data_ptr(), pos0, n,
                                  rows.data_ptr(), _stream(stream)))
    return rows


def profile_hardware(w: Weights, n_tokens: int) -> ProfiledTimings:
    """harness.hpp:76-77, measured on the device."""
    t = capi.TimingsC()
    check(lib().hc_profile(w._h, n_tokens, C.byref(t)))
    return ProfiledTimings(t.io_h, t.io_kv, t.c_h, t.c_token, t.n_layers)


def timings_from_timeline(tl: "Timeline", base: ProfiledTimings) -> ProfiledTimings:
    """profile_hardware refined on a measured restore (hc_timings_from_timeline):
    each kind the timeline holds events of takes its per-event busy time."""
    if tl._c is None:
        raise ValueError("timings_from_timeline: needs a device timeline")
    t = base._c()
    check(lib().hc_timings_from_timeline(C.byref(tl._c), C.byref(t)))
    return ProfiledTimings(t.io_h, t.io_kv, t.c_h, t.c_token, t.n_layers)


def measure_h2d(bytes_: int, reps: int = 5, device: int = 0) -> float:
    out = C.c_double()
    check(lib().hc_measure_h2d(device, bytes_, reps, C.byref(out)))
    return out.value


# ----------------------------------------------------------------- serving
class Strategy(IntEnum):
    """harness.hpp:14"""
    HCACHE = 0
    KV_OFFLOAD = 1
    RECOMPUTE = 2
    IDEAL = 3


class SavingMode(IntEnum):
    """harness.hpp:17 (device meaning: see hc_saving_mode)."""
    TWO_STAGE = 0
    DIRECT = 1
    OFF = 2


class TraceKind(IntEnum):
    CONVERSATION = 0
    LONG_CONTEXT = 1


@dataclass
class Request:
    """trace.hpp:11-19"""
    session_id: str
    round: int = 1
    history_tokens: int = 0
    context: List[int] = field(default_factory=list)
    prompt: List[int] = field(default_factory=list)
    output_budget: int = 1
    arrival_s: float = 0.0


@dataclass
class TraceParams:
    """trace.hpp:21-36"""
    n_sessions: int = 4
    rounds: int = 3
    mean_input: float = 66.8
    mean_output: float = 358.8
    arrival_rate_per_s: float = 0.1
    round_gap_s: float = 30.0
    ctx_min: int = 4096
    ctx_max: int = 16384
    lc_mean_input: float = 44.7
    lc_mean_output: float = 50.2
    lc_max_io: int = 99
    vocab: int = 1024

    def validate(self):
        """trace.cpp:44-53"""
        if self.n_sessions < 1 or self.rounds < 1 or self.vocab < 1:
            raise ValueError("TraceParams: counts must be >= 1")
        if min(self.mean_input, self.mean_output, self.lc_mean_input, self.lc_mean_output) < 1:
            raise ValueError("TraceParams: means must be >= 1")
        if self.arrival_rate_per_s <= 0 or self.round_gap_s < 0:
            raise ValueError("TraceParams: bad arrival parameters")
        if self.ctx_min < 1 or self.ctx_max < self.ctx_min:
            raise ValueError("TraceParams: bad context range")


@dataclass
class Trace:
    kind: TraceKind
    params: TraceParams
    seed: int
    requests: List[Request]


class _TraceRng:
    """The trace generator's splitmix64 stream (trace.cpp:11-39)."""
    M = (1 << 64) - 1

    def __init__(self, seed):
        self.s = (seed ^ 0xA5A5A5A5DEADBEEF) & self.M

    def next(self):
        self.s = (self.s + 0x9E3779B97F4A7C15) & self.M
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & self.M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & self.M
        return z ^ (z >> 31)

    def uniform(self):
        return float(self.next() >> 11) * 2.0 ** -53

    def geometric(self, mean):
        p = 1.0 / max(1.0, mean)
        u = max(self.uniform(), 1e-300)
        return 1 + int(math.floor(math.log(u) / math.log(1.0 - p)))

    def exponential(self, rate):
        return -math.log(max(self.uniform(), 1e-300)) / rate

    def uniform_int(self, lo, hi):
        return lo + int(self.next() % (hi - lo + 1))

    def tokens(self, n, vocab):
        return [int(self.next() % vocab) for _ in range(n)]


def gen_trace(kind: TraceKind, params: TraceParams, seed: int) -> Trace:
    """gen_trace (trace.cpp:55-100): Poisson session starts, geometric prompt
    and output lengths, conversation rounds round_gap_s apart (or one
    long-context request per session); sorted by arrival (stable)."""
    params.validate()
    rng = _TraceRng(seed)
    reqs = []
    arrival = 0.0
    for s in range(params.n_sessions):
        arrival += rng.exponential(params.arrival_rate_per_s)
        sid = f"sess{s}"
        if kind == TraceKind.CONVERSATION:
            history = 0
            for r in range(1, params.rounds + 1):
                prompt = rng.tokens(rng.geometric(params.mean_input), params.vocab)
                budget = rng.geometric(params.mean_output)
                reqs.append(Request(sid, r, history, [], prompt, budget,
                                    arrival + float(r - 1) * params.round_gap_s))
                history += len(prompt) + budget
        else:
            ctx = rng.tokens(rng.uniform_int(params.ctx_min, params.ctx_max), params.vocab)
            prompt = rng.tokens(min(params.lc_max_io, rng.geometric(params.lc_mean_input)),
                                params.vocab)
            budget = min(params.lc_max_io, rng.geometric(params.lc_mean_output))
            reqs.append(Request(sid, 1, len(ctx), ctx, prompt, budget, arrival))
    reqs.sort(key=lambda r: r.arrival_s)  # stable, like std::stable_sort
    return Trace(kind, params, seed, reqs)


@dataclass
class RequestMetrics:
    """harness.hpp:27-36"""
    session_id: str
    round: int
    arrival_s: float
    history_tokens: int
    restore_s: float
    ttft_s: float
    tbt_s: float
    generated: int


@dataclass
class Metrics:
    """harness.hpp:38-55 + the device engine's extras."""
    strategy: Strategy
    per_request: List[RequestMetrics]
    outputs: List[List[int]]
    ttft_p50: float = 0.0
    ttft_p95: float = 0.0
    tbt_mean: float = 0.0
    tbt_p50: float = 0.0
    tbt_p95: float = 0.0
    restore_tokens_per_s: float = 0.0
    storage_bytes_per_token: float = 0.0
    saved_bytes: int = 0
    saved_tokens: int = 0
    backpressure_stalls: int = 0
    busy_s: float = 0.0
    save_stall_s: float = 0.0
    persist_wait_s: float = 0.0
    decode_steps: int = 0
    decode_tokens: int = 0


def _percentile(xs, p):
    """percentile (harness.cpp:36-44)."""
    if not xs:
        return 0.0
    xs = sorted(xs)
    idx = p * (len(xs) - 1)
    lo = int(idx)
    hi = min(lo + 1, len(xs) - 1)
    frac = idx - lo
    return xs[lo] * (1 - frac) + xs[hi] * frac


def metrics_to_csv(m: "Metrics") -> str:
    """Metrics::to_csv (harness.cpp:153-163): full-precision per-request rows."""
    rows = [f"# strategy={m.strategy.name}",
            "session,round,arrival_s,history,restore_s,ttft_s,tbt_s,generated"]
    for r in m.per_request:
        rows.append(f"{r.session_id},{r.round},{r.arrival_s!r},{r.history_tokens},"
                    f"{r.restore_s!r},{r.ttft_s!r},{r.tbt_s!r},{r.generated}")
    return "\n".join(rows) + "\n"


def metrics_from_csv(text: str) -> "Metrics":
    """Metrics::from_csv (harness.cpp:165-187) + finalize_aggregates
    (harness.cpp:133-151)."""
    strategy, per = Strategy.IDEAL, []
    for line in text.splitlines():
        if not line:
            continue
        if line.startswith("# strategy="):
            strategy = Strategy[line[len("# strategy="):]]
            continue
        if line.startswith("session,"):
            continue
        f = line.split(",")
        if len(f) != 8:
            raise RuntimeError("metrics csv: bad row: " + line)
        per.append(RequestMetrics(f[0], int(f[1]), float(f[2]), int(f[3]), float(f[4]),
                                  float(f[5]), float(f[6]), int(f[7])))
    ttft = [r.ttft_s for r in per]
    tbt = [r.tbt_s for r in per if r.generated > 1]
    hist = sum(r.history_tokens for r in per)
    rest = sum(r.restore_s for r in per)
    return Metrics(strategy, per, [], _percentile(ttft, 0.5), _percentile(ttft, 0.95),
                   sum(tbt) / len(tbt) if tbt else 0.0, _percentile(tbt, 0.5),
                   _percentile(tbt, 0.95), hist / rest if rest > 0 else 0.0)


@dataclass
class RunOptions:
    """harness.hpp:60-65 for the device engine. num_pages: KV page pool (all
    layers); None sizes it for the worst case of the trace."""
    strategy: Strategy = Strategy.HCACHE
    saving: SavingMode = SavingMode.TWO_STAGE
    hcache_plan: Optional[RestorationPlan] = None
    page_size: int = 64
    num_pages: Optional[int] = None
    max_batch: int = 0


def run(trace, w: Weights, store: StorageManager, opt: RunOptions, stream=None) -> Metrics:
    """run (harness.cpp:189-429) on the GPU through hc_serve_run: restore ->
    prefill -> continuous-batching decode over the trace, the clock advanced
    by measured phase durations."""
    reqs = trace.requests if isinstance(trace, Trace) else list(trace)
    n = len(reqs)
    keep = []
    arr = (capi.RequestC * max(n, 1))()
    hist, need, active_need = {}, [], []
    for i, r in enumerate(reqs):
        ctx = (C.c_int32 * max(len(r.context), 1))(*r.context)
        pr = (C.c_int32 * max(len(r.prompt), 1))(*r.prompt)
        sid = r.session_id.encode()
        keep += [ctx, pr, sid]
        arr[i] = capi.RequestC(sid, r.round, len(r.context), ctx, len(r.prompt), r.output_budget,
                               pr, r.arrival_s)
        h = hist.get(r.session_id, 0) or len(r.context)
        need.append(-(-(h + len(r.prompt) + r.output_budget) // opt.page_size))
        hist[r.session_id] = h + len(r.prompt) + r.output_budget
    num_pages = opt.num_pages
    if num_pages is None:
        cap = opt.max_batch + 1 if opt.max_batch > 0 else n
        num_pages = max(1, sum(sorted(need, reverse=True)[:cap]))
    p = opt.hcache_plan or RestorationPlan.make(w.cfg.n_layers, w.cfg.n_layers, Complement.NONE)
    o = capi.ServeOptsC(int(opt.strategy), int(opt.saving), p._c, opt.page_size, num_pages,
                        opt.max_batch, 0)
    per = (capi.RequestMetricsC * max(n, 1))()
    outs = (C.c_int32 * max(1, sum(r.output_budget for r in reqs)))()
    m = capi.ServeMetricsC()
    check(lib().hc_serve_run(store._h, w._h, arr, n, C.byref(o), per, outs, C.byref(m),
                             _stream(stream)))
    pr_list, out_list, off = [], [], 0
    for i, r in enumerate(reqs):
        q = per[i]
        pr_list.append(RequestMetrics(r.session_id, q.round, q.arrival_s, q.history_tokens,
                                      q.restore_s, q.ttft_s, q.tbt_s, q.generated))
        out_list.append(list(outs[off:off + r.output_budget]))
        off += r.output_budget
    return Metrics(opt.strategy, pr_list, out_list, m.ttft_p50, m.ttft_p95, m.tbt_mean, m.tbt_p50,
                   m.tbt_p95, m.restore_tokens_per_s, m.storage_bytes_per_token, m.saved_bytes,
                   m.saved_tokens, m.backpressure_stalls, m.busy_s, m.save_stall_s,
                   m.persist_wait_s, m.decode_steps, m.decode_tokens)


def report(sets: Sequence[Metrics], csv: bool = False) -> str:
    """report (harness.cpp:492-525): one row per strategy, TTFT ratio vs HCACHE."""
    hc = next((m for m in sets if m.strategy == Strategy.HCACHE), None)
    rows = []
    if csv:
        rows.append("strategy,requests,ttft_p50_s,ttft_p95_s,tbt_mean_s,restore_tok_per_s,"
                    "bytes_per_token,ttft_vs_hcache")
    else:
        rows.append(f"{'strategy':<12}{'reqs':>6}{'ttft_p50':>14}{'ttft_p95':>14}{'tbt_mean':>14}"
                    f"{'restore_tok/s':>16}{'bytes/tok':>12}{'vs_hc':>10}")
    for m in sets:
        ratio = m.ttft_p50 / hc.ttft_p50 if hc and hc.ttft_p50 > 0 else 0.0
        if csv:
            rows.append(f"{m.strategy.name},{len(m.per_request)},{m.ttft_p50!r},{m.ttft_p95!r},"
                        f"{m.tbt_mean!r},{m.restore_tokens_per_s!r},{m.storage_bytes_per_token!r},"
                        f"{ratio!r}")
        else:
            rows.append(f"{m.strategy.name:<12}{len(m.per_request):>6}{m.ttft_p50:>14.5g}"
                        f"{m.ttft_p95:>14.5g}{m.tbt_mean:>14.5g}{m.restore_tokens_per_s:>16.5g}"
                        f"{m.storage_bytes_per_token:>12.5g}{ratio:>10.2f}")
    return "\n".join(rows) + "\n"
