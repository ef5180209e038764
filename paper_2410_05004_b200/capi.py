"""ctypes binding of the C ABI declared in include/hcache_b200.h.

The library is the in-tree ``paper_2410_05004_b200/lib/libhcache_b200.so``
built by ``__graft_entry__.build()``. There is no fallback: if the library is
missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HC_LIB_PATH") or os.path.join(HERE, "lib", "libhcache_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(HERE), "include", "hcache_b200.h")

HC_OK, HC_EINVAL, HC_ENOENT, HC_EINCOMPLETE, HC_EAGAIN, HC_ECUDA, HC_ENCCL, HC_ERUNTIME, \
    HC_ENOMEM = range(9)
HC_DTYPE_F32, HC_DTYPE_BF16, HC_DTYPE_F16 = 0, 1, 2
HC_STATE_HIDDEN, HC_STATE_KV = 0, 1
HC_METHOD_HIDDEN, HC_METHOD_KV_OFFLOAD, HC_METHOD_RECOMPUTE = 0, 1, 2
HC_COMPLEMENT_NONE, HC_COMPLEMENT_KV_OFFLOAD, HC_COMPLEMENT_RECOMPUTE, HC_COMPLEMENT_MIXED = \
    0, 1, 2, 3
HC_LANE_IO, HC_LANE_COMPUTE = 0, 1
EVENT_KINDS = ["fetch_hidden", "fetch_kv", "project", "recompute", "scatter", "gather", "fetch",
               "compute"]
HC_CHUNK_TOKENS = 64
HC_MAX_LAYERS = 256
HC_MAX_EVENTS = 4 * HC_MAX_LAYERS
HC_MAX_SESSION_ID = 128

i32, i64, u64, f64, f32 = C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_float
vp, cp = C.c_void_p, C.c_char_p


class ModelConfigC(C.Structure):
    _fields_ = [(n, i32) for n in ("n_layers", "d_hidden", "n_heads", "n_kv_heads", "d_ffn",
                                   "vocab_size", "max_seq", "elem_bytes", "norm_enabled",
                                   "rope_enabled")]


class KvPagesC(C.Structure):
    _fields_ = [("n_layers", i32), ("page_size", i32), ("num_pages", i32), ("d_kv", i32),
                ("dtype", i32), ("k_layers", C.POINTER(vp)), ("v_layers", C.POINTER(vp))]


class PlanC(C.Structure):
    _fields_ = [("n_layers", i32), ("l_h", i32), ("l_o", i32), ("complement", i32),
                ("l_kv", i32), ("l_re", i32), ("layer_assignment", C.c_uint8 * HC_MAX_LAYERS)]


class TimingsC(C.Structure):
    _fields_ = [("io_h", f64), ("io_kv", f64), ("c_h", f64), ("c_token", f64), ("n_layers", i32)]


class EventC(C.Structure):
    _fields_ = [("lane", i32), ("layer", i32), ("kind", i32), ("pad_", i32), ("start_s", f64),
                ("end_s", f64)]


class TimelineC(C.Structure):
    _fields_ = [("n_events", i32), ("pad_", i32), ("total_s", f64), ("fill_s", f64),
                ("events", EventC * HC_MAX_EVENTS)]


class PipelineJobC(C.Structure):
    _fields_ = [("layer", i32), ("has_io", i32), ("has_compute", i32), ("io_kind", i32),
                ("compute_kind", i32), ("pad_", i32), ("io_s", f64), ("compute_s", f64)]


class PoolDescC(C.Structure):
    _fields_ = [("device_count", i32), ("pad_", i32), ("bw_bytes_per_s", f64),
                ("read_latency_s", f64)]


class SessionSeedC(C.Structure):
    _fields_ = [("session_id", cp), ("config_hash", u64), ("n_layers", i32), ("d_hidden", i32),
                ("d_kv", i32), ("elem_bytes", i32), ("dtype", i32), ("pad_", i32),
                ("plan", C.POINTER(PlanC)), ("tokens", C.POINTER(i32)), ("n_tokens", i64)]


class ManifestC(C.Structure):
    _fields_ = [("session_id", C.c_char * HC_MAX_SESSION_ID), ("config_hash", u64),
                ("n_tokens", i32), ("n_layers", i32), ("d_hidden", i32), ("d_kv", i32),
                ("elem_bytes", i32), ("dtype", i32), ("device_count", i32),
                ("chunk_tokens", i32), ("finalized", i32), ("pad_", i32), ("n_token_ids", i64),
                ("plan", PlanC)]


class RestoreOptsC(C.Structure):
    _fields_ = [("prefetch_depth", i32), ("timeline", i32), ("split_tokens", i32),
                ("peer_gather", i32)]


class RequestC(C.Structure):
    _fields_ = [("session_id", cp), ("round", i32), ("n_context", i32), ("context", C.POINTER(i32)),
                ("n_prompt", i32), ("output_budget", i32), ("prompt", C.POINTER(i32)),
                ("arrival_s", f64)]


class ServeOptsC(C.Structure):
    _fields_ = [("strategy", i32), ("saving", i32), ("plan", PlanC), ("page_size", i32),
                ("num_pages", i32), ("max_batch", i32), ("pad_", i32)]


class RequestMetricsC(C.Structure):
    _fields_ = [("round", i32), ("history_tokens", i32), ("generated", i32), ("pad_", i32),
                ("arrival_s", f64), ("restore_s", f64), ("ttft_s", f64), ("tbt_s", f64)]


class ServeMetricsC(C.Structure):
    _fields_ = [("ttft_p50", f64), ("ttft_p95", f64), ("tbt_mean", f64), ("tbt_p50", f64),
                ("tbt_p95", f64), ("restore_tokens_per_s", f64), ("storage_bytes_per_token", f64),
                ("saved_bytes", u64), ("saved_tokens", u64), ("backpressure_stalls", u64),
                ("busy_s", f64), ("save_stall_s", f64), ("persist_wait_s", f64),
                ("decode_steps", i64), ("decode_tokens", i64)]


P = C.POINTER
_PROTOS = {
    "hc_last_error": (cp, []),
    "hc_version": (cp, []),
    "hc_abi_version": (i32, []),
    "hc_device_count": (i32, []),
    "hc_config_validate": (i32, [P(ModelConfigC)]),
    "hc_config_hash": (u64, [P(ModelConfigC)]),
    "hc_weights_create": (i32, [P(ModelConfigC), i32, i32, i32, P(vp)]),
    "hc_weights_destroy": (None, [vp]),
    "hc_weights_set_layer_kv": (i32, [vp, i32, vp]),
    "hc_weights_set_layer_full": (i32, [vp, i32, vp, vp, vp, vp, vp]),
    "hc_weights_set_embedding": (i32, [vp, vp]),
    "hc_project_hidden_to_kv": (i32, [vp, i32, vp, i64, i32, vp, vp, i32, vp]),
    "hc_project_to_pages": (i32, [vp, i32, vp, i64, vp, i32, P(KvPagesC), vp, i32, vp]),
    "hc_kv_scatter_to_pages": (i32, [vp, i64, i32, vp, i32, P(KvPagesC), vp, i32, vp]),
    "hc_fill_symmetric": (i32, [vp, i64, u64, u64, f32, i32, vp]),
    "hc_chunk_tokens": (i32, []),
    "hc_device_for_chunk": (i32, [i32, i32, i32]),
    "hc_timings_validate": (i32, [P(TimingsC)]),
    "hc_plan_make": (i32, [i32, i32, i32, P(PlanC)]),
    "hc_plan_make_mixed": (i32, [i32, i32, i32, P(PlanC)]),
    "hc_plan_serialize": (i32, [P(PlanC), cp, i32]),
    "hc_plan_parse": (i32, [cp, P(PlanC)]),
    "hc_plan_closed_form": (i32, [P(TimingsC), P(PlanC)]),
    "hc_makespan": (i32, [P(PlanC), P(TimingsC), P(f64)]),
    "hc_brute_force_plan": (i32, [P(TimingsC), P(PlanC)]),
    "hc_plan_three_way": (i32, [P(TimingsC), i32, P(PlanC), P(f64)]),
    "hc_plan_token_split": (i32, [P(TimingsC), i32, P(PlanC), i32, P(i32), P(f64)]),
    "hc_timeline_lane_busy": (f64, [P(TimelineC), i32]),
    "hc_timings_from_timeline": (i32, [P(TimelineC), P(TimingsC)]),
    "hc_timeline_bubble_fraction": (i32, [P(TimelineC), P(f64)]),
    "hc_simulate_pipeline": (i32, [P(PipelineJobC), i32, i32, P(TimelineC)]),
    "hc_store_create": (i32, [P(PoolDescC), C.c_size_t, P(vp)]),
    "hc_store_reserve": (i32, [vp, C.c_size_t]),
    "hc_store_destroy": (None, [vp]),
    "hc_store_create_session": (i32, [vp, P(SessionSeedC)]),
    "hc_store_reopen_for_append": (i32, [vp, cp, P(i32), i64]),
    "hc_store_snapshot": (i32, [vp, cp, i32, i32, vp, i64, i32, i32, i32, vp]),
    "hc_store_drain": (i32, [vp, i64, P(i64)]),
    "hc_store_drain_all": (i32, [vp]),
    "hc_store_finalize": (i32, [vp, cp]),
    "hc_store_open": (i32, [vp, cp, P(ManifestC)]),
    "hc_store_layer_info": (i32, [vp, cp, i32, i32, P(i32), P(i32)]),
    "hc_store_tokens": (i32, [vp, cp, P(i32), i64, P(i64)]),
    "hc_store_read_layer": (i32, [vp, cp, i32, i32, vp, i64, i32, vp]),
    "hc_store_read_layer_range": (i32, [vp, cp, i32, i32, i32, i32, vp, i64, i32, vp]),
    "hc_store_chunk_info": (i32, [vp, cp, i32, i32, i32, P(i32), P(vp), P(i64)]),
    "hc_store_device_chunk_counts": (i32, [vp, P(i64), i32]),
    "hc_store_start_daemon": (i32, [vp]),
    "hc_store_stop_daemon": (i32, [vp]),
    "hc_store_buffer_bytes": (C.c_size_t, [vp]),
    "hc_store_pinned": (i32, [vp]),
    "hc_store_buffer_capacity": (C.c_size_t, [vp]),
    "hc_store_backpressure_events": (u64, [vp]),
    "hc_store_simulated_read_seconds_tokens": (f64, [vp, i32, i32, i32]),
    "hc_restore": (i32, [vp, cp, vp, P(PlanC), P(RestoreOptsC), P(KvPagesC), vp, vp,
                         P(TimelineC)]),
    "hc_restore_batch": (i32, [vp, P(cp), i32, vp, P(RestoreOptsC), P(KvPagesC), vp, i32, vp,
                               P(TimelineC)]),
    "hc_project_multi_source": (i32, [vp, i32, i32, P(vp), P(i64), P(KvPagesC), vp, i32, vp]),
    "hc_stream_wait_flag": (i32, [vp, vp, C.c_uint32]),
    "hc_store_snapshot_range": (i32, [vp, cp, i32, i32, i64, vp, i64, i32, i32, i32, vp]),
    "hc_shard_range": (i32, [i64, i32, i32, P(i64), P(i64)]),
    "hc_shard_heads": (i32, [i32, i32, i32, P(i32), P(i32)]),
    "hc_peer_group_create": (i32, [i32, i32, i32, i32, i64, i32, P(vp)]),
    "hc_peer_group_destroy": (None, [vp]),
    "hc_peer_group_blob_size": (C.c_size_t, []),
    "hc_peer_group_export": (i32, [vp, vp, C.c_size_t]),
    "hc_peer_group_import": (i32, [vp, P(vp)]),
    "hc_peer_group_ready": (i32, [vp]),
    "hc_restore_sharded": (i32, [vp, vp, cp, vp, P(PlanC), P(RestoreOptsC), P(KvPagesC), vp, vp,
                                 P(TimelineC)]),
    "hc_stream_signal_flags": (i32, [vp, P(vp), i32, C.c_uint32]),
    "hc_serve_run": (i32, [vp, vp, P(RequestC), i32, P(ServeOptsC), P(RequestMetricsC), vp,
                           P(ServeMetricsC), vp]),
    "hc_forward_batch": (i32, [vp, vp, i32, vp, vp, P(KvPagesC), vp, i32, vp, vp, vp]),
    "hc_kv_gather_rows": (i32, [P(KvPagesC), i32, vp, i32, i64, vp, vp]),
    "hc_restore_token_wise": (i32, [vp, cp, vp, i32, P(KvPagesC), vp, vp, P(TimelineC)]),
    "hc_restore_resident": (i32, [vp, P(vp), i64, vp, i32, P(KvPagesC), vp, i32, vp]),
    "hc_prefill_layers": (i32, [vp, vp, i64, i32, i32, P(KvPagesC), vp, vp]),
    "hc_prefill": (i32, [vp, vp, i64, P(KvPagesC), vp, vp, P(i32), vp]),
    "hc_profile": (i32, [vp, i32, P(TimingsC)]),
    "hc_measure_h2d": (i32, [i32, C.c_size_t, i32, P(f64)]),
    "hc_bench_project": (i32, [vp, i32, vp, i64, i32, vp, P(f64), P(f64)]),
    "hc_attention_dense": (i32, [vp, i32, i32, i32, i32, vp, vp, i32, vp, vp]),
    "hc_gemm_epilogue": (i32, [i32, vp, vp, i32, i32, i32, vp, vp, vp, vp, vp, i32, vp]),
}

_lib = None


def lib():
    """The loaded C-ABI library (loads on first use; raises when missing)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _PROTOS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def header_symbols():
    """Function names declared in include/hcache_b200.h."""
    text = open(HEADER_PATH).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hc_[a-z0-9_]+)\s*\(", text)))


class HCacheError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{msg} (hc_status {status})")
        self.status = status


class InvalidArgument(HCacheError, ValueError):
    """std::invalid_argument in the reference."""


class NotFound(HCacheError):
    """std::runtime_error (missing manifest / chunk) in the reference."""


class Incomplete(HCacheError):
    """std::runtime_error (session not finalized) in the reference."""


class CudaError(HCacheError):
    pass


def check(status):
    if status == HC_OK:
        return
    msg = lib().hc_last_error().decode(errors="replace")
    cls = {HC_EINVAL: InvalidArgument, HC_ENOENT: NotFound, HC_EINCOMPLETE: Incomplete,
           HC_ECUDA: CudaError}.get(status, HCacheError)
    raise cls(status, msg)
