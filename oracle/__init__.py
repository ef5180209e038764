"""Parity oracle for the HCache restoration path -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package, and only as the checker
(or the timed CPU baseline). The product path never routes through it.

Two libraries:

* ``Oracle`` -- our C restatement (``hc_oracle.c``) of the reference routines,
  each citing the reference file:line it follows. Travels to the GPU box as a
  prebuilt ``_build/libhc_oracle.so``.
* ``Reference`` -- the unmodified reference (``/root/reference/proj/src``)
  compiled by ``oracle/Makefile`` into ``_ref/libhcache_ref.so`` with our
  ``ref_shim.cpp`` glue. Present wherever the build container produced it.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libhc_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libhcache_ref.so")

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


def _nthreads(n=None):
    return int(n or os.cpu_count() or 1)


class _Timings(C.Structure):
    _fields_ = [("io_h", C.c_double), ("io_kv", C.c_double), ("c_h", C.c_double),
                ("c_token", C.c_double), ("n_layers", C.c_int)]


class _Plan(C.Structure):
    _fields_ = [("l_h", C.c_int), ("l_o", C.c_int), ("complement", C.c_int)]


class _Job(C.Structure):
    _fields_ = [("layer", C.c_int), ("io_s", C.c_double), ("compute_s", C.c_double),
                ("has_io", C.c_int), ("has_compute", C.c_int)]


class _Event(C.Structure):
    _fields_ = [("lane", C.c_int), ("layer", C.c_int), ("job", C.c_int),
                ("start_s", C.c_double), ("end_s", C.c_double)]


class _Config(C.Structure):
    _fields_ = [("n_layers", C.c_int), ("d_hidden", C.c_int), ("n_heads", C.c_int),
                ("d_ffn", C.c_int), ("vocab_size", C.c_int), ("max_seq", C.c_int),
                ("norm_enabled", C.c_int), ("rope_enabled", C.c_int)]


def bf16_round(x: np.ndarray) -> np.ndarray:
    """float32 -> nearest bf16 (RNE) -> float32, vectorised."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    out = r.astype(np.uint32).view(np.float32)
    nan = np.isnan(x)
    if nan.any():
        out = out.copy()
        out[nan] = np.nan
    return out.reshape(x.shape)


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """float32 -> bf16 bit patterns (uint16), RNE."""
    return (bf16_round(x).view(np.uint32) >> 16).astype(np.uint16)


def bf16_from_bits(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


class Oracle:
    """ctypes binding of hc_oracle.c (the C restatement)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library missing: {path} (run make -C oracle)")
        L = self.lib = C.CDLL(path)
        L.hco_splitmix64_at.restype = C.c_uint64
        L.hco_splitmix64_at.argtypes = [C.c_uint64, C.c_uint64]
        L.hco_symmetric_at.restype = C.c_float
        L.hco_symmetric_at.argtypes = [C.c_uint64, C.c_uint64, C.c_float]
        L.hco_fill_symmetric.argtypes = [_f32p, C.c_size_t, C.c_uint64, C.c_uint64, C.c_float]
        L.hco_fill_symmetric_bf16.argtypes = [_f32p, C.c_size_t, C.c_uint64, C.c_uint64,
                                              C.c_float, C.c_int]
        L.hco_init_model.restype = C.c_size_t
        L.hco_init_model.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_void_p]
        L.hco_float_to_half.restype = C.c_uint16
        L.hco_float_to_half.argtypes = [C.c_float]
        L.hco_half_to_float.restype = C.c_float
        L.hco_half_to_float.argtypes = [C.c_uint16]
        L.hco_float_to_bf16.restype = C.c_uint16
        L.hco_float_to_bf16.argtypes = [C.c_float]
        L.hco_bf16_to_float.restype = C.c_float
        L.hco_bf16_to_float.argtypes = [C.c_uint16]
        L.hco_layer_norm.argtypes = [_f32p, C.c_int64, C.c_int, _f32p]
        L.hco_matmul_wt.argtypes = [_f32p, C.c_int64, C.c_int, _f32p, C.c_int, _f32p, C.c_int]
        L.hco_apply_rope.argtypes = [_f32p, C.c_int64, C.c_int, C.c_int, C.c_int]
        L.hco_rope_table.argtypes = [C.c_int, C.c_int, _f32p, _f32p]
        L.hco_project_hidden_to_kv.argtypes = [_f32p, C.c_int64, C.c_int, _f32p, _f32p, C.c_int,
                                               C.c_int, C.c_int, C.c_int, C.c_int, _f32p, _f32p,
                                               C.c_int]
        L.hco_prefill.restype = C.c_int
        L.hco_prefill.argtypes = [C.POINTER(_Config), _f32p, _i32p, C.c_int64, C.c_void_p,
                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
        L.hco_prefill_layers.argtypes = [C.POINTER(_Config), _f32p, _i32p, C.c_int64, C.c_int,
                                         C.c_int, _f32p, _f32p, C.c_int]
        L.hco_block_forward.argtypes = [C.POINTER(_Config), _f32p, _f32p, _f32p, _f32p, _f32p,
                                        _f32p, _f32p, C.c_int64, _f32p, _f32p, C.c_int]
        L.hco_device_for_chunk.restype = C.c_int
        L.hco_device_for_chunk.argtypes = [C.c_int, C.c_int, C.c_int]
        L.hco_num_chunks.restype = C.c_int
        L.hco_num_chunks.argtypes = [C.c_int]
        L.hco_plan_closed_form.argtypes = [C.POINTER(_Timings), C.POINTER(_Plan)]
        L.hco_brute_force_plan.argtypes = [C.POINTER(_Timings), C.POINTER(_Plan)]
        L.hco_makespan.restype = C.c_double
        L.hco_makespan.argtypes = [C.POINTER(_Plan), C.POINTER(_Timings)]
        L.hco_simulate_pipeline.restype = C.c_int
        L.hco_simulate_pipeline.argtypes = [C.POINTER(_Job), C.c_int, C.c_int, C.POINTER(_Event),
                                            C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.hco_conversation_history.restype = C.c_int
        L.hco_conversation_history.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double,
                                               C.c_double, C.c_int, C.c_uint64, _i32p]
        L.hco_fnv1a.restype = C.c_uint64
        L.hco_fnv1a.argtypes = [C.c_void_p, C.c_size_t]

    # generators
    def symmetric(self, n, seed, offset=0, bound=1.0):
        out = np.empty(int(n), np.float32)
        self.lib.hco_fill_symmetric(out, out.size, seed, offset, bound)
        return out

    def symmetric_bf16(self, n, seed, offset=0, bound=1.0, nthreads=None):
        """bf16_round(symmetric(...)), generated on all host threads."""
        out = np.empty(int(n), np.float32)
        self.lib.hco_fill_symmetric_bf16(out, out.size, seed, offset, bound, _nthreads(nthreads))
        return out

    def init_model(self, n_layers, d, d_ffn, vocab, seed):
        n = self.lib.hco_init_model(n_layers, d, d_ffn, vocab, seed, None)
        out = np.empty(n, np.float32)
        self.lib.hco_init_model(n_layers, d, d_ffn, vocab, seed, out.ctypes.data)
        return out

    @staticmethod
    def split_weights(flat, n_layers, d, d_ffn, vocab):
        """Views into an init_model flat buffer (model.cpp:175-194 order)."""
        dd, df = d * d, d * d_ffn
        emb = flat[: vocab * d].reshape(vocab, d)
        layers = []
        base = vocab * d
        for _ in range(n_layers):
            lw = {}
            for name, size, shape in (("wq", dd, (d, d)), ("wk", dd, (d, d)), ("wv", dd, (d, d)),
                                      ("wo", dd, (d, d)), ("fc1", df, (d_ffn, d)),
                                      ("fc2", df, (d, d_ffn))):
                lw[name] = flat[base: base + size].reshape(shape)
                base += size
            layers.append(lw)
        return emb, layers

    # math
    def layer_norm(self, x):
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty_like(x)
        self.lib.hco_layer_norm(x, x.shape[0], x.shape[1], out)
        return out

    def matmul_wt(self, x, w, nthreads=None):
        x = np.ascontiguousarray(x, np.float32)
        w = np.ascontiguousarray(w, np.float32)
        y = np.empty((x.shape[0], w.shape[0]), np.float32)
        self.lib.hco_matmul_wt(x, x.shape[0], x.shape[1], w, w.shape[0], y, _nthreads(nthreads))
        return y

    def apply_rope(self, x, n_heads, start_pos=0):
        x = np.array(x, np.float32, order="C", copy=True)
        self.lib.hco_apply_rope(x, x.shape[0], x.shape[1], n_heads, start_pos)
        return x

    def rope_table(self, n_pos, d_head):
        c = np.empty((n_pos, d_head // 2), np.float32)
        s = np.empty_like(c)
        self.lib.hco_rope_table(n_pos, d_head, c, s)
        return c, s

    def project(self, h, wk, wv, n_kv_heads, start_pos=0, norm=True, rope=True, nthreads=None):
        """project_hidden_to_kv (model.cpp:219-235) -> (K, V) float32."""
        h = np.ascontiguousarray(h, np.float32)
        wk = np.ascontiguousarray(wk, np.float32)
        wv = np.ascontiguousarray(wv, np.float32)
        n, d = h.shape
        d_kv = wk.shape[0]
        k = np.empty((n, d_kv), np.float32)
        v = np.empty((n, d_kv), np.float32)
        self.lib.hco_project_hidden_to_kv(h, n, d, wk, wv, d_kv, n_kv_heads, start_pos,
                                          int(norm), int(rope), k, v, _nthreads(nthreads))
        return k, v

    def prefill(self, cfg: dict, weights, tokens, nthreads=None, want=("inputs", "k", "v")):
        c = _Config(cfg["n_layers"], cfg["d_hidden"], cfg["n_heads"], cfg["d_ffn"],
                    cfg["vocab_size"], cfg.get("max_seq", 4096), int(cfg.get("norm", 1)),
                    int(cfg.get("rope", 1)))
        tokens = np.ascontiguousarray(tokens, np.int32)
        n, d, L = tokens.size, c.d_hidden, c.n_layers
        outs = {}
        for key in ("inputs", "k", "v"):
            outs[key] = np.empty((L, n, d), np.float32) if key in want else None
        final = np.empty((n, d), np.float32)
        ptr = lambda a: None if a is None else a.ctypes.data  # noqa: E731
        nxt = self.lib.hco_prefill(C.byref(c), np.ascontiguousarray(weights, np.float32), tokens,
                                   n, ptr(outs["inputs"]), ptr(outs["k"]), ptr(outs["v"]),
                                   final.ctypes.data, _nthreads(nthreads))
        outs["final"] = final
        outs["next_token"] = nxt
        return outs

    def prefill_layers(self, cfg: dict, weights, tokens, lb, le, nthreads=None):
        c = _Config(cfg["n_layers"], cfg["d_hidden"], cfg["n_heads"], cfg["d_ffn"],
                    cfg["vocab_size"], cfg.get("max_seq", 4096), int(cfg.get("norm", 1)),
                    int(cfg.get("rope", 1)))
        tokens = np.ascontiguousarray(tokens, np.int32)
        n, d, L = tokens.size, c.d_hidden, c.n_layers
        k = np.zeros((L, n, d), np.float32)
        v = np.zeros((L, n, d), np.float32)
        self.lib.hco_prefill_layers(C.byref(c), np.ascontiguousarray(weights, np.float32), tokens,
                                    n, lb, le, k, v, _nthreads(nthreads))
        return k, v

    def block_forward(self, cfg: dict, lw: dict, x, nthreads=None):
        """block_forward (model.cpp:102-115) of one layer with explicit
        weights lw = {wq, wk, wv, wo, fc1, fc2}; x (n x d float32) is updated
        in place; returns the layer's (K, V)."""
        c = _Config(1, cfg["d_hidden"], cfg["n_heads"], cfg["d_ffn"], cfg.get("vocab_size", 1),
                    cfg.get("max_seq", 4096), int(cfg.get("norm", 1)), int(cfg.get("rope", 1)))
        assert x.dtype == np.float32 and x.flags["C_CONTIGUOUS"]
        n = x.shape[0]
        k = np.empty_like(x)
        v = np.empty_like(x)
        w = {key: np.ascontiguousarray(lw[key], np.float32)
             for key in ("wq", "wk", "wv", "wo", "fc1", "fc2")}
        self.lib.hco_block_forward(C.byref(c), w["wq"], w["wk"], w["wv"], w["wo"], w["fc1"],
                                   w["fc2"], x, n, k, v, _nthreads(nthreads))
        return k, v

    # indexing / planner / pipeline
    def device_for_chunk(self, layer, chunk, ndev):
        return self.lib.hco_device_for_chunk(layer, chunk, ndev)

    def num_chunks(self, n):
        return self.lib.hco_num_chunks(n)

    def plan(self, io_h, io_kv, c_h, c_token, n_layers, brute=False):
        t = _Timings(io_h, io_kv, c_h, c_token, n_layers)
        p = _Plan()
        fn = self.lib.hco_brute_force_plan if brute else self.lib.hco_plan_closed_form
        if fn(C.byref(t), C.byref(p)) != 0:
            raise ValueError("ProfiledTimings: nonpositive timing")
        return (p.l_h, p.l_o, p.complement), self.lib.hco_makespan(C.byref(p), C.byref(t))

    def makespan(self, l_h, l_o, comp, io_h, io_kv, c_h, c_token):
        t = _Timings(io_h, io_kv, c_h, c_token, l_h + l_o)
        p = _Plan(l_h, l_o, comp)
        return self.lib.hco_makespan(C.byref(p), C.byref(t))

    def simulate_pipeline(self, jobs, depth):
        """jobs: list of (layer, io_s, compute_s, has_io, has_compute)."""
        arr = (_Job * max(1, len(jobs)))(*[_Job(*j) for j in jobs])
        ev = (_Event * max(1, 2 * len(jobs)))()
        total, fill = C.c_double(), C.c_double()
        k = self.lib.hco_simulate_pipeline(arr, len(jobs), depth, ev, C.byref(total), C.byref(fill))
        if k < 0:
            raise ValueError("simulate_pipeline failed")
        events = [(ev[i].lane, ev[i].layer, ev[i].start_s, ev[i].end_s) for i in range(k)]
        return events, total.value, fill.value

    def conversation_history(self, n_sessions, rounds, seed, mean_input=66.8, mean_output=358.8,
                             arrival_rate=0.1, vocab=1024):
        out = np.empty(n_sessions * rounds, np.int32)
        self.lib.hco_conversation_history(n_sessions, rounds, mean_input, mean_output,
                                          arrival_rate, vocab, seed, out)
        return out

    def fnv1a(self, arr):
        arr = np.ascontiguousarray(arr)
        return int(self.lib.hco_fnv1a(arr.ctypes.data, arr.nbytes))


class Reference:
    """ctypes binding of the reference compiled from source (oracle/_ref)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"reference library missing: {path}")
        L = self.lib = C.CDLL(path)
        L.ref_init_model.argtypes = [C.c_int] * 5 + [C.c_ulonglong, _f32p]
        L.ref_prefill.restype = C.c_int
        L.ref_prefill.argtypes = [C.c_int] * 8 + [C.c_ulonglong, _i32p, C.c_int] + [C.c_void_p] * 4
        L.ref_prefill_layers.argtypes = [C.c_int] * 8 + [C.c_ulonglong, _i32p, C.c_int, C.c_int,
                                                         C.c_int, _f32p, _f32p]
        L.ref_project.argtypes = [_f32p, C.c_int, C.c_int, _f32p, _f32p, C.c_int, C.c_int, C.c_int,
                                  C.c_int, C.c_int, _f32p, _f32p]
        L.ref_project_timed.restype = C.c_double
        L.ref_project_timed.argtypes = [_f32p, C.c_int, C.c_int, _f32p, _f32p, C.c_int, C.c_int,
                                        C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int]
        L.ref_apply_rope.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_int]
        L.ref_float_to_half.restype = C.c_ushort
        L.ref_float_to_half.argtypes = [C.c_float]
        L.ref_half_to_float.restype = C.c_float
        L.ref_half_to_float.argtypes = [C.c_ushort]
        L.ref_device_for_chunk.argtypes = [C.c_int, C.c_int, C.c_int]
        L.ref_plan.argtypes = [C.c_double] * 4 + [C.c_int, C.c_int] + [C.POINTER(C.c_int)] * 3 + [
            C.POINTER(C.c_double)]
        L.ref_plan_serialize.argtypes = [C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_int]
        L.ref_simulate_pipeline.restype = C.c_int
        L.ref_simulate_pipeline.argtypes = [C.c_int, _i32p, _f64p, _f64p, _i32p, _i32p, C.c_int,
                                            _i32p, _i32p, _f64p, _f64p, C.POINTER(C.c_double),
                                            C.POINTER(C.c_double)]
        L.ref_conversation_history.argtypes = [C.c_int, C.c_int, C.c_ulonglong, _i32p]
        L.ref_gen_trace.restype = C.c_int
        L.ref_gen_trace.argtypes = [C.c_int, C.c_int, C.c_int, C.c_ulonglong, C.c_int, _i32p,
                                    C.c_void_p, C.c_void_p]
        L.ref_restore_wall.restype = C.c_double
        L.ref_restore_wall.argtypes = [C.c_int] * 7 + [C.c_ulonglong, C.c_char_p,
                                                       C.POINTER(C.c_double)]

    def init_model(self, n_layers, d, n_heads, d_ffn, vocab, seed):
        n = vocab * d + n_layers * (4 * d * d + 2 * d * d_ffn)
        out = np.empty(n, np.float32)
        if self.lib.ref_init_model(n_layers, d, n_heads, d_ffn, vocab, seed, out) != 0:
            raise RuntimeError("ref_init_model failed")
        return out

    def prefill(self, cfg: dict, seed, tokens):
        tokens = np.ascontiguousarray(tokens, np.int32)
        n, d, L = tokens.size, cfg["d_hidden"], cfg["n_layers"]
        inp = np.empty((L, n, d), np.float32)
        k = np.empty_like(inp)
        v = np.empty_like(inp)
        final = np.empty((n, d), np.float32)
        nxt = self.lib.ref_prefill(L, d, cfg["n_heads"], cfg["d_ffn"], cfg["vocab_size"],
                                   cfg.get("max_seq", 4096), int(cfg.get("norm", 1)),
                                   int(cfg.get("rope", 1)), seed, tokens, n, inp.ctypes.data,
                                   k.ctypes.data, v.ctypes.data, final.ctypes.data)
        return {"inputs": inp, "k": k, "v": v, "final": final, "next_token": nxt}

    def prefill_layers(self, cfg: dict, seed, tokens, lb, le):
        tokens = np.ascontiguousarray(tokens, np.int32)
        n, d, L = tokens.size, cfg["d_hidden"], cfg["n_layers"]
        k = np.zeros((L, n, d), np.float32)
        v = np.zeros_like(k)
        rc = self.lib.ref_prefill_layers(L, d, cfg["n_heads"], cfg["d_ffn"], cfg["vocab_size"],
                                         cfg.get("max_seq", 4096), int(cfg.get("norm", 1)),
                                         int(cfg.get("rope", 1)), seed, tokens, n, lb, le, k, v)
        if rc != 0:
            raise RuntimeError("ref_prefill_layers failed")
        return k, v

    def project(self, h, wk, wv, n_kv_heads, start_pos=0, norm=True, rope=True):
        h = np.ascontiguousarray(h, np.float32)
        wk = np.ascontiguousarray(wk, np.float32)
        wv = np.ascontiguousarray(wv, np.float32)
        n, d = h.shape
        k = np.empty((n, wk.shape[0]), np.float32)
        v = np.empty_like(k)
        if self.lib.ref_project(h, n, d, wk, wv, wk.shape[0], n_kv_heads, start_pos, int(norm),
                                int(rope), k, v) != 0:
            raise RuntimeError("ref_project failed")
        return k, v

    def project_timed(self, h, wk, wv, n_kv_heads, start_pos=0, norm=True, rope=True,
                      nthreads=None, keep=False):
        h = np.ascontiguousarray(h, np.float32)
        wk = np.ascontiguousarray(wk, np.float32)
        wv = np.ascontiguousarray(wv, np.float32)
        n, d = h.shape
        k = np.empty((n, wk.shape[0]), np.float32) if keep else None
        v = np.empty_like(k) if keep else None
        dt = self.lib.ref_project_timed(h, n, d, wk, wv, wk.shape[0], n_kv_heads, start_pos,
                                        int(norm), int(rope), None if k is None else k.ctypes.data,
                                        None if v is None else v.ctypes.data, _nthreads(nthreads))
        return (dt, k, v) if keep else dt

    def apply_rope(self, x, n_heads, start_pos=0):
        x = np.array(x, np.float32, order="C", copy=True)
        self.lib.ref_apply_rope(x, x.shape[0], x.shape[1], n_heads, start_pos)
        return x

    def plan(self, io_h, io_kv, c_h, c_token, n_layers, brute=False):
        lh, lo, comp, ms = C.c_int(), C.c_int(), C.c_int(), C.c_double()
        if self.lib.ref_plan(io_h, io_kv, c_h, c_token, n_layers, int(brute), C.byref(lh),
                             C.byref(lo), C.byref(comp), C.byref(ms)) != 0:
            raise ValueError("ProfiledTimings: nonpositive timing")
        return (lh.value, lo.value, comp.value), ms.value

    def plan_serialize(self, n_layers, l_h, comp):
        buf = C.create_string_buffer(128)
        self.lib.ref_plan_serialize(n_layers, l_h, comp, buf, 128)
        return buf.value.decode()

    def simulate_pipeline(self, jobs, depth):
        n = len(jobs)
        layer = np.array([j[0] for j in jobs], np.int32)
        io = np.array([j[1] for j in jobs], np.float64)
        cs = np.array([j[2] for j in jobs], np.float64)
        hio = np.array([j[3] for j in jobs], np.int32)
        hc = np.array([j[4] for j in jobs], np.int32)
        el = np.zeros(2 * n + 1, np.int32)
        ey = np.zeros(2 * n + 1, np.int32)
        es = np.zeros(2 * n + 1, np.float64)
        ee = np.zeros(2 * n + 1, np.float64)
        total, fill = C.c_double(), C.c_double()
        k = self.lib.ref_simulate_pipeline(n, layer, io, cs, hio, hc, depth, el, ey, es, ee,
                                           C.byref(total), C.byref(fill))
        if k < 0:
            raise ValueError("simulate_pipeline failed")
        return [(int(el[i]), int(ey[i]), float(es[i]), float(ee[i])) for i in range(k)], \
            total.value, fill.value

    def conversation_history(self, n_sessions, rounds, seed):
        out = np.empty(n_sessions * rounds, np.int32)
        self.lib.ref_conversation_history(n_sessions, rounds, seed, out)
        return out

    def gen_trace(self, kind, n_sessions, rounds, seed, max_out=4096):
        """(meta [k x 6], arrival [k], token-hash [k]) in arrival order."""
        meta = np.empty((max_out, 6), np.int32)
        arr = np.empty(max_out, np.float64)
        hsh = np.empty(max_out, np.uint64)
        k = self.lib.ref_gen_trace(kind, n_sessions, rounds, seed, max_out, meta, arr.ctypes.data,
                                   hsh.ctypes.data)
        if k < 0:
            raise RuntimeError("ref_gen_trace failed")
        return meta[:k], arr[:k], hsh[:k]

    def restore_wall(self, n_layers, d, n_heads, d_ffn, vocab, n, elem_bytes, seed, root):
        diff = C.c_double()
        t = self.lib.ref_restore_wall(n_layers, d, n_heads, d_ffn, vocab, n, elem_bytes, seed,
                                      root.encode(), C.byref(diff))
        return t, diff.value


def have_reference() -> bool:
    return os.path.exists(REF_SO)
