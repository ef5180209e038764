#!/usr/bin/env python
"""Benchmark of the B200 HCache restoration path (BASELINE.json metric:
restored KV tokens/s and restore latency, % of PCIe/GEMM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config llama2-7b]
    python bench.py --impl reference ...   # reference CPU implementation

N=1 workload (configs[1]): Llama-2-7B shape (32 layers, d=4096, 32 heads,
MHA), one 4096-token context restored from hidden states. Synthetic bf16
hidden states and random-init weights (splitmix64 generators, no network).

* ``value``  -- restored tokens/s of the north-star path: ``hc_restore`` of
  the session from the pinned-host chunk store, executing the bubble-free
  scheduler's plan (hc_plan_three_way on hc_profile's measured PCIe / K1 / K6
  timings). Every step copies the planned layers' hidden states
  host->device (copy engine) inside the timed region, overlapped with K1
  and the K6 recompute prefix. Device time (CUDA events), steps back to back.
* ``e2e``    -- the same public call as a user sees it: per step hc_restore,
  a device->host read of restored rows and a stream synchronisation, host
  clock.
* ``resident`` -- hidden states already in HBM: K1 (row stats + LN-fold
  tcgen05 GEMM + RoPE -> paged KV) over all layers (the kernel-bound leg).
* ``parity`` -- the restored cache of the benchmarked plan checked against
  the oracle after the timed region (oracle/parity.py).
* The KV-offload and recompute paths of the same codebase are timed
  alongside; ``cpu_baseline`` times the reference's own code on the host.
* N>1 (torchrun, or ``--gpus N`` which spawns the ranks itself): head-sharded
  restore (north star (4)): each rank fetches 1/N of every layer's token
  chunks over its own PCIe link, the all-gather is fused into K1 over peer
  memory and each rank projects only its own KV heads.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (layers, d, heads, kv_heads, d_ffn, tokens, rope)
    "tiny": (4, 512, 8, 8, 2048, 1024, True),
    "llama2-7b": (32, 4096, 32, 32, 11008, 4096, True),
    "llama2-13b": (40, 5120, 40, 40, 13824, 16384, True),
    # configs[3]: the 32 round-4 conversations of gen_trace (BATCH_TRACES), n = their max
    "opt-30b": (48, 7168, 56, 56, 28672, 3338, False),
    "llama2-70b": (80, 8192, 64, 8, 28672, 32768, True),
}
DEFAULT_CONFIG = "llama2-7b"
# configs restored as a batch of sessions: gen_trace(CONVERSATION, n_sessions,
# rounds, seed) and the contexts (history tokens) of its last-round requests
BATCH_TRACES = {"opt-30b": dict(n_sessions=32, rounds=4, seed=7)}
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        d["_source"] = "measured (MEASURED_PEAKS.json)"
        return d
    d = dict(FALLBACK_PEAKS)
    d["_source"] = "fallback (B200_PROFILING.md)"
    return d


def host_cpu():
    """CPU model and usable thread count of this host (printed with the CPU
    baseline numbers)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        threads = len(os.sched_getaffinity(0))
    except AttributeError:
        threads = os.cpu_count() or 1
    return {"model": model, "threads": threads, "logical_cpus": os.cpu_count()}


def workload_config(args, cfg, world=1):
    """The `config` object of the JSON line -- identical for the GPU arm and
    the reference arm of the same workload (plan and planner details are
    reported under "planner", not here)."""
    L, d, heads, kvh, _, n, rope = cfg
    name = args.config + (" (configs[1])" if args.config == "llama2-7b" else "")
    c = {"workload": name, "layers": L, "d_hidden": d, "heads": heads, "kv_heads": kvh,
         "tokens": n, "rope": rope, "page_size": 64,
         "l2": "inputs larger than L2 (hidden states + weights per step exceed 126 MB)"}
    if args.config in BATCH_TRACES:
        tr = BATCH_TRACES[args.config]
        c["trace"] = (f"gen_trace(CONVERSATION, n_sessions={tr['n_sessions']}, "
                      f"rounds={tr['rounds']}, seed={tr['seed']}), round-{tr['rounds']} contexts")
    c["parallelism"] = f"head-sharded x{world}" if world > 1 else "single GPU"
    return c


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled DURING the timed
    region: NVML every 5 ms (nvidia_ml_py), nvidia-smi as the fallback."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
            "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index):
        self.index, self.samples, self._stop = index, [], threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self._physical_index(index))
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self._nvml = None

    @staticmethod
    def _physical_index(index):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            try:
                return int(vis.split(",")[index])
            except (ValueError, IndexError):
                pass
        return index

    def _run(self):
        while not self._stop.is_set():
            try:
                if self._nvml is not None:
                    nv = self._nvml
                    sm = float(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                    try:
                        bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                    except AttributeError:
                        bits = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
                    self.samples.append((sm, self.max_mhz,
                                         sorted(k for k, b in self.BITS.items() if bits & b)))
                    self._stop.wait(0.005)
                    continue
                out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                      f"--query-gpu={self.Q}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    f = [x.strip() for x in out.split(",")]
                    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                             "sw_power_cap"]
                    self.samples.append((float(f[0]), float(f[1]),
                                         [names[i] for i in range(4)
                                          if len(f) > 2 + i and f[2 + i].lower() == "active"]))
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [s[0] for s in self.samples]
        reasons = sorted({r for s in self.samples for r in s[2]})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(s[1] for s in self.samples),
                "sm_min_mhz": float(min(sm)), "reasons": reasons, "samples": len(self.samples),
                "source": "nvml" if self._nvml is not None else "nvidia-smi"}


# ------------------------------------------------------------ CPU baseline
def cpu_reference_sample(cfg, target_s=10.0, max_tokens=1024, fixed_tokens=None):
    """Reference project_hidden_to_kv (oracle/_ref = the reference compiled
    from source, else the oracle port) on one layer x m tokens of the same
    workload, fanned out over all host threads. Returns (tok/s, desc), or
    (seconds, desc) with fixed_tokens=m."""
    from oracle import Oracle, Reference, bf16_round, have_reference
    L, d, heads, kvh, _, n, rope = cfg
    dh = d // heads
    o = Oracle()
    threads = host_cpu()["threads"]
    d_kv = kvh * dh
    wk = bf16_round(o.symmetric(d_kv * d, 1234, 0, 1 / np.sqrt(d))).reshape(d_kv, d)
    wv = bf16_round(o.symmetric(d_kv * d, 1234, d_kv * d, 1 / np.sqrt(d))).reshape(d_kv, d)
    kind = "reference" if have_reference() else "port"
    ref = Reference() if kind == "reference" else None

    def run(m):
        h = bf16_round(o.symmetric(m * d, 7, 0, 1.7320508)).reshape(m, d)
        if ref is not None:
            return ref.project_timed(h, wk, wv, kvh, 0, True, rope, nthreads=threads)
        t0 = time.perf_counter()
        o.project(h, wk, wv, kvh, 0, True, rope, nthreads=threads)
        return time.perf_counter() - t0

    if fixed_tokens:
        m = fixed_tokens
        dt = run(m)
    else:
        m = max(threads, 16)
        dt = run(m)
        # grow the sample until it is ~target_s of CPU work (bounded)
        while dt < target_s / 4 and m < max_tokens:
            m = min(max_tokens, m * 4)
            dt = run(m)
    desc = {"kind": kind, "cores": threads, "sample_tokens": m, "sample_layers": 1,
            "sample_s": dt, "host_cpu": host_cpu()["model"],
            "sample": f"project_hidden_to_kv of 1 layer x {m} tokens (d={d}, "
                      f"d_kv={d_kv}) on {threads} threads; tok/s = m / (sample_s x {L} layers)"}
    if fixed_tokens:
        return dt, desc
    return m / (dt * L), desc  # one context needs L layers of this projection per token


def cpu_config1_restore():
    """BASELINE.md section 3, CPU baseline 1: configs[0] (4 layers, d=512, 8
    heads, 1K tokens) through the reference's own restore() in WallClock mode
    (restore.cpp:133-220: one compute thread + one IO thread, as shipped; the
    chunk files on /dev/shm), and the same projection fanned out over every
    host thread (project_hidden_to_kv is pure). Needs the
    reference compiled from source (oracle/_ref)."""
    from oracle import Oracle, Reference, bf16_round, have_reference
    if not have_reference():
        return {"unavailable": "oracle/_ref (the reference built from source) not present"}
    ref, o = Reference(), Oracle()
    L, d, heads, dffn, vocab, n = 4, 512, 8, 2048, 1024, 1024
    root = os.path.join("/dev/shm" if os.path.isdir("/dev/shm") else "/tmp",
                        f"hc_ref_restore_{os.getpid()}")
    t, diff = ref.restore_wall(L, d, heads, dffn, vocab, n, 4, 1234, root)
    threads = host_cpu()["threads"]
    wb = 1 / np.sqrt(np.float32(d))
    dt = 0.0
    for layer in range(L):
        h = bf16_round(o.symmetric(n * d, 7, layer * n * d, 1.7320508)).reshape(n, d)
        wk = bf16_round(o.symmetric(d * d, 1234 + layer, 0, wb)).reshape(d, d)
        wv = bf16_round(o.symmetric(d * d, 1234 + layer, d * d, wb)).reshape(d, d)
        dt += ref.project_timed(h, wk, wv, heads, 0, True, True, nthreads=threads)
    return {"config": "configs[0]: 4 layers, d=512, 8 heads, 1024 tokens",
            "restore_wall_s": t, "restore_wall_tok_s": n / t if t > 0 else None,
            "restore_threads": "1 compute + 1 IO (as shipped)",
            "restore_max_abs_diff_vs_prefill": diff,
            "project_all_cores_s": dt, "project_all_cores_tok_s": n / dt, "cores": threads}


def run_reference_arm(args, cfg, rank, world):
    """--impl reference: the reference's project_hidden_to_kv (compiled from
    its own sources, oracle/_ref; the oracle port when absent) on the host
    cores. A step is one bounded sample of the workload -- one layer of m
    tokens -- so ms_per_step is the real time of a step; `value` is the
    restored-tokens/s rate that sample implies for the whole context (a
    context needs L such layers per token). Rank 0 only."""
    if rank != 0:
        return
    L, _, _, _, _, n, _ = cfg
    m = 512
    times = []
    desc = None
    for i in range(args.warmup + args.steps):
        dt, desc = cpu_reference_sample(cfg, fixed_tokens=m)
        if i >= args.warmup:
            times.append(dt)
    dt = float(np.mean(times))
    v = m / (dt * L)
    host = host_cpu()
    line = {"impl": "reference", "metric": "restored_kv_tokens_per_s", "value": v,
            "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": workload_config(args, cfg, world),
            "step": f"one sample: project_hidden_to_kv of 1 layer x {m} tokens on "
                    f"{desc['cores']} threads",
            "extrapolated": {"restore_ms_per_context": dt * 1e3 * L * n / m,
                             "note": f"sample time x {L} layers x {n}/{m} tokens (exact in FLOPs)"},
            "host_cpu": host,
            "cpu_baseline": dict(desc, value=v, unit="tokens/s"),
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    if not args.no_cpu_baseline:
        line["config1_full_restore"] = cpu_config1_restore()
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm
def verify_restore(kv, table, plan, cfg, tokens, split, kv_rows, m=32):
    """Parity of the benchmarked restore (run after the timed region, on the
    cache the last timed step wrote), against the oracle on the same
    synthetic inputs (oracle/parity.py):

    * HIDDEN layers (and the KV layers, whose stored rows are K1 outputs):
      token slices [s, s+m) at the start, middle and end of four sampled
      layers vs project_hidden_to_kv at start_pos = s -- north-star metric
      |g - r| / max(|r|, 1e-2 rms(r)) <= 1e-2;
    * KV_OFFLOAD layers: the restored pages equal the stored [K|V] rows bit
      for bit;
    * RECOMPUTE layers: rows [0, m) (causal: they depend on tokens < m only)
      vs the oracle's fp32 prefill_layers of those m tokens -- stated K6
      tolerance max |g - r| / rms(r) <= 5e-2 (bf16 operands),
      the north-star metric reported alongside."""
    import torch
    from oracle import Oracle
    from oracle import parity as P
    from paper_2410_05004_b200 import hcache as H
    L, d, heads, kvh, dffn, n, rope = cfg
    d_kv = kvh * (d // heads)
    o = Oracle()
    meth = list(plan.layer_assignment)
    hid = [layer for layer, x in enumerate(meth) if x == H.LayerMethod.HIDDEN]
    kvl = [layer for layer, x in enumerate(meth) if x == H.LayerMethod.KV_OFFLOAD]
    rel = [layer for layer, x in enumerate(meth) if x == H.LayerMethod.RECOMPUTE]
    out = {"tolerances": {"hidden_max_rel": 1e-2, "recompute_norm_err": 5e-2,
                          "kv": "bit-exact"}, "slice_tokens": m}
    t0 = time.perf_counter()
    # projected layers: up to four, spread over the plan's HIDDEN (+KV) layers
    proj = sorted(set(hid + kvl))
    pick = sorted({proj[int(round(k * (len(proj) - 1) / 3))] for k in range(4)}) if proj else []
    starts = sorted({max(split, 0) // 64 * 64 if split else 0, (n // 2) // 64 * 64, n - m})
    worst = 0.0
    for layer in pick:
        k, v = kv.gather(layer, table, n)
        for s0 in starts:
            if layer == len(rel) and split and s0 < split:
                continue  # recomputed part of the split layer
            kr, vr = P.hidden_kv(o, layer, n, d, d_kv, kvh, s0, m, rope)
            g_k = k[s0:s0 + m].float().cpu().numpy()
            g_v = v[s0:s0 + m].float().cpu().numpy()
            worst = max(worst, P.max_rel_err(g_k, kr), P.max_rel_err(g_v, vr))
    out["hidden_layers_checked"] = pick
    out["hidden_slices"] = starts
    out["hidden_max_rel"] = worst
    # KV-offload layers: bit-exact against the stored rows
    exact = True
    for layer in kvl:
        k, v = kv.gather(layer, table, n)
        exact &= bool(torch.equal(torch.cat([k, v], 1), kv_rows[layer]))
    out["kv_layers"] = kvl
    out["kv_bitexact"] = exact if kvl else None
    # RECOMPUTE prefix: rows [0, m) of every recomputed layer
    if rel:
        ref = P.recompute_kv(o, d, heads, dffn, tokens[:m], len(rel), rope)
        ne, mr = 0.0, 0.0
        for layer in rel:
            k, v = kv.gather(layer, table, m)
            g_k, g_v = k.float().cpu().numpy(), v.float().cpu().numpy()
            kr, vr = ref[layer]
            ne = max(ne, P.norm_err(g_k, kr), P.norm_err(g_v, vr))
            mr = max(mr, P.max_rel_err(g_k, kr), P.max_rel_err(g_v, vr))
        out.update(recompute_layers=rel, recompute_norm_err=ne, recompute_max_rel=mr)
    else:
        out.update(recompute_layers=[], recompute_norm_err=None, recompute_max_rel=None)
    out["ok"] = bool(worst <= 1e-2 and exact and
                     (out["recompute_norm_err"] is None or out["recompute_norm_err"] <= 5e-2))
    out["check_s"] = time.perf_counter() - t0
    return out


def verify_batch(kv, tables, plan, cfg, lens, tokens, m=16):
    """Parity of the benchmarked batch restore (configs[3]) against the
    oracle, after its timed region: HIDDEN layers of the longest, median and
    shortest sessions on token slices at both ends (each session's rows are
    its own positions 0..n-1; the synthetic hidden rows of layer l are the
    seed-(7+l) stream over the concatenated sessions), north-star metric;
    RECOMPUTE layers on the first m tokens of the longest session vs the
    oracle's fp32 prefill (stated normwise tolerance); KV layers are K1
    outputs stored and scattered (bit-exact by construction, not re-checked
    here)."""
    from oracle import Oracle
    from oracle import parity as P
    from paper_2410_05004_b200 import hcache as H
    L, d, heads, kvh, dffn, _, rope = cfg
    d_kv = kvh * (d // heads)
    o = Oracle()
    t0 = time.perf_counter()
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    order = sorted(range(len(lens)), key=lambda s_: lens[s_])
    sess = sorted({order[-1], order[len(order) // 2], order[0]})
    meth = list(plan.layer_assignment)
    hid = [x for x, y in enumerate(meth) if y == H.LayerMethod.HIDDEN]
    rel = [x for x, y in enumerate(meth) if y == H.LayerMethod.RECOMPUTE]
    pick = sorted({hid[0], hid[len(hid) // 2], hid[-1]}) if hid else []
    worst = 0.0
    for layer in pick:
        wk, wv = P.layer_wkv(o, layer, d, d_kv)
        for s_ in sess:
            n = lens[s_]
            k, v = kv.gather(layer, tables[s_], n)
            for i0 in sorted({0, max(0, n - m)}):
                mm = min(m, n - i0)
                h = P.sym(o, mm * d, P.SEED_HIDDEN + layer, int(offs[s_] + i0) * d,
                          P.HIDDEN_BOUND).reshape(mm, d)
                kr, vr = o.project(h, wk, wv, kvh, i0, True, rope)
                worst = max(worst, P.max_rel_err(k[i0:i0 + mm].float().cpu().numpy(), kr),
                            P.max_rel_err(v[i0:i0 + mm].float().cpu().numpy(), vr))
    out = {"tolerances": {"hidden_max_rel": 1e-2, "recompute_norm_err": 5e-2},
           "sessions_checked": sess, "hidden_layers_checked": pick, "slice_tokens": m,
           "hidden_max_rel": worst}
    ne = None
    if rel:
        s_ = order[-1]
        mm = min(m, lens[s_])
        ref = P.recompute_kv(o, d, heads, dffn, tokens[s_][:mm], len(rel), rope)
        ne = 0.0
        for layer in rel:
            k, v = kv.gather(layer, tables[s_], mm)
            kr, vr = ref[layer]
            ne = max(ne, P.norm_err(k.float().cpu().numpy(), kr),
                     P.norm_err(v.float().cpu().numpy(), vr))
    out.update(recompute_layers=rel, recompute_norm_err=ne,
               ok=bool(worst <= 1e-2 and (ne is None or ne <= 5e-2)),
               check_s=time.perf_counter() - t0)
    return out


def qkv_weights(fill, layer, d, d_kv, full):
    """[W_k;W_v] of a layer (seed 1234+layer) and, for the full block, W_q
    (seed 5000+layer) laid out right before it in one allocation, so the
    recompute path projects Q, K and V with one GEMM (hc_weights_set_layer_full
    fuses them when W_q immediately precedes [W_k;W_v])."""
    if not full:
        return fill((2 * d_kv, d), 1234 + layer), None
    qkv = fill((d + 2 * d_kv, d), 0)
    fill(qkv[:d], 5000 + layer)
    fill(qkv[d:], 1234 + layer)
    return qkv[d:], qkv[:d]


def run_ours(args, cfg, rank, world):
    import torch
    from paper_2410_05004_b200 import capi
    from paper_2410_05004_b200 import hcache as H
    from paper_2410_05004_b200.capi import check, lib

    L, d, heads, kvh, dffn, n, rope = cfg
    dev = local_device()
    torch.cuda.set_device(dev)
    if world > 1 or args.sharded:
        from paper_2410_05004_b200 import sharded
        args.workload_config = workload_config(args, cfg, world)
        return sharded.bench(args, cfg, rank, world, dev, ClockSampler, peaks())

    stream = torch.cuda.current_stream().cuda_stream
    vocab = 32000
    mc = H.ModelConfig(n_layers=L, d_hidden=d, n_heads=heads, n_kv_heads=kvh, d_ffn=dffn,
                       vocab_size=vocab, max_seq=max(n, 4096), rope_enabled=rope)
    w = H.Weights(mc)
    d_kv = w.d_kv
    bound = float(np.float32(1) / np.sqrt(np.float32(d)))

    def fill(shape, seed):
        # seeds: oracle/parity.py (the CPU side of the parity check); shape
        # may be an existing bf16 tensor (filled in place)
        t = shape if torch.is_tensor(shape) else torch.empty(shape, dtype=torch.bfloat16,
                                                              device="cuda")
        check(lib().hc_fill_symmetric(t.data_ptr(), t.numel(), seed, 0, bound, 1, stream))
        return t
    emb = fill((vocab, d), 99)
    w.set_embedding(emb)
    full = not args.no_recompute and kvh == heads
    for layer in range(L):
        wkv, wq = qkv_weights(fill, layer, d, d_kv, full)
        w.set_layer_kv(layer, wkv)
        if full:
            w.set_layer_full(layer, wq, wkv, fill((d, d), 6000 + layer),
                             fill((dffn, d), 7000 + layer), fill((d, dffn), 8000 + layer))
    page = 64
    n_pages = (n + page - 1) // page
    kv = H.KvCache(L, n_pages, page, d_kv)
    table = torch.arange(n_pages, dtype=torch.int32, device="cuda")
    hid = torch.empty((L, n, d), dtype=torch.bfloat16, device="cuda")
    check(lib().hc_fill_symmetric(hid.data_ptr(), hid.numel(), 7, 0, 1.7320508, 1, stream))
    hptrs = (C.c_void_p * L)(*[hid[layer].data_ptr() for layer in range(L)])
    tokens = [(i * 11 + 1) % vocab for i in range(n)]

    # bubble-free scheduler on measured PCIe / GEMM / recompute timings
    prof = H.profile_hardware(w, n)
    prof.n_layers = L
    if not full:
        # no full block weights (GQA configs here): RECOMPUTE is unavailable,
        # the planner splits between hidden states and KV offload only
        prof.c_token = H.RECOMPUTE_UNAVAILABLE
    plan, plan_ms = H.plan_three_way(prof, layer_bytes=n * d * 2)
    prof0 = prof
    all_h = H.RestorationPlan.make(L, L, H.Complement.NONE)
    all_kv = H.RestorationPlan.make(L, 0, H.Complement.KV_OFFLOAD)

    # pinned-host chunk store: the sessions (saved from the device, D2H)
    store = H.StorageManager(H.DevicePool(1), buffer_capacity_bytes=4 << 30)
    kv_rows = {}  # the [K|V] rows stored for the plan's KV-offload layers (parity)
    kv_rows_all = {}  # ... and for the all-KV session's (the strict plan's parity)

    def save(sid, p, keep=None):
        store.create_session(H.SessionSeed(sid, mc.hash(), L, d, 2, p, tokens, d_kv=d_kv))
        for layer, m in enumerate(p.layer_assignment):
            if m == H.LayerMethod.HIDDEN:
                rows = hid[layer]
                kind = H.StateKind.HIDDEN
            elif m == H.LayerMethod.KV_OFFLOAD:
                k_, v_ = kv.gather(layer, table, n)
                rows = torch.cat([k_, v_], 1).contiguous()
                kind = H.StateKind.KV
                if keep is not None:
                    keep[layer] = rows
            else:
                continue
            while not store.snapshot(sid, layer, kind, rows):
                store.drain()
        store.finalize(sid)

    def resident_step():
        check(lib().hc_restore_resident(w._h, hptrs, n, None, 1, C.byref(kv.desc),
                                        table.data_ptr(), 0, stream))

    opts = capi.RestoreOptsC(0, 0, 0)
    host_ck = torch.empty(16 * d_kv, dtype=torch.bfloat16, pin_memory=True)

    def restore_step(sid, p, o=opts):
        check(lib().hc_restore(store._h, sid, w._h, C.byref(p._c), C.byref(o),
                               C.byref(kv.desc), table.data_ptr(), stream, None))
        # device->host read of the step's result: 16 restored K rows of the last layer
        host_ck.copy_(kv.k[L - 1].view(-1)[: 16 * d_kv], non_blocking=True)

    d_tok = torch.tensor(tokens, dtype=torch.int32, device="cuda")

    def recompute_step():
        # the RECOMPUTE baseline: token ids host->device, K6 over every layer
        d_tok.copy_(torch.tensor(tokens, dtype=torch.int32), non_blocking=False)
        check(lib().hc_prefill_layers(w._h, d_tok.data_ptr(), n, 0, L, C.byref(kv.desc),
                                      table.data_ptr(), stream))
        host_ck.copy_(kv.k[L - 1].view(-1)[: 16 * d_kv], non_blocking=True)

    resident_step()
    torch.cuda.synchronize()
    # the planner's costs refined on the restore itself: hc_profile times the
    # recompute under back-to-back K6 layers (the hardest power-cap case); a
    # restore's prefix shares the part with the DMA and the K1s. Restore the
    # plan with a timeline, take each kind's per-event busy time
    # (hc_timings_from_timeline), re-plan, until the plan is stable.
    calibration = []
    split_pick = 0
    if full and not os.environ.get("HC_NO_CALIBRATE"):
        tried = {}  # plan record -> (plan, median synchronous restore ms)

        def measure(p, sid, o=None, saved=False):
            # back-to-back restores first: the timed loop's sustained power
            # state (its clock under the cap) is the one the plan must fit;
            # then the synchronous latency (the e2e leg's measure) and one
            # restore with a timeline (no overlap with a previous step's tail)
            o = o or opts
            if not saved:
                save(sid, p)
            for _ in range(max(8, args.steps)):
                restore_step(sid.encode(), p, o)
            lat = []
            for _ in range(5):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                restore_step(sid.encode(), p, o)
                torch.cuda.synchronize()
                lat.append((time.perf_counter() - t0) * 1e3)
            res = H.restore(store, sid, w, p, H.ThrottleConfig(0, True), kv, table)
            return float(np.median(lat)), res

        cand, n_sid = plan, 0
        for it in range(3):
            if cand.serialize() in tried:
                break
            lat, res = measure(cand, f"cal{n_sid}")
            n_sid += 1
            tried[cand.serialize()] = (cand, lat)
            prof = H.timings_from_timeline(res.timeline, prof)
            prof.n_layers = L
            nxt, nxt_ms = H.plan_three_way(prof, layer_bytes=n * d * 2)
            calibration.append({"plan": cand.serialize(), "restore_ms": lat,
                                "timeline_ms": res.timeline.total_s * 1e3,
                                "c_token_ms": prof.c_token * 1e3, "c_h_ms": prof.c_h * 1e3,
                                "io_h_ms": prof.io_h * 1e3, "replan": nxt.serialize(),
                                "replan_predicted_ms": nxt_ms * 1e3})
            cand = nxt
        # the model's choice and its neighbours (one recompute layer more /
        # fewer), measured: at balanced lanes the pipeline model cannot
        # separate plans a few percent apart
        for dre in (-1, 1):
            l_re = cand.l_re + dre
            l_h = cand.l_h - dre
            if l_re < 0 or l_h < 0:
                continue
            q = H.RestorationPlan.make_mixed(l_re, l_h, cand.l_kv)
            if q.serialize() in tried:
                continue
            lat, _ = measure(q, f"cal{n_sid}")
            n_sid += 1
            tried[q.serialize()] = (q, lat)
            calibration.append({"plan": q.serialize(), "restore_ms": lat, "neighbour": True})
        model_plan, model_ms = H.plan_three_way(prof, layer_bytes=n * d * 2)
        plan, best_ms = min(tried.values(), key=lambda x: x[1])
        plan_ms = model_ms if plan.serialize() == model_plan.serialize() else None
        # the token split of the chosen plan's first hidden layer, measured too
        split_try, _ = H.plan_token_split(prof, plan, n, layer_bytes=n * d * 2)
        if split_try:
            sid = [k for k, (q, _) in enumerate(tried.values()) if q.serialize() == plan.serialize()]
            lat, _ = measure(plan, f"cal{sid[0]}", capi.RestoreOptsC(0, 0, split_try), saved=True)
            calibration.append({"plan": plan.serialize(), "split_tokens": split_try,
                                "restore_ms": lat})
            if lat < best_ms * 0.995:
                split_pick = split_try
    # B200 extension: split the first hidden layer between the recompute
    # prefix and the link where that balances the two lanes
    # (opt-in, HC_SPLIT=1: interleaved A/B runs on B200 did not separate it
    # from run-to-run noise, scripts/ab_split.sh)
    split, split_ms = split_pick, plan_ms
    if full and os.environ.get("HC_SPLIT") == "1":
        split, split_ms = H.plan_token_split(prof, plan, n, layer_bytes=n * d * 2)
    opts_plan = capi.RestoreOptsC(0, 0, split)
    save(b"hcache".decode(), plan, keep=kv_rows)
    if plan.serialize() != all_h.serialize():
        save("all_hidden", all_h)
    save("kv_offload", all_kv, keep=kv_rows_all)
    sid_plan = b"hcache"
    sid_allh = b"hcache" if plan.serialize() == all_h.serialize() else b"all_hidden"

    def e2e_step():
        restore_step(sid_plan, plan, opts_plan)

    def timed(fn, steps):
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
        ev[0].record()
        for i in range(steps):
            fn()
            ev[i + 1].record()
        torch.cuda.synchronize()
        if os.environ.get("HC_STEP_TIMES"):  # per-step device times (diagnostics)
            print("step_ms", [round(ev[i].elapsed_time(ev[i + 1]), 3) for i in range(steps)],
                  file=sys.stderr)
        return ev[0].elapsed_time(ev[-1]) / steps

    def latency(fn, steps):
        # the user-visible latency of the public call: hc_restore + the D2H
        # read of its result + the stream synchronisation, host clock per step
        out = []
        for _ in range(steps):
            torch.cuda.synchronize()
            t = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            out.append((time.perf_counter() - t) * 1e3)
        return float(np.mean(out)), float(np.median(out))

    # the dominant kernel (K1) timed alone, before the timed legs heat the
    # part into its power cap: 20 launches back to back on its stream, best of
    # three (against the burst peak, which MEASURED_PEAKS takes the same way)
    torch.cuda.synchronize()
    time.sleep(2.0)
    k1_alone = []
    for _ in range(3):
        a_ms, b_ms = C.c_double(), C.c_double()
        check(lib().hc_bench_project(w._h, L - 1, hid[L - 1].data_ptr(), n, 20, stream,
                                     C.byref(a_ms), C.byref(b_ms)))
        k1_alone.append(b_ms.value)
    k1_alone_ms = min(k1_alone)

    for _ in range(args.warmup):
        resident_step()
        e2e_step()
    torch.cuda.synchronize()

    with ClockSampler(dev) as clk:
        # headline: restores from the pinned-host store, back to back, device
        # time (the resident leg runs the tensor cores at ~1.5 PFLOP/s and
        # leaves the part power-capped for a while, so it goes last)
        ms_restore = timed(e2e_step, args.steps)
        ms_e2e, ms_e2e_p50 = latency(e2e_step, args.steps)
        ms_resident = timed(resident_step, args.steps)
    clocks = clk.summary()
    # parity of the benchmarked restore: one more step of the plan, then the
    # restored cache is checked against the oracle (not timed)
    e2e_step()
    torch.cuda.synchronize()
    parity = verify_restore(kv, table, plan, cfg, tokens, split, kv_rows)
    # same-codebase baselines (not part of the headline timed region)
    for _ in range(2):
        restore_step(sid_allh, all_h)
        restore_step(b"kv_offload", all_kv)
    ms_allh = timed(lambda: restore_step(sid_allh, all_h), max(3, args.steps // 2))
    ms_kv = timed(lambda: restore_step(b"kv_offload", all_kv), max(3, args.steps // 2))
    torch.cuda.synchronize()
    # the strict plan: every layer restored within the north-star elementwise
    # bound (no RECOMPUTE layer, whose stated tolerance is normwise); the
    # faster of all-hidden and all-KV, checked like the headline plan
    strict_sid, strict_plan, strict_ms = ((sid_allh, all_h, ms_allh) if ms_allh <= ms_kv
                                          else (b"kv_offload", all_kv, ms_kv))
    restore_step(strict_sid, strict_plan)
    torch.cuda.synchronize()
    strict_par = verify_restore(kv, table, strict_plan, cfg, tokens, 0,
                                kv_rows if strict_sid == sid_plan else kv_rows_all)
    e2e_step()  # the cache holds the headline plan's restore again
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    restore_step(sid_plan, plan, opts_plan)
    enqueue_ms = (time.perf_counter() - t0) * 1e3  # host time to enqueue one restore
    torch.cuda.synchronize()
    ms_re = None
    if full:
        recompute_step()
        ms_re = timed(recompute_step, max(3, args.steps // 2))

    launches_restore = count_launches(e2e_step)
    launches_resident = count_launches(resident_step)
    # dominant kernel (K1): per-launch times with events on its stream
    stats_ms, k1_ms = C.c_double(), C.c_double()
    check(lib().hc_bench_project(w._h, L - 1, hid[L - 1].data_ptr(), n, 20, stream,
                                 C.byref(stats_ms), C.byref(k1_ms)))
    flop = 4.0 * n * d * d_kv
    pk = peaks()
    k1_tflops = flop / (k1_alone_ms * 1e-3) / 1e12
    k1_capped_tflops = flop / (k1_ms.value * 1e-3) / 1e12
    h2d = H.measure_h2d(256 << 20, 5, dev)

    # restore timeline of one e2e step (fill / bubble / lane busy)
    res = H.restore(store, sid_plan.decode(), w, plan, H.ThrottleConfig(0, True, split), kv,
                    table)
    tl = res.timeline
    if os.environ.get("HC_DUMP_TIMELINE"):
        with open(os.environ["HC_DUMP_TIMELINE"], "w") as f:
            f.write(tl.export_text())
    h_bytes = L * n * d * 2
    h_bytes_plan = (plan.l_h * n - split) * d * 2 + plan.l_kv * n * 2 * d_kv * 2 + \
        (4 * n if plan.l_re or split else 0)
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "k1_traffic.json")
    if os.path.exists(tpath):  # ncu --set full capture of this kernel (scripts/profile_r2.sh)
        t = json.load(open(tpath))
        if t.get("config") == args.config:
            traffic = t.get("dram_bytes_per_launch")
            traffic_src = f"{t.get('source')}; {t.get('build')}"

    cpu_tok_s, cpu_desc = cpu_reference_sample(cfg) if not args.no_cpu_baseline else (None, {})
    if cpu_tok_s is not None:
        cpu_desc["config1_full_restore"] = cpu_config1_restore()
    value = n / (ms_restore * 1e-3)
    roof_gemm_s = L * flop / (pk["bf16_tflops"] * 1e12)
    roof_pcie_s = h_bytes / h2d
    roof_s = max(roof_pcie_s, roof_gemm_s)
    line = {
        "metric": "restored_kv_tokens_per_s", "value": value, "unit": "tokens/s",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_restore,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (splitmix64 bf16 hidden states + random-init weights)",
        "config": workload_config(args, cfg),
        "measures": "value: hc_restore of the planned session from the pinned-host chunk store "
                    "(H2D copies inside), steps back to back, CUDA events; e2e: the same call "
                    "as a user sees it -- per step hc_restore + D2H read of the result + stream "
                    "sync, host clock; resident: hidden states already in HBM (K1 only)",
        "restore_latency_ms": {"restore": ms_restore, "e2e": ms_e2e, "e2e_p50": ms_e2e_p50,
                               "resident": ms_resident, "all_hidden": ms_allh,
                               "kv_offload": ms_kv, "recompute": ms_re,
                               "host_enqueue": enqueue_ms},
        "resident": {"value": n / (ms_resident * 1e-3), "unit": "tokens/s",
                     "ms_per_step": ms_resident},
        "speedup": {"hcache_vs_kv_offload": ms_kv / ms_restore,
                    "hcache_vs_recompute": (ms_re / ms_restore) if ms_re else None,
                    "hcache_vs_all_hidden": ms_allh / ms_restore},
        "planner": {"profiled": {"io_h_ms": prof0.io_h * 1e3, "io_kv_ms": prof0.io_kv * 1e3,
                                 "c_h_ms": prof0.c_h * 1e3, "c_token_ms": prof0.c_token * 1e3},
                    "calibrated": {"io_h_ms": prof.io_h * 1e3, "io_kv_ms": prof.io_kv * 1e3,
                                   "c_h_ms": prof.c_h * 1e3, "c_token_ms": prof.c_token * 1e3},
                    "calibration": calibration,
                    "plan": plan.serialize(), "split_tokens": split,
                    "how": "hc_plan_three_way (+ hc_plan_token_split) on hc_profile, refined on "
                           "timelines of the restore itself (hc_timings_from_timeline) until "
                           "the plan is stable; the model's plan, its +-1 recompute-layer "
                           "neighbours and its token split are then measured (synchronous "
                           "restore latency after back-to-back restores) and the fastest kept",
                    "predicted_ms": plan_ms * 1e3 if plan_ms else None,
                    "predicted_with_split_ms": split_ms * 1e3 if split_ms else None},
        "parity": parity,
        "strict_plan": {
            "plan": strict_plan.serialize(), "restore_ms": strict_ms,
            "value": n / (strict_ms * 1e-3), "unit": "tokens/s",
            "hidden_max_rel": strict_par["hidden_max_rel"],
            "kv_bitexact": strict_par["kv_bitexact"], "ok": strict_par["ok"],
            "note": "every layer within the north-star max relative error 1e-2 (no "
                    "recomputed layer); the headline plan trades that for its recompute "
                    "prefix's stated normwise tolerance"},
        "e2e": {"value": n / (ms_e2e * 1e-3), "unit": "tokens/s", "h2d_bytes_per_step": h_bytes_plan,
                "d2h_bytes_per_step": int(host_ck.numel() * 2)},
        "path_roofline": {
            "bound": "pcie", "unit": "GB/s", "peak": h2d / 1e9,
            "peak_source": "measured pinned H2D 256 MiB",
            "achieved": h_bytes_plan / (ms_restore * 1e-3) / 1e9,
            "frac": h_bytes_plan / (ms_restore * 1e-3) / h2d,
            "all_hidden_roofline_ms": 1e3 * roof_s,
            "frac_vs_all_hidden_roofline": roof_s / (ms_restore * 1e-3),
            "note": "north-star roofline = max(hidden bytes / PCIe, FLOPs / tensor peak); the "
                    "plan recomputes some layers, so it can beat the all-hidden bound"},
        "roofline": {"bound": "tensor", "kernel": "k1_restore_kv", "achieved": k1_tflops,
                     "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
                     "frac": k1_tflops / pk["bf16_tflops"],
                     "peak_kind": "burst (K1 timed alone: 20 launches back to back on its "
                                  "stream, CUDA events, best of 3, after a 2 s rest -- the "
                                  "way MEASURED_PEAKS takes the burst peak)",
                     "peak_source": pk["_source"], "traffic": traffic,
                     "traffic_source": traffic_src,
                     "flop_per_launch": flop, "k1_ms": k1_alone_ms,
                     "power_capped": {"k1_ms": k1_ms.value, "achieved": k1_capped_tflops,
                                      "frac_of_sustained": k1_capped_tflops / pk.get(
                                          "bf16_tflops_sustained", pk["bf16_tflops"]),
                                      "how": "the same 20 launches after the timed legs, at "
                                             "the sw_power_cap clock, against the sustained "
                                             "peak"},
                     "row_stats_ms": stats_ms.value},
        "timeline": {"total_ms": tl.total_s * 1e3, "fill_ms": tl.fill_s * 1e3,
                     "io_busy_ms": tl.lane_busy(H.Lane.IO) * 1e3,
                     "compute_busy_ms": tl.lane_busy(H.Lane.COMPUTE) * 1e3,
                     "bubble_fraction": tl.bubble_fraction(),
                     "lane_busy": "union of each lane's event intervals"},
        # our kernels launched in the timed region: per headline step the
        # planned restore's launches (counted from a CUPTI trace of one step),
        # 2 x steps restores (back to back + synchronous) and steps resident
        # steps
        "gpu_launches": args.steps * (2 * launches_restore + launches_resident),
        "gpu_launches_per_step": {"restore": launches_restore, "resident": launches_resident,
                                  "how": "CUPTI kernel records (torch.profiler) of one call, "
                                         "kernels in namespace hc::"},
        "clocks": clocks,
    }
    if cpu_tok_s is not None:
        line["cpu_baseline"] = dict(cpu_desc, value=cpu_tok_s, unit="tokens/s")
    print(json.dumps(line), flush=True)


def count_launches(fn):
    """Kernel launches of ours (namespace hc::) one call of fn makes, from a
    CUPTI activity trace (torch.profiler) -- the per-step count behind the
    bench line's gpu_launches."""
    import warnings

    import torch
    from torch.profiler import ProfilerActivity, profile
    warnings.filterwarnings("ignore", message=".*Profiler clears events.*")
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    return sum(1 for e in prof.events()
               if e.device_type.name == "CUDA" and "hc::" in e.name and "Memcpy" not in e.name)


def restore_launches(plan):
    """Kernel launches of one hc_restore of `plan` (the K6 prefix: one
    embedding, per layer 2 x (statistics + mean-shift check), 5 GEMMs and the
    attention; per hidden layer statistics + mean-shift check + K1; per KV
    layer one scatter)."""
    return (10 * plan.l_re + 1 if plan.l_re else 0) + 3 * plan.l_h + plan.l_kv


def run_ours_batch(args, cfg, rank, world):
    """configs[3]: a batch of sessions (OPT-30B shape, no RoPE) restored
    concurrently -- hc_restore_batch executing the three-way plan (RECOMPUTE
    prefix as one ragged forward, grouped K1 per HIDDEN layer) from the
    pinned store; resident K1 over the concatenated rows; KV offload and
    recompute of the same batch in the same codebase."""
    import torch
    from paper_2410_05004_b200 import hcache as H
    from paper_2410_05004_b200.capi import check, lib

    if world > 1 and rank != 0:
        return
    L, d, heads, kvh, dffn, _, rope = cfg
    tr = BATCH_TRACES[args.config]
    trace = H.gen_trace(H.TraceKind.CONVERSATION,
                        H.TraceParams(n_sessions=tr["n_sessions"], rounds=tr["rounds"]),
                        tr["seed"])
    lens = [q.history_tokens for q in trace.requests if q.round == tr["rounds"]]
    S, total = len(lens), sum(lens)
    dev = local_device()
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream().cuda_stream
    vocab, page = 32000, 64
    mc = H.ModelConfig(n_layers=L, d_hidden=d, n_heads=heads, n_kv_heads=kvh, d_ffn=dffn,
                       vocab_size=vocab, max_seq=4096, rope_enabled=rope)
    w = H.Weights(mc)
    d_kv = w.d_kv
    bound = float(np.float32(1) / np.sqrt(np.float32(d)))

    def fill(shape, seed, b=bound):
        t = shape if torch.is_tensor(shape) else torch.empty(shape, dtype=torch.bfloat16,
                                                              device="cuda")
        check(lib().hc_fill_symmetric(t.data_ptr(), t.numel(), seed, 0, b, 1, stream))
        return t
    w.set_embedding(fill((vocab, d), 99))
    full = not args.no_recompute
    for layer in range(L):
        wkv, wq = qkv_weights(fill, layer, d, d_kv, full)
        w.set_layer_kv(layer, wkv)
        if full:
            w.set_layer_full(layer, wq, wkv, fill((d, d), 6000 + layer),
                             fill((dffn, d), 7000 + layer), fill((d, dffn), 8000 + layer))
    # pages: each session its own run of pages (no padding to the longest)
    npg = [(n + page - 1) // page for n in lens]
    stride = max(npg)
    first = np.concatenate([[0], np.cumsum(npg)])
    tab = np.zeros((S, stride), dtype=np.int32)
    for s_ in range(S):
        tab[s_, :npg[s_]] = np.arange(first[s_], first[s_ + 1])
    tables = torch.from_numpy(tab).cuda()
    kv = H.KvCache(L, int(first[-1]), page, d_kv)
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    cu = torch.from_numpy(offs.astype(np.int32)).cuda()
    tokens = [[(i * 11 + 1 + 7 * s_) % vocab for i in range(n)] for s_, n in enumerate(lens)]

    def hidden(layer):  # the layer's synthetic hidden states of every session, [total, d]
        return fill((total, d), 7 + layer, 1.7320508)

    def timed(fn, steps):
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
        ev[0].record()
        for i in range(steps):
            fn()
            ev[i + 1].record()
        torch.cuda.synchronize()
        if os.environ.get("HC_STEP_TIMES"):  # per-step device times (diagnostics)
            print("step_ms", [round(ev[i].elapsed_time(ev[i + 1]), 3) for i in range(steps)],
                  file=sys.stderr)
        return ev[0].elapsed_time(ev[-1]) / steps

    host_ck = torch.empty(16 * d_kv, dtype=torch.bfloat16, pin_memory=True)

    def read_back():  # device->host read of the step's result (16 K rows, last layer)
        host_ck.copy_(kv.k[L - 1].view(-1)[: 16 * d_kv], non_blocking=True)

    # resident leg (also c_h for the planner): K1 over the concatenated rows,
    # eight distinct resident layer buffers cycled (no L2 reuse: 0.6 GB each)
    res_bufs = [hidden(layer) for layer in range(min(L, 8))]
    hptrs = (C.c_void_p * L)(*[res_bufs[layer % len(res_bufs)].data_ptr() for layer in range(L)])

    def resident_step():
        check(lib().hc_restore_resident(w._h, hptrs, total, cu.data_ptr(), S, C.byref(kv.desc),
                                        tables.data_ptr(), stride, stream))
    for _ in range(args.warmup):
        resident_step()
    ms_resident = timed(resident_step, args.steps)
    del res_bufs
    # recompute leg (also c_token): ragged forward of every session from position 0
    flat = torch.tensor([t for ts in tokens for t in ts], dtype=torch.int32)
    d_flat = torch.empty_like(flat, device="cuda")

    def recompute_step():
        d_flat.copy_(flat, non_blocking=False)
        H.forward_batch(w, d_flat, lens, [0] * S, kv, tables)
        read_back()
    ms_re = None
    if full:
        recompute_step()
        ms_re = timed(recompute_step, max(3, args.steps // 3))
    h2d = H.measure_h2d(256 << 20, 5, dev)
    prof = H.ProfiledTimings(io_h=total * d * 2 / h2d, io_kv=total * 2 * d_kv * 2 / h2d,
                             c_h=ms_resident * 1e-3 / L,
                             c_token=(ms_re * 1e-3 / L) if ms_re else H.RECOMPUTE_UNAVAILABLE, n_layers=L)
    plan, plan_ms = H.plan_three_way(prof, L)
    all_h = H.RestorationPlan.make(L, L, H.Complement.NONE)
    all_kv = H.RestorationPlan.make(L, 0, H.Complement.KV_OFFLOAD)

    def save(p):
        store = H.StorageManager(H.DevicePool(1), buffer_capacity_bytes=4 << 30)
        for s_, n in enumerate(lens):
            store.create_session(H.SessionSeed(f"s{s_}", mc.hash(), L, d, 2, p, tokens[s_],
                                               d_kv=d_kv))
        for layer, m in enumerate(p.layer_assignment):
            if m == H.LayerMethod.RECOMPUTE:
                continue
            rows = hidden(layer)
            if m == H.LayerMethod.KV_OFFLOAD:
                rows = torch.cat([rows[:, :d_kv], rows[:, :d_kv]], 1).contiguous()  # KV-row bytes
            kind = H.StateKind.HIDDEN if m == H.LayerMethod.HIDDEN else H.StateKind.KV
            for s_ in range(S):
                while not store.snapshot(f"s{s_}", layer, kind, rows[offs[s_]:offs[s_ + 1]]):
                    store.drain()
            store.drain_all()
        for s_ in range(S):
            store.finalize(f"s{s_}")
        return store
    sids = [f"s{s_}" for s_ in range(S)]

    def restore_step(store):
        H.restore_batch(store, sids, w, H.ThrottleConfig(0, False), kv, tables)
        read_back()

    parity = {}
    launches = {}

    def leg(p, steps, check=False):
        store = save(p)
        for _ in range(2):
            restore_step(store)
        with ClockSampler(dev) as clk:
            ms = timed(lambda: restore_step(store), steps)
        if check:  # the restored cache of the benchmarked plan vs the oracle
            launches["restore"] = count_launches(lambda: restore_step(store))
            torch.cuda.synchronize()
            parity.update(verify_batch(kv, tables, p, cfg, lens, tokens))
        # the public call as a user sees it: per step the batch restore, the
        # D2H read of its result and a stream sync, host clock (mean)
        walls = []
        for _ in range(steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            restore_step(store)
            torch.cuda.synchronize()
            walls.append((time.perf_counter() - t0) * 1e3)
        tl = H.restore_batch(store, sids, w, H.ThrottleConfig(0, True), kv, tables).timeline
        store.close()
        return ms, float(np.mean(walls)), clk.summary(), tl
    # the model's plan and its +-1 recompute-layer neighbours, each measured
    # on its own store (the restore's prefix runs at a different clock than
    # the back-to-back recompute leg that priced c_token); the fastest is
    # the benchmarked plan
    def counts(p):
        a = list(p.layer_assignment)
        return (sum(x == H.LayerMethod.RECOMPUTE for x in a),
                sum(x == H.LayerMethod.KV_OFFLOAD for x in a))
    model_plan = plan
    calibration = []
    if full:
        l_re0, l_kv0 = counts(plan)
        measured = {}

        def measure_re(l_re):  # restore time of the plan with l_re recompute layers
            if l_re not in measured:
                cand = plan if l_re == l_re0 else \
                    H.RestorationPlan.make_mixed(l_re, L - l_re - l_kv0, l_kv0)
                st = save(cand)
                restore_step(st)
                ms_c = timed(lambda: restore_step(st), 2)
                st.close()
                calibration.append({"plan": cand.serialize(), "restore_ms": ms_c})
                measured[l_re] = (ms_c, cand)
            return measured[l_re][0]
        ok = lambda r: 0 <= r and L - r - l_kv0 >= 1  # noqa: E731
        for r in (l_re0 - 1, l_re0, l_re0 + 1):
            if ok(r):
                measure_re(r)
        # walk on while the best is at an edge of what was measured (<= 3 more)
        for _ in range(3):
            r_best = min(measured, key=lambda r: measured[r][0])
            step = -1 if r_best == min(measured) else (1 if r_best == max(measured) else 0)
            if step == 0 or not ok(r_best + step):
                break
            measure_re(r_best + step)
        plan = min(measured.values(), key=lambda x: x[0])[1]
    ms_e2e, wall_e2e, clocks, tl = leg(plan, args.steps, check=True)
    ms_allh = ms_e2e if plan.serialize() == all_h.serialize() else \
        leg(all_h, max(3, args.steps // 2))[0]
    ms_kv = leg(all_kv, max(3, args.steps // 2))[0]

    stats_ms, k1_ms = C.c_double(), C.c_double()
    hb = hidden(L - 1)
    check(lib().hc_bench_project(w._h, L - 1, hb.data_ptr(), total, 5, stream,
                                 C.byref(stats_ms), C.byref(k1_ms)))
    del hb
    flop = 4.0 * total * d * d_kv
    pk = peaks()
    k1_tflops = flop / (k1_ms.value * 1e-3) / 1e12
    h_bytes = L * total * d * 2
    h_bytes_plan = plan.l_h * total * d * 2 + plan.l_kv * total * 2 * d_kv * 2 + \
        (4 * total if plan.l_re else 0)
    roof_gemm_s = L * flop / (pk["bf16_tflops"] * 1e12)
    roof_pcie_s = h_bytes / h2d
    cpu_tok_s, cpu_desc = cpu_reference_sample(cfg) if not args.no_cpu_baseline else (None, {})
    line = {
        "metric": "restored_kv_tokens_per_s", "value": total / (ms_e2e * 1e-3),
        "unit": "tokens/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_e2e, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (splitmix64 bf16 hidden states + random-init weights; "
                "session lengths from gen_trace)",
        "config": dict(workload_config(args, cfg), sessions=S, tokens=total,
                       max_session_tokens=max(lens)),
        "measures": "value: hc_restore_batch of the 32 planned sessions from the pinned-host "
                    "store (H2D inside), steps back to back, device time; e2e: the same public "
                    "call per step with a D2H read of its result and a stream sync, host clock; "
                    "resident: hidden states already in HBM (K1 only)",
        "parity": parity,
        "restore_latency_ms": {"restore": ms_e2e, "e2e": wall_e2e, "resident": ms_resident,
                               "all_hidden": ms_allh, "kv_offload": ms_kv, "recompute": ms_re},
        "resident": {"value": total / (ms_resident * 1e-3), "unit": "tokens/s",
                     "ms_per_step": ms_resident},
        "speedup": {"hcache_vs_kv_offload": ms_kv / ms_e2e,
                    "hcache_vs_recompute": (ms_re / ms_e2e) if ms_re else None,
                    "hcache_vs_all_hidden": ms_allh / ms_e2e},
        "planner": {"profiled": {"io_h_ms": prof.io_h * 1e3, "io_kv_ms": prof.io_kv * 1e3,
                                 "c_h_ms": prof.c_h * 1e3, "c_token_ms": prof.c_token * 1e3},
                    "plan": plan.serialize(), "model_plan": model_plan.serialize(),
                    "calibration": calibration,
                    "how": "hc_plan_three_way on measured PCIe, batched K1 and batched "
                           "recompute per layer (model_plan); it and its +-1 recompute-layer "
                           "neighbours are then measured (calibration) and the fastest kept",
                    "predicted_ms": plan_ms * 1e3 if plan_ms else None},
        "e2e": {"value": total / (wall_e2e * 1e-3), "unit": "tokens/s",
                "h2d_bytes_per_step": h_bytes_plan, "d2h_bytes_per_step": int(host_ck.numel() * 2)},
        "path_roofline": {"bound": "pcie", "unit": "GB/s",
                          "achieved": h_bytes_plan / (ms_e2e * 1e-3) / 1e9,
                          "peak": h2d / 1e9, "peak_source": "measured pinned H2D 256 MiB",
                          "frac": h_bytes_plan / (ms_e2e * 1e-3) / h2d,
                          "all_hidden_roofline_ms": 1e3 * max(roof_pcie_s, roof_gemm_s),
                          "frac_vs_all_hidden_roofline":
                              max(roof_pcie_s, roof_gemm_s) / (ms_e2e * 1e-3)},
        "roofline": {"bound": "tensor", "kernel": "k1_restore_kv (ragged batch)",
                     "achieved": k1_tflops, "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
                     "frac": k1_tflops / pk["bf16_tflops"], "peak_source": pk["_source"],
                     "traffic": None, "flop_per_launch": flop, "k1_ms": k1_ms.value,
                     "row_stats_ms": stats_ms.value},
        "timeline": {"total_ms": tl.total_s * 1e3, "fill_ms": tl.fill_s * 1e3,
                     "io_busy_ms": tl.lane_busy(H.Lane.IO) * 1e3,
                     "compute_busy_ms": tl.lane_busy(H.Lane.COMPUTE) * 1e3,
                     "bubble_fraction": tl.bubble_fraction(),
                     "lane_busy": "union of each lane's event intervals"},
        # the batch restores of the timed region (back to back + synchronous)
        "gpu_launches": 2 * args.steps * launches.get("restore", restore_launches(plan)),
        "clocks": clocks,
    }
    if cpu_tok_s is not None:
        line["cpu_baseline"] = dict(cpu_desc, value=cpu_tok_s, unit="tokens/s")
    print(json.dumps(line), flush=True)


def local_device():
    """This rank's GPU: LOCAL_RANK (ranks beyond the visible devices share
    them -- e.g. `--gpus 2` on a one-GPU box runs both ranks on it, the peer
    mappings still going through CUDA IPC)."""
    import torch
    if "HC_FORCE_DEVICE" in os.environ:
        return int(os.environ["HC_FORCE_DEVICE"])
    return int(os.environ.get("LOCAL_RANK", 0)) % max(1, torch.cuda.device_count())


def spawn_ranks(n):
    """`bench.py --gpus N` without a launcher: run N ranks with
    torch.distributed.run on this node (127.0.0.1) and relay rank 0's line."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=dict(os.environ, HC_SPAWNED="1"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="run the head-sharded (N>1) path even at world size 1 (testing)")
    ap.add_argument("--no-recompute", action="store_true",
                    help="skip full-block weights (no RECOMPUTE complement / baseline)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    cfg = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        return run_reference_arm(args, cfg, rank, max(world, args.gpus))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    if world != args.gpus and "WORLD_SIZE" in os.environ and args.gpus != 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.config in BATCH_TRACES and not args.sharded and world == 1:
        return run_ours_batch(args, cfg, rank, world)
    return run_ours(args, cfg, rank, world)


if __name__ == "__main__":
    main()
