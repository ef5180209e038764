"""Head-sharded multi-GPU restoration (north star (4)) -- host side.

Every GPU needs the full [n x d] hidden state of a layer (each KV head
contracts over all of d), while the projection output shards by KV head. The
data path is the C ABI's ``hc_restore_sharded`` (csrc/sharded.cpp): rank r of
N fetches its 128-row aligned token range of each HIDDEN layer over its own
PCIe link into an HBM slot every other rank has mapped (CUDA IPC over
NVLink), publishes the range's LayerNorm statistics, and every rank's K1
reads all ranges' A tiles straight from the owners' slots (the all-gather
fused into the GEMM) for its own KV heads. KV_OFFLOAD layers fetch only the
rank's heads' [K|V] rows. Chunk indexing is the reference's (chunk c = tokens
[64c, 64c+64), device (L + c) % ndev, storage.cpp:29-31).

This module holds what sits around that call:

* ``save_shard``  -- one rank's save path: its token range of each HIDDEN
  layer (hc_store_snapshot_range) and its heads' KV rows of each KV layer;
* ``plan_sharded`` -- the bubble-free planner at N GPUs: per-rank costs
  (PCIe measured with every rank copying at once, K1 on the rank's heads,
  the recompute of a layer -- replicated: every rank runs the RECOMPUTE
  prefix for all heads, since a layer's attention needs every head, and
  keeps its own heads' K/V), the three-way planner, one plan agreed by all
  ranks;
* ``restore_layers`` -- the orchestration in plain host terms (fetch own
  range, all-gather, project own heads), which the gloo CPU test runs with
  the oracle as the projection;
* ``bench`` -- ``bench.py --gpus N``: one process per GPU, timing = max over
  ranks.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import time
from dataclasses import dataclass
from typing import Callable, List, Tuple

from .capi import HC_CHUNK_TOKENS


def shard_ranges(n_tokens: int, world: int) -> Tuple[List[Tuple[int, int]], int]:
    """Chunk-aligned contiguous token ranges per rank and the padded shard
    size (tokens) every rank contributes to an all-gather (host reference of
    the partition; the device path uses the 128-row aligned hc_shard_range)."""
    if n_tokens < 1 or world < 1:
        raise ValueError("shard_ranges: n_tokens and world must be >= 1")
    chunks = (n_tokens + HC_CHUNK_TOKENS - 1) // HC_CHUNK_TOKENS
    per = (chunks + world - 1) // world
    out = []
    for r in range(world):
        c0, c1 = min(chunks, r * per), min(chunks, (r + 1) * per)
        out.append((min(n_tokens, c0 * HC_CHUNK_TOKENS), min(n_tokens, c1 * HC_CHUNK_TOKENS)))
    return out, per * HC_CHUNK_TOKENS


def head_range(n_kv_heads: int, world: int, rank: int) -> Tuple[int, int]:
    """KV heads [begin, begin+count) projected by `rank`."""
    if n_kv_heads % world:
        raise ValueError(f"head sharding needs n_kv_heads ({n_kv_heads}) % world ({world}) == 0")
    c = n_kv_heads // world
    return rank * c, c


@dataclass
class ShardPlan:
    n_tokens: int
    world: int
    rank: int
    ranges: List[Tuple[int, int]]
    shard_tokens: int

    @staticmethod
    def make(n_tokens, world, rank):
        ranges, shard = shard_ranges(n_tokens, world)
        return ShardPlan(n_tokens, world, rank, ranges, shard)

    @property
    def mine(self):
        return self.ranges[self.rank]


def restore_layers(layers: List[int], plan: ShardPlan,
                   fetch: Callable[[int, int, int, object], None],
                   allgather: Callable[[object, object], None],
                   project: Callable[[int, object], None],
                   alloc_full: Callable[[], object], shard_view: Callable[[object, int], object],
                   depth: int = 2):
    """Host-side orchestration of one rank (the CPU reference of what
    hc_restore_sharded does on the device).

    fetch(layer, tok_begin, tok_end, dst_shard) fills this rank's shard;
    allgather(shard, full) assembles [world * shard_tokens x d] in `full`;
    project(layer, full) projects this rank's heads. Buffers cycle through a
    ring of `depth` full-size buffers."""
    ring = [alloc_full() for _ in range(max(1, depth))]
    b, e = plan.mine
    for i, layer in enumerate(layers):
        full = ring[i % len(ring)]
        mine = shard_view(full, plan.rank)
        if e > b:
            fetch(layer, b, e, mine)
        allgather(mine, full)
        project(layer, full)


def save_shard(store, sid: str, seed, plan, rank: int, world: int,
               hidden_rows: Callable[[int, int, int], object],
               kv_rows: Callable[[int], object]):
    """One rank's save path (storage.cpp:129-149 per rank): the session
    (every token id, so positions and chunk indices are the context's) with
    this rank's token range [b, e) of each HIDDEN layer -- hidden_rows(layer,
    b, e) -> rows -- and its own heads' [K|V] rows of each KV layer --
    kv_rows(layer) -> n x 2*d_kv_local rows."""
    from . import hcache as H
    n = len(seed.tokens)
    b, e = H.shard_range(n, world, rank)
    store.create_session(seed)
    for layer, m in enumerate(plan.layer_assignment):
        if m == H.LayerMethod.HIDDEN:
            if e > b:
                rows = hidden_rows(layer, b, e)
                while not store.snapshot(sid, layer, H.StateKind.HIDDEN, rows, tok_begin=b):
                    store.drain()
        elif m == H.LayerMethod.KV_OFFLOAD:
            rows = kv_rows(layer)
            while not store.snapshot(sid, layer, H.StateKind.KV, rows):
                store.drain()
        # RECOMPUTE layers store nothing: every rank recomputes them from the
        # session's token ids
    store.finalize(sid)


def plan_sharded(io_h_rank: List[float], io_kv_rank: List[float], c_h_rank: List[float],
                 n_layers: int, depth: int = 2, c_token_rank: List[float] = None):
    """The three-way planner at N GPUs: every rank's lanes must finish, so a
    layer costs the slowest rank's fetch (io_h: its token range, io_kv: its
    heads' KV rows, both measured with all ranks copying at once), K1 (its
    heads over all n rows) and recompute (the whole layer, replicated on every
    rank; None = unavailable, e.g. without the full block weights).
    Deterministic in its inputs, so ranks that share them agree."""
    from . import hcache as H
    c_tok = max(c_token_rank) if c_token_rank else H.RECOMPUTE_UNAVAILABLE
    t = H.ProfiledTimings(io_h=max(io_h_rank), io_kv=max(io_kv_rank), c_h=max(c_h_rank),
                          c_token=c_tok, n_layers=n_layers)
    return H.plan_three_way(t, prefetch_depth=max(1, depth - 1)) + (t,)


def bench(args, cfg, rank, world, dev, clock_sampler=None, peaks=None):
    """bench.py --gpus N: head-sharded restore of one context over N ranks
    (strong scaling), every rank calling hc_restore_sharded. Prints the JSON
    line on rank 0."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from . import hcache as H
    from .capi import check, lib

    if not dist.is_initialized():
        for k, v in (("RANK", "0"), ("WORLD_SIZE", "1"), ("LOCAL_RANK", "0"),
                     ("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29517")):
            os.environ.setdefault(k, v)
        # the control plane only (handle exchange, barriers, max over ranks):
        # the data path is peer memory, no collective library call
        dist.init_process_group("gloo")
    L, d, heads, kvh, dffn, n, rope = cfg
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream().cuda_stream
    hb, hc = H.shard_heads(kvh, world, rank)
    dh = d // heads
    d_kv_all = kvh * dh
    vocab = 32000
    mc = H.ModelConfig(n_layers=L, d_hidden=d, n_heads=heads, n_kv_heads=kvh, d_ffn=dffn,
                       vocab_size=vocab, max_seq=max(n, 4096), rope_enabled=rope)
    w = H.Weights(mc, hb, hc, dev)
    bound = float(np.float32(1) / np.sqrt(np.float32(d)))
    a, c = hb * dh, (hb + hc) * dh
    # the RECOMPUTE complement needs the whole block on every rank (the prefix
    # is replicated); MHA models as at N=1 (bench.py), not GQA-70B's 140 GB
    full = not getattr(args, "no_recompute", False) and kvh == heads
    keep = []

    def fill(t, seed):
        check(lib().hc_fill_symmetric(t.data_ptr(), t.numel(), seed, 0, bound, 1, stream))
        return t

    def new(shape):
        return torch.empty(shape, dtype=torch.bfloat16, device="cuda")
    if full:
        keep.append(fill(new((vocab, d)), 99))
        w.set_embedding(keep[-1])
    for layer in range(L):
        # [W_q ; W_k ; W_v] (bench.py seeds; the fused Q/K/V GEMM of the prefix)
        qkv = new((d + 2 * d_kv_all, d)) if full else new((2 * d_kv_all, d))
        q_rows = d if full else 0
        full_w = fill(qkv[q_rows:], 1234 + layer)
        mine = torch.cat([full_w[a:c], full_w[d_kv_all + a: d_kv_all + c]]).contiguous()
        w.set_layer_kv(layer, mine)
        keep.append(mine)
        if full:
            fill(qkv[:d], 5000 + layer)
            blk = [fill(new((d, d)), 6000 + layer), fill(new((dffn, d)), 7000 + layer),
                   fill(new((d, dffn)), 8000 + layer)]
            w.set_layer_full(layer, qkv[:d], full_w, *blk)
            keep += [qkv] + blk
        del full_w, qkv
    page = 64
    n_pages = (n + page - 1) // page
    kv = H.KvCache(L, n_pages, page, w.d_kv)
    table = torch.arange(n_pages, dtype=torch.int32, device="cuda")
    ranges = [H.shard_range(n, world, r) for r in range(world)]
    b, e = ranges[rank]
    rows_max = max(1, max(y - x for x, y in ranges))
    # staging slots: enough for the IO lane to run ahead through a RECOMPUTE
    # prefix (every HIDDEN layer when it fits in ~4 GiB), at least 2
    slot_bytes = rows_max * d * 2
    depth = int(max(2, min(L, (4 << 30) // max(1, slot_bytes)))) if full else 2
    group = H.PeerGroup(world, rank, d, rows_max, depth=depth, device=dev,
                        exchange=H.PeerGroup.torch_exchange())
    tokens = [(i * 11 + 1) % 32000 for i in range(n)]

    def layer_hidden(layer):  # the synthetic layer input of every token (bench.py seeds)
        h = torch.empty((n, d), dtype=torch.bfloat16, device="cuda")
        check(lib().hc_fill_symmetric(h.data_ptr(), h.numel(), 7, layer * n * d, 1.7320508, 1,
                                      stream))
        return h

    def max_over_ranks(x):
        t = torch.tensor([float(x)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- per-rank costs for the planner
    # PCIe with every rank copying at once (ranks share host memory / PCIe
    # switches: the aggregate, not N x one GPU's), per-rank bytes of a layer
    def concurrent_h2d(nbytes, reps=5):
        dist.barrier()
        torch.cuda.synchronize()
        bw = H.measure_h2d(nbytes, reps, dev)
        t = nbytes / bw
        slowest = max_over_ranks(t)
        return bw, world * nbytes / slowest  # this rank's, aggregate
    probe = max(64 << 20, rows_max * d * 2)
    bw_rank, bw_agg = concurrent_h2d(probe)
    bw_min = -max_over_ranks(-bw_rank)
    io_h = rows_max * d * 2 / bw_min
    io_kv = n * 2 * w.d_kv * 2 / bw_min
    hb_probe = layer_hidden(0)
    stats_ms, k1_ms = C.c_double(), C.c_double()
    check(lib().hc_bench_project(w._h, 0, hb_probe.data_ptr(), n, 10, stream, C.byref(stats_ms),
                                 C.byref(k1_ms)))
    del hb_probe
    c_h = max_over_ranks(k1_ms.value * 1e-3)
    c_tok = None
    if full:  # one rank's recompute of a whole layer (all heads), max over ranks
        dist.barrier()
        c_tok = max_over_ranks(H.profile_hardware(w, n).c_token)
    plan, plan_s, prof = plan_sharded([io_h], [io_kv], [c_h], L, depth,
                                      [c_tok] if c_tok else None)
    # every rank computed the same plan from the same maxima; check it
    plans = [None] * world
    dist.all_gather_object(plans, plan.serialize())
    if len(set(plans)) != 1:
        raise RuntimeError(f"ranks disagree on the plan: {plans}")
    all_h = H.RestorationPlan.make(L, L, H.Complement.NONE)
    all_kv = H.RestorationPlan.make(L, 0, H.Complement.KV_OFFLOAD)

    # ---- this rank's share of the sessions (pinned host store)
    store = H.StorageManager(H.DevicePool(1), buffer_capacity_bytes=2 << 30)
    kv_saved = {}

    def kv_rows(layer):
        k_, v_ = H.project_hidden_to_kv(w, layer, layer_hidden(layer), 0)
        return torch.cat([k_, v_], 1).contiguous()

    def save(sid, p, keep_kv=False):
        def kvr(layer):
            r = kv_rows(layer)
            if keep_kv:
                kv_saved[layer] = r
            return r
        save_shard(store, sid, H.SessionSeed(sid, mc.hash(), L, d, 2, p, tokens, d_kv=w.d_kv),
                   p, rank, world, lambda layer, x, y: layer_hidden(layer)[x:y].contiguous(), kvr)
    save("hcache", plan, keep_kv=True)
    sids = {"hcache": plan}
    if plan.serialize() != all_h.serialize():
        save("all_hidden", all_h)
        sids["all_hidden"] = all_h
    if plan.serialize() != all_kv.serialize():
        save("kv_offload", all_kv)
        sids["kv_offload"] = all_kv
    all_re = H.RestorationPlan.make(L, 0, H.Complement.RECOMPUTE)
    if full:  # the recompute baseline: every layer recomputed on every rank
        save("recompute", all_re)
        sids["recompute"] = all_re
    torch.cuda.synchronize()
    throttle = H.ThrottleConfig(0, False)
    host_ck = torch.empty(16 * w.d_kv, dtype=torch.bfloat16, pin_memory=True)

    throttle_copy = H.ThrottleConfig(0, False, 0, 1)  # copy-engine gather, then K1

    def step(sid, thr=None):
        H.restore_sharded(group, store, sid, w, sids[sid], thr or throttle, kv, table, stream)
        host_ck.copy_(kv.k[L - 1].view(-1)[: 16 * w.d_kv], non_blocking=True)

    def timed(sid, steps, thr=None):
        dist.barrier()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(steps):
            step(sid, thr)
        ev1.record()
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1) / steps
        dist.barrier()
        return max_over_ranks(ms)

    def latency(sid, steps):
        out = []
        for _ in range(steps):
            dist.barrier()
            torch.cuda.synchronize()
            t = time.perf_counter()
            step(sid)
            torch.cuda.synchronize()
            out.append(max_over_ranks((time.perf_counter() - t) * 1e3))
        return float(np.mean(out))

    for _ in range(args.warmup):
        for sid in sids:
            step(sid)
    torch.cuda.synchronize()
    # calibration (as the single-GPU bench does): the model's plan against
    # the all-hidden plan, both measured; the faster is the headline
    calib = {"hcache": timed("hcache", 3)}
    if "all_hidden" in sids:
        calib["all_hidden"] = timed("all_hidden", 3)
    head = min(calib, key=calib.get)
    plan_head = sids[head]
    clk = clock_sampler(dev) if clock_sampler else None
    if clk:
        clk.__enter__()
    ms = timed(head, args.steps)
    ms_e2e = latency(head, args.steps)
    if clk:
        clk.__exit__(None, None, None)
    clocks = clk.summary() if clk else {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
    legs = {}
    for sid in ("all_hidden", "kv_offload"):
        legs[sid] = timed(sid, max(3, args.steps // 2)) if sid in sids else ms
    legs["recompute"] = None
    if "recompute" in sids:
        step("recompute")
        legs["recompute"] = timed("recompute", 3)
    # the all-gather-then-GEMM baseline of the fused peer-memory K1: the same
    # plan with every owner's range gathered by the copy engines first
    legs["copy_gather"] = None
    if plan_head.l_h:
        step(head, throttle_copy)
        legs["copy_gather"] = timed(head, max(3, args.steps // 2), throttle_copy)
    from bench import count_launches
    n_launch = count_launches(lambda: step(head))
    n_launch = int(max_over_ranks(n_launch))
    # parity of this rank's heads after one more restore of the plan
    step(head)
    torch.cuda.synchronize()
    par = _verify_shard(kv, table, plan_head, cfg, hb, hc, kv_saved, w.d_kv, tokens)
    pars = [None] * world
    dist.all_gather_object(pars, par)
    tl = H.restore_sharded(group, store, head, w, plan_head, H.ThrottleConfig(0, True), kv, table,
                           stream, timeline=True)
    tl_total = max_over_ranks(tl.total_s * 1e3)
    if rank == 0:
        pk = peaks or {"bf16_tflops": 1617.3, "_source": "fallback"}
        flop = 4.0 * n * d * w.d_kv
        k1_tflops = flop / (c_h) / 1e12
        h_bytes = L * n * d * 2  # the context's hidden states, all ranks together
        plan_bytes = (plan_head.l_h * n * d * 2 + plan_head.l_kv * n * 2 * d_kv_all * 2)
        roof_pcie_s = h_bytes / bw_agg
        roof_gemm_s = L * 4.0 * n * d * d_kv_all / (world * pk["bf16_tflops"] * 1e12)
        roof_s = max(roof_pcie_s, roof_gemm_s)
        parity = {"ranks": pars,
                  "hidden_max_rel": max(p_["hidden_max_rel"] for p_ in pars),
                  "kv_bitexact": (all(p_["kv_bitexact"] for p_ in pars)
                                  if pars[0]["kv_bitexact"] is not None else None),
                  "recompute_norm_err": max((p_["recompute_norm_err"] or 0.0) for p_ in pars),
                  "ok": all(p_["ok"] for p_ in pars),
                  "tolerances": {"hidden_max_rel": 1e-2, "kv": "bit-exact",
                                 "recompute_norm_err": 5e-2}}
        line = {
            "metric": "restored_kv_tokens_per_s", "value": n / (ms * 1e-3), "unit": "tokens/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (splitmix64 bf16 hidden states + random-init weights)",
            "config": args.workload_config,
            "measures": "value: hc_restore_sharded on every rank from its pinned-host share of "
                        "the session (its token range of each hidden layer, its heads' KV rows; "
                        "H2D inside), steps back to back, CUDA events, max over ranks; e2e: per "
                        "step the call + a D2H read + sync, host clock, max over ranks",
            "restore_latency_ms": {"restore": ms, "e2e": ms_e2e, "all_hidden": legs["all_hidden"],
                                   "kv_offload": legs["kv_offload"],
                                   "recompute": legs["recompute"],
                                   "copy_gather": legs["copy_gather"],
                                   "timeline_total": tl_total},
            "speedup": {"hcache_vs_kv_offload": legs["kv_offload"] / ms,
                        "hcache_vs_all_hidden": legs["all_hidden"] / ms,
                        "hcache_vs_recompute": (legs["recompute"] / ms
                                                if legs["recompute"] else None),
                        "recompute_note": "the recompute path at N ranks is replicated (every "
                                          "rank runs every layer for all heads)",
                        "fused_vs_copy_gather": (legs["copy_gather"] / ms
                                                 if legs["copy_gather"] else None)},
            "planner": {"plan": plan_head.serialize(), "model_plan": plan.serialize(),
                        "calibration_ms": calib,
                        "per_rank_ms": {"io_h": io_h * 1e3, "io_kv": io_kv * 1e3,
                                        "c_h": c_h * 1e3,
                                        "c_token": c_tok * 1e3 if c_tok else None},
                        "predicted_ms": plan_s * 1e3, "staging_slots": depth,
                        "how": "hc_plan_three_way on the slowest rank's measured costs (PCIe "
                               "with all ranks copying at once; c_token = a whole layer's "
                               "recompute, the RECOMPUTE prefix being replicated on every "
                               "rank); the model plan and the all-hidden plan are then both "
                               "measured and the faster is the headline (calibration_ms)" +
                               ("" if c_tok else "; RECOMPUTE unavailable (no full "
                                "block weights: GQA or --no-recompute)")},
            "pcie": {"per_rank_gbs": bw_rank / 1e9, "slowest_rank_gbs": bw_min / 1e9,
                     "aggregate_gbs": bw_agg / 1e9, "probe_bytes": probe,
                     "how": f"hc_measure_h2d on every rank at once after a barrier; aggregate = "
                            f"{world} x bytes / slowest rank's time"},
            "parity": parity,
            "e2e": {"value": n / (ms_e2e * 1e-3), "unit": "tokens/s",
                    "h2d_bytes_per_step": int(plan_bytes),
                    "d2h_bytes_per_step": int(world * host_ck.numel() * 2)},
            "path_roofline": {"bound": "pcie" if roof_pcie_s >= roof_gemm_s else "tensor",
                              "all_hidden_roofline_ms": roof_s * 1e3,
                              "frac_vs_all_hidden_roofline": roof_s / (ms * 1e-3),
                              "achieved_pcie_gbs": plan_bytes / (ms * 1e-3) / 1e9,
                              "frac_of_aggregate_pcie": plan_bytes / (ms * 1e-3) / bw_agg,
                              "note": "north-star roofline max(hidden bytes / aggregate PCIe, "
                                      "FLOPs / (N x tensor peak))"},
            "roofline": {"bound": "tensor", "kernel": "k1_restore_kv (this rank's heads)",
                         "achieved": k1_tflops, "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
                         "frac": k1_tflops / pk["bf16_tflops"], "peak_source": pk["_source"],
                         "traffic": None, "flop_per_launch": flop, "k1_ms": c_h * 1e3},
            # our kernels in the timed region: every rank's restores (back to
            # back + synchronous), counted from a CUPTI trace of one step
            "gpu_launches": 2 * args.steps * world * n_launch,
            "gpu_launches_per_step_and_rank": n_launch,
            "clocks": clocks,
        }
        if not args.no_cpu_baseline:
            from bench import cpu_reference_sample
            tok_s, desc = cpu_reference_sample(cfg)
            line["cpu_baseline"] = dict(desc, value=tok_s, unit="tokens/s")
        print(json.dumps(line), flush=True)
    dist.barrier()
    group.close()
    dist.barrier()
    dist.destroy_process_group()


def _verify_shard(kv, table, plan, cfg, hb, hc, kv_saved, d_kv_local, tokens, m=32):
    """This rank's heads after the benchmarked restore: HIDDEN layers on
    token slices vs the oracle's project_hidden_to_kv (north-star metric),
    KV layers bit-exact against the stored rows, RECOMPUTE layers on rows
    [0, m) vs the oracle's fp32 prefill of those tokens (stated K6 tolerance;
    oracle/parity.py seeds)."""
    import numpy as np
    import torch

    from oracle import Oracle
    from oracle import parity as P

    from . import hcache as H
    L, d, heads, kvh, dffn, n, rope = cfg
    dh = d // heads
    a, c = hb * dh, (hb + hc) * dh
    o = Oracle()
    meth = list(plan.layer_assignment)
    hid = [x for x, y in enumerate(meth) if y == H.LayerMethod.HIDDEN]
    kvl = [x for x, y in enumerate(meth) if y == H.LayerMethod.KV_OFFLOAD]
    rel = [x for x, y in enumerate(meth) if y == H.LayerMethod.RECOMPUTE]
    pick = sorted({hid[int(round(k * (len(hid) - 1) / 2))] for k in range(3)}) if hid else []
    worst = 0.0
    starts = sorted({0, (n // 2) // 64 * 64, max(0, n - m)})
    for layer in pick:
        k, v = kv.gather(layer, table, n)
        wk, wv = P.layer_wkv(o, layer, d, kvh * dh)
        for s0 in starts:
            h = P.hidden_rows(o, layer, n, d, s0, min(m, n - s0))
            kr, vr = o.project(h, np.ascontiguousarray(wk[a:c]), np.ascontiguousarray(wv[a:c]),
                               hc, s0, True, rope)
            worst = max(worst, P.max_rel_err(k[s0:s0 + len(h)].float().cpu().numpy(), kr),
                        P.max_rel_err(v[s0:s0 + len(h)].float().cpu().numpy(), vr))
    exact = None
    if kvl:
        exact = True
        for layer in kvl:
            k, v = kv.gather(layer, table, n)
            exact &= bool(torch.equal(torch.cat([k, v], 1), kv_saved[layer]))
    ne = None
    if rel:
        ref = P.recompute_kv(o, d, heads, dffn, tokens[:m], len(rel), rope)
        ne = 0.0
        for layer in rel:
            k, v = kv.gather(layer, table, m)
            kr, vr = ref[layer]
            ne = max(ne, P.norm_err(k.float().cpu().numpy(), kr[:, a:c]),
                     P.norm_err(v.float().cpu().numpy(), vr[:, a:c]))
    return {"heads": [hb, hb + hc], "hidden_layers_checked": pick, "hidden_max_rel": worst,
            "kv_layers": len(kvl), "kv_bitexact": exact, "recompute_layers": rel,
            "recompute_norm_err": ne,
            "ok": bool(worst <= 1e-2 and exact is not False and (ne is None or ne <= 5e-2))}
