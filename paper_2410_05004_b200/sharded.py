"""Head-sharded multi-GPU restoration (north star (4)).

Every GPU needs the full [n x d] hidden state of a layer (each KV head
contracts over all of d), while the projection output shards by KV head. So,
per layer, on each of the N ranks (one process per GPU):

  IO      fetch this rank's chunk-aligned 1/N of the layer's tokens over its
          own PCIe link (hc_store_read_layer_range on the copy stream);
  gather  all-gather the N shards over NVLink (NCCL, torch.distributed) into
          the full hidden matrix;
  compute K1 for this rank's KV heads only (hc_project_to_pages).

The three stages run on three streams and are pipelined across layers
(fetch L+1 || all-gather L || K1 L-1) with a bounded staging ring. Chunk
indexing is the reference's (chunk c = tokens [64c, 64c+64), device
(L + c) % ndev, storage.cpp:29-31); shards are whole chunks so ranks never
split one. Timing is device time, max over ranks.

The stages are functions so the same orchestration runs on gloo + CPU in the
tests (host reads, gloo all-gather, oracle projection).
"""
from __future__ import annotations

import ctypes as C
import os
import time
from dataclasses import dataclass
from typing import Callable, List, Tuple

from .capi import HC_CHUNK_TOKENS


def shard_ranges(n_tokens: int, world: int) -> Tuple[List[Tuple[int, int]], int]:
    """Chunk-aligned contiguous token ranges per rank and the padded shard
    size (tokens) every rank contributes to the all-gather."""
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
    """Host-side orchestration shared by the CPU (gloo) and GPU (NCCL) paths.

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


# ------------------------------------------------------------------ GPU path
class GpuShardedRestorer:
    """NCCL + copy engine + K1 pipeline for one rank (torch.distributed must
    be initialised with the nccl backend; one process per GPU)."""

    def __init__(self, store, sid: str, weights, kv, page_table, n_tokens: int, d: int,
                 depth: int = 3):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.world, self.rank = dist.get_world_size(), dist.get_rank()
        self.store, self.sid, self.w, self.kv, self.table = store, sid, weights, kv, page_table
        self.n, self.d = n_tokens, d
        self.plan = ShardPlan.make(n_tokens, self.world, self.rank)
        rows = self.plan.shard_tokens * self.world
        self.ring = [torch.empty((rows, d), dtype=torch.bfloat16, device="cuda")
                     for _ in range(max(2, depth))]
        self.copy = torch.cuda.Stream()
        self.comm = torch.cuda.Stream()
        self.compute = torch.cuda.current_stream()

    def _shard(self, full):
        s = self.plan.shard_tokens
        return full[self.rank * s:(self.rank + 1) * s]

    def restore(self, layers: List[int], resident_shards=None):
        """Enqueue the pipelined restore of `layers`. resident_shards: optional
        per-layer HBM tensors holding this rank's shard (skips PCIe)."""
        import ctypes as Cc
        torch = self.torch
        from .capi import check, lib
        b, e = self.plan.mine
        consumed = [None] * len(self.ring)
        start = torch.cuda.Event()
        start.record(self.compute)
        self.copy.wait_event(start)
        for i, layer in enumerate(layers):
            slot = i % len(self.ring)
            full = self.ring[slot]
            mine = self._shard(full)
            if consumed[slot] is not None:
                self.copy.wait_event(consumed[slot])
            with torch.cuda.stream(self.copy):
                if e > b:
                    if resident_shards is not None:
                        mine[: e - b].copy_(resident_shards[layer][: e - b], non_blocking=True)
                    else:
                        check(lib().hc_store_read_layer_range(
                            self.store._h, self.sid.encode(), layer, 0, b, e, mine.data_ptr(),
                            (e - b) * self.d * 2, 1, self.copy.cuda_stream))
                fetched = torch.cuda.Event()
                fetched.record(self.copy)
            self.comm.wait_event(fetched)
            with torch.cuda.stream(self.comm):
                self.dist.all_gather_into_tensor(full, mine)
                gathered = torch.cuda.Event()
                gathered.record(self.comm)
            self.compute.wait_event(gathered)
            check(lib().hc_project_to_pages(self.w._h, layer, full.data_ptr(), self.n, None, 1,
                                            Cc.byref(self.kv.desc), self.table.data_ptr(), 0,
                                            self.compute.cuda_stream))
            done = torch.cuda.Event()
            done.record(self.compute)
            consumed[slot] = done


def bench(args, cfg, rank, world, dev, clock_sampler=None, peaks=None):
    """bench.py --gpus N (torchrun): head-sharded restore of one context
    (strong scaling). Prints the JSON line on rank 0. clock_sampler: context
    manager class sampling nvidia-smi clocks (bench.ClockSampler); peaks: the
    measured-peaks dict."""
    import json

    import numpy as np
    import torch
    import torch.distributed as dist

    from . import hcache as H
    from .capi import check, lib

    if not dist.is_initialized():
        # a plain `python bench.py --sharded` (no torchrun): a world of one
        for k, v in (("RANK", "0"), ("WORLD_SIZE", "1"), ("LOCAL_RANK", "0"),
                     ("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29517")):
            os.environ.setdefault(k, v)
        backend = os.environ.get("HC_DIST_BACKEND", "nccl")  # gloo: 2 ranks on one GPU (tests)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    L, d, heads, kvh, dffn, n, rope = cfg
    stream = torch.cuda.current_stream().cuda_stream
    hb, hc = head_range(kvh, world, rank)
    mc = H.ModelConfig(n_layers=L, d_hidden=d, n_heads=heads, n_kv_heads=kvh, d_ffn=dffn,
                       max_seq=max(n, 4096), rope_enabled=rope)
    w = H.Weights(mc, hb, hc, dev)
    dh = d // heads
    bound = float(np.float32(1) / np.sqrt(np.float32(d)))
    for layer in range(L):
        full_w = torch.empty((2 * kvh * dh, d), dtype=torch.bfloat16, device="cuda")
        check(lib().hc_fill_symmetric(full_w.data_ptr(), full_w.numel(), 1234 + layer, 0, bound,
                                      1, stream))
        a, c = hb * dh, (hb + hc) * dh
        w.set_layer_kv(layer, torch.cat([full_w[a:c], full_w[kvh * dh + a: kvh * dh + c]]).contiguous())
    page = 64
    n_pages = (n + page - 1) // page
    kv = H.KvCache(L, n_pages, page, w.d_kv)
    table = torch.arange(n_pages, dtype=torch.int32, device="cuda")
    # every rank's store holds the session (stand-in for shared storage); each
    # rank reads only its chunk-aligned token range
    store = H.StorageManager(H.DevicePool(1), buffer_capacity_bytes=4 << 30)
    plan = H.RestorationPlan.make(L, L, H.Complement.NONE)
    store.create_session(H.SessionSeed("bench", mc.hash(), L, d, 2, plan, list(range(n)),
                                       d_kv=kvh * dh))
    shard = ShardPlan.make(n, world, rank)
    b, e = shard.mine
    resident = []
    for layer in range(L):
        hrows = torch.empty((n, d), dtype=torch.bfloat16, device="cuda")
        check(lib().hc_fill_symmetric(hrows.data_ptr(), hrows.numel(), 7, layer * n * d,
                                      1.7320508, 1, stream))
        while not store.snapshot("bench", layer, H.StateKind.HIDDEN, hrows):
            store.drain()
        resident.append(hrows[b:e].clone() if e > b else hrows[:0].clone())
    store.finalize("bench")
    torch.cuda.synchronize()
    # default: the all-gather fused into K1 over peer memory (CUDA IPC over
    # NVLink); HC_SHARD_MODE=nccl selects the NCCL all-gather pipeline
    mode = os.environ.get("HC_SHARD_MODE", "peer")
    if mode == "peer":
        try:
            r = PeerShardedRestorer(store, "bench", w, kv, table, n, d)
        except Exception as exc:  # noqa: BLE001  (IPC mapping unavailable)
            print(f"[rank {rank}] peer mapping failed ({exc}); using the NCCL all-gather",
                  flush=True)
            mode = "nccl"
    if mode != "peer":
        r = GpuShardedRestorer(store, "bench", w, kv, table, n, d)
    if mode == "peer":
        # resident shards live in this rank's range of the aligned split
        b, e = r.ranges[rank]
        resident = [None] * L
        for layer in range(L):
            hrows = torch.empty((n, d), dtype=torch.bfloat16, device="cuda")
            check(lib().hc_fill_symmetric(hrows.data_ptr(), hrows.numel(), 7, layer * n * d,
                                          1.7320508, 1, stream))
            resident[layer] = hrows[b:e].clone() if e > b else hrows[:0].clone()
        torch.cuda.synchronize()

    host_ck = torch.empty(16 * w.d_kv, dtype=torch.bfloat16, pin_memory=True)

    def timed(resident_mode, steps):
        dist.barrier()
        torch.cuda.synchronize()
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(steps):
            r.restore(list(range(L)), resident if resident_mode else None)
            if not resident_mode:  # e2e: device->host read of the step's result
                host_ck.copy_(kv.k[L - 1].view(-1)[: 16 * w.d_kv], non_blocking=True)
        z.record()
        torch.cuda.synchronize()
        ms = torch.tensor([a.elapsed_time(z) / steps], device="cuda")
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        dist.barrier()
        return float(ms.item())

    for _ in range(args.warmup):
        r.restore(list(range(L)), resident)
        r.restore(list(range(L)))
    clk = clock_sampler(dev) if clock_sampler else None
    if clk:
        clk.__enter__()
    ms_e2e = timed(False, args.steps)
    ms_res = timed(True, args.steps)
    if clk:
        clk.__exit__(None, None, None)
    clocks = clk.summary() if clk else {"sm_mhz": None, "sm_max_mhz": None,
                                        "reasons": ["unsampled"]}
    h2d = H.measure_h2d(256 << 20, 5, dev) / 1e9
    if rank == 0:
        h_bytes = L * n * d * 2
        line = {"metric": "restored_kv_tokens_per_s", "value": n / (ms_res * 1e-3),
                "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms_res, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "bf16",
                "data": "synthetic (splitmix64 bf16 hidden states + random-init weights)",
                "config": {"workload": args.config + " head-sharded", "layers": L,
                           "d_hidden": d, "kv_heads": kvh, "tokens": n,
                           "parallelism": f"head-sharded x{world} + " + (
                               "all-gather fused into K1 over peer memory" if mode == "peer"
                               else "NCCL all-gather"),
                           "l2": "inputs larger than L2"},
                "restore_latency_ms": {"resident": ms_res, "e2e": ms_e2e},
                "e2e": {"value": n / (ms_e2e * 1e-3), "unit": "tokens/s",
                        "h2d_bytes_per_step": h_bytes // world,
                        "d2h_bytes_per_step": int(host_ck.numel() * 2)},
                "gpu_launches": args.steps * 2 * L,  # resident leg: row statistics + K1 per layer
                "clocks": clocks,
                "roofline": {"bound": "pcie", "unit": "GB/s",
                             "achieved": h_bytes / world / (ms_e2e * 1e-3) / 1e9,
                             "peak": h2d, "peak_source": "measured pinned H2D 256 MiB (this rank)",
                             "frac": h_bytes / world / (ms_e2e * 1e-3) / 1e9 / h2d,
                             "traffic": None},
                "note": "value: shards resident in HBM (all-gather + K1); e2e: each rank "
                        "fetches its 1/N over PCIe; times are max over ranks"}
        print(json.dumps(line), flush=True)
    if isinstance(r, PeerShardedRestorer):
        r.close()
    dist.barrier()
    dist.destroy_process_group()


# ------------------------------------------- GPU path, all-gather in K1 (peer)
def aligned_ranges(n_tokens: int, world: int, align: int = 128) -> List[Tuple[int, int]]:
    """Contiguous token ranges per rank, boundaries multiples of `align` rows
    (the K1 tile: one M tile reads one rank's range) and hence of the 64-token
    chunk."""
    if n_tokens < 1 or world < 1:
        raise ValueError("aligned_ranges: n_tokens and world must be >= 1")
    blocks = (n_tokens + align - 1) // align
    per = (blocks + world - 1) // world
    return [(min(n_tokens, r * per * align), min(n_tokens, (r + 1) * per * align))
            for r in range(world)]


class PeerShardedRestorer:
    """Head-sharded restore with the all-gather fused into K1 over peer memory.

    Rank r fetches only its token range of each layer (its own PCIe link) into
    a slot of a small staging ring; every rank's K1 (hc_project_multi_source)
    reads the A tiles of all ranges straight from the owners' slots, which are
    mapped into each process with CUDA IPC (NVLink on a multi-GPU node). No
    gathered n x d copy exists. Slot hand-off is stream-ordered through flags
    in device memory: the owner stores the slot's epoch into every rank's
    `ready` flag after the fetch; each consumer stores it into the owner's
    `consumed` flag after its K1; each side waits on its own memory
    (hc_stream_wait_flag). torch.distributed (any backend; gloo suffices) is
    used once, to exchange the IPC handles."""

    def __init__(self, store, sid: str, weights, kv, page_table, n_tokens: int, d: int,
                 depth: int = 2, group=None):
        import torch
        import torch.distributed as dist
        from torch.multiprocessing.reductions import reduce_tensor
        self.torch = torch
        self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        if self.world > 8:
            raise ValueError("peer all-gather: at most 8 ranks (K1 sources)")
        self.store, self.sid, self.w, self.kv, self.table = store, sid, weights, kv, page_table
        self.n, self.d, self.depth = n_tokens, d, max(1, depth)
        self.ranges = aligned_ranges(n_tokens, self.world)
        b, e = self.ranges[self.rank]
        rows = max(1, e - b)
        self.slots = [torch.empty((rows, d), dtype=torch.bfloat16, device="cuda")
                      for _ in range(self.depth)]
        # flags[0][src][slot]: epoch of src's slot ready; flags[1][c][slot]:
        # epoch consumer c finished with MY slot
        self.flags = torch.zeros((2, self.world, self.depth), dtype=torch.int32, device="cuda")
        mine = [reduce_tensor(t) for t in self.slots + [self.flags]]
        allh = [None] * self.world
        dist.all_gather_object(allh, mine, group=group)
        self._peer = []  # keep the mapped tensors alive
        self.peer_slots, self.peer_flags = [], []
        for r in range(self.world):
            if r == self.rank:
                ts = self.slots + [self.flags]
            else:
                ts = [fn(*args) for fn, args in allh[r]]
                self._peer.append(ts)
            self.peer_slots.append(ts[:-1])
            self.peer_flags.append(ts[-1])
        self.copy = torch.cuda.Stream()
        self.step = 0
        dist.barrier(group=group)

    def close(self, group=None):
        """Unmap the peers' buffers (before any producer process exits)."""
        import torch.distributed as dist
        self.torch.cuda.synchronize()
        self._peer.clear()
        self.peer_slots, self.peer_flags = [], []
        self.torch.cuda.ipc_collect()
        dist.barrier(group=group)

    def _flag_ptr(self, owner: int, kind: int, who: int, slot: int) -> int:
        f = self.peer_flags[owner]
        return f.data_ptr() + ((kind * self.world + who) * self.depth + slot) * 4

    def restore(self, layers: List[int], resident_shards=None, stream=None):
        """Enqueue the restore of `layers` on `stream` (default: current)."""
        import ctypes as Cc
        torch = self.torch
        from .capi import check, lib
        compute = stream or torch.cuda.current_stream()
        b, e = self.ranges[self.rank]
        row_begin = (Cc.c_int64 * (self.world + 1))(*([r[0] for r in self.ranges] + [self.n]))
        start = torch.cuda.Event()
        start.record(compute)
        self.copy.wait_event(start)
        P = Cc.c_void_p
        for layer in layers:
            g = self.step
            self.step += 1
            s, ep = g % self.depth, g // self.depth + 1
            # IO lane: my slot is free once every consumer finished epoch ep-1
            if ep > 1:
                for c in range(self.world):
                    check(lib().hc_stream_wait_flag(self.copy.cuda_stream,
                                                    self._flag_ptr(self.rank, 1, c, s), ep - 1))
            if e > b:
                dst = self.slots[s]
                if resident_shards is not None:
                    with torch.cuda.stream(self.copy):
                        dst[: e - b].copy_(resident_shards[layer][: e - b], non_blocking=True)
                else:
                    check(lib().hc_store_read_layer_range(
                        self.store._h, self.sid.encode(), layer, 0, b, e, dst.data_ptr(),
                        (e - b) * self.d * 2, 1, self.copy.cuda_stream))
            ready = (P * self.world)(*[self._flag_ptr(r, 0, self.rank, s)
                                       for r in range(self.world)])
            check(lib().hc_stream_signal_flags(self.copy.cuda_stream, ready, self.world, ep))
            # compute lane: every range of this layer is in place -> fused K1
            for src in range(self.world):
                check(lib().hc_stream_wait_flag(compute.cuda_stream,
                                                self._flag_ptr(self.rank, 0, src, s), ep))
            srcs = (P * self.world)(*[self.peer_slots[r][s].data_ptr()
                                      for r in range(self.world)])
            check(lib().hc_project_multi_source(self.w._h, layer, self.world, srcs, row_begin,
                                                Cc.byref(self.kv.desc), self.table.data_ptr(), 0,
                                                compute.cuda_stream))
            done = (P * self.world)(*[self._flag_ptr(r, 1, self.rank, s)
                                      for r in range(self.world)])
            check(lib().hc_stream_signal_flags(compute.cuda_stream, done, self.world, ep))
        end = torch.cuda.Event()
        end.record(self.copy)
        compute.wait_event(end)
