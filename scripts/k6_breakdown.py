#!/usr/bin/env python
"""Per-kernel breakdown of one K6 (recompute) layer of the 7B shape under
sustained load: hc_prefill_layers over 4 full layers (+ the projection-only
last one) back to back for ~1.5 s, then a torch.profiler (CUPTI) capture of
a few more calls. Prints each kernel's mean duration per layer in launch
order -- in-situ numbers at the power-capped clock, unlike ncu's serialised
replay.

    python scripts/k6_breakdown.py [--n 4096] [--out gpurun_out/k6_breakdown.json]
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--layers", type=int, default=5)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "k6_breakdown.json"))
    args = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile

    from paper_2410_05004_b200 import hcache as H
    from paper_2410_05004_b200.capi import check, lib

    L, d, heads, dffn, n, vocab = args.layers, 4096, 32, 11008, args.n, 32000
    torch.cuda.set_device(0)
    s = torch.cuda.current_stream().cuda_stream
    b = float(np.float32(1) / np.sqrt(np.float32(d)))

    def fill(shape, seed):
        t = torch.empty(shape, dtype=torch.bfloat16, device="cuda")
        check(lib().hc_fill_symmetric(t.data_ptr(), t.numel(), seed, 0, b, 1, s))
        return t
    cfg = H.ModelConfig(n_layers=L, d_hidden=d, n_heads=heads, d_ffn=dffn, vocab_size=vocab,
                        max_seq=max(4096, n))
    w = H.Weights(cfg)
    keep = [fill((vocab, d), 1)]
    w.set_embedding(keep[0])
    for layer in range(L):
        # [W_q ; W_k ; W_v] in one allocation (the fused Q/K/V GEMM) unless HC_QKV_SPLIT
        qkv = fill((3 * d, d), 10 + layer)
        if os.environ.get("HC_QKV_SPLIT"):
            qkv = torch.cat([qkv[:d].clone(), torch.zeros((64, d), dtype=qkv.dtype, device="cuda"),
                             qkv[d:]])
            wq, wkv = qkv[:d], qkv[d + 64:]
        else:
            wq, wkv = qkv[:d], qkv[d:]
        t = [wq, fill((d, d), 30 + layer), fill((dffn, d), 40 + layer),
             fill((d, dffn), 50 + layer)]
        keep += [qkv] + t
        w.set_layer_kv(layer, wkv)
        w.set_layer_full(layer, t[0], wkv, t[1], t[2], t[3])
    kv = H.KvCache(L, n // 64, 64, d)
    table = torch.arange(n // 64, dtype=torch.int32, device="cuda")
    tok = torch.randint(0, vocab, (n,), dtype=torch.int32, device="cuda")

    def call():
        check(lib().hc_prefill_layers(w._h, tok.data_ptr(), n, 0, L, C.byref(kv.desc),
                                      table.data_ptr(), s))
    t0 = time.time()
    while time.time() - t0 < 1.5:
        call()
        torch.cuda.synchronize()
    reps = 6
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    for _ in range(reps):
        call()
    host_ms = (time.perf_counter() - h0) * 1e3 / reps  # enqueue only (GPU still running)
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        call()
    e.record()
    torch.cuda.synchronize()
    call_ms = a.elapsed_time(e) / reps
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            call()
        torch.cuda.synchronize()
    evs = [x for x in prof.events() if x.device_type.name == "CUDA" and "Memcpy" not in x.name
           and "Memset" not in x.name]
    evs.sort(key=lambda x: x.time_range.start)
    per_call = len(evs) // reps
    names = [x.name for x in evs[:per_call]]
    dur = np.array([x.time_range.elapsed_us() for x in evs[:per_call * reps]]).reshape(reps, -1)
    rows = []
    for i, nm in enumerate(names):
        rows.append({"i": i, "kernel": nm[:90], "us": float(dur[:, i].mean())})
    span = (evs[per_call * reps - 1].time_range.end - evs[0].time_range.start) / reps
    out = {"n": n, "layers": L, "call_ms_events": call_ms, "host_enqueue_ms": host_ms, "kernels_per_call": per_call,
           "kernel_sum_us": float(dur.sum(1).mean()), "span_us": span, "kernels": rows}
    for r in rows:
        print(f"{r['i']:3d} {r['us']:9.1f} us  {r['kernel']}")
    print(f"host enqueue {host_ms:.3f} ms/call; call {call_ms:.3f} ms (events), kernel sum {out['kernel_sum_us']:.1f} us, "
          f"span {span:.1f} us")
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(out, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
