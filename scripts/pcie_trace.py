#!/usr/bin/env python
"""Profiler evidence for the restore's PCIe loads: one
7B e2e restore (the bench's synthetic session, planner plan) under
torch.profiler -- CUPTI activity records of every H2D copy the C-ABI library
issues (bytes, start, end) and of every kernel -- summarised as achieved
PCIe GB/s per copy and over the restore, link-busy fraction, and the share
of copy time that overlaps K1 / K6 kernels.

    python scripts/pcie_trace.py [--out profiles/r2_pcie_trace.json] [--trace t.json]
"""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "r2_pcie_trace.json"))
    ap.add_argument("--trace", default=None)
    ap.add_argument("--plan", default=None, help="e.g. 8,23,1 (l_re,l_h,l_kv); default planner")
    ap.add_argument("--kernels", action="store_true", help="list every kernel launch")
    args = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile

    from paper_2410_05004_b200 import capi
    from paper_2410_05004_b200 import hcache as H
    from paper_2410_05004_b200.capi import check, lib

    L, d, heads, dffn, n, vocab = 32, 4096, 32, 11008, 4096, 32000
    torch.cuda.set_device(0)
    stream = torch.cuda.current_stream().cuda_stream
    mc = H.ModelConfig(n_layers=L, d_hidden=d, n_heads=heads, d_ffn=dffn, vocab_size=vocab,
                       max_seq=4096)
    w = H.Weights(mc)
    bound = float(np.float32(1) / np.sqrt(np.float32(d)))

    def fill(shape, seed):
        t = shape if torch.is_tensor(shape) else torch.empty(shape, dtype=torch.bfloat16,
                                                              device="cuda")
        check(lib().hc_fill_symmetric(t.data_ptr(), t.numel(), seed, 0, bound, 1, stream))
        return t
    keep = [fill((vocab, d), 99)]
    w.set_embedding(keep[0])
    for layer in range(L):
        qkv = fill((3 * d, d), 0)  # [W_q ; W_k ; W_v]: the fused Q/K/V GEMM
        keep.append(qkv)
        wq, wkv = fill(qkv[:d], 5000 + layer), fill(qkv[d:], 1234 + layer)
        w.set_layer_kv(layer, wkv)
        w.set_layer_full(layer, wq, wkv, fill((d, d), 6000 + layer),
                         fill((dffn, d), 7000 + layer), fill((d, dffn), 8000 + layer))
    kv = H.KvCache(L, n // 64, 64, d)
    table = torch.arange(n // 64, dtype=torch.int32, device="cuda")
    hid = torch.empty((L, n, d), dtype=torch.bfloat16, device="cuda")
    check(lib().hc_fill_symmetric(hid.data_ptr(), hid.numel(), 7, 0, 1.7320508, 1, stream))
    tokens = [(i * 11 + 1) % vocab for i in range(n)]
    if args.plan:
        re, h, k = (int(x) for x in args.plan.split(","))
        plan = H.RestorationPlan.make_mixed(re, h, k)
    else:
        prof = H.profile_hardware(w, n)
        prof.n_layers = L
        plan, _ = H.plan_three_way(prof, layer_bytes=n * d * 2)
    store = H.StorageManager(H.DevicePool(1), buffer_capacity_bytes=4 << 30)
    store.create_session(H.SessionSeed("p", mc.hash(), L, d, 2, plan, tokens))
    for layer, m in enumerate(plan.layer_assignment):
        if m == H.LayerMethod.HIDDEN:
            rows, kind = hid[layer], H.StateKind.HIDDEN
        elif m == H.LayerMethod.KV_OFFLOAD:
            k_, v_ = H.project_hidden_to_kv(w, layer, hid[layer], 0)
            rows, kind = torch.cat([k_, v_], 1).contiguous(), H.StateKind.KV
        else:
            continue
        while not store.snapshot("p", layer, kind, rows):
            store.drain()
    store.finalize("p")
    opts = capi.RestoreOptsC(0, 0, 0)

    def restore():
        check(lib().hc_restore(store._h, b"p", w._h, C.byref(plan._c), C.byref(opts),
                               C.byref(kv.desc), table.data_ptr(), stream, None))
    for _ in range(5):
        restore()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as p:
        restore()
        torch.cuda.synchronize()
    path = args.trace or os.path.join(ROOT, "gpurun_out", "pcie_trace_chrome.json")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    p.export_chrome_trace(path)
    ev = json.load(open(path))["traceEvents"]
    copies = [e for e in ev if e.get("cat") == "gpu_memcpy" and "HtoD" in e.get("name", "")]
    kernels = [e for e in ev if e.get("cat") == "kernel"]
    if not copies:
        raise SystemExit("no H2D copies recorded")
    t0 = min(e["ts"] for e in copies + kernels)
    cp = sorted(((e["ts"] - t0, e["ts"] - t0 + e["dur"], e.get("args", {}).get("bytes", 0))
                 for e in copies))
    kn = sorted(((e["ts"] - t0, e["ts"] - t0 + e["dur"], e["name"]) for e in kernels))

    def union(iv):
        tot, cur = 0.0, None
        for a, b in sorted(iv):
            if cur and a < cur[1]:
                cur[1] = max(cur[1], b)
                continue
            if cur:
                tot += cur[1] - cur[0]
            cur = [a, b]
        return tot + (cur[1] - cur[0] if cur else 0.0)

    def overlap(a_iv, b_iv):  # length of union(a) intersect union(b)
        pts = []
        for a, b in a_iv:
            for c, d_ in b_iv:
                lo, hi = max(a, c), min(b, d_)
                if hi > lo:
                    pts.append((lo, hi))
        return union(pts)
    span = max(b for _, b, _ in cp + kn) - min(a for a, _, _ in cp + kn)  # us
    busy = union([(a, b) for a, b, _ in cp])
    total_bytes = sum(x for _, _, x in cp)
    k1 = [(a, b) for a, b, nm in kn if "tc_gemm" in nm]
    per_copy = [x / (b - a) / 1e3 for a, b, x in cp if b > a and x >= (1 << 20)]
    out = {
        "what": "one hc_restore of the 7B session (bench synthetic model, 4096 tokens) under "
                "torch.profiler (CUPTI activity: memcpy + kernel records)",
        "plan": plan.serialize(),
        "h2d_copies": len(cp), "h2d_bytes": total_bytes,
        "restore_span_ms": span / 1e3,
        "link_busy_ms": busy / 1e3,
        "link_busy_fraction": busy / span,
        "achieved_gbs_over_busy": total_bytes / (busy * 1e-6) / 1e9,
        "achieved_gbs_over_span": total_bytes / (span * 1e-6) / 1e9,
        "per_copy_gbs": {"n": len(per_copy), "median": float(np.median(per_copy)) if per_copy else None,
                         "min": float(min(per_copy)) if per_copy else None,
                         "max": float(max(per_copy)) if per_copy else None},
        "copy_time_overlapping_kernels_ms": overlap([(a, b) for a, b, _ in cp],
                                                    [(a, b) for a, b, _ in kn]) / 1e3,
        "copy_time_overlapping_gemms_ms": overlap([(a, b) for a, b, _ in cp], k1) / 1e3,
        "kernels": len(kn),
        "first_copy_start_us": cp[0][0], "last_copy_end_us": max(b for _, b, _ in cp),
        "first_kernel_start_us": kn[0][0] if kn else None,
        "last_kernel_end_us": max(b for _, b, _ in kn) if kn else None,
    }
    if args.kernels:  # the compute lane's launches in order (name, start, duration)
        out["kernel_list"] = [{"name": nm[:60], "start_us": round(a, 1), "us": round(b - a, 1)}
                              for a, b, nm in kn]
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
