"""Decode-step probe: one hc_forward_batch of B sequences x 1 token on the
7B shape; device time (CUDA events) vs host enqueue time."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2410_05004_b200 import hcache as H
from serve_bench import build_weights

B = int(os.environ.get("B", 16))
ctx = int(os.environ.get("CTX", 512))
reps = int(os.environ.get("REPS", 20))
stream = torch.cuda.current_stream().cuda_stream
mc, w, keep = build_weights(32, 4096, 32, 11008, 32000, 8192, stream)
page = 64
stride = (ctx + 64 + page - 1) // page
kv = H.KvCache(32, B * stride, page, 4096)
tables = torch.arange(B * stride, dtype=torch.int32, device="cuda").view(B, stride)
toks = torch.randint(0, 32000, (B,), dtype=torch.int32, device="cuda")
inputs = torch.empty((32, B, 4096), dtype=torch.bfloat16, device="cuda")
for _ in range(3):
    H.forward_batch(w, toks, [1] * B, [ctx] * B, kv, tables, inputs)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
t0 = time.perf_counter()
for _ in range(reps):
    H.forward_batch(w, toks, [1] * B, [ctx] * B, kv, tables, inputs)
t1 = time.perf_counter()
e1.record()
torch.cuda.synchronize()
print(f"B={B} ctx={ctx}: device {e0.elapsed_time(e1) / reps:.3f} ms/step, host enqueue "
      f"{(t1 - t0) * 1e3 / reps:.3f} ms/step")

if os.environ.get("KPROF"):
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(5):
            H.forward_batch(w, toks, [1] * B, [ctx] * B, kv, tables, inputs)
        torch.cuda.synchronize()
    agg = {}
    for e in prof.events():
        if e.device_type.name != "CUDA":
            continue
        k = e.name[:60]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
    tot = sum(v[1] for v in agg.values())
    print(f"warm kernel time per step: {tot / 5:.1f} us")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:12]:
        print(f"  {v[1] / 5:9.1f} us/step {v[0] // 5:5d}/step {k}")
