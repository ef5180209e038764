"""Causal prefill attention probe (hc_attention_dense -> tcgen05 kernel)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2410_05004_b200.capi import check, lib

s = torch.cuda.current_stream().cuda_stream
cases = ((4096, 32), (16384, 40), (1024, 32))
if len(sys.argv) > 1:
    cases = tuple(c for c in cases if c[0] == int(sys.argv[1]))
for n, heads in cases:
    dh = 128
    q = torch.randn(n, heads * dh, device="cuda").bfloat16()
    k = torch.randn(n, heads * dh, device="cuda").bfloat16()
    v = torch.randn(n, heads * dh, device="cuda").bfloat16()
    o = torch.empty_like(q)
    f = lambda: check(lib().hc_attention_dense(q.data_ptr(), n, heads, heads, dh, k.data_ptr(),
                                               v.data_ptr(), heads * dh, o.data_ptr(), s))
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = int(os.environ.get("REPS", 10))
    clk = None
    if os.environ.get("CLOCKS"):  # median SM clock over the loop (nvml)
        from bench import ClockSampler
        clk = ClockSampler(torch.cuda.current_device()).__enter__()
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    if clk is not None:
        clk.__exit__()
        print(clk.summary())
    us = e0.elapsed_time(e1) / reps * 1e3
    flops = 4.0 * n * n * heads * dh / 2
    print(f"n={n:6d} heads={heads}: {us:8.1f} us  {flops / us / 1e6:7.1f} TFLOP/s (causal)")
