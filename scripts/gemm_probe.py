"""Skinny-GEMM probe: hc_gemm_epilogue (RESID) at decode shapes; us/launch and
effective weight-streaming GB/s."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2410_05004_b200.capi import check, lib

s = torch.cuda.current_stream().cuda_stream
for (m, n, k) in [(16, 4096, 4096), (16, 4096, 11008), (16, 11008, 4096), (16, 8192, 4096),
                  (64, 4096, 4096), (128, 4096, 4096), (1, 4096, 4096), (256, 4096, 4096)]:
    a = torch.randn(m, k, device="cuda").bfloat16()
    b = torch.randn(n, k, device="cuda").bfloat16() * 0.01
    x = torch.zeros(m, n, device="cuda")
    xb = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
    f = lambda: check(lib().hc_gemm_epilogue(1, a.data_ptr(), b.data_ptr(), m, n, k, x.data_ptr(),
                                             xb.data_ptr(), None, None, None, 0, s))
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 50
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / reps * 1e3
    print(f"M={m:4d} N={n:6d} K={k:6d}: {us:8.1f} us  W {n * k * 2 / us / 1e3:7.1f} GB/s")
