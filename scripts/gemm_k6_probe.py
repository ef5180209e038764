"""The K6 GEMM shapes of a 7B layer (4096 tokens) through hc_gemm_epilogue
(RESID: x += C, xb = bf16(x); GELU: xb = bf16(gelu(C))), each timed alone
back to back (CUDA events), beside cuBLAS's plain GEMM (scripts/cublas_ref.py).
HC_GEMM_SPLIT=1 allows the tail split of the last wave."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2410_05004_b200.capi import check, lib

s = torch.cuda.current_stream().cuda_stream
for name, mode, (m, n, k) in [("O  RESID", 1, (4096, 4096, 4096)), ("FC1 GELU", 2, (4096, 11008, 4096)),
                              ("FC2 RESID", 1, (4096, 4096, 11008)), ("QKV-size RESID", 1, (4096, 12288, 4096))]:
    a = torch.randn(m, k, device="cuda").bfloat16()
    b = (torch.randn(n, k, device="cuda") * 0.01).bfloat16()
    x = torch.zeros(m, n, device="cuda")
    xb = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
    f = lambda: check(lib().hc_gemm_epilogue(mode, a.data_ptr(), b.data_ptr(), m, n, k, x.data_ptr(),
                                             xb.data_ptr(), None, None, None, 0, s))
    for _ in range(10):
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
    print(f"{name:16s} M={m} N={n:6d} K={k:6d}: {us:8.1f} us  {2.0 * m * n * k / us / 1e6:7.1f} TFLOP/s")
