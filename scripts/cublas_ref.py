"""cuBLAS (torch.matmul, bf16) on the K6 GEMM shapes of a 7B layer at 4096
tokens, for comparison with the pair kernel's in-situ times: plain GEMMs,
no epilogue (no LayerNorm fold, RoPE, residual or GELU)."""
import torch

torch.cuda.set_device(0)
shapes = {"QKV (N=12288, K=4096)": (4096, 12288, 4096), "O (N=4096, K=4096)": (4096, 4096, 4096),
          "FC1 (N=11008, K=4096)": (4096, 11008, 4096), "FC2 (N=4096, K=11008)": (4096, 4096, 11008),
          "K1 (N=8192, K=4096)": (4096, 8192, 4096)}
for name, (m, n, k) in shapes.items():
    a = torch.randn(m, k, device="cuda").bfloat16()
    b = torch.randn(n, k, device="cuda").bfloat16()
    for _ in range(20):
        c = a @ b.t()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 50
    e0.record()
    for _ in range(reps):
        c = a @ b.t()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / reps * 1e3
    print(f"{name:24s} {us:8.1f} us  {2.0 * m * n * k / us / 1e6:7.1f} TFLOP/s")
