"""Row-statistics kernel probe: one layer's hidden states (7B shape, n=4096)
and the 32-layer batched launch of hc_restore_resident's prologue."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2410_05004_b200 import hcache as H
from paper_2410_05004_b200.capi import check, lib

n, d, L = 4096, 4096, 32
cfg = H.ModelConfig(n_layers=1, d_hidden=d, n_heads=32, d_ffn=4 * d, max_seq=n)
w = H.Weights(cfg)
w.set_layer_kv(0, (torch.randn(2 * d, d, device="cuda") / 64).bfloat16())
hid = torch.randn(n, d, device="cuda").bfloat16()
s = torch.cuda.current_stream().cuda_stream
a, b = C.c_double(), C.c_double()
for _ in range(2):
    check(lib().hc_bench_project(w._h, 0, hid.data_ptr(), n, 20, s, C.byref(a), C.byref(b)))
print(f"row stats {a.value * 1e3:.1f} us, K1 {b.value * 1e3:.1f} us (n={n}, d={d})")
