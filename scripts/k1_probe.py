#!/usr/bin/env python
"""K1 on the 7B bench layer (4096 tokens, d=4096, [W_k;W_v] 8192 x 4096) with
the bench's synthetic data, `iters` launches via hc_bench_project: the
target of the ncu --set full capture in scripts/profile_r2.sh."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2410_05004_b200 import hcache as H
    from paper_2410_05004_b200.capi import check, lib
    n, d, iters = 4096, 4096, int(sys.argv[1]) if len(sys.argv) > 1 else 3
    torch.cuda.set_device(0)
    s = torch.cuda.current_stream().cuda_stream
    w = H.Weights(H.ModelConfig(n_layers=1, d_hidden=d, n_heads=32, d_ffn=11008, max_seq=4096))
    wkv = torch.empty((2 * d, d), dtype=torch.bfloat16, device="cuda")
    check(lib().hc_fill_symmetric(wkv.data_ptr(), wkv.numel(), 1234, 0,
                                  float(1 / np.sqrt(np.float32(d))), 1, s))
    w.set_layer_kv(0, wkv)
    h = torch.empty((n, d), dtype=torch.bfloat16, device="cuda")
    check(lib().hc_fill_symmetric(h.data_ptr(), h.numel(), 7, 0, 1.7320508, 1, s))
    a, b = C.c_double(), C.c_double()
    check(lib().hc_bench_project(w._h, 0, h.data_ptr(), n, iters, s, C.byref(a), C.byref(b)))
    print(f"row_stats {a.value * 1e3:.1f} us, K1 {b.value * 1e3:.1f} us "
          f"({4.0 * n * d * 2 * d / (b.value * 1e-3) / 1e12:.0f} TFLOP/s)")


if __name__ == "__main__":
    main()
