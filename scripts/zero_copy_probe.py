"""Design probe: K1 reading its A operand (the hidden states) straight from
pinned host memory over PCIe (TMA on the UVA host address; no staging copy)
vs the restore's copy-engine H2D into HBM followed by K1 from HBM. 7B layer,
4096 tokens. Prints per-layer times; the parity of the two outputs."""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2410_05004_b200 import hcache as H
    from paper_2410_05004_b200.capi import check, lib
    n, d = 4096, 4096
    torch.cuda.set_device(0)
    s = torch.cuda.current_stream().cuda_stream
    w = H.Weights(H.ModelConfig(n_layers=1, d_hidden=d, n_heads=32, d_ffn=11008, max_seq=4096))
    wkv = torch.empty((2 * d, d), dtype=torch.bfloat16, device="cuda")
    check(lib().hc_fill_symmetric(wkv.data_ptr(), wkv.numel(), 1234, 0,
                                  float(1 / np.sqrt(np.float32(d))), 1, s))
    w.set_layer_kv(0, wkv)
    hd = torch.empty((n, d), dtype=torch.bfloat16, device="cuda")
    check(lib().hc_fill_symmetric(hd.data_ptr(), hd.numel(), 7, 0, 1.7320508, 1, s))
    hh = hd.cpu().pin_memory()  # UVA: the host pointer is a device-visible address
    k0, v0 = H.project_hidden_to_kv(w, 0, hd, 0)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]

    def timed(fn, reps=10):
        fn()
        torch.cuda.synchronize()
        ev[0].record()
        for _ in range(reps):
            fn()
        ev[1].record()
        torch.cuda.synchronize()
        return ev[0].elapsed_time(ev[1]) / reps

    k = torch.empty_like(k0)
    v = torch.empty_like(v0)

    def zero_copy():  # row statistics + K1, A read over PCIe
        check(lib().hc_project_hidden_to_kv(w._h, 0, hh.data_ptr(), n, 0, k.data_ptr(),
                                            v.data_ptr(), 1, s))

    stage = torch.empty_like(hd)

    def staged():  # copy engine H2D, then statistics + K1 from HBM
        stage.copy_(hh, non_blocking=True)
        check(lib().hc_project_hidden_to_kv(w._h, 0, stage.data_ptr(), n, 0, k.data_ptr(),
                                            v.data_ptr(), 1, s))

    def k1_hbm():
        check(lib().hc_project_hidden_to_kv(w._h, 0, hd.data_ptr(), n, 0, k.data_ptr(),
                                            v.data_ptr(), 1, s))

    def h2d_only():
        stage.copy_(hh, non_blocking=True)

    out = {}
    for name, fn in (("k1_from_hbm", k1_hbm), ("h2d_copy_engine", h2d_only),
                     ("staged_h2d_then_k1", staged), ("zero_copy_k1_over_pcie", zero_copy)):
        out[name] = timed(fn)
        print(f"{name:24s} {out[name]:8.3f} ms", flush=True)
    zero_copy()
    torch.cuda.synchronize()
    print("zero-copy K/V == HBM K/V:", bool(torch.equal(k, k0) and torch.equal(v, v0)))
    print("pcie GB/s (zero copy, A bytes once):", n * d * 2 / (out["zero_copy_k1_over_pcie"] * 1e-3) / 1e9)


if __name__ == "__main__":
    main()
