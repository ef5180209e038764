"""Resident restore (hc_restore_resident) vs 32 x K1: host enqueue time and
device time of one step (Llama-2-7B shape, 4096 tokens)."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2410_05004_b200 import hcache as H
from paper_2410_05004_b200.capi import check, lib

L, d, n, page = 32, 4096, 4096, 64
s = torch.cuda.current_stream().cuda_stream
cfg = H.ModelConfig(n_layers=L, d_hidden=d, n_heads=32, d_ffn=11008, max_seq=n)
w = H.Weights(cfg)
keep = []
for l in range(L):
    t = (torch.randn(2 * d, d, device="cuda") / 64).bfloat16()
    keep.append(t)
    w.set_layer_kv(l, t)
hid = torch.randn(L, n, d, device="cuda").bfloat16()
hptrs = (C.c_void_p * L)(*[hid[l].data_ptr() for l in range(L)])
kv = H.KvCache(L, n // page, page, d)
table = torch.arange(n // page, dtype=torch.int32, device="cuda")


def step():
    check(lib().hc_restore_resident(w._h, hptrs, n, None, 1, C.byref(kv.desc), table.data_ptr(),
                                    0, s))


for _ in range(3):
    step()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 10
a.record()
t0 = time.perf_counter()
for _ in range(reps):
    step()
host = (time.perf_counter() - t0) / reps * 1e3
b.record()
torch.cuda.synchronize()
dev = a.elapsed_time(b) / reps
st, k1 = C.c_double(), C.c_double()
check(lib().hc_bench_project(w._h, 0, hid[0].data_ptr(), n, 20, s, C.byref(st), C.byref(k1)))
print(f"resident: device {dev:.3f} ms/step, host enqueue {host:.3f} ms/step; "
      f"K1 {k1.value:.4f} ms x {L} = {k1.value * L:.3f} ms, stats {st.value * 1e3:.1f} us")
