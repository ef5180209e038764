"""Steady-state e2e restore latency of three-way plans around the planner's
choice (7B, 4096 tokens): back-to-back hc_restore calls, CUDA events."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2410_05004_b200 import capi
from paper_2410_05004_b200 import hcache as H
from paper_2410_05004_b200.capi import check, lib
from serve_bench import build_weights

stream = torch.cuda.current_stream().cuda_stream
L, d, n = 32, 4096, 4096
mc, w, keep = build_weights(L, d, 32, 11008, 32000, 8192, stream)
kv = H.KvCache(L, n // 64, 64, d)
table = torch.arange(n // 64, dtype=torch.int32, device="cuda")
hid = torch.empty((L, n, d), dtype=torch.bfloat16, device="cuda")
check(lib().hc_fill_symmetric(hid.data_ptr(), hid.numel(), 7, 0, 1.7320508, 1, stream))
prof = H.profile_hardware(w, n)
prof.n_layers = L
best, best_ms = H.plan_three_way(prof, L)
print("planner:", best.serialize(), "predicted", best_ms)
store = H.StorageManager(H.DevicePool(1), buffer_capacity_bytes=4 << 30)
opts = capi.RestoreOptsC(0, 0)
tokens = [(i * 11 + 1) % 32000 for i in range(n)]
res = {}
for l_re in (4, 5, 6, 7, 8, 9, 10):
    p = H.RestorationPlan.make_mixed(l_re, L - l_re, 0)
    sid = f"p{l_re}"
    store.create_session(H.SessionSeed(sid, mc.hash(), L, d, 2, p, tokens))
    for layer in range(l_re, L):
        while not store.snapshot(sid, layer, H.StateKind.HIDDEN, hid[layer]):
            store.drain()
    store.finalize(sid)
    f = lambda: check(lib().hc_restore(store._h, sid.encode(), w._h, C.byref(p._c), C.byref(opts),
                                       C.byref(kv.desc), table.data_ptr(), stream, None))
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        f()
    e1.record()
    torch.cuda.synchronize()
    res[l_re] = e0.elapsed_time(e1) / 20
    print(f"l_re={l_re}: {res[l_re]:.3f} ms/restore (loop of 20)", flush=True)
