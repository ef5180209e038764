import os, sys, time, json, ctypes as C
sys.argv = ["bench.py", "--steps", "3", "--warmup", "3", "--no-cpu-baseline"]
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import bench
# monkeypatch: capture restore_step via a small harness after bench setup is too invasive;
# instead time hc_restore directly with events per step using the bench's pieces
from paper_2410_05004_b200 import hcache as H, capi
from paper_2410_05004_b200.capi import check, lib
L, d, heads, kvh, dffn, n, rope = bench.CONFIGS["llama2-7b"]
s = torch.cuda.current_stream().cuda_stream
mc = H.ModelConfig(n_layers=L, d_hidden=d, n_heads=heads, d_ffn=dffn, vocab_size=32000, max_seq=4096)
w = H.Weights(mc)
b = float(np.float32(1) / np.sqrt(np.float32(d)))
keep = []
def fill(shape, seed):
    t = torch.empty(shape, dtype=torch.bfloat16, device="cuda")
    check(lib().hc_fill_symmetric(t.data_ptr(), t.numel(), seed, 0, b, 1, s)); keep.append(t); return t
for l in range(L):
    wkv = fill((2*d, d), 10+l); w.set_layer_kv(l, wkv)
    w.set_layer_full(l, fill((d, d), 20+l), wkv, fill((d, d), 30+l), fill((dffn, d), 40+l), fill((d, dffn), 50+l))
w.set_embedding(fill((32000, d), 3))
kv = H.KvCache(L, n // 64, 64, d); table = torch.arange(n // 64, dtype=torch.int32, device="cuda")
store = H.StorageManager(H.DevicePool(1), 4 << 30)
plan = H.RestorationPlan.make(L, 26, H.Complement.RECOMPUTE)
store.create_session(H.SessionSeed("s", 1, L, d, 2, plan, list(range(n))))
hid = torch.empty((n, d), dtype=torch.bfloat16, device="cuda")
for l in range(6, L):
    check(lib().hc_fill_symmetric(hid.data_ptr(), hid.numel(), 7, l, 1.7, 1, s)); torch.cuda.synchronize()
    assert store.snapshot("s", l, H.StateKind.HIDDEN, hid); store.drain()
store.finalize("s")
opts = capi.RestoreOptsC(0, 0)
def step():
    check(lib().hc_restore(store._h, b"s", w._h, C.byref(plan._c), C.byref(opts), C.byref(kv.desc), table.data_ptr(), s, None))
for _ in range(3): step()
torch.cuda.synchronize()
evs = [torch.cuda.Event(enable_timing=True) for _ in range(11)]
evs[0].record()
hs = []
for i in range(10):
    t0 = time.perf_counter(); step(); hs.append((time.perf_counter()-t0)*1e3)
    evs[i+1].record()
torch.cuda.synchronize()
print("per-step GPU ms", [round(evs[i].elapsed_time(evs[i+1]), 3) for i in range(10)])
print("host enqueue ms", [round(x, 3) for x in hs])
res = H.restore(store, "s", w, plan, H.ThrottleConfig(0, True), kv, table)
print("single timed", res.timeline.total_s * 1e3, "fill", res.timeline.fill_s * 1e3)
# synchronous per step
ts = []
for i in range(5):
    torch.cuda.synchronize(); a = torch.cuda.Event(enable_timing=True); z = torch.cuda.Event(enable_timing=True)
    a.record(); step(); z.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(z))
print("isolated steps", [round(x, 3) for x in ts])

# after a hot resident-style burst
hptrs = (C.c_void_p * L)(*[hid.data_ptr()] * L)
for i in range(30):
    check(lib().hc_restore_resident(w._h, hptrs, n, None, 1, C.byref(kv.desc), table.data_ptr(), 0, s))
ts = []
a = torch.cuda.Event(enable_timing=True); z = torch.cuda.Event(enable_timing=True)
a.record()
for i in range(10): step()
z.record(); torch.cuda.synchronize()
print("after hot burst, per step", a.elapsed_time(z) / 10)
