import sys, os, ctypes as C
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2410_05004_b200 import hcache as H
from paper_2410_05004_b200.capi import check, lib
L, d, heads, dffn, n, vocab = 2, 4096, 32, 11008, 4096, 32000  # layer 0 full, layer 1 K/V only
s = torch.cuda.current_stream().cuda_stream
b = float(np.float32(1) / np.sqrt(np.float32(d)))
def fill(shape, seed):
    t = torch.empty(shape, dtype=torch.bfloat16, device="cuda")
    check(lib().hc_fill_symmetric(t.data_ptr(), t.numel(), seed, 0, b, 1, s)); return t
cfg = H.ModelConfig(n_layers=L, d_hidden=d, n_heads=heads, d_ffn=dffn, vocab_size=vocab, max_seq=4096)
w = H.Weights(cfg); emb = fill((vocab, d), 1); w.set_embedding(emb)
keep = []
for l in range(L):
    wkv = fill((2*d, d), 10+l); t = [fill((d,d),20+l), fill((d,d),30+l), fill((dffn,d),40+l), fill((d,dffn),50+l)]
    keep += [wkv] + t; w.set_layer_kv(l, wkv); w.set_layer_full(l, t[0], wkv, t[1], t[2], t[3])
kv = H.KvCache(L, n // 64, 64, d); table = torch.arange(n // 64, dtype=torch.int32, device="cuda")
tok = torch.randint(0, vocab, (n,), dtype=torch.int32, device="cuda")
for i in range(4):
    check(lib().hc_prefill_layers(w._h, tok.data_ptr(), n, 0, 2, C.byref(kv.desc), table.data_ptr(), s))
torch.cuda.synchronize()
a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for i in range(5):
    check(lib().hc_prefill_layers(w._h, tok.data_ptr(), n, 0, 2, C.byref(kv.desc), table.data_ptr(), s))
e.record(); torch.cuda.synchronize(); print("K6 layer ms", a.elapsed_time(e) / 5)
