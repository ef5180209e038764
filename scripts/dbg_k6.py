import sys, os, math
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
from oracle import Oracle, bf16_round
from paper_2410_05004_b200 import hcache as H
from test_recompute_gpu import gpu_prefill
o = Oracle()
L_, d, heads, dffn, vocab, seed, n = 2, 256, 4, 512, 256, 21, 200
dh = d // heads
flat = bf16_round(o.init_model(L_, d, dffn, vocab, seed))
emb_np, layers = o.split_weights(flat, L_, d, dffn, vocab)
cfg = H.ModelConfig(n_layers=L_, d_hidden=d, n_heads=heads, d_ffn=dffn, vocab_size=vocab, max_seq=1024)
w = H.Weights(cfg)
to = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(torch.bfloat16).cuda()
emb = to(emb_np); w.set_embedding(emb)
keep = []
for L, lw in enumerate(layers):
    wkv = to(np.concatenate([lw["wk"], lw["wv"]])); keep.append(wkv)
    w.set_layer_kv(L, wkv)
    t = [to(lw["wq"]), to(lw["wo"]), to(lw["fc1"]), to(lw["fc2"])]; keep += t
    w.set_layer_full(L, t[0], wkv, t[1], t[2], t[3])
tokens = [(i * 7 + 3) % vocab for i in range(n)]
kv, table, inputs, _ = gpu_prefill(w, cfg, tokens, page=32)
ref = o.prefill(dict(n_layers=L_, d_hidden=d, n_heads=heads, d_ffn=dffn, vocab_size=vocab), flat, np.array(tokens, np.int32))
# torch fp32 layer 0
x = torch.from_numpy(emb_np[tokens]).cuda()
def ln(x): 
    m = x.mean(1, keepdim=True); v = ((x-m)**2).mean(1, keepdim=True); return (x-m)/torch.sqrt(v+1e-5)
lw = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in layers[0].items()}
a = ln(x)
q, k, v = a @ lw["wq"].T, a @ lw["wk"].T, a @ lw["wv"].T
cs, sn = o.rope_table(n, dh); cs = torch.from_numpy(cs).cuda(); sn = torch.from_numpy(sn).cuda()
def rope(t):
    t = t.view(n, heads, dh // 2, 2); a_, b_ = t[..., 0], t[..., 1]
    c = cs[:, None, :]; s = sn[:, None, :]
    return torch.stack([a_*c - b_*s, a_*s + b_*c], -1).view(n, d)
q, k = rope(q), rope(k)
print("K0 gpu vs torch", ((kv.gather(0, table, n)[0].float() - k).abs().max() / k.abs().max()).item())
print("K0 oracle vs torch", (np.abs(ref["k"][0] - k.cpu().numpy()).max() / k.abs().max()).item())
qh = q.view(n, heads, dh).transpose(0,1); kh = k.view(n, heads, dh).transpose(0,1); vh = v.view(n, heads, dh).transpose(0,1)
s_ = qh @ kh.transpose(1,2) / math.sqrt(dh)
s_ = s_.masked_fill(torch.triu(torch.ones(n,n,dtype=torch.bool,device="cuda"),1), float("-inf"))
mix = (torch.softmax(s_, -1) @ vh).transpose(0,1).reshape(n, d)
x = x + mix @ lw["wo"].T
f = ln(x); h1 = torch.nn.functional.gelu(f @ lw["fc1"].T); x = x + h1 @ lw["fc2"].T
g1 = inputs[1].float()
print("x1 gpu vs torch", ((g1 - x).abs().max() / x.abs().max()).item())
print("x1 oracle vs torch", (np.abs(ref["inputs"][1] - x.cpu().numpy()).max() / x.abs().max()).item())
print("x1 gpu vs oracle", (np.abs(ref["inputs"][1] - g1.cpu().numpy()).max() / np.abs(ref["inputs"][1]).max()).item())
print(g1[:2, :6]); print(x[:2, :6]); print(ref["inputs"][1][:2, :6])
