"""K4 (KV-offload scatter) probe: 4096 [K_row | V_row] rows of a Llama-2-7B
layer (2 x 4096 bf16) into a paged cache (64-token pages, shuffled page
table). Prints the event-timed launch and the HBM bandwidth it implies
(algorithmic bytes: rows read + K/V written = 4 * n * d_kv * 2)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2410_05004_b200 import hcache as H
from paper_2410_05004_b200.capi import check, lib

n, d_kv, page = 4096, 4096, 64
kv = H.KvCache(1, n // page, page, d_kv)
table = torch.randperm(n // page, generator=torch.Generator().manual_seed(3)).to(torch.int32).cuda()
rows = torch.randn(n, 2 * d_kv, device="cuda").bfloat16()
s = torch.cuda.current_stream().cuda_stream


def step():
    check(lib().hc_kv_scatter_to_pages(rows.data_ptr(), n, 0, None, 1, C.byref(kv.desc),
                                       table.data_ptr(), 0, s))


for _ in range(5):
    step()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    step()
b.record()
torch.cuda.synchronize()
us = a.elapsed_time(b) / 20 * 1e3
byt = 4 * n * d_kv * 2
print(f"K4 scatter: {us:.1f} us/launch, {byt / us / 1e3:.0f} GB/s algorithmic ({byt / 1e6:.1f} MB)")
k, v = kv.gather(0, table, n)
assert torch.equal(k, rows[:, :d_kv]) and torch.equal(v, rows[:, d_kv:])
