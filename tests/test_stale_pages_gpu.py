"""Paged KV caches are caller memory that may hold anything past a
sequence's last token (a recycled page, a freed buffer's bytes -- half of an
fp32 word is a bf16 NaN 1 time in 256). Masked keys must not reach the
output: with P = 0, a P x V product over a stale NaN row is still NaN. Every
attention path (the tcgen05 prefill kernel, the batched "extend" forward,
split-KV decode) runs once over pages poisoned with NaN / Inf bit patterns
and once over zeroed pages: K/V, layer inputs and next tokens must agree bit
for bit."""
import ctypes as C

import pytest

from test_recompute_gpu import build

pytestmark = pytest.mark.gpu

CFG = dict(n_layers=2, d_hidden=512, n_heads=8, d_ffn=1024, vocab_size=1024, max_seq=8192)


def _kv(H, cfg, w, n_pages, page, poison):
    import torch
    kv = H.KvCache(cfg.n_layers, n_pages, page, w.d_kv)
    if poison:
        for t in kv.k + kv.v:
            bits = torch.full(t.shape, 0x7FC0, dtype=torch.int16, device="cuda")  # bf16 NaN
            bits[..., 1::3] = 0x7F80  # +Inf
            t.view(torch.int16).copy_(bits)
    return kv


# (5000 tokens: 160 attention items over the persistent CTAs, several per CTA,
# the heaviest ending in a partial key tile)
@pytest.mark.parametrize("n", [40, 100, 130, 200, 777, 5000])
def test_prefill_ignores_stale_page_rows(cuda, n):
    import torch
    from paper_2410_05004_b200 import hcache as H
    from paper_2410_05004_b200.capi import check, lib
    cfg, w = build(CFG, 1234)
    page = 64
    n_pages = (n + page - 1) // page + 1
    toks = torch.tensor([(i * 11 + 1) % 1024 for i in range(n)], dtype=torch.int32, device="cuda")
    table = torch.arange(n_pages, dtype=torch.int32, device="cuda").flip(0).contiguous()
    out = []
    for poison in (False, True):
        kv = _kv(H, cfg, w, n_pages, page, poison)
        inputs = torch.empty((cfg.n_layers, n, cfg.d_hidden), dtype=torch.bfloat16, device="cuda")
        nxt = C.c_int32(-1)
        check(lib().hc_prefill(w._h, toks.data_ptr(), n, C.byref(kv.desc), table.data_ptr(),
                               inputs.data_ptr(), C.byref(nxt),
                               torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        out.append((kv, inputs, nxt.value))
    (k0, i0, t0), (k1, i1, t1) = out
    assert torch.isfinite(i1.float()).all()
    assert torch.equal(i0, i1) and t0 == t1
    for layer in range(cfg.n_layers):
        a0, b0 = k0.gather(layer, table, n)
        a1, b1 = k1.gather(layer, table, n)
        assert torch.equal(a0, a1) and torch.equal(b0, b1), layer


@pytest.mark.parametrize("prefix,new", [([40, 130], [1, 1]), ([64, 100], [30, 7])])
def test_continuation_ignores_stale_page_rows(cuda, prefix, new):
    import torch
    from paper_2410_05004_b200 import hcache as H
    cfg, w = build(CFG, 1234)
    page = 64
    B = len(prefix)
    stride = max((a + b + page - 1) // page for a, b in zip(prefix, new)) + 1
    tables = torch.arange(B * stride, dtype=torch.int32).view(B, stride).cuda()
    res = []
    for poison in (False, True):
        kv = _kv(H, cfg, w, B * stride, page, poison)
        toks = [[(i * 7 + s) % 1024 for i in range(a + b)] for s, (a, b) in enumerate(zip(prefix, new))]
        flat = torch.tensor([t for s, ts in enumerate(toks) for t in ts[: prefix[s]]],
                            dtype=torch.int32, device="cuda")
        H.forward_batch(w, flat, prefix, [0] * B, kv, tables)
        flat2 = torch.tensor([t for s, ts in enumerate(toks) for t in ts[prefix[s]:]],
                             dtype=torch.int32, device="cuda")
        nxt = H.forward_batch(w, flat2, new, prefix, kv, tables)
        torch.cuda.synchronize()
        res.append((kv, nxt.cpu().tolist()))
    (k0, n0), (k1, n1) = res
    assert n0 == n1
    for s in range(B):
        for layer in range(cfg.n_layers):
            a0, b0 = k0.gather(layer, tables[s], prefix[s] + new[s])
            a1, b1 = k1.gather(layer, tables[s], prefix[s] + new[s])
            assert torch.equal(a0, a1) and torch.equal(b0, b1), (s, layer)
