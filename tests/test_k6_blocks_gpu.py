"""K6 building blocks vs plain PyTorch fp32 references of the same op
(attention_forward model.cpp:237-288 per head; GEMM epilogues)."""
import math

import pytest

pytestmark = pytest.mark.gpu


def _attn_ref(q, k, v, n_heads, n_kv_heads, dh):
    import torch
    n = q.shape[0]
    qf = q.float().view(n, n_heads, dh).transpose(0, 1)
    kf = k.float().view(n, n_kv_heads, dh).transpose(0, 1)
    vf = v.float().view(n, n_kv_heads, dh).transpose(0, 1)
    g = n_heads // n_kv_heads
    kf = kf.repeat_interleave(g, 0)
    vf = vf.repeat_interleave(g, 0)
    s = qf @ kf.transpose(1, 2) / math.sqrt(dh)
    mask = torch.triu(torch.ones(n, n, dtype=torch.bool, device=q.device), 1)
    s = s.masked_fill(mask, float("-inf"))
    return (torch.softmax(s, -1) @ vf).transpose(0, 1).reshape(n, n_heads * dh)


@pytest.mark.parametrize("n,heads,kvh,dh", [(1, 2, 2, 64), (64, 2, 2, 64), (200, 4, 4, 64),
                                            (333, 4, 2, 128), (1024, 8, 8, 64), (130, 8, 1, 128)])
def test_attention_dense_vs_torch(cuda, n, heads, kvh, dh):
    import torch
    from paper_2410_05004_b200 import capi
    g = torch.Generator(device="cuda").manual_seed(n)
    q = torch.randn(n, heads * dh, device="cuda", generator=g).bfloat16()
    k = torch.randn(n, kvh * dh, device="cuda", generator=g).bfloat16()
    v = torch.randn(n, kvh * dh, device="cuda", generator=g).bfloat16()
    out = torch.empty(n, heads * dh, device="cuda", dtype=torch.bfloat16)
    capi.check(capi.lib().hc_attention_dense(q.data_ptr(), n, heads, kvh, dh, k.data_ptr(),
                                             v.data_ptr(), kvh * dh, out.data_ptr(),
                                             torch.cuda.current_stream().cuda_stream))
    ref = _attn_ref(q, k, v, heads, kvh, dh)
    torch.cuda.synchronize()
    err = (out.float() - ref).abs().max().item() / ref.abs().max().item()
    assert err < 2e-2, err


@pytest.mark.parametrize("n,heads,kvh", [(4096, 16, 16), (4608, 40, 40), (4133, 32, 32),
                                         (4096, 32, 32), (4133, 32, 8)])
def test_attention_block_orders_vs_torch(cuda, n, heads, kvh):
    """The launch shapes of the two-tile kernel: the persistent CTAs for a
    sequence whose K/V fit in L2 -- one item per CTA (4096 x 16 heads: 128
    items), several per CTA (4096 x 32 heads = the 7B layer, 544 items at
    4133 tokens, where every CTA's heaviest items also carry the partial
    last key tile, and a GQA variant) -- and the head-major grid once K/V
    outgrow the 80 MB L2 budget (4608 x 40 heads = 94 MB)."""
    import torch
    from paper_2410_05004_b200 import capi
    dh = 128
    g = torch.Generator(device="cuda").manual_seed(n + heads + kvh)
    q = torch.randn(n, heads * dh, device="cuda", generator=g).bfloat16()
    k = torch.randn(n, kvh * dh, device="cuda", generator=g).bfloat16()
    v = torch.randn(n, kvh * dh, device="cuda", generator=g).bfloat16()
    out = torch.empty(n, heads * dh, device="cuda", dtype=torch.bfloat16)
    capi.check(capi.lib().hc_attention_dense(q.data_ptr(), n, heads, kvh, dh, k.data_ptr(),
                                             v.data_ptr(), kvh * dh, out.data_ptr(),
                                             torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    grp = heads // kvh
    for h0 in range(0, heads, 8):  # the fp32 reference eight heads at a time
        sl = slice(h0 * dh, (h0 + 8) * dh)
        kh0, kh1 = h0 // grp, (h0 + 8 + grp - 1) // grp
        ksl = slice(kh0 * dh, kh1 * dh)
        ref = _attn_ref(q[:, sl], k[:, ksl], v[:, ksl], 8, kh1 - kh0, dh)
        err = (out[:, sl].float() - ref).abs().max().item() / ref.abs().max().item()
        assert err < 2e-2, (h0, err)


@pytest.mark.parametrize("n,heads,kvh", [(4133, 32, 32), (4096, 32, 8)])
def test_attention_persistent_equals_grid_bitwise(cuda, n, heads, kvh):
    """The persistent kernel (default for a sequence whose K/V fit in L2) and
    the grid kernel (taken under CUDA-graph capture, which cannot hold the
    persistent schedule's upload) run the same per-tile arithmetic: their
    outputs are bit-identical."""
    import torch
    from paper_2410_05004_b200 import capi
    dh = 128
    g = torch.Generator(device="cuda").manual_seed(7 * n + heads)
    q = torch.randn(n, heads * dh, device="cuda", generator=g).bfloat16()
    k = torch.randn(n, kvh * dh, device="cuda", generator=g).bfloat16()
    v = torch.randn(n, kvh * dh, device="cuda", generator=g).bfloat16()
    outs = [torch.full((n, heads * dh), float("nan"), device="cuda", dtype=torch.bfloat16)
            for _ in range(2)]

    def run(o, stream):
        capi.check(capi.lib().hc_attention_dense(q.data_ptr(), n, heads, kvh, dh, k.data_ptr(),
                                                 v.data_ptr(), kvh * dh, o.data_ptr(), stream))
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        run(outs[0], s.cuda_stream)  # persistent
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            run(outs[1], s.cuda_stream)  # grid (captured)
        graph.replay()
    s.synchronize()
    assert not torch.isnan(outs[0].float()).any()
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("m,n,k,split", [
    (200, 256, 512, 0), (1024, 512, 2048, 0), (130, 4096, 256, 0),
    # decode shapes: narrow tiles + compact smem ring, and the K-split path
    # (uneven slices: 64 K blocks over 9 slices, 172 over 9, one row)
    (16, 256, 512, 0), (40, 4096, 4096, 0), (16, 4096, 4096, 1), (16, 4096, 11008, 1),
    (1, 512, 1088, 1), (100, 11008, 4096, 1)])
def test_gemm_epilogues_vs_torch(cuda, mode, m, n, k, split):
    import torch
    from paper_2410_05004_b200 import capi
    g = torch.Generator(device="cuda").manual_seed(m + n)
    a = torch.randn(m, k, device="cuda", generator=g).bfloat16()
    b = (torch.randn(n, k, device="cuda", generator=g) / math.sqrt(k)).bfloat16()
    x = torch.randn(m, n, device="cuda", generator=g)
    x0 = x.clone()
    xb = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    mean = a.float().mean(1).contiguous()
    rstd = (1 / torch.sqrt(a.float().var(1, unbiased=False) + 1e-5)).contiguous()
    colsum = b.float().sum(1).contiguous()
    fold = mode == 2
    capi.check(capi.lib().hc_gemm_epilogue(mode | (0x100 if split else 0), a.data_ptr(), b.data_ptr(), m, n, k,
                                           x.data_ptr(), xb.data_ptr(),
                                           mean.data_ptr() if fold else None,
                                           rstd.data_ptr() if fold else None,
                                           colsum.data_ptr() if fold else None, 0,
                                           torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    c = a.float() @ b.float().t()
    if mode == 1:
        want = x0 + c
        assert torch.allclose(x, want, rtol=1e-4, atol=1e-4)
        assert torch.equal(xb, x.bfloat16())
    else:
        ln = (a.float() - mean[:, None]) * rstd[:, None]
        want = torch.nn.functional.gelu(ln @ b.float().t())
        err = (xb.float() - want).abs().max().item() / want.abs().max().item()
        assert err < 1e-2, err


def test_attention_many_lengths_vs_torch(cuda):
    """A serving run sees many context lengths: the persistent kernel keeps
    a schedule per shape for up to 64 shapes, later shapes take the grid
    kernel. 80 distinct lengths, each checked against the fp32 reference."""
    import torch
    from paper_2410_05004_b200 import capi
    heads, dh = 8, 128
    g = torch.Generator(device="cuda").manual_seed(5)
    for n in range(600, 680):
        q = torch.randn(n, heads * dh, device="cuda", generator=g).bfloat16()
        k = torch.randn(n, heads * dh, device="cuda", generator=g).bfloat16()
        v = torch.randn(n, heads * dh, device="cuda", generator=g).bfloat16()
        out = torch.empty(n, heads * dh, device="cuda", dtype=torch.bfloat16)
        capi.check(capi.lib().hc_attention_dense(q.data_ptr(), n, heads, heads, dh, k.data_ptr(),
                                                 v.data_ptr(), heads * dh, out.data_ptr(),
                                                 torch.cuda.current_stream().cuda_stream))
        ref = _attn_ref(q, k, v, heads, heads, dh)
        err = (out.float() - ref).abs().max().item() / ref.abs().max().item()
        assert err < 2e-2, (n, err)
