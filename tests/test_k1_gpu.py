"""K1 (LN-fold tcgen05 projection + RoPE + paged store) vs the oracle's
project_hidden_to_kv (reference model.cpp:219-235) on identical bf16 inputs.

Tolerances (north star): bf16 K/V outputs, max relative error <= 1e-2 with
relative error |g-r| / max(|r|, tau), tau = 1e-2 * rms(r); fp32 outputs,
normwise max|g-r| / rms(r) <= 2e-4 (accumulation order only)."""
import numpy as np
import pytest

from hc_testutil import (F32_NORM_TOL, REL_TOL, cpu_hidden, cpu_wkv, dev_hidden, dev_wkv,
                         max_rel_err, norm_err)

pytestmark = pytest.mark.gpu


def _weights(cfg, layers, head_begin=0, head_count=None, seed_layers=None):
    from paper_2410_05004_b200 import hcache as H
    w = H.Weights(cfg, head_begin, head_count or 0)
    keep = []
    for L in range(cfg.n_layers):
        if layers is not None and L not in layers:
            continue
        wkv = dev_wkv(cfg.d_hidden, cfg.kv_heads() * cfg.d_head(), L, head_begin,
                      w.kv_head_count if head_count else None, cfg.d_head())
        keep.append(wkv)
        w.set_layer_kv(L, wkv)
    return w


SHAPES = [
    # n, d, n_heads, n_kv_heads, start, norm, rope
    (200, 256, 4, 4, 0, True, True),
    (1, 256, 4, 4, 0, True, True),
    (7, 128, 2, 2, 3, True, True),
    (129, 512, 8, 8, 0, True, True),
    (300, 1024, 16, 4, 11, True, True),      # GQA
    (64, 192, 3, 3, 0, False, True),          # d not a multiple of 64, norm off
    (77, 256, 8, 8, 500, True, False),        # rope off, d_head 32
    (1000, 512, 8, 2, 0, True, True),
]


@pytest.mark.parametrize("n,d,nh,nkv,start,norm,rope", SHAPES)
def test_k1_dense_matches_oracle(cuda, oracle, n, d, nh, nkv, start, norm, rope):
    import torch
    from paper_2410_05004_b200 import hcache as H
    cfg = H.ModelConfig(n_layers=1, d_hidden=d, n_heads=nh, n_kv_heads=nkv, d_ffn=4 * d,
                        max_seq=4096, norm_enabled=norm, rope_enabled=rope)
    w = _weights(cfg, None)
    h = dev_hidden(n, d)
    k32, v32 = H.project_hidden_to_kv(w, 0, h, start, torch.float32)
    k16, v16 = H.project_hidden_to_kv(w, 0, h, start, torch.bfloat16)
    torch.cuda.synchronize()
    hc = cpu_hidden(oracle, n, d)
    wk, wv = cpu_wkv(oracle, d, nkv * cfg.d_head(), 0)
    kr, vr = oracle.project(hc, wk, wv, nkv, start, norm, rope)
    assert norm_err(k32.cpu().numpy(), kr) < F32_NORM_TOL
    assert norm_err(v32.cpu().numpy(), vr) < F32_NORM_TOL
    assert max_rel_err(k16.float().cpu().numpy(), kr) < REL_TOL
    assert max_rel_err(v16.float().cpu().numpy(), vr) < REL_TOL


def test_k1_paged_equals_dense(cuda):
    import torch
    from paper_2410_05004_b200 import hcache as H
    cfg = H.ModelConfig(n_layers=2, d_hidden=512, n_heads=8, d_ffn=2048, max_seq=4096)
    w = _weights(cfg, None)
    n, page = 1000, 16
    kv = H.KvCache(2, num_pages=128, page_size=page, d_kv=512)
    perm = torch.randperm(128, generator=torch.Generator().manual_seed(0))[: (n + page - 1) // page]
    table = perm.to(torch.int32).cuda()
    h = dev_hidden(n, 512)
    from paper_2410_05004_b200 import capi
    import ctypes as C
    for L in range(2):
        capi.check(capi.lib().hc_project_to_pages(w._h, L, h.data_ptr(), n, None, 1,
                                                  C.byref(kv.desc), table.data_ptr(), 0,
                                                  torch.cuda.current_stream().cuda_stream))
        kd, vd = H.project_hidden_to_kv(w, L, h, 0)
        kp, vp = kv.gather(L, table, n)
        torch.cuda.synchronize()
        assert torch.equal(kp, kd) and torch.equal(vp, vd)
    # pages not in the table stay untouched
    unused = sorted(set(range(128)) - set(perm.tolist()))
    assert kv.k[0][unused].abs().sum().item() == 0


def test_k1_ragged_batch_positions_restart(cuda):
    """Concatenated sequences (config 4 layout): each restarts at position 0."""
    import ctypes as C

    import torch
    from paper_2410_05004_b200 import capi
    from paper_2410_05004_b200 import hcache as H
    cfg = H.ModelConfig(n_layers=1, d_hidden=256, n_heads=4, d_ffn=1024, max_seq=2048)
    w = _weights(cfg, None)
    lens = [5, 130, 64, 1, 300]
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    total, page = int(cu[-1]), 64
    stride = max((x + page - 1) // page for x in lens)
    tables = torch.zeros((len(lens), stride), dtype=torch.int32)
    nxt = 0
    for s, x in enumerate(lens):
        for p in range((x + page - 1) // page):
            tables[s, p] = nxt
            nxt += 1
    tables = tables.cuda()
    kv = H.KvCache(1, num_pages=nxt, page_size=page, d_kv=256)
    h = dev_hidden(total, 256)
    d_cu = torch.from_numpy(cu).cuda()
    capi.check(capi.lib().hc_project_to_pages(w._h, 0, h.data_ptr(), total, d_cu.data_ptr(),
                                              len(lens), C.byref(kv.desc), tables.data_ptr(),
                                              stride, torch.cuda.current_stream().cuda_stream))
    for s, x in enumerate(lens):
        kd, vd = H.project_hidden_to_kv(w, 0, h[cu[s]:cu[s + 1]].contiguous(), 0)
        kp, vp = kv.gather(0, tables[s], x)
        torch.cuda.synchronize()
        assert torch.equal(kp, kd) and torch.equal(vp, vd), s


def test_k1_head_sharded_slices(cuda, oracle):
    """a GPU projecting KV heads [b, b+c) equals that slice."""
    import torch
    from paper_2410_05004_b200 import hcache as H
    cfg = H.ModelConfig(n_layers=1, d_hidden=512, n_heads=8, n_kv_heads=4, d_ffn=2048,
                        max_seq=1024)
    n = 256
    h = dev_hidden(n, 512)
    full = _weights(cfg, None)
    kf, vf = H.project_hidden_to_kv(full, 0, h, 0, torch.float32)
    for b, c in ((0, 1), (1, 2), (3, 1)):
        ws = _weights(cfg, None, b, c)
        ks, vs = H.project_hidden_to_kv(ws, 0, h, 0, torch.float32)
        torch.cuda.synchronize()
        dh = cfg.d_head()
        assert torch.allclose(ks, kf[:, b * dh:(b + c) * dh], rtol=1e-5, atol=1e-5)
        assert torch.allclose(vs, vf[:, b * dh:(b + c) * dh], rtol=1e-5, atol=1e-5)


def _sampled_slices_check(oracle, cfg, n, layer, slices, head_begin=0, head_count=None):
    """Full-size K1 on the GPU; the oracle checks sampled token slices [s, s+m)
    at start_pos = s (rows are independent)."""
    import torch
    from paper_2410_05004_b200 import hcache as H
    w = H.Weights(cfg, head_begin, head_count or 0)
    d, dh = cfg.d_hidden, cfg.d_head()
    wkv = dev_wkv(d, cfg.kv_heads() * dh, layer, head_begin, head_count, dh)
    # weights are registered for `layer` only
    w.set_layer_kv(layer, wkv)
    h = dev_hidden(n, d)
    k, v = H.project_hidden_to_kv(w, layer, h, 0, torch.bfloat16)
    torch.cuda.synchronize()
    wk, wv = cpu_wkv(oracle, d, cfg.kv_heads() * dh, layer, head_begin, head_count, dh)
    nkv = head_count or cfg.kv_heads()
    for s, m in slices:
        hc = cpu_hidden(oracle, m, d, row0=s)
        kr, vr = oracle.project(hc, wk, wv, nkv, s, cfg.norm_enabled, cfg.rope_enabled)
        assert max_rel_err(k[s:s + m].float().cpu().numpy(), kr) < REL_TOL, (s, m)
        assert max_rel_err(v[s:s + m].float().cpu().numpy(), vr) < REL_TOL, (s, m)


def test_config2_llama7b_sampled(cuda, oracle):
    from paper_2410_05004_b200 import hcache as H
    cfg = H.ModelConfig(n_layers=32, d_hidden=4096, n_heads=32, d_ffn=11008, max_seq=4096)
    _sampled_slices_check(oracle, cfg, 4096, 31, [(0, 40), (2000, 37), (4096 - 33, 33)])


def test_config5_llama70b_gqa_head_sharded_sampled(cuda, oracle):
    from paper_2410_05004_b200 import hcache as H
    cfg = H.ModelConfig(n_layers=80, d_hidden=8192, n_heads=64, n_kv_heads=8, d_ffn=28672,
                        max_seq=32768)
    # N=8: this GPU projects KV head 5 of 8 over the full 32K context
    _sampled_slices_check(oracle, cfg, 32768, 3, [(0, 16), (32768 - 24, 24), (17000, 16)], 5, 1)


def test_config4_opt30b_no_rope_sampled(cuda, oracle):
    from paper_2410_05004_b200 import hcache as H
    cfg = H.ModelConfig(n_layers=48, d_hidden=7168, n_heads=56, d_ffn=28672, max_seq=4096,
                        rope_enabled=False)
    _sampled_slices_check(oracle, cfg, 3338, 0, [(0, 20), (3338 - 17, 17)])


@pytest.mark.parametrize("offset", [8.0, -40.0])
def test_k1_layernorm_large_mean(cuda, oracle, offset):
    """Rows whose mean dwarfs their spread (|mean| / sigma ~ 80-400): the row
    statistics must not cancel (the reference takes mean and variance in
    double, model.cpp:43-61; K1's statistics use sums of x - x0 per row)."""
    import torch
    from oracle import bf16_round
    from paper_2410_05004_b200 import hcache as H
    n, d, nh = 300, 1024, 8
    cfg = H.ModelConfig(n_layers=1, d_hidden=d, n_heads=nh, d_ffn=4 * d, max_seq=4096)
    w = _weights(cfg, None)
    hc = bf16_round(np.float32(offset) + np.float32(0.1) * cpu_hidden(oracle, n, d))
    h = torch.from_numpy(hc).cuda().bfloat16()
    assert np.array_equal(h.float().cpu().numpy(), hc)  # exactly the oracle's input
    k16, v16 = H.project_hidden_to_kv(w, 0, h, 0, torch.bfloat16)
    torch.cuda.synchronize()
    wk, wv = cpu_wkv(oracle, d, d, 0)
    kr, vr = oracle.project(hc, wk, wv, nh, 0, True, True)
    assert max_rel_err(k16.float().cpu().numpy(), kr) < REL_TOL
    assert max_rel_err(v16.float().cpu().numpy(), vr) < REL_TOL
