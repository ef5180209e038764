"""hc_project_multi_source: K1 with its A operand spread over several
buffers (the building block of the head-sharded restore's fused all-gather,
SURVEY 8e). On one process the rows split over separate buffers must give the
single-source projection bit for bit (row boundaries on 128-row tiles, empty
trailing ranges, up to 8 sources); rows with |mean| >> sigma take the same
mean-shift guard as the single-GPU path and stay within the north-star bound
of the oracle. The multi-process protocol is tests/test_sharded_restore_gpu.py."""
import pytest

pytestmark = pytest.mark.gpu

L, D, HEADS = 3, 512, 8


def _setup(rank, world, n):
    import torch
    from paper_2410_05004_b200 import hcache as H
    from paper_2410_05004_b200.sharded import head_range
    from hc_testutil import dev_hidden, dev_wkv
    hb, hc = head_range(HEADS, world, rank)
    dh = D // HEADS
    cfg = H.ModelConfig(n_layers=L, d_hidden=D, n_heads=HEADS, d_ffn=4 * D, max_seq=2048)
    w = H.Weights(cfg, hb, hc)
    for layer in range(L):
        w.set_layer_kv(layer, dev_wkv(D, D, layer, hb, hc, dh))
    hid = [dev_hidden(n, D, seed=70 + layer) for layer in range(L)]
    n_pages = (n + 63) // 64
    table = torch.randperm(n_pages, generator=torch.Generator().manual_seed(9)).to(
        torch.int32).cuda()
    return cfg, w, hid, table, n_pages


def test_multi_source_projection_matches_single(cuda):
    import ctypes as C

    import torch
    from paper_2410_05004_b200 import capi
    from paper_2410_05004_b200 import hcache as H
    n = 900
    cfg, w, hid, table, n_pages = _setup(0, 1, n)
    for bounds in ([0, 256, 640, 900], [0, 128, 900], [0, 900, 900, 900],
                   [0, 128, 256, 384, 512, 640, 768, 896, 900]):
        kv = H.KvCache(L, n_pages, 64, w.d_kv)
        ref = H.KvCache(L, n_pages, 64, w.d_kv)
        s = torch.cuda.current_stream().cuda_stream
        for layer in range(L):
            parts = [hid[layer][a:b].clone() for a, b in zip(bounds[:-1], bounds[1:])]
            srcs = (C.c_void_p * len(parts))(*[p_.data_ptr() if p_.numel() else 0 for p_ in parts])
            rb = (C.c_int64 * len(bounds))(*bounds)
            capi.check(capi.lib().hc_project_multi_source(w._h, layer, len(parts), srcs, rb,
                                                          C.byref(kv.desc), table.data_ptr(), 0, s))
            capi.check(capi.lib().hc_project_to_pages(w._h, layer, hid[layer].data_ptr(), n, None, 1,
                                                      C.byref(ref.desc), table.data_ptr(), 0, s))
            torch.cuda.synchronize()
            assert torch.equal(kv.k[layer], ref.k[layer]) and torch.equal(kv.v[layer], ref.v[layer])
    with pytest.raises(ValueError):  # interior boundary off the 128-row tile
        bad = (C.c_int64 * 3)(0, 100, 900)
        srcs = (C.c_void_p * 2)(hid[0].data_ptr(), hid[0].data_ptr())
        capi.check(capi.lib().hc_project_multi_source(w._h, 0, 2, srcs, bad, C.byref(kv.desc),
                                                      table.data_ptr(), 0, s))


def test_multi_source_large_mean_rows(cuda, oracle):
    """|mean| / sigma ~ 80 on every row (the LayerNorm fold's cancellation
    case): the statistics flag the matrix, the rows are mean-shifted into a
    local copy (the sources -- other GPUs' buffers -- are never written) and
    K1 reads that; K/V within the north-star bound of the oracle, sources
    untouched."""
    import ctypes as C

    import torch
    from hc_testutil import REL_TOL, cpu_wkv, max_rel_err
    from paper_2410_05004_b200 import capi
    from paper_2410_05004_b200 import hcache as H
    n = 640
    cfg, w, hid, table, n_pages = _setup(0, 1, n)
    x = (hid[1].float() + 80.0).to(torch.bfloat16)
    bounds = [0, 256, 512, 640]
    parts = [x[a:b].clone() for a, b in zip(bounds[:-1], bounds[1:])]
    before = [p_.clone() for p_ in parts]
    kv = H.KvCache(L, n_pages, 64, w.d_kv)
    s = torch.cuda.current_stream().cuda_stream
    srcs = (C.c_void_p * 3)(*[p_.data_ptr() for p_ in parts])
    rb = (C.c_int64 * 4)(*bounds)
    capi.check(capi.lib().hc_project_multi_source(w._h, 1, 3, srcs, rb, C.byref(kv.desc),
                                                  table.data_ptr(), 0, s))
    torch.cuda.synchronize()
    assert all(torch.equal(a, b) for a, b in zip(parts, before))
    kr, vr = oracle.project(x.float().cpu().numpy(), *cpu_wkv(oracle, D, D, 1), HEADS)
    k, v = kv.gather(1, table, n)
    err = max(max_rel_err(k.float().cpu().numpy(), kr), max_rel_err(v.float().cpu().numpy(), vr))
    assert err <= REL_TOL, err
    # and identical to the single-source path, which takes the same guard
    ref = H.KvCache(L, n_pages, 64, w.d_kv)
    capi.check(capi.lib().hc_project_to_pages(w._h, 1, x.data_ptr(), n, None, 1,
                                              C.byref(ref.desc), table.data_ptr(), 0, s))
    torch.cuda.synchronize()
    assert torch.equal(kv.k[1], ref.k[1]) and torch.equal(kv.v[1], ref.v[1])
