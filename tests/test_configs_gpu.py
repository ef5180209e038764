"""BASELINE configs 3-5 at their real shapes and context lengths (2-3 layers
each so the pinned store stays ~1 GB): full restores through hc_restore /
hc_restore_batch, checked on sampled token slices against the oracle (rows
are independent) and bit-exact where the data is moved, not
computed (KV-offload layers, page placement)."""
import numpy as np
import pytest

from hc_testutil import REL_TOL, cpu_hidden, cpu_wkv, dev_hidden, dev_wkv, golden, max_rel_err

pytestmark = pytest.mark.gpu


def _check_slices(oracle, kv, table, layer, n, d, d_kv_all, heads, seed, slices, rope=True,
                  head_begin=0, head_count=None, d_head=None, seq_offset=0):
    wk, wv = cpu_wkv(oracle, d, d_kv_all, layer, head_begin, head_count, d_head)
    k_all, v_all = kv.gather(layer, table, n)
    for s, m in slices:
        hc = cpu_hidden(oracle, m, d, seed=seed, row0=seq_offset + s)
        kr, vr = oracle.project(hc, wk, wv, head_count or heads, s, True, rope)
        assert max_rel_err(k_all[s:s + m].float().cpu().numpy(), kr) < REL_TOL, (layer, s)
        assert max_rel_err(v_all[s:s + m].float().cpu().numpy(), vr) < REL_TOL, (layer, s)


def test_config3_llama13b_16k_hidden_plus_kv_offload(cuda, oracle):
    """Config 3: 13B shape, 16K context, a plan mixing hidden-state restore
    and KV-offload layers (forced: on one B200 the planner prefers a
    recompute complement, SURVEY finding 5)."""
    import torch
    from paper_2410_05004_b200 import hcache as H
    L, d, heads, n, page = 3, 5120, 40, 16384, 64
    cfg = H.ModelConfig(n_layers=L, d_hidden=d, n_heads=heads, d_ffn=13824, max_seq=n)
    w = H.Weights(cfg)
    for layer in range(L):
        w.set_layer_kv(layer, dev_wkv(d, d, layer))
    plan = H.RestorationPlan.make(L, 2, H.Complement.KV_OFFLOAD)  # 2H + 1KV
    store = H.StorageManager(H.DevicePool(4), buffer_capacity_bytes=1 << 30)
    store.create_session(H.SessionSeed("c3", cfg.hash(), L, d, 2, plan, list(range(n))))
    for layer in range(2):
        assert store.snapshot("c3", layer, H.StateKind.HIDDEN, dev_hidden(n, d, seed=30 + layer))
        store.drain()
    kvrows = dev_hidden(n, 2 * d, seed=99)
    assert store.snapshot("c3", 2, H.StateKind.KV, kvrows)
    store.finalize("c3")
    n_pages = n // page
    table = torch.randperm(n_pages, generator=torch.Generator().manual_seed(3)).to(torch.int32).cuda()
    kv = H.KvCache(L, n_pages, page, d)
    res = H.restore(store, "c3", w, plan, H.ThrottleConfig(), kv, table)
    torch.cuda.synchronize()
    for layer in range(2):
        _check_slices(oracle, kv, table, layer, n, d, d, heads, 30 + layer,
                      [(0, 8), (8191, 9), (n - 8, 8)])
    k, v = kv.gather(2, table, n)
    assert torch.equal(k, kvrows[:, :d]) and torch.equal(v, kvrows[:, d:])
    kinds = [e.kind for e in res.timeline.events]
    assert kinds.count("fetch_hidden") == 2 and kinds.count("fetch_kv") == 1


def test_config4_opt30b_ragged_batch_of_32_sessions(cuda, oracle):
    """Config 4: OPT-30B shape (no RoPE), the 32 round-4 conversations of
    gen_trace(seed 7) (golden: sum n = 44,145) restored concurrently by one
    grouped K1 per layer."""
    import torch
    from paper_2410_05004_b200 import hcache as H
    lens = golden("trace.json")["history"][3::4]
    assert sum(lens) == 44145 and len(lens) == 32
    L, d, heads, page = 2, 7168, 56, 64
    cfg = H.ModelConfig(n_layers=L, d_hidden=d, n_heads=heads, d_ffn=28672, max_seq=4096,
                        rope_enabled=False)
    w = H.Weights(cfg)
    for layer in range(L):
        w.set_layer_kv(layer, dev_wkv(d, d, layer))
    plan = H.RestorationPlan.make(L, L, H.Complement.NONE)
    store = H.StorageManager(H.DevicePool(4), buffer_capacity_bytes=1 << 30)
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    total = int(offs[-1])
    hid = [dev_hidden(total, d, seed=40 + layer) for layer in range(L)]
    for s, n in enumerate(lens):
        store.create_session(H.SessionSeed(f"sess{s}", cfg.hash(), L, d, 2, plan, list(range(n))))
        for layer in range(L):
            assert store.snapshot(f"sess{s}", layer, H.StateKind.HIDDEN,
                                  hid[layer][offs[s]:offs[s + 1]])
        store.drain()
        store.finalize(f"sess{s}")
    stride = max((n + page - 1) // page for n in lens)
    tables = torch.randperm(32 * stride, generator=torch.Generator().manual_seed(4)).to(
        torch.int32).view(32, stride).cuda()
    kv = H.KvCache(L, 32 * stride, page, d)
    res = H.restore_batch(store, [f"sess{s}" for s in range(32)], w, H.ThrottleConfig(), kv,
                          tables)
    torch.cuda.synchronize()
    assert sum(e.kind == "project" for e in res.timeline.events) == L
    for s in (0, 7, 31, int(np.argmax(lens))):
        n = lens[s]
        for layer in range(L):
            _check_slices(oracle, kv, tables[s], layer, n, d, d, heads, 40 + layer,
                          [(0, 4), (max(0, n - 5), min(5, n))], rope=False,
                          seq_offset=int(offs[s]))


def test_config5_llama70b_gqa_32k_head_shard(cuda, oracle):
    """Config 5: 70B GQA shape (8 KV heads), 32K context; this GPU restores
    KV head 2 of 8 (N=8 head sharding) from the full hidden states."""
    import torch
    from paper_2410_05004_b200 import hcache as H
    L, d, heads, kvh, n, page = 2, 8192, 64, 8, 32768, 64
    dh = d // heads
    cfg = H.ModelConfig(n_layers=L, d_hidden=d, n_heads=heads, n_kv_heads=kvh, d_ffn=28672,
                        max_seq=n)
    w = H.Weights(cfg, 2, 1)
    for layer in range(L):
        w.set_layer_kv(layer, dev_wkv(d, kvh * dh, layer, 2, 1, dh))
    plan = H.RestorationPlan.make(L, L, H.Complement.NONE)
    store = H.StorageManager(H.DevicePool(2), buffer_capacity_bytes=1 << 30)
    store.create_session(H.SessionSeed("c5", cfg.hash(), L, d, 2, plan, list(range(n)),
                                       d_kv=kvh * dh))
    for layer in range(L):
        assert store.snapshot("c5", layer, H.StateKind.HIDDEN, dev_hidden(n, d, seed=50 + layer))
        store.drain()
    store.finalize("c5")
    table = torch.arange(n // page, dtype=torch.int32, device="cuda")
    kv = H.KvCache(L, n // page, page, dh)
    H.restore(store, "c5", w, plan, H.ThrottleConfig(), kv, table)
    torch.cuda.synchronize()
    for layer in range(L):
        _check_slices(oracle, kv, table, layer, n, d, kvh * dh, heads, 50 + layer,
                      [(0, 4), (20000, 4), (n - 4, 4)], head_begin=2, head_count=1, d_head=dh)
