"""hc_restore_sharded: the head-sharded multi-GPU restore behind the C ABI
(north star (4); include/hcache_b200.h "multi-GPU").

The ranks run as separate processes on the test box's one GPU: their staging
slots and flags are mapped into each other with CUDA IPC exactly as across
GPUs (hc_peer_group_export / _import, blobs exchanged over gloo), the slot
hand-off runs through the device flags, and every rank's store holds only its
own share of the session (its token range of each HIDDEN layer,
hc_store_snapshot_range; its heads' [K|V] rows of each KV layer). Checks:

* every rank's K/V (its heads) equal, bit for bit, a single-process K1 over
  the whole hidden rows (HIDDEN layers) and the stored rows (KV layers),
  through several wraps of the slot ring, for 2 and 4 ranks, uneven ranges;
* rows with |mean| >> sigma (the LayerNorm fold's cancellation case): each
  owner mean-shifts its own range in place, consumers read its statistics;
  K/V match the oracle's project_hidden_to_kv within the north-star bound
  (|g - r| / max(|r|, 1e-2 rms) <= 1e-2) on every rank's heads;
* world 1 is the single-GPU executor (hc_restore)."""
import socket

import pytest

pytestmark = pytest.mark.gpu

L, D, HEADS = 3, 512, 8


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _hidden(layer, n, large_mean):
    from hc_testutil import dev_hidden
    h = dev_hidden(n, D, seed=70 + layer)
    if large_mean and layer == 1:
        # |mean| / sigma ~ 80 on every row of layer 1 (stored as bf16)
        import torch
        h = (h.float() + 80.0 + torch.arange(n, device=h.device).float()[:, None] * 1e-3).to(
            torch.bfloat16)
    return h


def _worker(rank, world, port, n, large_mean, q, gather=None):
    try:
        import ctypes as C
        import os
        if gather:  # read once by the library, before the first restore
            os.environ["HC_SHARDED_GATHER"] = gather

        import torch
        import torch.distributed as dist
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        from hc_testutil import dev_wkv
        from paper_2410_05004_b200 import capi
        from paper_2410_05004_b200 import hcache as H
        hb, hc = H.shard_heads(HEADS, world, rank)
        dh = D // HEADS
        cfg = H.ModelConfig(n_layers=L, d_hidden=D, n_heads=HEADS, d_ffn=4 * D, max_seq=2048)
        w = H.Weights(cfg, hb, hc)
        for layer in range(L):
            w.set_layer_kv(layer, dev_wkv(D, D, layer, hb, hc, dh))
        n_pages = (n + 63) // 64
        table = torch.randperm(n_pages, generator=torch.Generator().manual_seed(9)).to(
            torch.int32).cuda()
        hid = [_hidden(layer, n, large_mean) for layer in range(L)]
        b, e = H.shard_range(n, world, rank)
        plan = H.RestorationPlan.make(L, L - 1, H.Complement.KV_OFFLOAD)  # 2 HIDDEN + 1 KV
        # this rank's share of the session
        kv_rows = {}
        store = H.StorageManager(H.DevicePool(2))
        store.create_session(H.SessionSeed("s", cfg.hash(), L, D, 2, plan, list(range(n)),
                                           d_kv=w.d_kv))
        for layer, m in enumerate(plan.layer_assignment):
            if m == H.LayerMethod.HIDDEN:
                if e > b:
                    assert store.snapshot("s", layer, H.StateKind.HIDDEN,
                                          hid[layer][b:e].contiguous(), tok_begin=b)
            else:
                k_, v_ = H.project_hidden_to_kv(w, layer, hid[layer], 0)
                kv_rows[layer] = torch.cat([k_, v_], 1).contiguous()
                assert store.snapshot("s", layer, H.StateKind.KV, kv_rows[layer])
        store.finalize("s")
        rows_max = max(H.shard_range(n, world, r)[1] - H.shard_range(n, world, r)[0]
                       for r in range(world))
        g = H.PeerGroup(world, rank, D, rows_max, depth=2, exchange=H.PeerGroup.torch_exchange())
        kv = H.KvCache(L, n_pages, 64, w.d_kv)
        for it in range(3):  # epochs wrap the 2-slot ring several times
            tl = H.restore_sharded(g, store, "s", w, plan, H.ThrottleConfig(), kv, table,
                                   timeline=(it == 2))
        torch.cuda.synchronize()
        assert sum(ev.kind == "project" for ev in tl.events) == L - 1
        # single-process reference: K1 over the whole rows / the stored KV rows
        ref = H.KvCache(L, n_pages, 64, w.d_kv)
        s = torch.cuda.current_stream().cuda_stream
        for layer in range(L - 1):
            capi.check(capi.lib().hc_project_to_pages(
                w._h, layer, hid[layer].data_ptr(), n, None, 1, C.byref(ref.desc),
                table.data_ptr(), 0, s))
        capi.check(capi.lib().hc_kv_scatter_to_pages(
            kv_rows[L - 1].data_ptr(), n, L - 1, None, 1, C.byref(ref.desc), table.data_ptr(), 0,
            s))
        torch.cuda.synchronize()
        exact = {layer: bool(torch.equal(kv.k[layer], ref.k[layer]) and
                             torch.equal(kv.v[layer], ref.v[layer])) for layer in range(L)}
        worst = None
        if large_mean:
            from hc_testutil import cpu_wkv, max_rel_err
            from oracle import Oracle
            o = Oracle()
            h = hid[1].float().cpu().numpy()
            kr, vr = o.project(h, *cpu_wkv(o, D, D, 1, hb, hc, dh), hc)
            k_, v_ = kv.gather(1, table, n)
            worst = max(max_rel_err(k_.float().cpu().numpy(), kr),
                        max_rel_err(v_.float().cpu().numpy(), vr))
        dist.barrier()
        g.close()
        dist.barrier()
        q.put((rank, exact, worst, None))
        dist.destroy_process_group()
    except Exception:  # noqa: BLE001
        import traceback
        q.put((rank, None, None, traceback.format_exc()))


def _run(world, n, large_mean=False, gather=None):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, large_mean, q, gather))
             for r in range(world)]
    for p in procs:
        p.start()
    res = []
    try:
        for _ in range(world):
            res.append(q.get(timeout=300))
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for rank, exact, worst, err in res:
        assert err is None, err
    return res


@pytest.mark.parametrize("world,n", [(2, 700), (2, 1024), (4, 1000)])
def test_sharded_restore_bit_exact(cuda, world, n):
    for rank, exact, _, _ in _run(world, n):
        assert all(exact.values()), (rank, exact)


def test_sharded_restore_copy_gather_fallback(cuda):
    """HC_SHARDED_GATHER=copy: the owners' ranges gathered by the copy
    engines into a local buffer, then K1 over it (the path taken where TMA
    cannot address a peer's memory) -- the same bits as the fused K1."""
    for rank, exact, _, _ in _run(2, 1024, gather="copy"):
        assert all(exact.values()), (rank, exact)


def test_sharded_restore_large_mean_rows(cuda):
    from hc_testutil import REL_TOL
    for rank, exact, worst, _ in _run(2, 768, large_mean=True):
        assert exact[0] and exact[2], (rank, exact)  # unflagged / KV layers bit-exact
        assert worst <= REL_TOL, (rank, worst)


def test_sharded_world_one_is_the_single_gpu_restore(cuda):
    import torch
    from hc_testutil import dev_hidden, dev_wkv
    from paper_2410_05004_b200 import hcache as H
    n = 500
    cfg = H.ModelConfig(n_layers=L, d_hidden=D, n_heads=HEADS, d_ffn=4 * D, max_seq=2048)
    w = H.Weights(cfg)
    for layer in range(L):
        w.set_layer_kv(layer, dev_wkv(D, D, layer))
    plan = H.RestorationPlan.make(L, L, H.Complement.NONE)
    store = H.StorageManager(H.DevicePool(1))
    store.create_session(H.SessionSeed("s", cfg.hash(), L, D, 2, plan, list(range(n))))
    hid = [dev_hidden(n, D, seed=5 + layer) for layer in range(L)]
    for layer in range(L):
        assert store.snapshot("s", layer, H.StateKind.HIDDEN, hid[layer])
    store.finalize("s")
    n_pages = (n + 63) // 64
    table = torch.arange(n_pages, dtype=torch.int32, device="cuda")
    g = H.PeerGroup(1, 0, D, n)
    kv = H.KvCache(L, n_pages, 64, D)
    H.restore_sharded(g, store, "s", w, plan, H.ThrottleConfig(), kv, table)
    ref = H.KvCache(L, n_pages, 64, D)
    H.restore(store, "s", w, plan, H.ThrottleConfig(), ref, table)
    torch.cuda.synchronize()
    for layer in range(L):
        assert torch.equal(kv.k[layer], ref.k[layer]) and torch.equal(kv.v[layer], ref.v[layer])


def _worker_recompute(rank, world, port, n, q):
    """A plan with a RECOMPUTE prefix at world > 1: every rank recomputes
    layers [0, 2) for all heads from the session's token ids (replicated
    prefix) and keeps its own heads; then one HIDDEN and one KV layer."""
    try:
        import ctypes as C

        import torch
        import torch.distributed as dist
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        from test_recompute_gpu import dev_init_model
        from paper_2410_05004_b200 import capi
        from paper_2410_05004_b200 import hcache as H
        LR, DFF, VOC = 4, 4 * D, 1024
        hb, hc = H.shard_heads(HEADS, world, rank)
        dh = D // HEADS
        a, c = hb * dh, (hb + hc) * dh
        kw = dict(n_layers=LR, d_hidden=D, n_heads=HEADS, d_ffn=DFF, vocab_size=VOC, max_seq=2048)
        cfg = H.ModelConfig(**kw)
        emb, layers = dev_init_model(LR, D, DFF, VOC, 17)
        w = H.Weights(cfg, hb, hc)
        w_all = H.Weights(cfg)
        for ww in (w, w_all):
            ww.set_embedding(emb)
        for layer, lw in enumerate(layers):
            wkv = lw["wkv"]
            mine = torch.cat([wkv[a:c], wkv[D + a:D + c]]).contiguous()
            w.set_layer_kv(layer, mine)
            w.set_layer_full(layer, lw["wq"], wkv, lw["wo"], lw["fc1"], lw["fc2"])
            w_all.set_layer_kv(layer, wkv)
            w_all.set_layer_full(layer, lw["wq"], wkv, lw["wo"], lw["fc1"], lw["fc2"])
            lw["mine"] = mine
        tokens = [(i * 11 + 1) % VOC for i in range(n)]
        n_pages = (n + 63) // 64
        table = torch.randperm(n_pages, generator=torch.Generator().manual_seed(3)).to(
            torch.int32).cuda()
        hid = {2: _hidden(2, n, False)}
        b, e = H.shard_range(n, world, rank)
        plan = H.RestorationPlan.make_mixed(2, 1, 1)  # RE RE H KV
        store = H.StorageManager(H.DevicePool(2))
        store.create_session(H.SessionSeed("s", cfg.hash(), LR, D, 2, plan, tokens, d_kv=w.d_kv))
        if e > b:
            assert store.snapshot("s", 2, H.StateKind.HIDDEN, hid[2][b:e].contiguous(),
                                  tok_begin=b)
        k3, v3 = H.project_hidden_to_kv(w, 3, _hidden(3, n, False), 0)
        kv3 = torch.cat([k3, v3], 1).contiguous()
        assert store.snapshot("s", 3, H.StateKind.KV, kv3)
        store.finalize("s")
        rows_max = max(H.shard_range(n, world, r)[1] - H.shard_range(n, world, r)[0]
                       for r in range(world))
        g = H.PeerGroup(world, rank, D, rows_max, depth=LR,
                        exchange=H.PeerGroup.torch_exchange())
        kv = H.KvCache(LR, n_pages, 64, w.d_kv)
        for it in range(2):
            tl = H.restore_sharded(g, store, "s", w, plan, H.ThrottleConfig(), kv, table,
                                   timeline=(it == 1))
        torch.cuda.synchronize()
        assert sum(ev.kind == "recompute" for ev in tl.events) == 2, [ev.kind for ev in tl.events]
        # reference: single-process prefill of all heads, this rank's columns
        full = H.KvCache(LR, n_pages, 64, D)
        s = torch.cuda.current_stream().cuda_stream
        tok = torch.tensor(tokens, dtype=torch.int32, device="cuda")
        capi.check(capi.lib().hc_prefill_layers(w_all._h, tok.data_ptr(), n, 0, 2,
                                                C.byref(full.desc), table.data_ptr(), s))
        ref = H.KvCache(LR, n_pages, 64, w.d_kv)
        capi.check(capi.lib().hc_project_to_pages(w._h, 2, hid[2].data_ptr(), n, None, 1,
                                                  C.byref(ref.desc), table.data_ptr(), 0, s))
        torch.cuda.synchronize()
        exact = {}
        for layer in (0, 1):
            fk, fv = full.gather(layer, table, n)
            k, v = kv.gather(layer, table, n)
            exact[layer] = bool(torch.equal(k, fk[:, a:c]) and torch.equal(v, fv[:, a:c]))
        k, v = kv.gather(2, table, n)
        rk, rv = ref.gather(2, table, n)
        exact[2] = bool(torch.equal(k, rk) and torch.equal(v, rv))
        k, v = kv.gather(3, table, n)
        exact[3] = bool(torch.equal(torch.cat([k, v], 1), kv3))
        dist.barrier()
        g.close()
        dist.barrier()
        q.put((rank, exact, None, None))
        dist.destroy_process_group()
    except Exception:  # noqa: BLE001
        import traceback
        q.put((rank, None, None, traceback.format_exc()))


@pytest.mark.parametrize("world,n", [(2, 640), (4, 1000)])
def test_sharded_restore_recompute_prefix(cuda, world, n):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_recompute, args=(r, world, port, n, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = []
    try:
        for _ in range(world):
            res.append(q.get(timeout=300))
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for rank, exact, _, err in res:
        assert err is None, err
        assert all(exact.values()), (rank, exact)
