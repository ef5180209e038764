"""Head-sharded restore with the all-gather fused into K1 over peer memory
(sharded.PeerShardedRestorer, hc_project_multi_source).

Two ranks run as two processes on the one GPU of the test box: their staging
slots are mapped into each other with CUDA IPC exactly as across GPUs, the
handles travel over gloo, the slot hand-off runs through the device flags.
Each rank's K/V (its KV heads) must equal, bit for bit, a single-process K1
over the concatenated hidden rows. Also: the multi-source projection on one
process with the rows split over separate buffers equals the single-source
projection (row boundaries on 128-row tiles, empty trailing ranges)."""
import os
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


def _worker(rank, world, port, n, q):
    try:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        from paper_2410_05004_b200 import capi
        from paper_2410_05004_b200 import hcache as H
        from paper_2410_05004_b200.sharded import PeerShardedRestorer
        cfg, w, hid, table, n_pages = _setup(rank, world, n)
        store = H.StorageManager(H.DevicePool(2))
        plan = H.RestorationPlan.make(L, L, H.Complement.NONE)
        store.create_session(H.SessionSeed("s", cfg.hash(), L, D, 2, plan, list(range(n))))
        for layer in range(L):
            assert store.snapshot("s", layer, H.StateKind.HIDDEN, hid[layer])
        store.finalize("s")
        kv = H.KvCache(L, n_pages, 64, w.d_kv)
        r = PeerShardedRestorer(store, "s", w, kv, table, n, D, depth=2)
        for _ in range(3):  # epochs wrap the 2-slot ring several times
            r.restore(list(range(L)))
        torch.cuda.synchronize()
        ref = H.KvCache(L, n_pages, 64, w.d_kv)
        import ctypes as C
        for layer in range(L):
            capi.check(capi.lib().hc_project_to_pages(
                w._h, layer, hid[layer].data_ptr(), n, None, 1, C.byref(ref.desc),
                table.data_ptr(), 0, torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        ok = all(torch.equal(kv.k[l_], ref.k[l_]) and torch.equal(kv.v[l_], ref.v[l_])
                 for l_ in range(L))
        dist.barrier()
        q.put((rank, ok, None))
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        import traceback
        q.put((rank, False, traceback.format_exc()))


@pytest.mark.parametrize("n", [700, 1024])
def test_peer_allgather_in_k1_two_processes(cuda, n):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = []
    try:
        for _ in range(2):
            res.append(q.get(timeout=240))
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for rank, ok, err in res:
        assert err is None, err
        assert ok, f"rank {rank}: peer-sharded K/V differ from the single-process K1"


def test_multi_source_projection_matches_single(cuda):
    import ctypes as C

    import torch
    from paper_2410_05004_b200 import capi
    from paper_2410_05004_b200 import hcache as H
    n = 900
    cfg, w, hid, table, n_pages = _setup(0, 1, n)
    for bounds in ([0, 256, 640, 900], [0, 128, 900], [0, 900, 900, 900]):
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
