"""GPU head-sharded pipeline (copy engine -> NCCL all-gather -> K1) at
world_size 1 (the GPU box has one GPU): the restored pages must equal the
single-GPU restore bit for bit."""
import os
import socket

import pytest

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_nccl_pipeline_world1_equals_single_gpu(cuda):
    import torch
    import torch.distributed as dist

    from hc_testutil import dev_hidden, dev_wkv
    from paper_2410_05004_b200 import hcache as H
    from paper_2410_05004_b200.sharded import GpuShardedRestorer

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        L, d, heads, n, page = 3, 512, 8, 900, 64
        cfg = H.ModelConfig(n_layers=L, d_hidden=d, n_heads=heads, d_ffn=4 * d, max_seq=1024)
        w = H.Weights(cfg)
        for layer in range(L):
            w.set_layer_kv(layer, dev_wkv(d, d, layer))
        store = H.StorageManager(H.DevicePool(2))
        plan = H.RestorationPlan.make(L, L, H.Complement.NONE)
        store.create_session(H.SessionSeed("s", cfg.hash(), L, d, 2, plan, list(range(n))))
        hid = [dev_hidden(n, d, seed=300 + layer) for layer in range(L)]
        for layer in range(L):
            assert store.snapshot("s", layer, H.StateKind.HIDDEN, hid[layer])
        store.finalize("s")
        n_pages = (n + page - 1) // page
        table = torch.arange(n_pages, dtype=torch.int32, device="cuda")
        kv1 = H.KvCache(L, n_pages, page, d)
        r = GpuShardedRestorer(store, "s", w, kv1, table, n, d)
        r.restore(list(range(L)))
        kv2 = H.KvCache(L, n_pages, page, d)
        H.restore(store, "s", w, plan, H.ThrottleConfig(), kv2, table)
        kv3 = H.KvCache(L, n_pages, page, d)
        r3 = GpuShardedRestorer(store, "s", w, kv3, table, n, d)
        r3.restore(list(range(L)), resident_shards=hid)
        torch.cuda.synchronize()
        for layer in range(L):
            assert torch.equal(kv1.k[layer], kv2.k[layer]) and torch.equal(kv1.v[layer], kv2.v[layer])
            assert torch.equal(kv3.k[layer], kv2.k[layer]) and torch.equal(kv3.v[layer], kv2.v[layer])
    finally:
        dist.destroy_process_group()
