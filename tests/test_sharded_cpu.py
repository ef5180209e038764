"""Head-sharded restore host logic on CPU: 2 processes over gloo run the real
orchestration (paper_2410_05004_b200.sharded.restore_layers) with host reads
from the real pinned-store code (hc_store_read_layer_range), a gloo
all-gather and the oracle projection of each rank's KV heads; the union of
the ranks' heads must equal the oracle's full projection bit for bit."""
import os
import socket

import numpy as np
import pytest

from paper_2410_05004_b200.sharded import ShardPlan, head_range, shard_ranges


def test_shard_ranges_chunk_aligned_cover():
    for n in (1, 63, 64, 65, 1000, 4096, 32768, 44145):
        for world in (1, 2, 3, 4, 8):
            ranges, shard = shard_ranges(n, world)
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            for (b0, e0), (b1, e1) in zip(ranges, ranges[1:]):
                assert e0 == b1
            for b, e in ranges:
                assert e - b <= shard and shard % 64 == 0
                if e > b:  # empty tail ranks fetch nothing
                    assert b % 64 == 0
                assert e == n or e % 64 == 0   # never splits a 64-token chunk
    with pytest.raises(ValueError):
        shard_ranges(0, 2)


def test_head_range():
    assert [head_range(8, 8, r) for r in range(8)] == [(r, 1) for r in range(8)]
    assert head_range(32, 4, 3) == (24, 8)
    with pytest.raises(ValueError):
        head_range(8, 3, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, d, kvh, dh, L, out_q):
    import ctypes as C

    import torch
    import torch.distributed as dist

    from oracle import Oracle, bf16_round
    from paper_2410_05004_b200 import capi
    from paper_2410_05004_b200 import hcache as H
    from paper_2410_05004_b200.sharded import ShardPlan, head_range, restore_layers

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = Oracle()
    # every rank's store holds the session (shared-storage stand-in), fp32
    store = H.StorageManager(H.DevicePool(3))
    store.create_session(H.SessionSeed("s", 1, L, d, 4,
                                       H.RestorationPlan.make(L, L, H.Complement.NONE),
                                       list(range(n))))
    hidden = [bf16_round(o.symmetric(n * d, 40 + layer, 0, 1.7320508)).reshape(n, d)
              for layer in range(L)]
    for layer in range(L):
        store.snapshot("s", layer, H.StateKind.HIDDEN, hidden[layer])
    store.finalize("s")
    plan = ShardPlan.make(n, world, rank)
    hb, hc = head_range(kvh, world, rank)
    got = {}

    def fetch(layer, b, e, dst):
        buf = np.empty((e - b, d), np.float32)
        capi.check(capi.lib().hc_store_read_layer_range(store._h, b"s", layer, 0, b, e,
                                                        buf.ctypes.data, buf.nbytes, 0, None))
        dst[: e - b] = torch.from_numpy(buf)

    def allgather(mine, full):
        dist.all_gather_into_tensor(full, mine)

    def project(layer, full):
        wk_all = bf16_round(o.symmetric(kvh * dh * d, 9 + layer, 0, 0.05)).reshape(kvh * dh, d)
        wv_all = bf16_round(o.symmetric(kvh * dh * d, 9 + layer, kvh * dh * d, 0.05)).reshape(kvh * dh, d)
        a, c = hb * dh, (hb + hc) * dh
        k, v = o.project(full[:n].numpy(), wk_all[a:c], wv_all[a:c], hc, 0, True, True, nthreads=2)
        got[layer] = (k, v)

    rows = plan.shard_tokens * world
    restore_layers(list(range(L)), plan, fetch, allgather, project,
                   alloc_full=lambda: torch.zeros((rows, d)),
                   shard_view=lambda full, r: full[r * plan.shard_tokens:(r + 1) * plan.shard_tokens])
    out_q.put((rank, hb, hc, {k: (v[0].tolist(), v[1].tolist()) for k, v in got.items()}))
    dist.barrier()
    dist.destroy_process_group()
    del C


@pytest.mark.parametrize("n", [200, 130, 64])
def test_two_rank_gloo_sharded_restore_matches_full_projection(n, oracle):
    import multiprocessing as mp

    from oracle import bf16_round
    d, kvh, dh, L, world = 64, 4, 16, 2, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, d, kvh, dh, L, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for layer in range(L):
        h = bf16_round(oracle.symmetric(n * d, 40 + layer, 0, 1.7320508)).reshape(n, d)
        wk = bf16_round(oracle.symmetric(kvh * dh * d, 9 + layer, 0, 0.05)).reshape(kvh * dh, d)
        wv = bf16_round(oracle.symmetric(kvh * dh * d, 9 + layer, kvh * dh * d, 0.05)).reshape(kvh * dh, d)
        kf, vf = oracle.project(h, wk, wv, kvh, 0, True, True)
        k = np.zeros_like(kf)
        v = np.zeros_like(vf)
        for rank, hb, hc, got in results:
            kr, vr = got[layer]
            k[:, hb * dh:(hb + hc) * dh] = np.array(kr, np.float32)
            v[:, hb * dh:(hb + hc) * dh] = np.array(vr, np.float32)
        np.testing.assert_array_equal(k, kf)
        np.testing.assert_array_equal(v, vf)


def test_shard_plan_mine():
    p = ShardPlan.make(1000, 4, 2)
    assert p.mine == p.ranges[2]
