"""Head-sharded restore host logic on CPU: 2 processes over gloo run the real
save path (sharded.save_shard: each rank's store holds only its own token
range, hc_store_snapshot_range) and orchestration (sharded.restore_layers)
with host reads from the real pinned-store code (hc_store_read_layer_range),
a gloo all-gather in place of the peer-memory reads and the oracle
projection of each rank's KV heads; the union of the ranks' heads must equal
the oracle's full projection bit for bit. Also the N-GPU planner's inputs."""
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
    from paper_2410_05004_b200.sharded import ShardPlan, head_range, restore_layers, save_shard

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = Oracle()
    hidden = [bf16_round(o.symmetric(n * d, 40 + layer, 0, 1.7320508)).reshape(n, d)
              for layer in range(L)]
    # this rank's store holds only its share: its token range of every
    # hidden layer (hc_store_snapshot_range), fp32 as the reference stores
    ranges = [H.shard_range(n, world, r) for r in range(world)]
    shard = max(e - b for b, e in ranges)
    plan = ShardPlan(n, world, rank, ranges, shard)
    store = H.StorageManager(H.DevicePool(3))
    rplan = H.RestorationPlan.make(L, L, H.Complement.NONE)
    save_shard(store, "s", H.SessionSeed("s", 1, L, d, 4, rplan, list(range(n))), rplan, rank,
               world, lambda layer, b, e: hidden[layer][b:e], None)
    man = store.open("s")
    b, e = plan.mine
    for layer in range(L):
        lc = man.find(layer, H.StateKind.HIDDEN)
        assert (lc.n_tokens if lc else 0) == (e if e > b else 0)
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


def test_plan_sharded_takes_the_slowest_rank_and_no_recompute():
    from paper_2410_05004_b200 import hcache as H
    from paper_2410_05004_b200.sharded import plan_sharded
    # 70B GQA at N=8: a rank's token range of hidden rows is 4x its heads' KV
    # bytes -> the planner picks KV offload for every layer (SURVEY finding 6)
    p, ms, t = plan_sharded([1.22e-3, 1.1e-3], [0.31e-3, 0.3e-3], [0.05e-3, 0.06e-3], 80)
    assert t.io_h == 1.22e-3 and t.c_h == 0.06e-3
    assert p.l_re == 0 and p.l_kv == 80
    # MHA at N=2: hidden rows are half the KV bytes -> mostly hidden
    p, ms, _ = plan_sharded([0.3e-3], [0.6e-3], [0.1e-3], 32)
    assert p.l_re == 0 and p.l_h >= 24
    assert all(m != H.LayerMethod.RECOMPUTE for m in p.layer_assignment)


def test_plan_sharded_with_replicated_recompute():
    """With the whole block on every rank the RECOMPUTE prefix is available
    at N > 1 (replicated: c_token is one rank's cost of a whole layer). A
    7B-like balance at N=2 (io_h halved, c_h halved, c_token not) still
    recomputes a prefix, fewer layers than at N=1; the plan is a function of
    the maxima over ranks only."""
    from paper_2410_05004_b200.sharded import plan_sharded
    n1, _, _ = plan_sharded([0.61e-3], [1.21e-3], [0.2e-3], 32, 33, [1.25e-3])
    n2, ms2, t2 = plan_sharded([0.305e-3, 0.3e-3], [0.6e-3, 0.6e-3], [0.1e-3, 0.11e-3], 32, 33,
                               [1.25e-3, 1.3e-3])
    assert t2.c_token == 1.3e-3 and t2.c_h == 0.11e-3
    assert n1.l_re > n2.l_re > 0
    p_none, ms_none, _ = plan_sharded([0.305e-3], [0.6e-3], [0.11e-3], 32, 33)
    assert p_none.l_re == 0 and ms2 < ms_none
